"""TEST INFRASTRUCTURE ONLY — ctypes access to the checkers.

* ``Oracle``: the C restatement (oracle/shotsim_oracle.c) over the product's
  flat program (include/shotsim_b200.h). Parity is "pinned" by
  tests/test_oracle.py against the Random123 KATs, the reference's uniform()
  values and the reference library itself.
* ``Reference``: the UNMODIFIED reference library compiled from
  /root/reference/proj/src by oracle/Makefile (oracle/_ref/libshotsim_ref.so),
  behind the test shim oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference legs) may import this module. The product never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libshotsim_oracle.so"
REF_SO = HERE / "_ref" / "libshotsim_ref.so"
REFERENCE_SRC = Path("/root/reference/proj")

_pu64 = C.POINTER(C.c_uint64)
_pd = C.POINTER(C.c_double)


def build(reference: bool = True) -> None:
    """Compile the oracle (and, when the reference sources are mounted, _ref)."""
    targets = ["oracle"]
    if reference and REFERENCE_SRC.exists():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), f"-j{os.cpu_count() or 4}", *targets], check=True)


class Oracle:
    def __init__(self):
        if not ORACLE_SO.exists():
            build(reference=False)
        lib = C.CDLL(str(ORACLE_SO), mode=os.RTLD_LOCAL)
        lib.oracle_philox.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        lib.oracle_uniform.restype = C.c_double
        lib.oracle_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        lib.oracle_run_shots.argtypes = [C.c_void_p, _pu64, C.c_uint64, C.c_uint64, C.c_uint, _pu64, _pd]
        lib.oracle_final_states.argtypes = [C.c_void_p, _pu64, C.c_uint64, C.c_uint64, _pd, _pu64]
        lib.oracle_run_branch.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, _pu64, _pu64, _pu64]
        lib.oracle_last_error.restype = C.c_char_p
        self.lib = lib

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"oracle error {rc}: {self.lib.oracle_last_error().decode()}")

    def philox(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        self.lib.oracle_philox(c, k, o)
        return list(o)

    def uniform(self, seed, shot, event) -> float:
        return self.lib.oracle_uniform(seed, shot, event)

    def run_shots(self, program, ids, seed, threads=1) -> np.ndarray:
        """program: paper_2308_03399_b200.Program (its flat C-ABI view)."""
        flat = program.flat()
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        out = np.empty(ids.size, dtype=np.uint64)
        self._check(self.lib.oracle_run_shots(C.byref(flat), ids.ctypes.data_as(_pu64), ids.size, seed, threads,
                                              out.ctypes.data_as(_pu64), None))
        return out

    def final_states(self, program, ids, seed):
        flat = program.flat()
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        amps = np.empty((ids.size, 1 << flat.num_qubits), dtype=np.complex128)
        cregs = np.empty(ids.size, dtype=np.uint64)
        self._check(self.lib.oracle_final_states(C.byref(flat), ids.ctypes.data_as(_pu64), ids.size, seed,
                                                 amps.ctypes.data_as(_pd), cregs.ctypes.data_as(_pu64)))
        return amps, cregs

    def run_branch(self, program, shots, seed, budget):
        flat = program.flat()
        out = np.empty(shots, dtype=np.uint64)
        peak, passes = C.c_uint64(), C.c_uint64()
        self._check(self.lib.oracle_run_branch(C.byref(flat), shots, seed, budget, out.ctypes.data_as(_pu64),
                                               C.byref(peak), C.byref(passes)))
        return out, peak.value, passes.value


class RefStats(C.Structure):
    _fields_ = [("dispatch_count", C.c_uint64), ("peak_states", C.c_uint64), ("passes", C.c_uint64),
                ("wall_seconds", C.c_double), ("counts_checksum", C.c_uint64), ("num_keys", C.c_uint64)]


class Reference:
    """The reference library itself (oracle/_ref)."""

    def __init__(self):
        if not REF_SO.exists():
            if not REFERENCE_SRC.exists():
                raise FileNotFoundError(f"{REF_SO} not built and /root/reference absent")
            build(reference=True)
        lib = C.CDLL(str(REF_SO), mode=os.RTLD_LOCAL)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_uniform.restype = C.c_double
        lib.ref_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        lib.ref_philox.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        lib.ref_select_kernels.argtypes = [C.c_char_p]
        lib.ref_run.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint, C.c_uint64,
                                C.c_uint64, _pu64, C.POINTER(RefStats)]
        lib.ref_single_shot.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_uint64, _pd, _pu64]
        lib.ref_run_ids.argtypes = [C.c_char_p, C.c_char_p, _pu64, C.c_uint64, C.c_uint64, C.c_uint, _pu64, _pd]
        lib.ref_batch_segments.argtypes = [C.c_char_p, C.c_char_p, _pu64, C.c_uint64, C.c_uint64, _pd, _pu64, _pu64]
        lib.ref_program_dump.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        lib.ref_exact_creg_distribution.argtypes = [C.c_char_p, C.c_char_p, _pu64, _pd, C.c_uint64, _pu64]
        lib.ref_exact_distribution.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_uint), C.c_uint, _pd]
        self.lib = lib
        self.select_kernels("scalar")  # canonical arithmetic order

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def select_kernels(self, which: str):
        self._check(self.lib.ref_select_kernels(which.encode()))

    def uniform(self, seed, shot, event) -> float:
        return self.lib.ref_uniform(seed, shot, event)

    def philox(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        self.lib.ref_philox(c, k, o)
        return list(o)

    def run(self, circuit, noise, strategy, shots, seed, workers=1, max_batch=0, budget=64):
        out = np.empty(shots, dtype=np.uint64)
        st = RefStats()
        self._check(self.lib.ref_run(circuit.encode(), noise.encode(), strategy.encode(), shots, seed, workers,
                                     max_batch, budget, out.ctypes.data_as(_pu64), C.byref(st)))
        return out, st

    def run_ids(self, circuit, noise, ids, seed, workers=1):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        out = np.empty(ids.size, dtype=np.uint64)
        secs = C.c_double()
        self._check(self.lib.ref_run_ids(circuit.encode(), noise.encode(), ids.ctypes.data_as(_pu64), ids.size,
                                         seed, workers, out.ctypes.data_as(_pu64), C.byref(secs)))
        return out, secs.value

    def single_shot(self, circuit, noise, shot, seed, n):
        amps = np.empty(1 << n, dtype=np.complex128)
        creg = C.c_uint64()
        self._check(self.lib.ref_single_shot(circuit.encode(), noise.encode(), shot, seed,
                                             amps.ctypes.data_as(_pd), C.byref(creg)))
        return amps, creg.value

    def batch_segments(self, circuit, noise, ids, seed, n):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        amps = np.empty((ids.size, 1 << n), dtype=np.complex128)
        cregs = np.empty(ids.size, dtype=np.uint64)
        disp = C.c_uint64()
        self._check(self.lib.ref_batch_segments(circuit.encode(), noise.encode(), ids.ctypes.data_as(_pu64),
                                                ids.size, seed, amps.ctypes.data_as(_pd),
                                                cregs.ctypes.data_as(_pu64), C.byref(disp)))
        return amps, cregs, disp.value

    def program_dump(self, circuit, noise) -> str:
        n = C.c_size_t()
        self._check(self.lib.ref_program_dump(circuit.encode(), noise.encode(), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self._check(self.lib.ref_program_dump(circuit.encode(), noise.encode(), buf, n.value + 1, None))
        return buf.value.decode()

    def exact_creg_distribution(self, circuit, noise):
        """exact_creg_distribution (density.cpp:291-306): {creg value: probability}."""
        n = C.c_uint64()
        self._check(self.lib.ref_exact_creg_distribution(circuit.encode(), noise.encode(), None, None, 0, C.byref(n)))
        keys = np.empty(n.value, dtype=np.uint64)
        probs = np.empty(n.value, dtype=np.float64)
        self._check(self.lib.ref_exact_creg_distribution(circuit.encode(), noise.encode(), keys.ctypes.data_as(_pu64),
                                                         probs.ctypes.data_as(_pd), n.value, C.byref(n)))
        return keys, probs

    def exact_distribution(self, circuit, noise, qubits):
        """exact_distribution (density.cpp:280-289) over `qubits` (qubits[0] = bit 0)."""
        q = (C.c_uint * len(qubits))(*qubits)
        out = np.empty(1 << len(qubits), dtype=np.float64)
        self._check(self.lib.ref_exact_distribution(circuit.encode(), noise.encode(), q, len(qubits),
                                                    out.ctypes.data_as(_pd)))
        return out
