"""Python host mirror of the reference's run API over the C ABI.

Mirrors ``RunOptions`` / ``RunResult`` / ``executor_by_name`` (exec.hpp:12-38)
and ``BatchState`` (exec_batch.hpp:22-84) so parity tests read like the
reference's own tests. Programs are built from the reference's lossless
circuit text + noise JSON (``Program.from_text``); every run executes on the
GPU through ``libshotsim_b200.so`` — there is no CPU execution path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, load


class Program:
    """An instrumented program (NoisyCircuit, program.hpp:42-70)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    @classmethod
    def from_text(cls, circuit_text: str, noise_json: str = "") -> "Program":
        h = C.c_void_p()
        check(load().ssb_program_from_text(circuit_text.encode(), noise_json.encode(), C.byref(h)))
        return cls(h.value)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                load().ssb_program_destroy(self._h)
            except Exception:
                pass
            self._h = C.c_void_p()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def flat(self) -> _lib.FlatProgram:
        f = _lib.FlatProgram()
        check(load().ssb_program_flat(self._h, C.byref(f)))
        return f

    def specialise_check(self, tile_qubits: int = 0) -> int:
        """Compiles the program's shape-specialised tile kernel with NVRTC
        (no GPU needed); returns the number of segment shapes."""
        n = C.c_uint32(0)
        check(load().ssb_program_specialise_check(self._h, tile_qubits, C.byref(n)))
        return n.value

    def fused_specialise_check(self) -> int:
        """Compiles the program's per-pass specialised fused-matrix kernels
        with NVRTC (no GPU needed); returns how many passes were specialised."""
        n = C.c_uint32(0)
        check(load().ssb_program_fused_specialise_check(self._h, C.byref(n)))
        return n.value

    def pass_map(self, tile_qubits: int = 0) -> np.ndarray:
        """Diagnostics: the streamed plan's tile pass of every op (-1: outside
        a pass), for `tile_qubits` local qubits (0: default). Host only."""
        f = self.flat()
        out = np.empty(f.num_ops, dtype=np.uint32)
        n = C.c_uint32(0)
        check(load().ssb_program_pass_map(self._h, tile_qubits, out.ctypes.data_as(C.POINTER(C.c_uint32)),
                                          f.num_ops, C.byref(n)))
        return out.astype(np.int64) - ((out == 0xFFFFFFFF) * (1 << 32))

    def fused_info(self, tile_qubits: int = 0) -> dict:
        """Diagnostics of the fused-matrix plan (host only)."""
        i = _lib.FusedInfoC()
        check(load().ssb_program_fused_info(self._h, tile_qubits, C.byref(i)))
        return {f: getattr(i, f) for f, _ in _lib.FusedInfoC._fields_ if f != "reserved"}

    def dump(self) -> str:
        n = C.c_size_t()
        check(load().ssb_program_dump(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(load().ssb_program_dump(self._h, buf, n.value + 1, None))
        return buf.value.decode()

    @property
    def num_qubits(self) -> int:
        return self.flat().num_qubits

    @property
    def num_clbits(self) -> int:
        return self.flat().num_clbits

    @property
    def num_events(self) -> int:
        return self.flat().num_events

    @property
    def has_measure(self) -> bool:
        return bool(self.flat().has_measure)

    @property
    def sampling_eligible(self) -> bool:
        return bool(self.flat().sampling_eligible)

    def ops(self) -> List[_lib.FlatOp]:
        f = self.flat()
        return [f.ops[i] for i in range(f.num_ops)]


@dataclass
class RunOptions:
    shots: int = 1
    seed: int = 0
    workers: int = 1            # GPUs for the executor shim; the Python API runs one engine
    max_batch_size: int = 0
    branch_budget: int = 64
    mem_limit_bytes: int = 0
    record_shot_values: bool = False
    check_norms: bool = False
    collect_leaf_stats: bool = False
    resident_max_qubits: int = 0  # tuning: 0 = engine default
    tile_qubits: int = 0
    profile: bool = False         # per-kernel-class CUDA-event timing in the stats
    interpret_only: bool = False  # never use the run-time shape-specialised tile kernel
    fused_matrices: bool = False  # 4x4 block fusion + guard band (ssb_run_options::fused_matrices)
    export_states: bool = False   # debug: RunResult.states = each shot's pre-sampling state

    def to_c(self) -> _lib.RunOptionsC:
        return _lib.RunOptionsC(self.max_batch_size, self.branch_budget, self.mem_limit_bytes,
                                int(self.check_norms), int(self.collect_leaf_stats),
                                self.resident_max_qubits, self.tile_qubits, int(self.profile),
                                int(self.interpret_only), int(self.fused_matrices), 0)


@dataclass
class BranchStats:
    peak_states: int = 0
    passes: int = 0
    leaf_shots: List[int] = field(default_factory=list)


@dataclass
class RunResult:
    counts: Dict[str, int]
    shot_values: Optional[np.ndarray]
    dispatch_count: int = 0
    peak_states: int = 0
    branch: BranchStats = field(default_factory=BranchStats)
    strategy: str = ""
    shots: int = 0
    seed: int = 0
    device_seconds: float = 0.0
    wall_seconds: float = 0.0
    fused_passes: int = 0
    specialised_shapes: int = 0
    sampling_serial_chunks: int = 0
    trunk_skipped: int = 0
    fused_blocks: int = 0
    guard_flagged: int = 0
    guard_delta: float = 0.0
    pass_seconds: float = 0.0     # profile=True: CUDA-event time of the fused passes
    special_seconds: float = 0.0
    sample_seconds: float = 0.0
    states: Optional[np.ndarray] = None


def bitstring(value: int, width: int) -> str:
    """result.cpp:7-13 — MSB first."""
    return format(value, "b").zfill(width)[-width:] if width else ""


def counts_from_values(values: Sequence[int], width: int, has_measure: bool) -> Dict[str, int]:
    """result.cpp:40-48."""
    vals = np.asarray(values, dtype=np.uint64)
    if not has_measure:
        return {"": int(vals.size)} if vals.size else {}
    uniq, cnt = np.unique(vals, return_counts=True)
    return {bitstring(int(u), width): int(c) for u, c in zip(uniq, cnt)}


def counts_checksum_of_values(values: np.ndarray, width: int, has_measure: bool):
    """counts_checksum (result.cpp:23-38) computed by the library; (checksum, keys)."""
    v = np.ascontiguousarray(values, dtype=np.uint64)
    cs, nk = C.c_uint64(), C.c_uint64()
    check(load().ssb_counts_checksum(v.ctypes.data_as(_lib._pu64), v.size, width, int(has_measure),
                                     C.byref(cs), C.byref(nk)))
    return cs.value, nk.value


class Engine:
    """One CUDA device (sm_100a)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(load().ssb_engine_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if self._h and self._h.value:
            load().ssb_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def stream(self) -> int:
        return load().ssb_engine_stream(self._h) or 0

    def _run(self, fn, program: Program, opts: RunOptions, shot_begin: int, shot_count: int, name: str):
        if opts.shots < 1 and shot_count is None:
            raise ValueError("shots must be >= 1")
        count = opts.shots if shot_count is None else shot_count
        values = np.empty(count, dtype=np.uint64)
        st = _lib.StatsC()
        co = opts.to_c()
        f = program.flat()
        states = None
        if opts.export_states:
            states = np.empty((count, 1 << f.num_qubits), dtype=np.complex128)
            co.states_out = states.ctypes.data_as(_lib._pd)
        leaves = np.empty(0, dtype=np.uint64)
        if opts.collect_leaf_stats:
            leaves = np.empty(4096, dtype=np.uint64)
            co.leaf_shots, co.leaf_shots_capacity = leaves.ctypes.data_as(_lib._pu64), leaves.size
        check(fn(self._h, program.handle, shot_begin, count, opts.seed, C.byref(co),
                 values.ctypes.data_as(_lib._pu64), C.byref(st)))
        if opts.collect_leaf_stats and st.num_leaves > leaves.size:  # rerun with room for every leaf
            leaves = np.empty(st.num_leaves, dtype=np.uint64)
            co.leaf_shots, co.leaf_shots_capacity = leaves.ctypes.data_as(_lib._pu64), leaves.size
            check(fn(self._h, program.handle, shot_begin, count, opts.seed, C.byref(co),
                     values.ctypes.data_as(_lib._pu64), C.byref(st)))
        r = RunResult(counts=counts_from_values(values, f.num_clbits, bool(f.has_measure)),
                      shot_values=values if opts.record_shot_values else None,
                      dispatch_count=st.dispatch_count, peak_states=st.peak_states,
                      branch=BranchStats(st.peak_states, st.passes,
                                         [int(x) for x in leaves[:st.num_leaves]]), strategy=name, shots=count,
                      seed=opts.seed, device_seconds=st.device_seconds, wall_seconds=st.wall_seconds,
                      fused_passes=st.fused_passes, specialised_shapes=st.specialised_shapes,
                      sampling_serial_chunks=st.sampling_serial_chunks,
                      trunk_skipped=st.trunk_skipped, fused_blocks=st.fused_blocks,
                      guard_flagged=st.guard_flagged, guard_delta=st.guard_delta,
                      pass_seconds=st.pass_seconds, special_seconds=st.special_seconds,
                      sample_seconds=st.sample_seconds, states=states)
        r._values = values
        return r

    def run_batch(self, program: Program, opts: RunOptions, shot_begin: int = 0,
                  shot_count: Optional[int] = None) -> RunResult:
        return self._run(load().ssb_run_batch, program, opts, shot_begin, shot_count, "gpu-batch")

    def run_branch(self, program: Program, opts: RunOptions, shot_begin: int = 0,
                   shot_count: Optional[int] = None) -> RunResult:
        if opts.branch_budget < 1:
            raise ValueError("branch budget must be >= 1")
        return self._run(load().ssb_run_branch, program, opts, shot_begin, shot_count, "gpu-branch")

    def run_batch_device(self, program: Program, opts: RunOptions, values_ptr: int, shot_begin: int,
                         shot_count: int) -> _lib.StatsC:
        st = _lib.StatsC()
        co = opts.to_c()
        check(load().ssb_run_batch_device(self._h, program.handle, shot_begin, shot_count, opts.seed,
                                          C.byref(co), C.c_void_p(values_ptr), C.byref(st)))
        return st

    def histogram_device(self, values_ptr: int, count: int, num_clbits: int, hist_ptr: int) -> None:
        check(load().ssb_histogram_device(self._h, C.c_void_p(values_ptr), count, num_clbits,
                                          C.c_void_p(hist_ptr)))


    # ---- exact density-matrix reference (density.hpp:56-68), n <= 10 ----
    def exact_creg_distribution(self, program: Program) -> Dict[int, float]:
        """exact_creg_distribution (density.cpp:291-306), evolved on this device."""
        n = C.c_uint64()
        check(load().ssb_exact_creg_distribution(self._h, program.handle, None, None, 0, C.byref(n)))
        keys = np.empty(n.value, dtype=np.uint64)
        probs = np.empty(n.value, dtype=np.float64)
        check(load().ssb_exact_creg_distribution(self._h, program.handle, keys.ctypes.data_as(_lib._pu64),
                                                 probs.ctypes.data_as(_lib._pd), n.value, C.byref(n)))
        return {int(k): float(p) for k, p in zip(keys, probs)}

    def exact_distribution(self, program: Program, qubits: Sequence[int]) -> np.ndarray:
        """exact_distribution (density.cpp:280-289) over `qubits` (qubits[0] = bit 0)."""
        q = (C.c_uint32 * max(1, len(qubits)))(*qubits)
        out = np.empty(1 << len(qubits), dtype=np.float64)
        check(load().ssb_exact_distribution(self._h, program.handle, q, len(qubits), out.ctypes.data_as(_lib._pd)))
        return out


def tvd_vs_exact(values: np.ndarray, num_clbits: int, has_measure: bool, exact: Dict[int, float]) -> float:
    """tvd_vs_exact (density.cpp:308-315) of per-shot register values against an exact distribution."""
    v = np.ascontiguousarray(values, dtype=np.uint64)
    keys = np.array(sorted(exact), dtype=np.uint64)
    probs = np.array([exact[int(k)] for k in keys], dtype=np.float64)
    out = C.c_double()
    check(load().ssb_tvd_vs_exact(v.ctypes.data_as(_lib._pu64), v.size, num_clbits, int(has_measure),
                                  keys.ctypes.data_as(_lib._pu64), probs.ctypes.data_as(_lib._pd), keys.size,
                                  C.byref(out)))
    return out.value


def _fp64_peak(engine) -> float:
    out = C.c_double(0.0)
    check(load().ssb_fp64_peak(engine._h, C.byref(out)))
    return out.value


class BatchState:
    """Operator-level batch over arbitrary shot ids (exec_batch.hpp:22-84)."""

    def __init__(self, engine: Engine, program: Program, shot_ids: Sequence[int], seed: int):
        ids = np.ascontiguousarray(shot_ids, dtype=np.uint64)
        h = C.c_void_p()
        check(load().ssb_batch_create(engine.handle, program.handle, ids.ctypes.data_as(_lib._pu64), ids.size,
                                      seed, C.byref(h)))
        self._h = h
        self.size = int(ids.size)
        self.n = program.num_qubits
        self._program = program
        self._engine = engine

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                load().ssb_batch_destroy(self._h)
            except Exception:
                pass
            self._h = C.c_void_p()

    def apply_op(self, op_index: int, u: Optional[Sequence[float]] = None) -> None:
        if u is None:
            check(load().ssb_batch_apply_op(self._h, op_index, None))
        else:
            arr = np.ascontiguousarray(u, dtype=np.float64)
            if arr.size != self.size:
                raise ValueError("need one draw per shot")
            check(load().ssb_batch_apply_op(self._h, op_index, arr.ctypes.data_as(_lib._pd)))

    def run(self) -> None:
        check(load().ssb_batch_run(self._h))

    def segments(self) -> np.ndarray:
        out = np.empty((self.size, 1 << self.n), dtype=np.complex128)
        check(load().ssb_batch_read(self._h, out.ctypes.data_as(_lib._pd), None))
        return out

    def cregs(self) -> np.ndarray:
        out = np.empty(self.size, dtype=np.uint64)
        check(load().ssb_batch_read(self._h, None, out.ctypes.data_as(_lib._pu64)))
        return out

    def write_segment(self, s: int, amps: np.ndarray) -> None:
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        check(load().ssb_batch_write_segment(self._h, s, a.ctypes.data_as(_lib._pd)))

    @property
    def dispatches(self) -> int:
        return int(load().ssb_batch_dispatches(self._h))


def executor_by_name(name: str):
    """``gpu-batch`` | ``gpu-branch`` -> fn(engine, program, options) (exec.hpp:32-35)."""
    if name == "gpu-batch":
        return lambda eng, prog, opts: eng.run_batch(prog, opts)
    if name == "gpu-branch":
        return lambda eng, prog, opts: eng.run_branch(prog, opts)
    raise _lib.ConfigError(_lib.SSB_ERR_CONFIG, f"unknown strategy: {name}")
