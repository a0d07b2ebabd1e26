"""ctypes binding of the C ABI (include/shotsim_b200.h) — the same calls a
reference-side FFI would make. Loads the in-tree
``lib/libshotsim_b200.so``; there is no fallback: a missing library raises."""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("SHOTSIM_B200_LIB", "")) if os.environ.get("SHOTSIM_B200_LIB") else \
    Path(__file__).resolve().parent / "lib" / "libshotsim_b200.so"

SSB_OK = 0
SSB_ERR_RUNTIME = 1
SSB_ERR_INVALID_ARGUMENT = 2
SSB_ERR_CONFIG = 3
SSB_ERR_CAPACITY = 4
SSB_ERR_DEGENERATE = 5
SSB_ERR_CUDA = 6

OP_GATE, OP_PAULI, OP_KRAUS, OP_MEASURE, OP_RESET, OP_BARRIER = range(6)
MAX_OP_QUBITS = 4
MATRIX_STRIDE = 32


class FlatOp(C.Structure):
    _fields_ = [
        ("kind", C.c_uint32), ("num_qubits", C.c_uint32),
        ("qubits", C.c_uint32 * MAX_OP_QUBITS), ("clbits", C.c_uint32 * MAX_OP_QUBITS),
        ("has_condition", C.c_uint32), ("gate_kind", C.c_uint32),
        ("cond_mask", C.c_uint64), ("cond_value", C.c_uint64), ("event", C.c_uint64),
        ("matrix", C.c_uint32), ("channel", C.c_uint32),
        ("term_begin", C.c_uint32), ("term_count", C.c_uint32),
    ]


class FlatTerm(C.Structure):
    _fields_ = [
        ("cumulative", C.c_double), ("x_mask", C.c_uint64), ("z_mask", C.c_uint64),
        ("num_y", C.c_uint32), ("x_max", C.c_uint32), ("identity", C.c_uint32), ("reserved", C.c_uint32),
    ]


class FlatChannel(C.Structure):
    _fields_ = [("arity", C.c_uint32), ("num_matrices", C.c_uint32),
                ("matrix_begin", C.c_uint32), ("reserved", C.c_uint32)]


class FlatProgram(C.Structure):
    _fields_ = [
        ("num_qubits", C.c_uint32), ("num_clbits", C.c_uint32), ("num_events", C.c_uint64),
        ("has_measure", C.c_uint32), ("sampling_eligible", C.c_uint32),
        ("terminal_measure_begin", C.c_uint64),
        ("num_ops", C.c_uint64), ("ops", C.POINTER(FlatOp)),
        ("num_terms", C.c_uint64), ("terms", C.POINTER(FlatTerm)),
        ("num_channels", C.c_uint64), ("channels", C.POINTER(FlatChannel)),
        ("num_matrices", C.c_uint64), ("matrices", C.POINTER(C.c_double)),
        ("num_sample_qubits", C.c_uint32), ("sample_qubits", C.POINTER(C.c_uint32)),
        ("num_sample_writes", C.c_uint32), ("sample_write_clbit", C.POINTER(C.c_uint32)),
        ("sample_write_pos", C.POINTER(C.c_uint32)),
    ]


class RunOptionsC(C.Structure):
    _fields_ = [
        ("max_batch_size", C.c_uint64), ("branch_budget", C.c_uint64), ("mem_limit_bytes", C.c_uint64),
        ("check_norms", C.c_uint32), ("collect_leaf_stats", C.c_uint32),
        ("resident_max_qubits", C.c_uint32), ("tile_qubits", C.c_uint32),
        ("profile", C.c_uint32), ("interpret_only", C.c_uint32),
        # ABI 2
        ("fused_matrices", C.c_uint32), ("reserved0", C.c_uint32),
        ("leaf_shots", C.POINTER(C.c_uint64)), ("leaf_shots_capacity", C.c_uint64),
        ("states_out", C.POINTER(C.c_double)),
    ]


class StatsC(C.Structure):
    _fields_ = [
        ("dispatch_count", C.c_uint64), ("peak_states", C.c_uint64), ("passes", C.c_uint64),
        ("fused_passes", C.c_uint64), ("device_seconds", C.c_double), ("wall_seconds", C.c_double),
        ("pass_seconds", C.c_double), ("pass_launches", C.c_uint64), ("special_seconds", C.c_double),
        ("sample_seconds", C.c_double), ("specialised_shapes", C.c_uint64),
        ("sampling_serial_chunks", C.c_uint64),
        ("trunk_skipped", C.c_uint64),
        # ABI 2
        ("num_leaves", C.c_uint64), ("fused_blocks", C.c_uint64), ("guard_flagged", C.c_uint64),
        ("guard_delta", C.c_double),
    ]


class FusedInfoC(C.Structure):
    _fields_ = [("ok", C.c_uint32), ("passes", C.c_uint32), ("blocks", C.c_uint32), ("groups", C.c_uint32),
                ("max_pass_blocks", C.c_uint32), ("reserved", C.c_uint32), ("err_bound", C.c_double)]


_vp = C.c_void_p
_u64 = C.c_uint64
_pu64 = C.POINTER(C.c_uint64)
_pd = C.POINTER(C.c_double)

# name -> (restype, argtypes); every symbol declared in include/shotsim_b200.h.
SIGNATURES = {
    "ssb_last_error": (C.c_char_p, []),
    "ssb_abi_version": (C.c_int, []),
    "ssb_program_from_text": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(_vp)]),
    "ssb_program_from_flat": (C.c_int, [C.POINTER(FlatProgram), C.POINTER(_vp)]),
    "ssb_program_destroy": (None, [_vp]),
    "ssb_program_flat": (C.c_int, [_vp, C.POINTER(FlatProgram)]),
    "ssb_program_dump": (C.c_int, [_vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ssb_counts_checksum": (C.c_int, [_pu64, _u64, C.c_uint32, C.c_uint32, _pu64, _pu64]),
    "ssb_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ssb_engine_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "ssb_engine_destroy": (None, [_vp]),
    "ssb_engine_stream": (_vp, [_vp]),
    "ssb_run_batch": (C.c_int, [_vp, _vp, _u64, _u64, _u64, C.POINTER(RunOptionsC), _pu64, C.POINTER(StatsC)]),
    "ssb_run_batch_device": (C.c_int, [_vp, _vp, _u64, _u64, _u64, C.POINTER(RunOptionsC), _vp,
                                       C.POINTER(StatsC)]),
    "ssb_run_branch": (C.c_int, [_vp, _vp, _u64, _u64, _u64, C.POINTER(RunOptionsC), _pu64, C.POINTER(StatsC)]),
    "ssb_histogram_device": (C.c_int, [_vp, _vp, _u64, C.c_uint32, _vp]),
    "ssb_fp64_peak": (C.c_int, [_vp, _pd]),
    "ssb_exact_creg_distribution": (C.c_int, [_vp, _vp, _pu64, _pd, _u64, _pu64]),
    "ssb_exact_distribution": (C.c_int, [_vp, _vp, C.POINTER(C.c_uint32), C.c_uint32, _pd]),
    "ssb_tvd_vs_exact": (C.c_int, [_pu64, _u64, C.c_uint32, C.c_uint32, _pu64, _pd, _u64, _pd]),
    "ssb_program_specialise_check": (C.c_int, [_vp, C.c_uint32, C.POINTER(C.c_uint32)]),
    "ssb_program_fused_specialise_check": (C.c_int, [_vp, C.POINTER(C.c_uint32)]),
    "ssb_program_fused_info": (C.c_int, [_vp, C.c_uint32, C.POINTER(FusedInfoC)]),
    "ssb_program_pass_map": (C.c_int, [_vp, C.c_uint32, C.POINTER(C.c_uint32), _u64, C.POINTER(C.c_uint32)]),
    "ssb_batch_create": (C.c_int, [_vp, _vp, _pu64, _u64, _u64, C.POINTER(_vp)]),
    "ssb_batch_destroy": (None, [_vp]),
    "ssb_batch_apply_op": (C.c_int, [_vp, _u64, _pd]),
    "ssb_batch_run": (C.c_int, [_vp]),
    "ssb_batch_read": (C.c_int, [_vp, _pd, _pu64]),
    "ssb_batch_write_segment": (C.c_int, [_vp, _u64, _pd]),
    "ssb_batch_dispatches": (_u64, [_vp]),
}

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(shotsim_b200 has no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL | os.RTLD_NOW)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class ShotsimError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


class ConfigError(ShotsimError):
    pass


class CapacityError(ShotsimError):
    pass


class DegenerateDistribution(ShotsimError):
    pass


class CudaUnavailable(ShotsimError):
    pass


_ERRORS = {SSB_ERR_CONFIG: ConfigError, SSB_ERR_CAPACITY: CapacityError,
           SSB_ERR_DEGENERATE: DegenerateDistribution, SSB_ERR_CUDA: CudaUnavailable}


def check(rc: int) -> None:
    if rc == SSB_OK:
        return
    msg = load().ssb_last_error().decode(errors="replace")
    if rc == SSB_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise _ERRORS.get(rc, ShotsimError)(rc, msg)
