"""shotsim_b200 — B200-native multi-shot statevector engine (batch-shots +
shot-branching, arXiv:2308.03399) behind the reference shotsim run API.

The product is the C++/CUDA library ``lib/libshotsim_b200.so`` (C ABI in
``include/shotsim_b200.h``); this package is its thin Python host mirror.
"""

from ._lib import (CapacityError, ConfigError, CudaUnavailable, DegenerateDistribution, LIB_PATH,
                   ShotsimError)
from .api import (BatchState, Engine, Program, RunOptions, RunResult, bitstring, counts_checksum_of_values,
                  counts_from_values, executor_by_name, tvd_vs_exact)

__all__ = [
    "BatchState", "Engine", "Program", "RunOptions", "RunResult", "bitstring", "counts_from_values",
    "counts_checksum_of_values", "executor_by_name", "tvd_vs_exact", "CapacityError", "ConfigError", "CudaUnavailable",
    "DegenerateDistribution", "ShotsimError", "LIB_PATH",
]
