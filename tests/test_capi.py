"""CPU: the C-ABI library loads, exports every symbol include/shotsim_b200.h
declares, and fails loudly (no CPU fallback) when no CUDA device exists."""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2308_03399_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "shotsim_b200.h"


def declared_symbols():
    return sorted(set(re.findall(r"SSB_API\s+[\w\s\*]+?\b(ssb_\w+)\s*\(", HEADER.read_text())))


def test_header_symbols_exported():
    lib = C.CDLL(str(_lib.LIB_PATH))
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "python binding out of sync with the header"


def test_abi_version():
    assert _lib.load().ssb_abi_version() == 2


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2308_03399_b200 import CudaUnavailable, Engine
    with pytest.raises(CudaUnavailable):
        Engine(0)


def test_flat_program_roundtrip():
    from paper_2308_03399_b200 import Program, circuits as cc
    p = Program.from_text(cc.quantum_volume(6, depth=3), cc.qv_noise())
    flat = p.flat()
    h = C.c_void_p()
    _lib.check(_lib.load().ssb_program_from_flat(C.byref(flat), C.byref(h)))
    q = Program(h.value)
    assert q.dump() == p.dump()


@pytest.mark.parametrize("key,tile", [("C2", 12), ("C4", 12), ("C5", 12), ("C2", 11)])
def test_shape_specialisation_compiles_without_gpu(key, tile):
    """The run-time specialiser's generated source (shape executors + the
    engine's embedded device headers) compiles with NVRTC for sm_100a."""
    from paper_2308_03399_b200 import Program, circuits as cc
    cfg = cc.CONFIGS[key]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    assert prog.specialise_check(tile) > 0


@pytest.mark.parametrize("key", ["C2", "C5"])
def test_fused_specialisation_compiles_without_gpu(key):
    """The per-pass specialised fused-matrix kernels (constant-bank block
    products, straight-line groups) compile with NVRTC for sm_100a."""
    from paper_2308_03399_b200 import Program, circuits as cc
    cfg = cc.CONFIGS[key]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    info = prog.fused_info(11)  # fused mode's default tile
    assert prog.fused_specialise_check() == info["passes"]


@pytest.mark.gpu
def test_integration_stub_runs_verbatim():
    """INTEGRATION.md §2's ctypes stub is executed as written (scripts/stub_check.py)."""
    import subprocess
    import sys
    from conftest import ROOT
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "stub_check.py")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "stub ok" in r.stdout, r.stderr[-2000:]
