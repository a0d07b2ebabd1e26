"""CPU checks of bench.py's roofline model: the unfused
reference op-stream bytes and the engine's executed FP64 op count."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2308_03399_b200 import Program, circuits as cc  # noqa: E402


def test_c2_algorithmic_bytes_match_survey():
    cfg = cc.CONFIGS["C2"]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    _, total = bench.algorithmic_bytes(prog)
    assert abs(total - 3.011e9) / 3.011e9 < 1e-3          # 3.011e9 B/shot


def test_c2_fp64_ops_per_shot():
    """1024 U gates x 24 rounded ops per amplitude pair x 2^15 pairs; CX and
    identity gates are free (register relabelings / skipped)."""
    cfg = cc.CONFIGS["C2"]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    assert bench.dp_ops_per_shot(prog) == 1024 * 24 * (1 << 15)


def test_entry_costs():
    assert bench._entry_cost(0.0, 0.0) == (0, False)
    assert bench._entry_cost(1.0, 0.0) == (0, True)
    assert bench._entry_cost(-1.0, 0.0) == (0, True)
    assert bench._entry_cost(0.5, 0.0) == (2, True)
    assert bench._entry_cost(0.0, 0.5) == (2, True)
    assert bench._entry_cost(0.5, 0.5) == (6, True)
