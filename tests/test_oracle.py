"""CPU: pin the oracle (C restatement) to the reference's golden vectors and,
when it is present, to the reference library itself (oracle/_ref)."""

import numpy as np
import pytest

from conftest import golden
from paper_2308_03399_b200 import Program, circuits as cc
from paper_2308_03399_b200.api import counts_checksum_of_values


def test_philox_random123_kats(oracle):
    for e in golden("rng_kat.json")["philox"]:
        assert oracle.philox(e["ctr"], e["key"]) == e["out"]
    # The published Random123 answers.
    assert oracle.philox([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_uniform_matches_reference_values(oracle):
    for e in golden("rng_kat.json")["uniform"]:
        assert oracle.uniform(e["seed"], e["shot"], e["event"]) == float.fromhex(e["u"])
    assert oracle.uniform(7, 0, 0) == 0.95459712616869996


def test_c1_ghz10_golden(oracle):
    g = golden("c1_ghz10.json")
    prog = Program.from_text(g["circuit"], g["noise"])
    vals = oracle.run_shots(prog, np.arange(g["shots"]), g["seed"])
    assert [int(v) for v in vals] == g["values"]
    cs, keys = counts_checksum_of_values(vals, 10, True)
    assert hex(cs) == g["checksum"] == "0xf73b2d20b1338848"
    assert keys == g["num_keys"] == 33


def test_random_programs_naive_and_branch(oracle):
    for g in golden("random_programs.json"):
        prog = Program.from_text(g["circuit"], g["noise"])
        vals = oracle.run_shots(prog, np.arange(g["shots"]), g["seed"])
        assert [int(v) for v in vals] == g["values"]
        for budget, st in g["branch"].items():
            bv, peak, passes = oracle.run_branch(prog, g["shots"], g["seed"], int(budget))
            assert [int(v) for v in bv] == g["values"]
            assert (peak, passes) == (st["peak_states"], st["passes"])


def test_dyn12_branch_statistics(oracle):
    g = golden("dyn12_branch.json")
    prog = Program.from_text(g["circuit"], g["noise"])
    for budget in ("1", "64"):
        st = g["budgets"][budget]
        bv, peak, passes = oracle.run_branch(prog, g["shots"], g["seed"], int(budget))
        assert (peak, passes) == (st["peak_states"], st["passes"])
        cs, _ = counts_checksum_of_values(bv, 12, True)
        assert hex(cs) == st["checksum"]
    assert [int(v) for v in bv] == g["values"]


def test_config_samples_c2(oracle):
    s = golden("config_samples.json")["C2"]
    cfg = cc.CONFIGS["C2"]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    vals = oracle.run_shots(prog, s["ids"], s["seed"], threads=4)
    assert [int(v) for v in vals] == s["values"]


def test_oracle_against_reference_library(oracle):
    """When the reference is built here, compare directly on fresh programs."""
    from oracle.oracle import REF_SO, Reference
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built")
    ref = Reference()
    rng = cc.SplitMix64(2024)
    for rep in range(12):
        circ = cc.random_mixed(rng, max_qubits=5)
        noise = cc.depolarizing_model(0.1, as_kraus=bool(rep % 2))
        prog = Program.from_text(circ, noise)
        v = oracle.run_shots(prog, np.arange(64), 77 + rep)
        rv, _ = ref.run(circ, noise, "naive", 64, 77 + rep)
        assert (v == rv).all()
        a, _ = oracle.final_states(prog, [5], 77 + rep)
        ra, _ = ref.single_shot(circ, noise, 5, 77 + rep, prog.num_qubits)
        assert np.array_equal(a[0], ra)
