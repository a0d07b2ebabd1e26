"""Bit-exact counts at the configs' own scale, against goldens the UNMODIFIED
reference produced with its scalar kernel table (tests/golden/make_scale_golden.py):

* C2 — all 1e5 shots of QV16 + depolarizing + readout (run_naive,
  exec_naive.cpp:131-161): every per-shot value, exact and fused-matrix modes;
* C3 — all 1e6 shots of dyn12 through shot-branching at budget 65536
  (run_branch, exec_branch.cpp:175-295): values hash, checksum, peak_states
  and passes, plus the batch executor's values hash;
* C4 — 64 shot ids of rnd20 + thermal Kraus; C5 — 8 shot ids of QV24
  (run_single_shot per id, exec_naive.cpp:88-129).
"""

import gzip
import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_2308_03399_b200 import Program, RunOptions, circuits as cc
from paper_2308_03399_b200.api import counts_checksum_of_values

pytestmark = pytest.mark.gpu


def sha(vals):
    return hashlib.sha256(np.ascontiguousarray(vals, dtype="<u8").tobytes()).hexdigest()


def prog_of(key, g):
    cfg = cc.CONFIGS[key]
    t, nz = cfg["circuit"](), cfg["noise"]()
    assert hashlib.sha256(t.encode()).hexdigest() == g["circuit_sha256"]
    assert hashlib.sha256(nz.encode()).hexdigest() == g["noise_sha256"]
    return Program.from_text(t, nz)


@pytest.mark.parametrize("mode", ["exact", "fused", "fused_jit"])
def test_c2_full_run(engine, monkeypatch, mode):
    fused = mode != "exact"
    if mode == "fused_jit":  # the per-pass run-time specialised fused kernels
        monkeypatch.setenv("SHOTSIM_B200_FUSED_JIT", "1")
    g = golden("scale_c2.json")
    want = np.frombuffer(gzip.decompress((GOLDEN / g["values_file"]).read_bytes()), dtype="<u2").astype(np.uint64)
    prog = prog_of("C2", g)
    r = engine.run_batch(prog, RunOptions(shots=g["shots"], seed=g["seed"], record_shot_values=True,
                                          fused_matrices=fused))
    got = np.asarray(r.shot_values)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"{bad.size} shots differ, first {bad[:5]}"
    assert sha(got) == g["values_sha256"]
    assert hex(counts_checksum_of_values(got, 16, True)[0]) == g["checksum"]
    if fused:
        assert r.fused_blocks > 0
    if mode == "fused_jit":
        assert r.specialised_shapes == r.fused_passes


def test_c3_full_branch_run(engine):
    g = golden("scale_c3.json")
    prog = prog_of("C3", g)
    r = engine.run_branch(prog, RunOptions(shots=g["shots"], seed=g["seed"], branch_budget=g["budget"],
                                           record_shot_values=True))
    got = np.asarray(r.shot_values)
    assert (r.branch.peak_states, r.branch.passes) == (g["peak_states"], g["passes"])
    assert hex(counts_checksum_of_values(got, 12, True)[0]) == g["checksum"]
    assert sha(got) == g["values_sha256"]
    b = engine.run_batch(prog, RunOptions(shots=g["shots"], seed=g["seed"], record_shot_values=True))
    assert sha(np.asarray(b.shot_values)) == g["values_sha256"]


@pytest.mark.parametrize("key,fused", [("C4", False), ("C5", False), ("C5", True)])
def test_large_config_shot_ids(engine, key, fused):
    """Reference values of sampled C4 / C5 shot ids; C5 also in fused-matrix
    mode (n >= 20: 11-qubit tiles by default, guard replays included)."""
    g = golden("scale_c45.json")[key]
    prog = prog_of(key, g)
    got = []
    ids = g["ids"]
    # contiguous runs of ids go through one call (several shots per wave)
    i = 0
    while i < len(ids):
        j = i
        while j + 1 < len(ids) and ids[j + 1] == ids[j] + 1:
            j += 1
        r = engine.run_batch(prog, RunOptions(shots=1, seed=g["seed"], record_shot_values=True, fused_matrices=fused),
                             shot_begin=ids[i], shot_count=j - i + 1)
        if fused:
            assert r.fused_blocks > 0
        got += [int(v) for v in r.shot_values]
        i = j + 1
    assert got == g["values"]
