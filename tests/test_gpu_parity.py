"""GPU parity: the sm_100a engine (through the C ABI) against the oracle and
the reference's golden fixtures. Integer results (per-shot register values,
counts, branch statistics) must be bit-exact; amplitudes must equal the
reference's exactly up to the sign of zero (numpy == treats -0.0 == 0.0),
which is stronger than north_star's 1e-10 relative bound (also asserted)."""

import numpy as np
import pytest

from conftest import golden
from paper_2308_03399_b200 import BatchState, CapacityError, Program, RunOptions, circuits as cc
from paper_2308_03399_b200.api import counts_checksum_of_values

pytestmark = pytest.mark.gpu

STREAMED = dict(resident_max_qubits=1, tile_qubits=3)   # force the HBM tile-pass path at tiny n


def values(res):
    return np.asarray(res._values)


def test_c1_ghz10_resident_and_branch(engine):
    g = golden("c1_ghz10.json")
    prog = Program.from_text(g["circuit"], g["noise"])
    for run in (engine.run_batch, engine.run_branch):
        r = run(prog, RunOptions(shots=1000, seed=1, record_shot_values=True))
        assert [int(v) for v in values(r)] == g["values"]
        cs, keys = counts_checksum_of_values(values(r), 10, True)
        assert hex(cs) == "0xf73b2d20b1338848" and keys == 33


def test_c1_streamed_path(engine):
    g = golden("c1_ghz10.json")
    prog = Program.from_text(g["circuit"], g["noise"])
    r = engine.run_batch(prog, RunOptions(shots=1000, seed=1, tile_qubits=6, resident_max_qubits=1))
    assert [int(v) for v in values(r)] == g["values"]


@pytest.mark.parametrize("mode", ["resident", "streamed", "branch1", "branch3", "branch64"])
def test_random_mixed_programs(engine, mode):
    for g in golden("random_programs.json"):
        prog = Program.from_text(g["circuit"], g["noise"])
        opts = RunOptions(shots=g["shots"], seed=g["seed"])
        if mode == "resident":
            r = engine.run_batch(prog, opts)
        elif mode == "streamed":
            r = engine.run_batch(prog, RunOptions(shots=g["shots"], seed=g["seed"], **STREAMED))
        else:
            budget = int(mode[len("branch"):])
            opts.branch_budget = budget
            r = engine.run_branch(prog, opts)
            st = g["branch"][str(budget)]
            assert (r.branch.peak_states, r.branch.passes) == (st["peak_states"], st["passes"])
        assert [int(v) for v in values(r)] == g["values"], g["circuit"]


def test_more_random_programs_vs_oracle(engine, oracle):
    rng = cc.SplitMix64(31337)
    for rep in range(40):
        circ = cc.random_mixed(rng, max_qubits=6)
        noise = cc.depolarizing_model(0.1, as_kraus=bool(rep % 2))
        prog = Program.from_text(circ, noise)
        want = oracle.run_shots(prog, np.arange(128), rep)
        for kw in ({}, STREAMED):
            r = engine.run_batch(prog, RunOptions(shots=128, seed=rep, **kw))
            assert (values(r) == want).all(), (circ, noise, kw)
        r = engine.run_branch(prog, RunOptions(shots=128, seed=rep, branch_budget=1 + rep % 5))
        assert (values(r) == want).all()


@pytest.mark.parametrize("n,tile", [(6, 3), (8, 5), (10, 10), (12, 11), (12, 12)])
def test_kraus_thermal_all_paths(engine, oracle, n, tile):
    """Kraus sites through the resident kernel, the streamed passes (decide
    step between passes, apply as the next pass's first micro-op) and the
    branch executor."""
    prog = Program.from_text(cc.random_layers(n, depth=4, seed=n), cc.thermal_noise(0.05, 0.1))
    want = oracle.run_shots(prog, np.arange(200), 3)
    for kw in ({}, dict(resident_max_qubits=1, tile_qubits=tile)):
        assert (values(engine.run_batch(prog, RunOptions(shots=200, seed=3, **kw))) == want).all()
    assert (values(engine.run_branch(prog, RunOptions(shots=200, seed=3, branch_budget=16))) == want).all()


@pytest.mark.parametrize("interpret_only", [False, True])
@pytest.mark.parametrize("tile", [11, 12])
def test_streamed_shapes_random_bursts(engine, oracle, tile, interpret_only):
    """Every gate kind, relabelings, conditionals and Pauli / Kraus noise through
    the HBM tile passes at tile sizes where the run-time shape-specialised
    kernel is used (and, interpret_only, the interpreter kernel)."""
    rng = cc.SplitMix64(4242 + tile)
    for rep in range(6):
        circ = cc.random_bursts(rng, n=12 + rep % 2)
        noise = cc.depolarizing_model(0.02 + 0.03 * (rep % 3), as_kraus=rep == 5)
        prog = Program.from_text(circ, noise)
        want = oracle.run_shots(prog, np.arange(96), 77 + rep, threads=8)
        r = engine.run_batch(prog, RunOptions(shots=96, seed=77 + rep, resident_max_qubits=1, tile_qubits=tile,
                                              interpret_only=interpret_only))
        assert (values(r) == want).all(), (rep, circ, noise)
        assert (r.specialised_shapes > 0) == (not interpret_only)


def test_qv14_streamed_default_tiles(engine, oracle):
    prog = Program.from_text(cc.quantum_volume(14, depth=6, seed=5), cc.qv_noise())
    want = oracle.run_shots(prog, np.arange(48), 9, threads=8)
    r = engine.run_batch(prog, RunOptions(shots=48, seed=9))
    assert (values(r) == want).all()
    assert r.fused_passes > 0


def test_c2_qv16_reference_sample(engine):
    s = golden("config_samples.json")["C2"]
    cfg = cc.CONFIGS["C2"]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    r = engine.run_batch(prog, RunOptions(shots=24, seed=1))
    assert [int(v) for v in values(r)] == s["values"][:24]
    assert r.specialised_shapes > 0
    r = engine.run_batch(prog, RunOptions(shots=24, seed=1, interpret_only=True))
    assert [int(v) for v in values(r)] == s["values"][:24] and r.specialised_shapes == 0
    r = engine.run_batch(prog, RunOptions(shots=1, seed=1), shot_begin=99_999, shot_count=1)
    assert int(values(r)[0]) == s["values"][24]


def test_c4_rnd20_reference_sample(engine):
    s = golden("config_samples.json")["C4"]
    cfg = cc.CONFIGS["C4"]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    got = []
    for sid in s["ids"]:
        got.append(int(values(engine.run_batch(prog, RunOptions(shots=1, seed=1), shot_begin=sid, shot_count=1))[0]))
    assert got == s["values"]


def test_c5_qv24_reference_sample(engine):
    s = golden("config_samples.json")["C5"]
    cfg = cc.CONFIGS["C5"]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    got = [int(values(engine.run_batch(prog, RunOptions(shots=1, seed=1), shot_begin=sid, shot_count=1))[0])
           for sid in s["ids"]]
    assert got == s["values"]


def test_dyn12_branch_statistics(engine):
    g = golden("dyn12_branch.json")
    prog = Program.from_text(g["circuit"], g["noise"])
    for budget, st in g["budgets"].items():
        r = engine.run_branch(prog, RunOptions(shots=g["shots"], seed=g["seed"], branch_budget=int(budget)))
        assert (r.branch.peak_states, r.branch.passes) == (st["peak_states"], st["passes"])
        assert hex(counts_checksum_of_values(values(r), 12, True)[0]) == st["checksum"]
    assert [int(v) for v in values(r)] == g["values"]
    b = engine.run_batch(prog, RunOptions(shots=g["shots"], seed=g["seed"]))
    assert [int(v) for v in values(b)] == g["values"]


def test_segments_equal_reference_states(engine, oracle):
    """BatchState op-at-a-time kernels vs reference final states (exact)."""
    rng = cc.SplitMix64(7)
    for rep in range(10):
        circ = cc.random_mixed(rng, max_qubits=5)
        prog = Program.from_text(circ, cc.depolarizing_model(0.1, as_kraus=bool(rep % 2)))
        ids = list(range(8 + rep))
        want, wregs = oracle.final_states(prog, ids, 1000 + rep)
        b = BatchState(engine, prog, ids, 1000 + rep)
        b.run()
        got = b.segments()
        assert np.array_equal(got, want)
        assert np.allclose(got, want, rtol=1e-10, atol=0)
        assert (b.cregs() == wregs).all()


def test_explicit_draws_pauli_site(engine):
    """test_exec_batch.cpp:62-87: per-shot branch selection with explicit u."""
    noise = '{"rules":[{"gates":["id"],"arity":1,"channel":{"type":"pauli","terms":[[0.99,"I"],[0.01,"X"]]}}]}'
    prog = Program.from_text("qubits 1\nclbits 0\nid q0\n", noise)
    b = BatchState(engine, prog, [0, 1], 0)
    b.apply_op(1, [0.5, 0.995])
    seg = b.segments()
    assert seg[0][0] == 1 and seg[1][1] == 1
    assert b.dispatches == 1
    idle = BatchState(engine, prog, [0, 1, 2], 0)
    idle.apply_op(1, [0.1, 0.2, 0.98])
    assert idle.dispatches == 0


def test_explicit_draws_amplitude_damping(engine):
    """test_exec_naive.cpp:112-149 via the batched Kraus op."""
    r = 0.5 ** 0.5
    noise = ('{"rules":[{"gates":["x"],"arity":1,"channel":{"type":"kraus","matrices":[[[1,0],[0,0],[0,0],[%r,0]],'
             '[[0,0],[%r,0],[0,0],[0,0]]]}}]}' % (r, r))
    prog = Program.from_text("qubits 1\nclbits 0\nx q0\n", noise)
    b = BatchState(engine, prog, [0, 1], 0)
    b.apply_op(0)
    b.apply_op(1, [0.25, 0.75])
    seg = b.segments()
    assert abs(seg[0][1] - 1) < 1e-12 and abs(seg[1][0] - 1) < 1e-12


def test_dispatch_count_independent_of_shots(engine):
    """test_exec_batch.cpp:178-187: QFT(4) + sampling = 13 logical dispatches."""
    prog = Program.from_text(cc.qft(4))
    for s in (1, 1024):
        b = BatchState(engine, prog, list(range(s)), 9)
        b.run()
        assert b.dispatches == 13


def test_perturbed_segment_does_not_leak(engine):
    prog = Program.from_text(cc.qft(3), cc.depolarizing_model(0.2))
    clean = BatchState(engine, prog, list(range(6)), 5)
    dirty = BatchState(engine, prog, list(range(6)), 5)
    seg = dirty.segments()[2].copy()
    seg[1] += 0.4 - 0.2j
    dirty.write_segment(2, seg)
    clean.run()
    dirty.run()
    a, b = clean.segments(), dirty.segments()
    for s in range(6):
        if s != 2:
            assert np.array_equal(a[s], b[s])


def test_capacity_error(engine):
    prog = Program.from_text(cc.quantum_volume(14, depth=1))
    with pytest.raises(CapacityError):
        engine.run_batch(prog, RunOptions(shots=64, seed=1, max_batch_size=64, mem_limit_bytes=1 << 20))


def test_shard_concatenation(engine, oracle):
    """Shots shard by id range: any split reproduces the single run."""
    prog = Program.from_text(cc.quantum_volume(8, depth=4), cc.qv_noise())
    whole = values(engine.run_batch(prog, RunOptions(shots=1000, seed=4)))
    parts = [values(engine.run_batch(prog, RunOptions(shots=1, seed=4), shot_begin=b, shot_count=c))
             for b, c in ((0, 300), (300, 1), (301, 699))]
    assert (np.concatenate(parts) == whole).all()
    assert (oracle.run_shots(prog, np.arange(1000), 4) == whole).all()


def test_exact_parallel_sampling_paths(engine, oracle, monkeypatch):
    """Terminal sampling over all qubits: the chunked exact-advance sampler and
    its sequential replay path (forced for every chunk) both give the
    reference's outcomes (statevector.cpp:185-197), at 12 and 14 qubits."""
    for n, depth in ((12, 3), (14, 2)):
        prog = Program.from_text(cc.quantum_volume(n, depth=depth, seed=8), cc.qv_noise())
        want = oracle.run_shots(prog, np.arange(64), 5, threads=8)
        r = engine.run_batch(prog, RunOptions(shots=64, seed=5, resident_max_qubits=1))
        assert (values(r) == want).all()
        if n == 14:  # 8 chunks per shot: some advance exactly in parallel
            assert r.sampling_serial_chunks < 64 * 8
        monkeypatch.setenv("SHOTSIM_B200_SAMPLE_SERIAL", "1")
        r = engine.run_batch(prog, RunOptions(shots=64, seed=5, resident_max_qubits=1))
        assert (values(r) == want).all()
        monkeypatch.delenv("SHOTSIM_B200_SAMPLE_SERIAL")


@pytest.mark.parametrize("n,tile,wave", [(8, 3, 0), (12, 10, 37), (14, 12, 0)])
def test_shared_trunk(engine, oracle, monkeypatch, n, tile, wave):
    """Shared noiseless trunk: shots run no pass before their first
    non-identity Pauli draw and copy the trunk state in then. Same values as
    the oracle and as the plain streamed run, across waves (max_batch_size)."""
    prog = Program.from_text(cc.quantum_volume(n, depth=5, seed=n), cc.depolarizing_model(0.004))
    shots = 160
    want = oracle.run_shots(prog, np.arange(shots), 21, threads=8)
    kw = dict(shots=shots, seed=21, resident_max_qubits=1, tile_qubits=tile, max_batch_size=wave)
    r = engine.run_batch(prog, RunOptions(**kw))
    assert (values(r) == want).all()
    assert 0 < r.trunk_skipped < shots * r.fused_passes
    monkeypatch.setenv("SHOTSIM_B200_NO_TRUNK", "1")
    r2 = engine.run_batch(prog, RunOptions(**kw))
    assert (values(r2) == want).all() and r2.trunk_skipped == 0


def test_shared_trunk_noiseless(engine, oracle, monkeypatch):
    """Without noise every shot's state is the trunk's: the passes run once per
    wave and only terminal sampling is per shot."""
    prog = Program.from_text(cc.quantum_volume(14, depth=4, seed=3), "")
    want = oracle.run_shots(prog, np.arange(200), 8, threads=8)
    r = engine.run_batch(prog, RunOptions(shots=200, seed=8))
    assert (values(r) == want).all()
    assert r.fused_passes > 0 and r.trunk_skipped == 200 * r.fused_passes
    monkeypatch.setenv("SHOTSIM_B200_NO_TRUNK", "1")
    assert (values(engine.run_batch(prog, RunOptions(shots=200, seed=8))) == want).all()


@pytest.mark.parametrize("direct", [False, True])
def test_kraus_probabilities_large_states(engine, oracle, monkeypatch, direct):
    """1q / 2q Kraus probabilities at n = 17: the shared-memory staged
    reductions (coalesced LDGSTS) and the direct per-thread kernels give the
    reference's blocked sums, hence the same choices."""
    if direct:
        monkeypatch.setenv("SHOTSIM_B200_EXPVAL1_DIRECT", "1")
        monkeypatch.setenv("SHOTSIM_B200_EXPVAL2_DIRECT", "1")
    prog = Program.from_text(cc.random_layers(17, depth=3, seed=17), cc.thermal_noise(0.05, 0.1))
    want = oracle.run_shots(prog, np.arange(32), 5, threads=8)
    assert (values(engine.run_batch(prog, RunOptions(shots=32, seed=5))) == want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("n,tile", [(6, 3), (8, 5)])
def test_kraus_long_channel_all_paths(engine, oracle, n, tile):
    """A 2q Kraus channel of 18 matrices (thermal tensor product, every matrix
    split in halves; tests/golden/make_density_golden.py): longer than any
    built-in channel, bit-exact on every path."""
    import json
    rules = json.loads(cc.thermal_noise(0.05, 0.1))["rules"]
    h = 0.5 ** 0.5
    rules[1]["channel"]["matrices"] = [[[h * x, h * y] for x, y in m] for m in rules[1]["channel"]["matrices"]
                                       for _ in (0, 1)]
    prog = Program.from_text(cc.random_layers(n, depth=4, seed=n), json.dumps({"rules": rules}))
    want = oracle.run_shots(prog, np.arange(200), 3)
    for kw in ({}, dict(resident_max_qubits=1, tile_qubits=tile)):
        assert (values(engine.run_batch(prog, RunOptions(shots=200, seed=3, **kw))) == want).all()
    assert (values(engine.run_branch(prog, RunOptions(shots=200, seed=3, branch_budget=16))) == want).all()


@pytest.mark.parametrize("epilogue", ["0", "1"])
def test_kraus_epilogue_parity(engine, oracle, monkeypatch, epilogue):
    """The opt-in tile-pass epilogue (the next Kraus site's matrix-0 partials
    from the preceding pass, exact sequential block sums) gives the
    reference's values for 1q and 2q channels, with several tiles per CTA."""
    monkeypatch.setenv("SHOTSIM_B200_EPILOGUE", epilogue)
    prog = Program.from_text(cc.random_layers(17, depth=2, seed=17), cc.thermal_noise(0.05, 0.1))
    want = oracle.run_shots(prog, np.arange(32), 5, threads=8)
    assert (values(engine.run_batch(prog, RunOptions(shots=32, seed=5))) == want).all()
