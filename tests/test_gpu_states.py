"""Amplitude-level parity of every executor path against the reference's own
BatchState states (oracle/_ref, ref_batch_segments over exec_batch.cpp:200-227;
the state terminal sampling reads, or the final state when the program is not
sampling-eligible), exported through ssb_run_options::states_out:

* the SM-resident program kernel (n <= 13),
* the HBM tile passes — run-time shape-specialised and interpreter builds,
* the shot-branching executor (each shot's leaf state).

Exact paths must be bit-identical (np.array_equal; only the sign of an exact
zero may differ) and within north_star's 1e-10 relative bound; the fused-
matrix mode (4x4 block products, FMA) must be within 1e-10 relative.
"""

import numpy as np
import pytest

from paper_2308_03399_b200 import Program, RunOptions, circuits as cc

pytestmark = pytest.mark.gpu

IDS = 6


def programs(n):
    return {
        "qv_pauli": (cc.quantum_volume(n, depth=4, seed=n), cc.qv_noise()),
        "layers_kraus": (cc.random_layers(n, depth=3, seed=n), cc.thermal_noise(0.05, 0.1)),
        "dynamic": (cc.dynamic(n, rounds=2), cc.depolarizing_model(0.03)),
    }


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Reference
    return Reference()


def rel_err(got, want):
    return np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)


PATHS = {
    "resident": (lambda n: n <= 13, dict()),
    "tile_jit": (lambda n: True, dict(resident_max_qubits=1, tile_qubits=10)),
    "tile_interp": (lambda n: True, dict(resident_max_qubits=1, tile_qubits=10, interpret_only=True)),
    "tile_default": (lambda n: n > 13, dict()),
    "tile_db": (lambda n: n == 14, dict(resident_max_qubits=1, tile_qubits=11)),  # SHOTSIM_B200_TILE_DB=1
    "branch": (lambda n: True, None),
}


@pytest.mark.parametrize("n", [12, 14, 16])
@pytest.mark.parametrize("path", list(PATHS))
def test_states_equal_reference(engine, ref, monkeypatch, n, path):
    ok, kw = PATHS[path]
    if path == "tile_db":  # the double-buffered specialised tile pass (A/B knob)
        monkeypatch.setenv("SHOTSIM_B200_TILE_DB", "1")
    if not ok(n):
        pytest.skip("path not used at this size")
    for name, (circ, noise) in programs(n).items():
        if n == 16 and name != "qv_pauli" and path != "tile_default":
            continue  # keep the reference's CPU side short; the qv case covers every path at 16
        want, wregs, _ = ref.batch_segments(circ, noise, list(range(IDS)), 11, n)
        prog = Program.from_text(circ, noise)
        if kw is None:
            r = engine.run_branch(prog, RunOptions(shots=IDS, seed=11, branch_budget=64, export_states=True))
        else:
            r = engine.run_batch(prog, RunOptions(shots=IDS, seed=11, export_states=True, **kw))
        assert np.array_equal(r.states, want), (path, name, n, max(rel_err(g, w) for g, w in zip(r.states, want)))
        assert max(rel_err(g, w) for g, w in zip(r.states, want)) <= 1e-10


def fused_kernel_env(monkeypatch, kernel):
    """fma: the static FMA build (default); mma: the tensor-core build;
    jit: the per-pass run-time specialised FMA kernels (fused_jit.cpp)."""
    if kernel == "mma":
        monkeypatch.setenv("SHOTSIM_B200_FUSED_MMA", "1")
    elif kernel == "jit":
        monkeypatch.setenv("SHOTSIM_B200_FUSED_JIT", "1")


@pytest.mark.parametrize("kernel", ["fma", "mma", "jit"])
@pytest.mark.parametrize("n", [14, 16])
def test_fused_states_within_bound(engine, ref, monkeypatch, n, kernel):
    """fused_matrices: amplitudes within 1e-10 relative of the reference."""
    fused_kernel_env(monkeypatch, kernel)
    circ, noise = programs(n)["qv_pauli"]
    want, _, _ = ref.batch_segments(circ, noise, list(range(IDS)), 11, n)
    r = engine.run_batch(Program.from_text(circ, noise),
                         RunOptions(shots=IDS, seed=11, export_states=True, fused_matrices=True))
    assert r.fused_blocks > 0
    if kernel == "jit":
        assert r.specialised_shapes == r.fused_passes
    errs = [rel_err(g, w) for g, w in zip(r.states, want)]
    assert max(errs) <= 1e-10, errs


@pytest.mark.parametrize("kernel", ["fma", "mma", "jit"])
@pytest.mark.parametrize("scale", ["1", "1e5"])
def test_fused_counts_equal_exact(engine, oracle, monkeypatch, scale, kernel):
    """fused_matrices gives the exact executor's (= the reference's) per-shot
    values. With the guard band widened 1e5-fold (test hook) a large share of
    shots falls inside it and is replayed through the exact executor — the
    replay path must give the same values."""
    monkeypatch.setenv("SHOTSIM_B200_GUARD_SCALE", scale)
    fused_kernel_env(monkeypatch, kernel)
    prog = Program.from_text(cc.quantum_volume(14, depth=8, seed=3), cc.qv_noise())
    want = oracle.run_shots(prog, np.arange(400), 19, threads=8)
    r = engine.run_batch(prog, RunOptions(shots=400, seed=19, fused_matrices=True, record_shot_values=True))
    assert r.fused_blocks > 0
    if kernel == "jit":
        assert r.specialised_shapes == r.fused_passes
    assert (np.asarray(r.shot_values) == want).all()
    if scale != "1":
        assert 0 < r.guard_flagged < 400
    else:
        assert r.guard_flagged <= 2


@pytest.mark.parametrize("tile", [10, 11, 12])
def test_fused_tile_sizes_equal_exact(engine, oracle, tile):
    """Every fused tile size (64 / 128 / 256-thread CTAs, one hexad per
    thread) gives the reference's per-shot values."""
    prog = Program.from_text(cc.quantum_volume(14, depth=8, seed=3), cc.qv_noise())
    want = oracle.run_shots(prog, np.arange(300), 23, threads=8)
    r = engine.run_batch(prog, RunOptions(shots=300, seed=23, fused_matrices=True, tile_qubits=tile,
                                          record_shot_values=True))
    assert r.fused_blocks > 0
    assert (np.asarray(r.shot_values) == want).all()


def test_fused_plan_cache_across_program_objects(engine, oracle, monkeypatch):
    """Fused plans are cached by program content: lowering the same circuit
    again (the plugin path) reuses the plan, a changed circuit does not, and
    both give the reference's values."""
    circ, noise = cc.quantum_volume(14, depth=6, seed=8), cc.qv_noise()
    want = oracle.run_shots(Program.from_text(circ, noise), np.arange(200), 29, threads=8)
    for _ in range(2):
        r = engine.run_batch(Program.from_text(circ, noise),
                             RunOptions(shots=200, seed=29, fused_matrices=True, record_shot_values=True))
        assert (np.asarray(r.shot_values) == want).all()
    other = cc.quantum_volume(14, depth=6, seed=9)
    want2 = oracle.run_shots(Program.from_text(other, noise), np.arange(200), 29, threads=8)
    r = engine.run_batch(Program.from_text(other, noise),
                         RunOptions(shots=200, seed=29, fused_matrices=True, record_shot_values=True))
    assert (np.asarray(r.shot_values) == want2).all()
