"""Exact density-matrix reference on the device.

Parity target: the reference's own exact_creg_distribution / exact_distribution
(proj/src/density.cpp:280-306), pinned as tests/golden/density_exact.json by
tests/golden/make_density_golden.py. Tolerance (floating point, SURVEY §8 /
north_star): |gpu - ref| <= 1e-10 * |ref| + 1e-15 per probability; keys exact.
The statistical gate is the reference's: executors within TVD 0.02 of the
exact distribution (acceptance_main.cpp:154-170, test_density.cpp:178-192).
"""

import numpy as np
import pytest

from conftest import golden

REL, ABS = 1e-10, 1e-15
CASES = golden("density_exact.json")["cases"]
ERRORS = golden("density_exact.json")["errors"]


def _by_name(name):
    return next(c for c in CASES if c["name"] == name)


# ---- CPU: fixture pins (reference known answers) and host arithmetic ------------
def test_fixture_known_answers():
    """test_density.cpp:106-172 examples, as recorded from the reference."""
    assert np.allclose(_by_name("qft3_noiseless")["marginal"], 0.125, rtol=1e-9)
    assert np.allclose(_by_name("h_flip")["marginal"], [0.5, 0.5], rtol=1e-12)
    assert np.allclose(_by_name("x_flip")["marginal"], [0.01, 0.99], rtol=1e-12)
    inter = _by_name("intermediate")
    assert inter["keys"] == [0b00, 0b11] and np.allclose(inter["probs"], [0.5, 0.5], rtol=1e-12)
    reset = _by_name("reset")
    assert reset["keys"] == [0] and abs(reset["probs"][0] - 1.0) < 1e-12
    for c in CASES:
        assert abs(sum(c["probs"]) - 1.0) < 1e-9, c["name"]


def test_fixture_matches_reference_library():
    """Re-derive a few fixtures from oracle/_ref (skipped where it is absent)."""
    from oracle.oracle import REF_SO, Reference
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built")
    ref = Reference()
    for name in ("qft3_depol", "dyn6_depol", "rnd5_thermal"):
        c = _by_name(name)
        keys, probs = ref.exact_creg_distribution(c["circuit"], c["noise"])
        assert [int(k) for k in keys] == c["keys"]
        assert [float(p) for p in probs] == c["probs"]


def test_tvd_host_arithmetic():
    """ssb_tvd_vs_exact (host half of the C ABI) = half the L1 distance."""
    from paper_2308_03399_b200 import tvd_vs_exact
    rng = np.random.default_rng(3)
    values = rng.integers(0, 8, size=5000).astype(np.uint64)
    exact = {0: 0.1, 1: 0.2, 2: 0.3, 5: 0.4, 9: 0.0}
    emp = np.bincount(values.astype(np.int64), minlength=10) / values.size
    want = 0.5 * sum(abs(emp[k] - exact.get(k, 0.0)) for k in range(10))
    assert abs(tvd_vs_exact(values, 4, True, exact) - want) < 1e-12
    assert tvd_vs_exact(np.array([], dtype=np.uint64), 4, True, {}) == 0.0


# ---- GPU: the device evolver against the reference --------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_exact_distribution_parity(engine, case):
    from paper_2308_03399_b200 import Program
    p = Program.from_text(case["circuit"], case["noise"])
    got = engine.exact_creg_distribution(p)
    assert sorted(got) == case["keys"]
    for k, want in zip(case["keys"], case["probs"]):
        assert abs(got[k] - want) <= REL * abs(want) + ABS, (case["name"], k, got[k], want)
    if "qubits" in case:
        m = engine.exact_distribution(p, case["qubits"])
        want = np.array(case["marginal"])
        assert np.all(np.abs(m - want) <= REL * np.abs(want) + ABS), case["name"]


@pytest.mark.gpu
@pytest.mark.parametrize("err", ERRORS, ids=[e["name"] for e in ERRORS])
def test_exact_distribution_errors(engine, err):
    from paper_2308_03399_b200 import CapacityError, Program
    p = Program.from_text(err["circuit"], err["noise"])
    exc = CapacityError if err["error"] == "CapacityError" else ValueError
    with pytest.raises(exc):
        engine.exact_creg_distribution(p)


@pytest.mark.gpu
def test_executors_within_tvd_of_exact(engine):
    """acceptance_main.cpp:154-170: qft 2..6 + depolarizing 1%, 50000 shots,
    seed 5, both GPU executors within TVD 0.02 of the exact distribution."""
    from paper_2308_03399_b200 import Program, RunOptions, tvd_vs_exact
    worst = 0.0
    for n in range(2, 7):
        c = _by_name("qft%d_depol" % n)
        p = Program.from_text(c["circuit"], c["noise"])
        exact = engine.exact_creg_distribution(p)
        f = p.flat()
        for run in (engine.run_batch, engine.run_branch):
            r = run(p, RunOptions(shots=50000, seed=5))
            worst = max(worst, tvd_vs_exact(r._values, f.num_clbits, bool(f.has_measure), exact))
    assert worst <= 0.02, worst


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ghz10_depol", "dyn6_depol", "rnd5_thermal", "qft4_depol_kraus", "qv8_readout",
                                  "rnd4_kraus18"])
def test_executors_match_exact_on_fixtures(engine, name):
    """The same statistical gate on the golden programs that exercise every op
    kind (Kraus channels, resets, conditions, intermediate measures, n = 10),
    with the exact distribution taken from the reference's fixture, 4e5 shots."""
    from paper_2308_03399_b200 import Program, RunOptions, tvd_vs_exact
    c = _by_name(name)
    p = Program.from_text(c["circuit"], c["noise"])
    exact = dict(zip(c["keys"], c["probs"]))
    f = p.flat()
    # QV is the batch path's workload; its 256-way noisy fan-out makes the
    # branch run slow without adding coverage, so it runs batch only.
    runs = (engine.run_batch,) if name == "qv8_readout" else (engine.run_batch, engine.run_branch)
    for run in runs:
        r = run(p, RunOptions(shots=400000, seed=9))
        assert tvd_vs_exact(r._values, f.num_clbits, bool(f.has_measure), exact) <= 0.02, (name, run.__name__)


@pytest.mark.gpu
def test_cpp_api(tmp_path):
    """The C++ drop-in (include/shotsim_b200.hpp): exact_creg_distribution,
    exact_distribution and tvd_vs_exact over Counts, compiled against the
    in-tree library like a reference-side caller would be."""
    import subprocess
    from conftest import ROOT
    exe = tmp_path / "density_api"
    lib = ROOT / "paper_2308_03399_b200" / "lib"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), str(ROOT / "tests" / "cpp" / "density_api.cpp"),
                    "-o", str(exe), "-L", str(lib), "-lshotsim_b200", f"-Wl,-rpath,{lib}"], check=True, timeout=300)
    c = _by_name("rnd5_thermal")
    (tmp_path / "c.txt").write_text(c["circuit"])
    (tmp_path / "n.json").write_text(c["noise"])
    out = subprocess.run([str(exe), str(tmp_path / "c.txt"), str(tmp_path / "n.json")], capture_output=True, text=True,
                         timeout=300, check=True).stdout.splitlines()
    rows = [l.split() for l in out if l[0].isdigit()]
    assert [int(k) for k, _ in rows] == c["keys"]
    for (_, p), want in zip(rows, c["probs"]):
        assert abs(float.fromhex(p) - want) <= REL * abs(want) + ABS
    marg = next(l for l in out if l.startswith("marginal0")).split()[1:]
    assert abs(sum(float.fromhex(x) for x in marg) - 1.0) < 1e-9
    assert float(next(l for l in out if l.startswith("tvd")).split()[1]) <= 0.02
    assert "capacity error" in out


@pytest.mark.gpu
def test_c_abi_argument_errors(engine):
    """C ABI contract of the checker: size query, capacity, bad qubits."""
    import ctypes as C
    from paper_2308_03399_b200 import CapacityError, Program, _lib
    c = _by_name("qft3_depol")
    p = Program.from_text(c["circuit"], c["noise"])
    lib = _lib.load()
    n = C.c_uint64()
    assert lib.ssb_exact_creg_distribution(engine.handle, p.handle, None, None, 0, C.byref(n)) == 0
    assert n.value == len(c["keys"])
    keys = (C.c_uint64 * 2)()
    probs = (C.c_double * 2)()
    rc = lib.ssb_exact_creg_distribution(engine.handle, p.handle, keys, probs, 2, C.byref(n))
    assert rc == _lib.SSB_ERR_CAPACITY
    with pytest.raises(ValueError):
        engine.exact_distribution(p, [5])
    big = Program.from_text(_by_name("ghz10_depol")["circuit"].replace("qubits 10", "qubits 11"), "")
    with pytest.raises(CapacityError):
        engine.exact_distribution(big, [0])
