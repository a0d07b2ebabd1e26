"""The C++ executor registry (include/shotsim_b200.hpp, csrc/host/executors.cpp)
compiled like a reference-side caller: workers keeps the reference's meaning
(a hint; shard g runs on device g % count, results identical for any value,
exec.hpp:24-27), engines persist across calls, and gpu-branch fills
BranchStats::leaf_shots (exec_branch.cpp:280)."""
import subprocess

import pytest

from conftest import ROOT
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

pytestmark = pytest.mark.gpu


def test_workers_invariance_and_leaf_stats(tmp_path):
    exe = tmp_path / "executors_workers"
    lib = ROOT / "paper_2308_03399_b200" / "lib"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "executors_workers.cpp"), "-o", str(exe), "-L", str(lib),
                    "-lshotsim_b200", f"-Wl,-rpath,{lib}"], check=True, timeout=300)
    (tmp_path / "c.txt").write_text(cc.dynamic(8, rounds=2))
    (tmp_path / "n.json").write_text(cc.depolarizing_model(0.02))
    r = subprocess.run([str(exe), str(tmp_path / "c.txt"), str(tmp_path / "n.json")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [l.split() for l in r.stdout.splitlines() if l.startswith("gpu-")]
    assert len(rows) == 6
    assert len({row[2] for row in rows}) == 1  # one checksum over strategies and worker counts
    for row in rows:
        if row[0] == "gpu-branch":
            assert int(row[7]) >= 1 and int(row[8]) == 2000  # leaves cover every shot
        else:
            assert int(row[7]) == 0


def test_leaf_shots_match_reference_shape(engine):
    """test_exec_branch.cpp:126-160: a noiseless program is one leaf holding
    every shot; budget 1 on a measuring program gives several passes whose
    leaves still add up to the shots."""
    r = engine.run_branch(Program.from_text(cc.ghz(5)), RunOptions(shots=4000, seed=1, collect_leaf_stats=True))
    assert r.branch.leaf_shots == [4000] and r.branch.passes == 1
    prog = Program.from_text("qubits 1\nclbits 1\nh q0\nmeasure q0 -> c0\nx q0 if 1==1\nmeasure q0 -> c0\n")
    r = engine.run_branch(prog, RunOptions(shots=1000, seed=2, branch_budget=1, collect_leaf_stats=True))
    assert r.branch.passes == 2 and sum(r.branch.leaf_shots) == 1000 and len(r.branch.leaf_shots) == 2
