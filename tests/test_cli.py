"""CLI drop-in for the reference's `run` / `validate` subcommands
(shotsim_main.cpp:38-67, 97-139): options, output format and exit codes."""
import subprocess

import pytest

from conftest import ROOT, golden
from paper_2308_03399_b200.api import counts_from_values

CLI = ROOT / "paper_2308_03399_b200" / "lib" / "shotsim_b200"


def cli(*args):
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=300)


@pytest.fixture(scope="module")
def c1_files(tmp_path_factory):
    g = golden("c1_ghz10.json")
    d = tmp_path_factory.mktemp("cli")
    (d / "c.txt").write_text(g["circuit"])
    (d / "n.json").write_text(g["noise"])
    return g, d / "c.txt", d / "n.json"


def test_validate(tmp_path, c1_files):
    r = cli("validate", "--circuit", c1_files[1])
    assert r.returncode == 0 and r.stdout == "ok\n"
    bad = tmp_path / "bad.txt"
    bad.write_text("qubits 2\nclbits 1\ncx q0,q0\nmeasure q1 -> c3\n")
    r = cli("validate", "--circuit", bad)
    assert r.returncode == 1 and r.stdout.startswith("instruction ")


def test_config_errors(c1_files):
    assert cli("run", "--circuit", c1_files[1], "--strategy", "naive").returncode == 3  # not a GPU executor
    assert cli("run", "--circuit", c1_files[1], "--shots", "-4").returncode == 3
    assert cli("run").returncode == 3  # --circuit is required
    assert cli("bench").returncode == 3
    assert cli("run", "--circuit", "/nonexistent.txt").returncode == 3


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["gpu-batch", "gpu-branch"])
def test_run_c1_counts(c1_files, strategy):
    g, circ, noise = c1_files
    r = cli("run", "--circuit", circ, "--noise-model", noise, "--strategy", strategy, "--shots", g["shots"],
            "--seed", g["seed"])
    assert r.returncode == 0, r.stderr
    got = {k: int(v) for k, v in (line.split() for line in r.stdout.splitlines())}
    want = counts_from_values(g["values"], 10, True)
    assert got == want
    assert list(got) == sorted(got)  # std::map order
    assert r.stderr.startswith(f"strategy={strategy} shots={g['shots']} seed={g['seed']} seconds=")
    assert ("dispatches=" in r.stderr) == (strategy == "gpu-batch")
    assert ("peak_states=" in r.stderr) == (strategy == "gpu-branch")
