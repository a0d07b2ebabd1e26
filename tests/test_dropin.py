"""The reference's own code drives the GPU executors (integration/exec_gpu.cpp
registered in executor_by_name, built from the unmodified reference sources by
oracle/Makefile `dropin`): run_bench's cross-strategy checksum gate over
{naive, batch, branch, gpu-batch, gpu-branch} (bench.cpp:171-187) and the
acceptance equivalence criterion (acceptance_main.cpp:79-118) over the GPU
executors."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
EXE = ROOT / "oracle" / "_ref" / "shotsim_dropin"


@pytest.mark.skipif(not EXE.exists(), reason="built here by __graft_entry__.build() (needs the reference sources)")
def test_reference_harness_drives_gpu_executors(tmp_path):
    r = subprocess.run([str(EXE), str(tmp_path / "bench.csv")], capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.splitlines()
    assert "bench pauli exit 0" in lines and "bench kraus exit 0" in lines
    eq = next(l for l in lines if l.startswith("equiv"))
    assert eq.endswith(" 0 mismatches") and int(eq.split()[1]) == 480
    rows = (tmp_path / "bench.csv").read_text().splitlines()
    assert any(",gpu-branch," in row for row in rows) and any(",gpu-batch," in row for row in rows)
