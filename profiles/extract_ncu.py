"""Summarise one `ncu --set full` capture (first profiled launch) into JSON.

usage: python profiles/extract_ncu.py <report.ncu-rep> <config-key> <shots-in-launch> [alg-bytes-per-shot]
Reads the report with `ncu -i ... --page raw --csv` (needs ncu on PATH)."""
import csv
import io
import json
import subprocess
import sys

rep, key, shots = sys.argv[1], sys.argv[2], int(sys.argv[3])
alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
units = dict(zip(rows[0], rows[1]))


def f(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


def bytes_of(k):
    v, u = f(k), units.get(k, "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return None if v is None else v * scale


dur_ms = f("gpu__time_duration.sum")
dur_scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(units.get("gpu__time_duration.sum"), 1.0)
dram = (bytes_of("dram__bytes_read.sum") or 0) + (bytes_of("dram__bytes_write.sum") or 0)
out = {
    "kernel": d.get("Kernel Name", "").split("(")[0],
    "shots_in_launch": shots,
    "duration_ms": dur_ms * dur_scale if dur_ms is not None else None,
    "dram_bytes_per_launch": dram,
    "dram_bytes_per_shot": dram / shots if shots else None,
    "fp64_pipe_active_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": f("sm__inst_executed.sum.pct_of_peak_sustained_elapsed"),
    "alu_pipe_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "lsu_pipe_pct": f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "registers_per_thread": f("launch__registers_per_thread"),
    "achieved_occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "shared_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "smem_wavefronts_pct": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "tensor_pipe_pct": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "grid": f("launch__grid_size"),
    "block": f("launch__block_size"),
}
if alg:
    out["algorithmic_bytes_per_launch"] = alg * shots
    out["traffic_over_algorithmic"] = dram / (alg * shots)
stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(k)
          for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
out["stalls_per_issue"] = {k: v for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0)) if v and v > 0.05}
print(json.dumps({key: out}, indent=1))
