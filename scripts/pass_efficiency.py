"""Per-pass FP64-pipe efficiency of a streamed run (diagnostics, not product
code): run under `ncu --metrics gpu__time_duration.sum --csv` with
SHOTSIM_B200_NO_TRUNK=1, then pass the CSV: python scripts/pass_efficiency.py
C2 2048 launches.csv [fp64_peak_ops]"""
import csv, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import dp_ops_per_op
from paper_2308_03399_b200 import Program, circuits as cc

key, shots, path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
peak = float(sys.argv[4]) if len(sys.argv) > 4 else 18.5e12
cfg = cc.CONFIGS[key]
prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
pm = prog.pass_map()
cost = np.array(dp_ops_per_op(prog), dtype=np.float64)
npass = int(pm.max()) + 1
dp = np.array([cost[pm == p].sum() for p in range(npass)])
nops = np.bincount(pm[pm >= 0], minlength=npass)
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
durs = [float(r[vi].replace(",", "")) for r in rows[1:] if "tile_pass" in r[ki]]
unit = [r for r in rows[1:] if "tile_pass" in r[ki]][0][hdr.index("Metric Unit")]
scale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}[unit]
durs = np.array(durs) * scale
print(f"{len(durs)} tile launches, {npass} passes per wave")
tot_t = tot_dp = 0.0
for i, t in enumerate(durs):
    p = i % npass
    eff = dp[p] * shots / t / peak if len(durs) == npass else float("nan")
    tot_t += t
    tot_dp += dp[p] * shots
    print(f"pass {p:3d} ops {nops[p]:4d} dp/shot {dp[p]:.3e} time {t*1e3:8.3f} ms  fp64 {eff:6.3f}")
print(f"total {tot_t*1e3:.1f} ms fp64 {tot_dp / tot_t / peak:.3f}")
