"""Repeat the C3 branch run (1e6 shots, budget 65536) in one process: spread."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
e = Engine(0)
cfg = cc.CONFIGS["C3"]
p = Program.from_text(cfg["circuit"](), cfg["noise"]())
shots = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
for rep in range(5):
    r = e.run_branch(p, RunOptions(shots=shots, seed=1, branch_budget=65536))
    print("rep", rep, "device_s %.3f" % r.device_seconds, "shots/s %.0f" % (shots / r.device_seconds), flush=True)
