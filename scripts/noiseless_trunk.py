"""Noiseless QV16 (C2 circuit without noise), 16384 shots: shared trunk on / off. Experiment driver."""
import os, sys, time
sys.path.insert(0, "/root/repo")
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
e = Engine(0)
p = Program.from_text(cc.CONFIGS["C2"]["circuit"](), "")
for mode in ("trunk", "plain", "trunk", "plain"):
    if mode == "plain": os.environ["SHOTSIM_B200_NO_TRUNK"] = "1"
    else: os.environ.pop("SHOTSIM_B200_NO_TRUNK", None)
    r = e.run_batch(p, RunOptions(shots=16384, seed=1))
    print("noiseless QV16", mode, round(16384 / r.device_seconds, 1), "shots/s", r.trunk_skipped)
