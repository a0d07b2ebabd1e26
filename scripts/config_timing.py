# quick GPU timing probe (not part of the product)
import sys, time
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
eng = Engine(0)
for key, shots in (("C1", 100000), ("C3", 100000), ("C2", 2048), ("C4", 256), ("C5", 16)):
    cfg = cc.CONFIGS[key]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    eng.run_batch(prog, RunOptions(shots=min(shots, 8), seed=1))
    r = eng.run_batch(prog, RunOptions(shots=shots, seed=1))
    print(key, "batch", shots, "shots", r.device_seconds, "s", shots / r.device_seconds, "shots/s", "launches", r.dispatch_count, "passes", r.fused_passes, "shapes", r.specialised_shapes, flush=True)
cfg = cc.CONFIGS["C3"]
prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
for b in (64, 65536):
    r = eng.run_branch(prog, RunOptions(shots=100000, seed=1, branch_budget=b))
    print("C3 branch", b, r.device_seconds, 100000 / r.device_seconds, "peak", r.branch.peak_states, "passes", r.branch.passes, flush=True)
