import sys; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
e = Engine(0)
cfg = cc.CONFIGS["C3"]; p = Program.from_text(cfg["circuit"](), cfg["noise"]())
for rep in range(4):
    r = e.run_batch(p, RunOptions(shots=100000, seed=1))
    print("C3 batch rep", rep, 100000 / r.device_seconds, flush=True)
cfg = cc.CONFIGS["C1"]; p = Program.from_text(cfg["circuit"](), cfg["noise"]())
for rep in range(3):
    r = e.run_batch(p, RunOptions(shots=100000, seed=1))
    print("C1 batch rep", rep, 100000 / r.device_seconds, flush=True)
