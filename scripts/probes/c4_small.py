import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
eng = Engine(0)
cfg = cc.CONFIGS["C4"]
prog = Program.from_text(cc.random_layers(20, depth=1, seed=2020), cfg["noise"]())
r = eng.run_batch(prog, RunOptions(shots=int(sys.argv[1]) if len(sys.argv) > 1 else 64, seed=1, profile=True))
print("shots/s", r.shots / r.device_seconds, "pass", r.pass_seconds, "shapes", r.specialised_shapes, flush=True)
