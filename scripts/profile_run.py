"""Profiling driver (ncu target): one batch of a config through the C ABI."""
import sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
key = sys.argv[1] if len(sys.argv) > 1 else "C2"
shots = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
cfg = cc.CONFIGS[key]
eng = Engine(0)
prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
mode = sys.argv[3] if len(sys.argv) > 3 else "batch"
if mode == "batch":
    r = eng.run_batch(prog, RunOptions(shots=shots, seed=1))
elif mode == "fused":
    r = eng.run_batch(prog, RunOptions(shots=shots, seed=1, fused_matrices=True))
else:  # branch:<budget>
    r = eng.run_branch(prog, RunOptions(shots=shots, seed=1, branch_budget=int(mode.split(":")[1])))
print(key, shots, "shots", r.device_seconds, "s", shots / r.device_seconds, "shots/s")
