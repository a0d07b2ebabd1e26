"""Wave size A/B for the fused C2 batch (GPU probe): shots per wave via
RunOptions.max_batch_size (default: 16 GiB of state = 16384 C2 shots)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
cfg = cc.CONFIGS["C2"]
prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
shots = 100000
for wave in (0, 8192, 32768, 50000, 0):
    eng.run_batch(prog, RunOptions(shots=2048, seed=1, fused_matrices=True))
    best = 0.0
    for _ in range(2):
        r = eng.run_batch(prog, RunOptions(shots=shots, seed=1, fused_matrices=True, max_batch_size=wave))
        best = max(best, shots / r.device_seconds)
    print(f"wave {wave or 'default'}: {best:.1f} shots/s", flush=True)
