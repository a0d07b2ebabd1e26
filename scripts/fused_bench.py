"""Fused-matrix batch throughput on C2 / C5 for library A/B runs (GPU probe,
not part of the product; SHOTSIM_B200_LIB selects the build). Prints
shots/s from the engine's CUDA events, best of 3, and a values checksum."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
tag = os.environ.get("TAG", os.environ.get("SHOTSIM_B200_LIB", "default"))
for item in sys.argv[1:] or ["C2:32768", "C5:64"]:
    key, shots = item.split(":")[0], int(item.split(":")[1])
    cfg = cc.CONFIGS[key]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    eng.run_batch(prog, RunOptions(shots=min(shots, 64), seed=1, fused_matrices=True))
    best, h = 0.0, ""
    for _ in range(3):
        r = eng.run_batch(prog, RunOptions(shots=shots, seed=1, fused_matrices=True, profile=True,
                                           record_shot_values=True))
        best = max(best, shots / r.device_seconds)
        h = hashlib.sha256(np.asarray(r.shot_values).tobytes()).hexdigest()[:12]
    print(f"{tag} {key} shots={shots} best {best:.1f} shots/s pass {r.pass_seconds:.3f}s values {h}", flush=True)
