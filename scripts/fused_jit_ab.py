"""A/B of the static fused_pass_kernel and the per-pass specialised kernels
(SHOTSIM_B200_FUSED_JIT=1, fused_jit.cpp) on C2 / C5 (GPU probe, not part of
the product): shots/s from the engine's CUDA events, values compared."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
which = sys.argv[1:] or ["C2:32768", "C5:64"]
for item in which:
    key, shots = item.split(":")[0], int(item.split(":")[1])
    cfg = cc.CONFIGS[key]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    out = {}
    for jit in ("0", "1", "0", "1"):
        os.environ["SHOTSIM_B200_FUSED_JIT"] = jit
        t0 = time.perf_counter()
        eng.run_batch(prog, RunOptions(shots=min(shots, 64), seed=1, fused_matrices=True))
        warm = time.perf_counter() - t0
        r = eng.run_batch(prog, RunOptions(shots=shots, seed=1, fused_matrices=True, profile=True,
                                           record_shot_values=True))
        v = np.asarray(r.shot_values)
        if jit in out:
            assert (out[jit] == v).all()
        out[jit] = v
        print(f"{key} jit={jit} shots={shots} {shots / r.device_seconds:.1f} shots/s device {r.device_seconds:.3f}s "
              f"pass {r.pass_seconds:.3f}s warm-up call {warm:.1f}s flagged {r.guard_flagged}", flush=True)
    print(key, "values equal:", bool((out["0"] == out["1"]).all()), flush=True)
