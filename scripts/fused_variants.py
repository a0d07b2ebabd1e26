"""Every build of the fused pass on C2 / C5 (GPU probe, not part of the
product): the default static FMA kernel and the opt-in variants selected by
environment knobs, each on a fresh Program (the plan caches its group size),
best of 3 from CUDA events, values compared with the default."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

VARIANTS = [
    ("fma (default)", {}, 0),
    ("fma 11-qubit tiles", {}, 11),
    ("octads (SHOTSIM_B200_FUSED_GROUP=3)", {"SHOTSIM_B200_FUSED_GROUP": "3"}, 0),
    ("double-buffered one CTA/SM (SHOTSIM_B200_FUSED_DB=1)", {"SHOTSIM_B200_FUSED_DB": "1"}, 0),
    ("FP64 tensor core (SHOTSIM_B200_FUSED_MMA=1)", {"SHOTSIM_B200_FUSED_MMA": "1"}, 0),
    ("per-pass NVRTC (SHOTSIM_B200_FUSED_JIT=1)", {"SHOTSIM_B200_FUSED_JIT": "1"}, 0),
]
KNOBS = {k for _, e, _ in VARIANTS for k in e}
eng = Engine(0)
for item in sys.argv[1:] or ["C2:32768", "C5:64"]:
    key, shots = item.split(":")[0], int(item.split(":")[1])
    cfg = cc.CONFIGS[key]
    ref = None
    for name, env, tile in VARIANTS:
        for k in KNOBS:
            os.environ.pop(k, None)
        os.environ.update(env)
        prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
        o = dict(seed=1, fused_matrices=True, tile_qubits=tile)
        eng.run_batch(prog, RunOptions(shots=min(shots, 64), **o))
        best, vals = 0.0, None
        for _ in range(3):
            r = eng.run_batch(prog, RunOptions(shots=shots, record_shot_values=True, profile=True, **o))
            best = max(best, shots / r.device_seconds)
            vals = np.asarray(r.shot_values)
        if ref is None:
            ref = vals
        print(f"{key} {name:55s} {best:10.1f} shots/s  passes {r.fused_passes:3d} flagged {r.guard_flagged} "
              f"values {'equal' if (vals == ref).all() else 'DIFFER'}", flush=True)
