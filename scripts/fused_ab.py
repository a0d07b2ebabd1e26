"""A/B of the exact and fused-matrix batch executors on C2 / C5 (GPU probe,
not part of the product): shots/s from the engine's CUDA events, pass time,
guard flags; values compared between the two modes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
which = sys.argv[1:] or ["C2:16384", "C5:64"]
for item in which:
    parts = item.split(":")
    key, shots = parts[0], int(parts[1])
    tile = int(parts[2]) if len(parts) > 2 else 0
    cfg = cc.CONFIGS[key]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    out = {}
    for fused in (False, True):
        eng.run_batch(prog, RunOptions(shots=min(shots, 64), seed=1, fused_matrices=fused, tile_qubits=tile))
        r = eng.run_batch(prog, RunOptions(shots=shots, seed=1, fused_matrices=fused, profile=True,
                                           record_shot_values=True, tile_qubits=tile))
        out[fused] = np.asarray(r.shot_values)
        print(f"{key} tile={tile} fused={int(fused)} shots={shots} {shots / r.device_seconds:.1f} shots/s "
              f"device {r.device_seconds:.3f}s passes {r.fused_passes} blocks {r.fused_blocks} "
              f"flagged {r.guard_flagged} delta {r.guard_delta:.3g} launches {r.dispatch_count}", flush=True)
    print(key, "values equal:", bool((out[False] == out[True]).all()), flush=True)
