"""C4 (rnd20 thermal Kraus, exact streamed batch) at several tile sizes and
with the tile-pass knobs (GPU probe): shots/s from CUDA events, pass / Kraus
split, values compared with the default."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
cfg = cc.CONFIGS["C4"]
shots = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ref = None
for tile in (12, 11, 13, 10):
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    eng.run_batch(prog, RunOptions(shots=8, seed=1, tile_qubits=tile))
    r = eng.run_batch(prog, RunOptions(shots=shots, seed=1, tile_qubits=tile, profile=True, record_shot_values=True))
    v = np.asarray(r.shot_values)
    ref = v if ref is None else ref
    print(f"C4 tile {tile}: {shots / r.device_seconds:.1f} shots/s pass {r.pass_seconds:.3f}s special "
          f"{r.special_seconds:.3f}s passes {r.fused_passes} values {'equal' if (v == ref).all() else 'DIFFER'}",
          flush=True)
