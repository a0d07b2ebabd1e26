"""C4 A/B (GPU probe): exact streamed executor with and without the tile-pass
epilogue that computes the next Kraus site's matrix-0 partials
(SHOTSIM_B200_NO_EPILOGUE=1 disables it); values compared."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
shots = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = cc.CONFIGS["C4"]
prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
out = {}
for off in ("1", "0"):
    os.environ["SHOTSIM_B200_EPILOGUE"] = "0" if off == "1" else "1"
    eng.run_batch(prog, RunOptions(shots=8, seed=1))
    r = eng.run_batch(prog, RunOptions(shots=shots, seed=1, profile=True, record_shot_values=True))
    out[off] = np.asarray(r.shot_values)
    print(f"C4 epilogue={'off' if off == '1' else 'on'} {shots / r.device_seconds:.1f} shots/s pass {r.pass_seconds:.3f}s "
          f"special {r.special_seconds:.3f}s launches {r.dispatch_count}", flush=True)
print("values equal:", bool((out["0"] == out["1"]).all()))
