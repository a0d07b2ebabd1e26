import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.oracle import Oracle
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
eng, orc = Engine(0), Oracle()
cases = [(17, 3, 17, 32, 5), (17, 1, 17, 32, 5), (17, 3, 17, 8, 5), (17, 2, 17, 8, 5), (20, 2, 20, 4, 1)]
for n, depth, cseed, shots, seed in cases:
    prog = Program.from_text(cc.random_layers(n, depth=depth, seed=cseed), cc.thermal_noise(0.05, 0.1))
    want = orc.run_shots(prog, np.arange(shots), seed, threads=8)
    for off in ("1", "0"):
        os.environ["SHOTSIM_B200_EPILOGUE"] = "0" if off == "1" else "1"
        try:
            r = eng.run_batch(prog, RunOptions(shots=shots, seed=seed, record_shot_values=True))
            got = np.asarray(r.shot_values)
            print(n, depth, shots, "epi", off == "0", "match" if (got == want).all() else f"MISMATCH {np.flatnonzero(got != want)[:8]}", flush=True)
        except Exception as e:
            print(n, depth, shots, "epi", off == "0", "error", e, flush=True)
    pm = prog.pass_map()
    print("  passes", int(pm.max()) + 1, flush=True)
