"""Times C2 on experiment builds (SHOTSIM_B200_LIB=<variant .so>): not product code."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys; sys.path.insert(0, %r)
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
e = Engine(0)
for key, shots, tile in %s:
    cfg = cc.CONFIGS[key]
    p = Program.from_text(cfg["circuit"](), cfg["noise"]())
    e.run_batch(p, RunOptions(shots=64, seed=1, tile_qubits=tile))
    best = 0
    for _ in range(2):
        r = e.run_batch(p, RunOptions(shots=shots, seed=1, tile_qubits=tile))
        best = max(best, shots / r.device_seconds)
    import json
    g = json.load(open(%r + "/tests/golden/config_samples.json")).get(key)
    ok = None
    if g and tile == 12:
        ok = [int(x) for x in e.run_batch(p, RunOptions(shots=24, seed=1))._values] == g["values"][:24]
    print(key, "parity", ok, "tile", tile, "shots", shots, "shots/s %%.1f" %% best, "passes", r.fused_passes, flush=True)
'''
work = sys.argv[2] if len(sys.argv) > 2 else '[("C2", 4096, 12), ("C2", 4096, 13), ("C5", 16, 12)]'
for v in sys.argv[1].split(","):
    env = dict(os.environ)
    if v != "main":
        env["SHOTSIM_B200_LIB"] = os.path.join(ROOT, "variants", v, "libshotsim_b200.so")
    print("== variant", v, flush=True)
    subprocess.run([sys.executable, "-c", CHILD % (ROOT, work, ROOT)], env=env)
