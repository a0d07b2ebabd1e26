"""Tuning sweep of the specialised tile kernel (SHOTSIM_B200_JIT_QPT/_MINB): C2
throughput and parity of the first 24 shots. Experiment driver, not product."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys; sys.path.insert(0, %r)
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
e = Engine(0)
cfg = cc.CONFIGS[%r]
p = Program.from_text(cfg["circuit"](), cfg["noise"]())
g = json.load(open(%r))[%r]
ok = [int(x) for x in e.run_batch(p, RunOptions(shots=len(g["values"]), seed=1), shot_begin=0)._values] == g["values"] if g["ids"] == list(range(len(g["ids"]))) else None
best = 0
for _ in range(2):
    r = e.run_batch(p, RunOptions(shots=%d, seed=1, tile_qubits=%d))
    best = max(best, %d / r.device_seconds)
print("shots/s %%.1f parity %%s shapes %%d passes %%d" %% (best, ok, r.specialised_shapes, r.fused_passes), flush=True)
'''
cfgkey = sys.argv[2] if len(sys.argv) > 2 else "C2"
shots = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
for combo in sys.argv[1].split(","):
    qpt, minb, tile = (combo.split("x") + ["12"])[:3]
    env = dict(os.environ, SHOTSIM_B200_JIT_QPT=qpt, SHOTSIM_B200_JIT_MINB=minb)
    print("== qpt", qpt, "minb", minb, "tile", tile, flush=True)
    subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfgkey, ROOT + "/tests/golden/config_samples.json", cfgkey,
                                                   shots, int(tile), shots)], env=env)
