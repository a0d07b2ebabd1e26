bash scripts/lib_ab.sh base tree base tree 2>&1 | tail -8
for t in 10 11 12; do
python - <<PY
import os,sys
sys.path.insert(0,'.')
import numpy as np
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
eng=Engine(0)
for key,shots in (("C2",32768),("C5",64)):
    cfg=cc.CONFIGS[key]; prog=Program.from_text(cfg["circuit"](), cfg["noise"]())
    eng.run_batch(prog, RunOptions(shots=64, seed=1, fused_matrices=True, tile_qubits=$t))
    best=0
    for _ in range(3):
        r=eng.run_batch(prog, RunOptions(shots=shots, seed=1, fused_matrices=True, tile_qubits=$t, profile=True))
        best=max(best, shots/r.device_seconds)
    print(key, "tile $t", round(best,1), "passes", r.fused_passes, flush=True)
PY
done
