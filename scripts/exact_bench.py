"""Exact-mode throughput on the configs for library A/B runs (GPU probe, not
part of the product; SHOTSIM_B200_LIB selects the build): C1 resident batch,
C2 / C5 exact streamed batch, C3 branch; best of 3 from CUDA events plus a
values checksum."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
tag = os.environ.get("TAG", "tree")
for item in sys.argv[1:] or ["C1:1000000", "C2:16384", "C3:1000000:branch", "C5:32"]:
    parts = item.split(":")
    key, shots = parts[0], int(parts[1])
    branch = len(parts) > 2 and parts[2] == "branch"
    cfg = cc.CONFIGS[key]
    prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
    run = (lambda o: eng.run_branch(prog, o)) if branch else (lambda o: eng.run_batch(prog, o))
    kw = {"branch_budget": 65536} if branch else {}
    run(RunOptions(shots=min(shots, 64), seed=1, **kw))
    best, h = 0.0, ""
    for _ in range(3):
        r = run(RunOptions(shots=shots, seed=1, record_shot_values=True, **kw))
        best = max(best, shots / r.device_seconds)
        h = hashlib.sha256(np.asarray(r.shot_values).tobytes()).hexdigest()[:12]
    print(f"{tag} {key}{' branch' if branch else ''} shots={shots} best {best:.1f} shots/s values {h}", flush=True)
