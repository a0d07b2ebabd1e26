"""Branch-mode sharding cost (GPU probe): C3 (dyn12, budget 65536) as one
run_branch over 1e6 shots vs the same shots in K contiguous chunks run back to
back on one GPU. sum(chunk times) / single time is the redundant subtree work
a K-way shot split (static or balanced) pays."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
cfg = cc.CONFIGS["C3"]
prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
shots, budget = 1_000_000, 65536
eng.run_branch(prog, RunOptions(shots=4096, seed=1, branch_budget=budget))
for _ in range(2):  # the second run is timed (the first sizes the engine's buffers)
    one = eng.run_branch(prog, RunOptions(shots=shots, seed=1, branch_budget=budget, record_shot_values=True))
ref = np.asarray(one.shot_values)
print(f"K=1 device {one.device_seconds:.3f}s peak {one.branch.peak_states} passes {one.branch.passes}", flush=True)
for K in (2, 4, 8):
    tot, vals, peaks, passes = 0.0, [], [], []
    for i in range(K):
        b, n = shots * i // K, shots * (i + 1) // K - shots * i // K
        r = eng.run_branch(prog, RunOptions(shots=n, seed=1, branch_budget=budget, record_shot_values=True),
                           shot_begin=b)
        tot += r.device_seconds
        vals.append(np.asarray(r.shot_values))
        peaks.append(r.branch.peak_states)
        passes.append(r.branch.passes)
    same = bool((np.concatenate(vals) == ref).all())
    print(f"K={K} sum {tot:.3f}s max-chunk {tot / K:.3f}s(avg) redundancy {tot / one.device_seconds:.2f} "
          f"ideal-{K}gpu speedup {one.device_seconds / (tot / K):.2f} peaks {peaks[:2]} passes {passes[:2]} "
          f"values equal {same}", flush=True)
