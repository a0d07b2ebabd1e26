"""In-process A/B of an engine environment switch (read at run time), e.g.
python scripts/env_ab.py SHOTSIM_B200_NO_TRUNK '[["C2",16384,"batch"]]'
Identical shot values required. Experiment driver, not product code."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

var = sys.argv[1]
work = json.loads(sys.argv[2])
e = Engine(0)
for key, shots, mode in work:
    cfg = cc.CONFIGS[key]
    p = Program.from_text(cfg["circuit"](), cfg["noise"]())
    run = e.run_branch if mode == "branch" else e.run_batch
    kw = dict(branch_budget=65536) if mode == "branch" else {}
    res = {}
    for on in (False, True, False, True):
        if on:
            os.environ[var] = "1"
        else:
            os.environ.pop(var, None)
        r = run(p, RunOptions(shots=shots, seed=3, record_shot_values=True, **kw))
        best = max(res.get(on, (0,))[0], shots / r.device_seconds)
        res[on] = (best, r._values.copy())
    print(json.dumps({"config": key, "mode": mode, "shots": shots, "identical": bool((res[True][1] == res[False][1]).all()),
                      "default": round(res[False][0], 2), var: round(res[True][0], 2),
                      "speedup_default": round(res[False][0] / res[True][0], 3)}), flush=True)
