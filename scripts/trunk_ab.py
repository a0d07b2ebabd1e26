"""A/B of the shared noiseless trunk (SHOTSIM_B200_NO_TRUNK) in one process:
identical shot values required, device time compared. Not product code."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

work = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [["C2", 16384], ["C5", 16]]
e = Engine(0)
for key, shots in work:
    cfg = cc.CONFIGS[key]
    p = Program.from_text(cfg["circuit"](), cfg["noise"]())
    res = {}
    for mode in ("trunk", "plain", "trunk", "plain"):
        if mode == "plain":
            os.environ["SHOTSIM_B200_NO_TRUNK"] = "1"
        else:
            os.environ.pop("SHOTSIM_B200_NO_TRUNK", None)
        r = e.run_batch(p, RunOptions(shots=shots, seed=7, record_shot_values=True))
        prev = res.get(mode)
        best = max(prev[0], shots / r.device_seconds) if prev else shots / r.device_seconds
        res[mode] = (best, r._values.copy(), r.trunk_skipped, r.fused_passes)
    same = bool((res["trunk"][1] == res["plain"][1]).all())
    print(json.dumps({"config": key, "shots": shots, "identical": same,
                      "trunk_shots_per_s": round(res["trunk"][0], 1), "plain_shots_per_s": round(res["plain"][0], 1),
                      "speedup": round(res["trunk"][0] / res["plain"][0], 3),
                      "trunk_skipped": res["trunk"][2], "shot_passes": shots * res["trunk"][3]}), flush=True)
