"""Probe: tile-pass epilogue (next Kraus site's matrix-0 partials) vs the
oracle, 1q-only and 2q-only thermal channels, streamed executor."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.oracle import Oracle
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
eng, orc = Engine(0), Oracle()
rules = json.loads(cc.thermal_noise(0.05, 0.1))["rules"]
for name, rr in (("1q", [rules[0]]), ("2q", [rules[1]]), ("mixed", rules)):
    noise = json.dumps({"rules": rr})
    for n in (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "12,14").split(",")):
        prog = Program.from_text(cc.random_layers(n, depth=1, seed=n), noise)
        want = orc.run_shots(prog, np.arange(8), 3, threads=8)
        for off in ("1", "0", "interp"):
            os.environ["SHOTSIM_B200_EPILOGUE"] = "1" if off in ("0", "interp") else "0"
            try:
                r = eng.run_batch(prog, RunOptions(shots=8, seed=3, resident_max_qubits=1, record_shot_values=True,
                                                   interpret_only=off == "interp"))
                ok = (np.asarray(r.shot_values) == want).all()
                print(name, n, "epilogue", {"1": "off", "0": "on", "interp": "on-interp"}[off], "match" if ok else "MISMATCH", flush=True)
            except Exception as e:
                print(name, n, "epilogue", {"1": "off", "0": "on", "interp": "on-interp"}[off], "error", e, flush=True)
