import sys, json
sys.path.insert(0, '.')
import numpy as np
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
eng = Engine(0)
progs = json.load(open('tests/golden/random_programs.json'))
which = sys.argv[1]
for i, g in enumerate(progs):
    prog = Program.from_text(g["circuit"], g["noise"])
    try:
        if which == "streamed":
            r = eng.run_batch(prog, RunOptions(shots=g["shots"], seed=g["seed"], resident_max_qubits=1, tile_qubits=3))
        else:
            r = eng.run_branch(prog, RunOptions(shots=g["shots"], seed=g["seed"], branch_budget=int(which)))
        ok = [int(v) for v in r._values] == g["values"]
        print(i, "ok" if ok else "MISMATCH", prog.num_qubits, flush=True)
        if not ok:
            print(g["circuit"], g["noise"]); print(list(r._values[:20])); print(g["values"][:20])
    except Exception as e:
        print(i, "ERR", e, prog.num_qubits); print(g["circuit"], g["noise"]); break
