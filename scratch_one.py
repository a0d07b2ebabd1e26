import sys, json
sys.path.insert(0, '.')
from paper_2308_03399_b200 import Engine, Program, RunOptions
eng = Engine(0)
g = json.load(open('tests/golden/random_programs.json'))[0]
prog = Program.from_text(g["circuit"], g["noise"])
if sys.argv[1] == "streamed":
    r = eng.run_batch(prog, RunOptions(shots=4, seed=g["seed"], resident_max_qubits=1, tile_qubits=3))
else:
    r = eng.run_branch(prog, RunOptions(shots=4, seed=g["seed"], branch_budget=3))
print(list(r._values), g["values"][:4])
