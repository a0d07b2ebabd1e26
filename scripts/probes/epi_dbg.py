import os, sys
sys.path.insert(0, '/root/repo')
os.environ['SHOTSIM_B200_EPI_CHECK'] = '1'
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc
eng = Engine(0)
for n in (12, 14):
    prog = Program.from_text(cc.random_layers(n, depth=1, seed=n), cc.thermal_noise(0.05, 0.1))
    try:
        eng.run_batch(prog, RunOptions(shots=4, seed=3, resident_max_qubits=1))
    except Exception as e:
        print('error', e)
