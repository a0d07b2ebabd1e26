"""C1 resident cost breakdown (GPU probe): shots/s of the resident batch
executor on GHZ10 variants — measure only, + H, + CX chain, + noise — to see
where the per-shot time goes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
N = 10


def circ(h, cx, measure=True):
    c = cc.CircuitText(N)
    if h:
        c.op("h", [0])
    for i in range(1, cx + 1):
        c.op("cx", [i - 1, i])
    if measure:
        c.measure_all()
    return c.text()


cases = [("measure only", circ(0, 0), ""), ("H", circ(1, 0), ""), ("GHZ", circ(1, 9), ""),
         ("GHZ no measure", circ(1, 9, False), ""), ("GHZ+depol", circ(1, 9), cc.depolarizing_model(0.01)),
         ("H+depol", circ(1, 0), cc.depolarizing_model(0.01)), ("H x9 (u)", None, "")]
hx = cc.CircuitText(N)
for q in range(N - 1):
    hx.op("h", [q])
hx.measure_all()
cases[-1] = ("H x9", hx.text(), "")
shots = 1_000_000
for name, c, nz in cases:
    prog = Program.from_text(c, nz)
    eng.run_batch(prog, RunOptions(shots=4096, seed=1))
    r = eng.run_batch(prog, RunOptions(shots=shots, seed=1, profile=True))
    print(f"{name:16s} {shots / r.device_seconds / 1e6:7.2f} M shots/s  {r.device_seconds * 1e3:7.2f} ms", flush=True)
