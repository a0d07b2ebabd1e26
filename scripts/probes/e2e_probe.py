"""e2e path timing breakdown (GPU probe): per step, host lowering, the
run_batch call's wall time and its device time, for C2 at 1e5 shots."""
import sys
import time

sys.path.insert(0, '.')
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc

eng = Engine(0)
cfg = cc.CONFIGS['C2']
ct, nz = cfg['circuit'](), cfg['noise']()
shots = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
p0 = Program.from_text(ct, nz)
eng.run_batch(p0, RunOptions(shots=shots, seed=1, fused_matrices=True))
import gc
for i in range(8):
    t0 = time.perf_counter()
    p = Program.from_text(ct, nz)
    t1 = time.perf_counter()
    r = eng.run_batch(p, RunOptions(shots=shots, seed=1, fused_matrices=True))
    t2 = time.perf_counter()
    del p
    t3 = time.perf_counter()
    n = gc.collect()
    t4 = time.perf_counter()
    print(f"step {i}: from_text {1e3 * (t1 - t0):.1f} ms  run_batch wall {1e3 * (t2 - t1):.1f} ms  "
          f"device {1e3 * r.device_seconds:.1f} ms  destroy {1e3 * (t3 - t2):.1f} ms  gc {1e3 * (t4 - t3):.1f} ms ({n})",
          flush=True)
