"""Per-config throughput report on one B200 (all five BASELINE.json configs):
shots/s (device time through the C ABI), the unfused-HBM algorithmic roofline
fraction and, for streamed configs, the FP64-pipe fraction
against the live-measured peak. Writes JSON lines to stdout.

  python scripts/config_report.py [C1,C2,...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (algorithmic_bytes, dp_ops_per_shot, measured_peak)
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc  # noqa: E402
from paper_2308_03399_b200.api import _fp64_peak  # noqa: E402

RUNS = {  # config -> (executor, shots per timed run, options)
    "C1": ("batch", 100_000, {}),
    "C2": ("batch", 16_384, {}),
    "C3": ("branch", 1_000_000, {"branch_budget": 65_536}),
    "C4": ("batch", 1_024, {}),
    "C5": ("batch", 64, {}),
}


def main():
    keys = sys.argv[1].split(",") if len(sys.argv) > 1 else list(RUNS)
    eng = Engine(0)
    hbm, _ = bench.measured_peak()
    dp_peak = _fp64_peak(eng)
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "config_samples.json")))
    for key in keys:
        mode, shots, extra = RUNS[key]
        cfg = cc.CONFIGS[key]
        prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
        run = eng.run_branch if mode == "branch" else eng.run_batch
        # Warm-up at the timed size (specialisation compile, engine buffers and
        # the branch slot pool reach their steady-state sizes), as bench.py does.
        run(prog, RunOptions(shots=shots, seed=1, **extra))
        t0 = time.perf_counter()
        r = run(prog, RunOptions(shots=shots, seed=1, **extra))
        wall = time.perf_counter() - t0
        rate = shots / r.device_seconds
        _, alg = bench.algorithmic_bytes(prog)
        line = {"config": key, "workload": cfg["name"], "executor": "gpu-" + mode, "shots": shots,
                "shots_per_s": rate, "wall_s": wall, "device_s": r.device_seconds,
                "alg_bytes_per_shot": alg, "hbm_alg_frac": rate * alg / (hbm * 1e9),
                "launches": r.dispatch_count, "fused_passes": r.fused_passes,
                "specialised_shapes": r.specialised_shapes}
        if mode == "branch":
            line.update(peak_states=r.branch.peak_states, passes=r.branch.passes)
        if prog.num_qubits > 13:
            dp = bench.dp_ops_per_shot(prog)
            # executed work only: (shot, pass) pairs the shared trunk covered are not run
            executed = 1.0 - r.trunk_skipped / max(1, shots * r.fused_passes)
            line.update(dp_ops_per_shot=dp, fp64_frac_whole_run=rate * dp * executed / dp_peak, fp64_peak=dp_peak,
                        trunk_skipped_frac=1.0 - executed)
        g = golden.get(key)
        if g:
            got = [int(run(prog, RunOptions(shots=1, seed=1, **extra), shot_begin=i, shot_count=1)._values[0])
                   for i in g["ids"][:4]]
            line["parity_sample"] = got == g["values"][:4]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
