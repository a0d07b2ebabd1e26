"""Per-config throughput report on one B200 (all five BASELINE.json configs),
each line with the SM clocks sampled DURING its timed run (bench.ClockSampler:
median under load, max, throttle reasons).

* shots/s from the engine's CUDA events (device time through the C ABI);
* streamed configs (C2, C4, C5): the dominant kernel's FP64-pipe and HBM
  fractions over the pass time, exact and fused-matrix executors;
* SM-resident configs (C1, C3): SURVEY §8(d)'s SM roofline
  min(smem 37.2 TB/s / alg bytes, FP64 37.2 TFLOP/s / alg FLOPs) per shot;
* a parity sample against the reference goldens.

  python scripts/config_report.py [C1,C2,...] > profiles/r02_configs.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (algorithmic_bytes, dp_ops_per_shot, measured_peak, ClockSampler)
from paper_2308_03399_b200 import Engine, Program, RunOptions, circuits as cc  # noqa: E402
from paper_2308_03399_b200.api import _fp64_peak  # noqa: E402

# config -> [(label, executor, shots per timed run, options)]
RUNS = {
    "C1": [("resident", "batch", 1_000_000, {}), ("branch", "branch", 1_000_000, {"branch_budget": 64})],
    "C2": [("fused", "batch", 100_000, {"fused_matrices": True}), ("exact", "batch", 16_384, {})],
    "C3": [("branch", "branch", 1_000_000, {"branch_budget": 65_536}), ("resident", "batch", 1_000_000, {})],
    "C4": [("exact", "batch", 1_024, {})],
    "C5": [("fused", "batch", 64, {"fused_matrices": True}), ("exact", "batch", 64, {})],
}
SMEM_BW = 148 * 128 * 1.965e9   # B/s: 128 B/clk/SM at the max SM clock
FP64_FLOPS = 148 * 64 * 2 * 1.965e9


def alg_flops(prog):
    """14 FLOP/amplitude per dense 1q gate, 30 per dense 2q gate."""
    f = prog.flat()
    A = 1 << f.num_qubits
    end = f.terminal_measure_begin if f.sampling_eligible else f.num_ops
    return sum((14 if f.ops[i].num_qubits == 1 else 30) * A for i in range(end) if f.ops[i].kind == 0)


def main():
    keys = sys.argv[1].split(",") if len(sys.argv) > 1 else list(RUNS)
    eng = Engine(0)
    hbm, _ = bench.measured_peak()
    dp_peak = _fp64_peak(eng)
    samples = json.load(open(os.path.join(ROOT, "tests", "golden", "config_samples.json")))
    for key in keys:
        cfg = cc.CONFIGS[key]
        prog = Program.from_text(cfg["circuit"](), cfg["noise"]())
        for label, mode, shots, extra in RUNS[key]:
            run = eng.run_branch if mode == "branch" else eng.run_batch
            run(prog, RunOptions(shots=shots, seed=1, **extra))  # warm-up at the timed size
            with bench.ClockSampler(0) as clocks:
                t0 = time.perf_counter()
                r = run(prog, RunOptions(shots=shots, seed=1, profile=True, **extra))
                wall = time.perf_counter() - t0
            rate = shots / r.device_seconds
            _, alg = bench.algorithmic_bytes(prog)
            line = {"config": key, "workload": cfg["name"], "executor": f"gpu-{mode} ({label})", "shots": shots,
                    "shots_per_s": rate, "wall_s": wall, "device_s": r.device_seconds,
                    "pass_s": r.pass_seconds, "sample_s": r.sample_seconds, "special_s": r.special_seconds,
                    "alg_bytes_per_shot": alg, "launches": r.dispatch_count, "clocks": clocks.summary()}
            A = 1 << prog.num_qubits
            if prog.num_qubits <= 13:
                fl = alg_flops(prog)
                sm_roof = min(SMEM_BW / alg, FP64_FLOPS / fl)
                line.update(sm_roofline_shots_s=sm_roof, sm_roofline_frac=rate / sm_roof, alg_flops_per_shot=fl)
            else:
                line["hbm_alg_frac_unfused"] = rate * alg / (hbm * 1e9)
                if r.fused_blocks:
                    dp = 16.0 * A * r.fused_blocks
                    by = 32.0 * A * r.fused_passes
                else:
                    dp = bench.dp_ops_per_shot(prog) * (1.0 - r.trunk_skipped / max(1, shots * r.fused_passes))
                    by = 32.0 * A * r.fused_passes
                line.update(dp_ops_per_shot=dp, fp64_frac_whole_run=rate * dp / dp_peak,
                            hbm_frac_whole_run=rate * by / (hbm * 1e9), fp64_peak=dp_peak,
                            fused_blocks=r.fused_blocks, passes=r.fused_passes, guard_flagged=r.guard_flagged)
            if mode == "branch":
                line.update(peak_states=r.branch.peak_states, branch_passes=r.branch.passes)
            g = samples.get(key)
            if g:
                got = [int(run(prog, RunOptions(shots=1, seed=1, **extra), shot_begin=i, shot_count=1)._values[0])
                       for i in g["ids"][:4]]
                line["parity_sample"] = got == g["values"][:4]
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
