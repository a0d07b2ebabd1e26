#!/usr/bin/env python3
"""Benchmark: shots/s of the noisy quantum-volume workload (BASELINE.json
metric, config C2: QV16 + depolarizing 1% + 1% readout, 1e5 shots, seed 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N ... bench.py --gpus N          (one rank per GPU)

One step = one pass of the hot path over one batch: the full instrumented
program for `shots` shots on every rank (weak scaling: rank r runs shot ids
[r*S, (r+1)*S)), then the dense counts histogram of the step (device kernel)
all-reduced over NCCL when N > 1 — the only cross-GPU exchange the path has.

`value`: device-resident inputs (program uploaded before timing), per-shot
register values left in HBM; CUDA events on the engine stream, max over ranks.
`e2e`: the same steps through the public C ABI from host buffers — circuit
text + noise JSON lowered and uploaded every step (ssb_program_from_text),
per-shot values copied back to pinned host memory (ssb_run_batch).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "shots/sec, noisy QV circuit, 1/2/4/8 B200; % of HBM/SM roofline"
UNIT = "shots/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--shots", type=int, default=0, help="override shots per GPU per step")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exact", action="store_true",
                    help="bit-exact-amplitude executor (no fused 4x4 blocks); default: fused_matrices")
    return ap.parse_args()


def workload(key, shots_override=0):
    from paper_2308_03399_b200 import circuits as cc
    cfg = cc.CONFIGS[key]
    return cfg, cfg["circuit"](), cfg["noise"](), (shots_override or cfg["shots"]), cfg["seed"]


def config_dict(key, cfg, shots, n_gpus, executor="gpu-batch", fused=True):
    desc = {
        "C1": "GHZ10 + depolarizing 1%",
        "C2": "QV16 (16 layers of SU(4) blocks) + depolarizing 1% + 1% readout flip",
        "C3": "dyn12 (4 rounds measure/reset/conditional) + depolarizing 1%",
        "C4": "rnd20 + thermal-relaxation Kraus (3-matrix 1q, 9-matrix 2q)",
        "C5": "QV24 + depolarizing 1%",
    }[key]
    return {"workload": f"{key} {cfg['name']}: {desc}", "shots_per_gpu_per_step": shots,
            "global_shots_per_step": shots * n_gpus, "seed": cfg["seed"], "executor": executor,
            "parallelism": f"shot-sharded x{n_gpus} (weak)",
            "l2": "inputs larger than L2: per-wave state 16 GiB >> 126 MB L2",
            "arithmetic": ("fp64 complex; fused 4x4 blocks with FMA (amplitudes within 1e-10 of the reference), "
                           "guard band + exact on-device replay on terminal sampling: bit-exact counts"
                           if fused else
                           "fp64 complex, reference scalar-table rounding (no FMA), bit-exact counts and amplitudes")}


# ---- algorithmic bytes -------------------------------------------
def algorithmic_bytes(program):
    """Per shot: gate 32A, expected non-identity Pauli 32A, Kraus 48A, measure 48A,
    reset 48A + 16A, terminal sampling 16A. Returns (pass_part, total)."""
    f = program.flat()
    A = 1 << f.num_qubits
    end = f.terminal_measure_begin if f.sampling_eligible else f.num_ops
    pass_b = other = 0.0
    for i in range(end):
        op = f.ops[i]
        if op.kind == 0:
            pass_b += 32 * A
        elif op.kind == 1:
            prev = 0.0
            p_nonid = 0.0
            for t in range(op.term_count):
                term = f.terms[op.term_begin + t]
                if not term.identity:
                    p_nonid += term.cumulative - prev
                prev = term.cumulative
            pass_b += 32 * A * p_nonid
        elif op.kind in (2, 3):
            other += 48 * A
        elif op.kind == 4:
            other += 64 * A
    if f.sampling_eligible:
        other += 16 * A
    return pass_b, pass_b + other


def _entry_cost(re, im):
    """Rounded FP64 ops of one complex product m*v in the engine's exact
    arithmetic (exact.cuh c_term): 0 for 0 / +-1, 2 for real or imaginary m,
    6 (4 DMUL + 2 DADD) for general m. Returns (ops, is_term)."""
    if re == 0.0 and im == 0.0:
        return 0, False
    if im == 0.0 and re in (1.0, -1.0):
        return 0, True
    if im == 0.0 or re == 0.0:
        return 2, True
    return 6, True


def dp_ops_per_shot(program):
    """FP64 ops (DMUL + DADD, no FMA) the fused tile passes execute per shot:
    per row, every nonzero term's product plus 2 DADD per complex add
    (row_apply / quad_apply*, exact.cuh). Pure permutations (CX, SWAP) and
    identity gates cost nothing; Pauli sites are sign / register moves."""
    return sum(dp_ops_per_op(program))


def dp_ops_per_op(program):
    """dp_ops_per_shot split per op of the program (0 for non-gates)."""
    f = program.flat()
    A = 1 << f.num_qubits
    end = f.terminal_measure_begin if f.sampling_eligible else f.num_ops
    out = [0] * f.num_ops
    for i in range(end):
        op = f.ops[i]
        if op.kind != 0:
            continue
        k = op.num_qubits
        d = 1 << k
        base = op.matrix * 32
        ops = 0
        identity = True
        for r in range(d):
            terms = 0
            for c in range(d):
                re, im = f.matrices[base + 2 * (r * d + c)], f.matrices[base + 2 * (r * d + c) + 1]
                cost, term = _entry_cost(re, im)
                ops += cost
                terms += term
                if (r == c) != (re == 1.0 and im == 0.0) or (r != c and term):
                    identity = False
            ops += 2 * max(terms - 1, 0)
        if not identity:
            out[i] = ops * (A >> k)
    return out


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key, shot_passes_per_launch):
    """Per-launch DRAM bytes of the dominant kernel: the committed ncu capture's
    measured bytes per (shot, pass) scaled to this run's shots per launch."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(key)
    if not d or d.get("dram_bytes_per_shot") is None:
        return None
    return d["dram_bytes_per_shot"] * shot_passes_per_launch


# ---- clocks ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(s[0]) for s in self.samples if num(s[0])]
        loaded = [num(s[0]) for s in self.samples if num(s[0]) and (num(s[6]) or 0) > 50] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": num(self.samples[0][1]), "reasons": reasons, "samples": len(self.samples)}


# ---- CPU baseline (the reference's own CPU implementation) ------------------------------
def cpu_baseline(circuit, noise, seed, budget_s, check_values=None):
    """Times the reference's run_single_shot path (oracle/_ref, built from the
    reference sources) on all host cores over shot ids [0, k) — a bounded
    sample of the same workload; shots are independent and keyed by id, so
    shots/s extrapolates linearly. Falls back to the oracle port."""
    import numpy as np
    cores = os.cpu_count() or 1
    try:
        from oracle.oracle import REF_SO, Reference
        if not REF_SO.exists():
            raise FileNotFoundError(REF_SO)
        ref = Reference()
        ref.select_kernels("auto")  # the reference's default (AVX2) table: its fastest CPU path
        run = lambda ids: ref.run_ids(circuit, noise, ids, seed, workers=cores)
        kind = "reference"
    except Exception:
        from oracle.oracle import Oracle
        from paper_2308_03399_b200 import Program
        o = Oracle()
        prog = Program.from_text(circuit, noise)

        def run(ids):
            t0 = time.perf_counter()
            v = o.run_shots(prog, ids, seed, threads=cores)
            return v, time.perf_counter() - t0
        kind = "port"
    k = cores
    vals, secs = run(np.arange(k))
    while secs < budget_s / 4 and k < 10_000_000:
        k = int(k * max(2.0, min(8.0, (budget_s / 2) / max(secs, 1e-3))))
        vals, secs = run(np.arange(k))
    parity = None
    if check_values is not None:
        m = min(len(check_values), k)
        parity = bool((np.asarray(check_values[:m], dtype=np.uint64) == vals[:m]).all())
    return {"value": k / secs, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"shot ids [0,{k}) of the same workload, {secs:.1f} s on {cores} host threads"
                      + (" (reference scalar/AVX2 auto table, run_single_shot per shot)" if kind == "reference" else ""),
            "parity_with_gpu_values": parity}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, circuit, noise, shots, seed = workload(args.config, args.shots)
    import numpy as np
    cores = os.cpu_count() or 1
    try:
        from oracle.oracle import REF_SO, Reference
        if not REF_SO.exists():
            raise FileNotFoundError(REF_SO)
        ref = Reference()
        ref.select_kernels("auto")
        run = lambda ids: ref.run_ids(circuit, noise, ids, seed, workers=cores)[1]
        kind = "reference"
    except Exception as e:  # the port of the reference path
        from oracle.oracle import Oracle
        from paper_2308_03399_b200 import Program
        o = Oracle()
        prog = Program.from_text(circuit, noise)

        def run(ids):
            t0 = time.perf_counter()
            o.run_shots(prog, ids, seed, threads=cores)
            return time.perf_counter() - t0
        kind = "port"
    # Size one step to ~3 s of CPU work.
    k = cores
    t = run(np.arange(k))
    k = max(cores, int(k * 3.0 / max(t, 1e-3)))
    for w in range(args.warmup):
        run(np.arange(w * k, (w + 1) * k))
    total = 0.0
    for s in range(args.steps):
        total += run(np.arange((args.warmup + s) * k, (args.warmup + s + 1) * k))
    value = k * args.steps / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": config_dict(args.config, cfg, k, 1, executor="reference run_single_shot (CPU, all host threads)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"{k} shot ids per step on {cores} host threads (reference CPU path)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    # SHOTSIM_BENCH_DIST_BACKEND=gloo (test hook): exercise the N>1 path with
    # several ranks sharing the visible GPUs (NCCL refuses duplicate GPUs).
    backend = os.environ.get("SHOTSIM_BENCH_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2308_03399_b200 import Engine, Program, RunOptions
    cfg, circuit, noise, shots, seed = workload(args.config, args.shots)
    eng = Engine(local)
    prog = Program.from_text(circuit, noise)
    nclb = prog.num_clbits
    from paper_2308_03399_b200.distributed import allreduce_histogram, weak_range
    begin, _ = weak_range(rank, shots)
    values = torch.empty(shots, dtype=torch.int64, device=f"cuda:{local}")
    hist = torch.zeros(1 << nclb, dtype=torch.int64, device=f"cuda:{local}") if nclb <= 24 else None
    stream = torch.cuda.ExternalStream(eng.stream, device=f"cuda:{local}")
    fused = not args.exact
    opts = RunOptions(seed=seed, fused_matrices=fused)
    prof = RunOptions(seed=seed, profile=True, fused_matrices=fused)

    def step(o):
        st = eng.run_batch_device(prog, o, values.data_ptr(), begin, shots)
        launches = st.dispatch_count
        if hist is not None:
            with torch.cuda.stream(stream):
                hist.zero_()
            eng.histogram_device(values.data_ptr(), shots, nclb, hist.data_ptr())
            launches += 1
            if world > 1:
                with torch.cuda.stream(stream):
                    allreduce_histogram(hist)  # NCCL over NVLink: the run's only collective
        return st, launches

    for _ in range(max(args.warmup, 0)):
        step(opts)
    torch.cuda.synchronize()

    # ---- timed region (device-resident inputs) ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    pass_s = other_s = 0.0
    pass_launches = launches = passes_per_wave = shapes = skipped = fused_blocks = flagged = 0
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            st, nl = step(prof)
            pass_s += st.pass_seconds
            pass_launches += st.pass_launches
            passes_per_wave = st.fused_passes
            shapes = st.specialised_shapes
            skipped += st.trunk_skipped
            fused_blocks = st.fused_blocks
            flagged += st.guard_flagged
            other_s += st.special_seconds + st.sample_seconds
            launches += nl
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed = ev0.elapsed_time(ev1) * 1e-3
    t = torch.tensor([elapsed], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())
    value = world * shots * args.steps / elapsed_max
    gpu_vals = values.cpu().numpy().astype(np.uint64)

    # ---- end-to-end through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        h_vals = np.empty(shots, dtype=np.uint64)
        flat = prog.flat()
        h2d = (flat.num_ops * 64 + flat.num_matrices * 256 + flat.num_terms * 24 + flat.num_channels * 16)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            p = Program.from_text(circuit, noise)  # host lowering + upload inside the step
            r = eng.run_batch(p, RunOptions(shots=shots, seed=seed, fused_matrices=fused), shot_begin=begin,
                              shot_count=shots)
            h_vals[:] = r._values
        e2e_s = time.perf_counter() - t0
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": world * shots * args.steps / float(t.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(8 * shots),
               "path": "ssb_program_from_text + ssb_run_batch (host values)"}
        assert (h_vals == gpu_vals).all(), "e2e values differ from the device-resident run"

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    pass_b, total_b = algorithmic_bytes(prog)
    peak, peak_src = measured_peak()
    from paper_2308_03399_b200.api import _fp64_peak
    dp_peak = _fp64_peak(eng)
    n_timed_shots = shots * args.steps
    A = 1 << prog.num_qubits
    roof = None
    if pass_s > 0 and fused_blocks:
        # Dominant kernel: fused_pass_kernel. Per shot it reads + writes the
        # state once per pass (32 A bytes) and applies every block as a dense
        # 4x4 complex matvec with FMA (16 DP instructions per amplitude).
        bytes_shot = 32.0 * A * passes_per_wave
        dp_shot = 16.0 * A * fused_blocks
        kname = "fused_pass_kernel (4x4 blocks, register groups)"
    elif pass_s > 0:
        # Exact mode: the tile passes read + write the state once per pass; DP
        # instructions are the engine's no-FMA arithmetic (dp_ops_per_shot).
        executed = max(0.0, 1.0 - skipped / (n_timed_shots * max(passes_per_wave, 1))) if passes_per_wave else 1.0
        bytes_shot = 32.0 * A * passes_per_wave * executed
        dp_shot = dp_ops_per_shot(prog) * executed
        kname = ("ssb_tile_pass_jit (run-time shape-specialised, %d shapes)" % shapes if shapes else "tile_pass_kernel") \
            if prog.num_qubits > 13 else "resident_kernel"
    if pass_s > 0:
        hbm_ach = bytes_shot * n_timed_shots / pass_s / 1e9
        dp_ach = dp_shot * n_timed_shots / pass_s
        hbm_frac, dp_frac = hbm_ach / peak, dp_ach / dp_peak
        fp64 = {"achieved": dp_ach / 1e12, "peak": dp_peak / 1e12, "unit": "T DP-op/s", "frac": dp_frac,
                "dp_ops_per_shot": dp_shot,
                "peak_source": "measured live: ssb_fp64_peak (independent DMUL/DADD chains, CUDA events; DFMA "
                               "issues at the same per-lane rate on the FP64 pipe)"}
        hbm = {"achieved": hbm_ach, "peak": peak, "unit": "GB/s", "frac": hbm_frac,
               "algorithmic_bytes_per_shot": bytes_shot, "peak_source": peak_src,
               "traffic": ncu_traffic(args.config + ("" if fused_blocks else "_exact"),
                                      n_timed_shots * passes_per_wave / max(pass_launches, 1)),
               "traffic_source": "profiles/ncu_summary.json (ncu --set full dram__bytes_read+write per shot-pass)"}
        lead = fp64 if dp_frac >= hbm_frac else hbm
        roof = {"bound": "fp64" if dp_frac >= hbm_frac else "hbm", "kernel": kname,
                "achieved": lead["achieved"], "peak": lead["peak"], "unit": lead["unit"], "frac": lead["frac"],
                "traffic": hbm["traffic"],
                "launches": pass_launches, "kernel_share_of_step": pass_s / max(elapsed, 1e-12),
                "fp64": fp64, "hbm": hbm,
                "fusion_gain": pass_b / bytes_shot if bytes_shot else None,
                "note": "frac = the binding unit of the dominant kernel (per-launch algorithmic work / its CUDA-event "
                        "time); fusion_gain = the reference's unfused op stream bytes (SURVEY 8(d)) / the bytes this "
                        "kernel must move"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, cfg, shots, world, fused=not args.exact), "e2e": e2e,
            "gpu_launches": launches, "guard_flagged": flagged,
            "roofline": roof, "clocks": clocks.summary()}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(circuit, noise, seed, args.cpu_seconds, check_values=gpu_vals)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
