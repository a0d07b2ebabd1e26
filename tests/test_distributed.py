"""World-size-2 gloo tests of the multi-GPU host logic (paper_2308_03399_b200.
distributed): shot sharding + the counts gather reproduce the single run.
Each rank computes its shard with the CPU oracle (no GPU here); on B200 the
same functions carry device values over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_03399_b200 import Program, circuits as cc
from paper_2308_03399_b200.api import counts_from_values
from paper_2308_03399_b200.distributed import ChunkQueue, gather_counts, run_balanced, shard_range, weak_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, circ, noise, shots, seed, wide, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        prog = Program.from_text(circ, noise)
        begin, count = shard_range(rank, world, shots)
        vals = Oracle().run_shots(prog, np.arange(begin, begin + count), seed)
        width = 30 if wide else prog.num_clbits  # wide: exercise the all-gather path
        counts = gather_counts(vals.astype(np.int64), width, True)
        out[rank] = counts
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for total in (0, 1, 7, 1000, 100_000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(r, world, total) for r in range(world)]
            assert sum(c for _, c in spans) == total
            assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    assert weak_range(3, 100) == (300, 100)
    with pytest.raises(ValueError):
        shard_range(2, 2, 10)


@pytest.mark.parametrize("wide", [False, True])
def test_two_rank_gather_equals_single_run(wide):
    circ, noise = cc.ghz(6), cc.depolarizing_model(0.05)
    shots, seed = 301, 11
    from oracle.oracle import Oracle
    prog = Program.from_text(circ, noise)
    want = counts_from_values(Oracle().run_shots(prog, np.arange(shots), seed), 30 if wide else prog.num_clbits,
                              True)
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _free_port(), circ, noise, shots, seed, wide, out), nprocs=2, join=True)
    assert out[0] == want and out[1] == want


def _engine_worker(rank, world, port, circ, noise, shots, seed, out):
    """One rank: its shard on the GPU engine (device values), the dense
    histogram built on the device (ssb_histogram_device), summed over ranks."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_2308_03399_b200 import Engine, RunOptions
        from paper_2308_03399_b200.distributed import allreduce_histogram, counts_from_histogram
        eng = Engine(0)
        prog = Program.from_text(circ, noise)
        begin, count = shard_range(rank, world, shots)
        vals = torch.empty(count, dtype=torch.int64, device="cuda:0")
        hist = torch.zeros(1 << prog.num_clbits, dtype=torch.int64, device="cuda:0")
        eng.run_batch_device(prog, RunOptions(seed=seed, fused_matrices=True), vals.data_ptr(), begin, count)
        eng.histogram_device(vals.data_ptr(), count, prog.num_clbits, hist.data_ptr())
        torch.cuda.synchronize()
        h = allreduce_histogram(hist.cpu())
        out[rank] = counts_from_histogram(h, prog.num_clbits, True)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_engine_histogram_equals_single_run():
    """The multi-GPU gather on the real device path: two ranks (gloo; both on
    the one GPU of the box) run their shot-id shards through the engine, build
    the histogram on the device and all-reduce it; the result equals the
    single-rank run's counts."""
    from paper_2308_03399_b200 import Engine, RunOptions
    circ, noise = cc.quantum_volume(14, depth=4, seed=2), cc.qv_noise()
    shots, seed = 3001, 5
    r = Engine(0).run_batch(Program.from_text(circ, noise), RunOptions(shots=shots, seed=seed))
    out = mp.Manager().dict()
    mp.spawn(_engine_worker, args=(2, _free_port(), circ, noise, shots, seed, out), nprocs=2, join=True)
    assert out[0] == r.counts and out[1] == r.counts


@pytest.mark.gpu
def test_bench_two_ranks_under_torchrun():
    """bench.py's N > 1 path (torchrun, weak shot sharding, barriers,
    max-over-ranks timing, device histogram all-reduce, rank-0 line) with two
    ranks sharing the box's GPU over gloo (NCCL refuses duplicate GPUs)."""
    import json
    import subprocess
    import sys
    from conftest import ROOT
    env = dict(os.environ, SHOTSIM_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1",
           "--warmup", "1", "--shots", "2048", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["global_shots_per_step"] == 4096 and line["value"] > 0


def _balanced_worker(rank, world, port, circ, noise, shots, seed, chunk, slow_rank, out):
    """One rank of a dynamically balanced run: chunks pulled from the store's
    counter; `slow_rank` sleeps per chunk (a loaded / slower GPU), so the
    other rank must take over the waiting chunks."""
    import time
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        prog = Program.from_text(circ, noise)
        orc = Oracle()

        def run_chunk(b, n):
            if rank == slow_rank:
                time.sleep(0.3)
            return orc.run_shots(prog, np.arange(b, b + n), seed)

        vals, mine = run_balanced(run_chunk, shots, chunk)
        out[rank] = (vals.tolist(), mine)
    finally:
        dist.destroy_process_group()


def test_chunk_queue_hands_out_each_chunk_once():
    class S:
        v = 0

        def add(self, k, n):
            S.v += n
            return S.v
    q = ChunkQueue(S(), 10, 4, "k")
    got = []
    while (c := q.next()) is not None:
        got.append(c)
    assert got == [(0, 4), (4, 4), (8, 2)] and q.num_chunks == 3
    assert ChunkQueue(S(), 0, 4, "z").num_chunks == 0
    with pytest.raises(ValueError):
        ChunkQueue(S(), 10, 0, "k")


def test_balanced_two_ranks_equal_single_run_and_shift_work():
    """Cross-rank load balancing (run_balanced): two gloo ranks pull shot
    chunks from one counter; the slow rank ends up with fewer chunks, and the
    merged per-shot values equal the single run's exactly."""
    circ, noise = cc.ghz(5), cc.depolarizing_model(0.05)
    shots, seed, chunk = 240, 3, 20
    from oracle.oracle import Oracle
    want = Oracle().run_shots(Program.from_text(circ, noise), np.arange(shots), seed)
    out = mp.Manager().dict()
    mp.spawn(_balanced_worker, args=(2, _free_port(), circ, noise, shots, seed, chunk, 1, out), nprocs=2,
             join=True)
    for r in (0, 1):
        assert out[r][0] == want.astype(np.int64).tolist()
    c0, c1 = out[0][1], out[1][1]
    assert sorted(c0 + c1) == [(b, chunk) for b in range(0, shots, chunk)]
    assert len(c0) > len(c1) >= 1


def _balanced_engine_worker(rank, world, port, circ, noise, shots, seed, chunk, budget, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_03399_b200 import Engine, RunOptions
        eng = Engine(0)
        prog = Program.from_text(circ, noise)

        def run_chunk(b, n):
            r = eng.run_branch(prog, RunOptions(shots=n, seed=seed, branch_budget=budget, record_shot_values=True),
                               shot_begin=b)
            return np.asarray(r.shot_values)

        vals, mine = run_balanced(run_chunk, shots, chunk)
        out[rank] = (vals.tolist(), mine)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_balanced_branch_two_ranks_equal_single_run():
    """gpu-branch under the cross-rank chunk balancer (two ranks sharing the
    box's GPU): the merged values equal one run_branch over all shots."""
    from paper_2308_03399_b200 import Engine, RunOptions
    circ, noise = cc.dynamic(10, rounds=3), cc.thermal_noise(0.02, 0.05)
    shots, seed, chunk, budget = 6000, 9, 500, 64
    want = Engine(0).run_branch(Program.from_text(circ, noise),
                                RunOptions(shots=shots, seed=seed, branch_budget=budget, record_shot_values=True))
    out = mp.Manager().dict()
    mp.spawn(_balanced_engine_worker, args=(2, _free_port(), circ, noise, shots, seed, chunk, budget, out), nprocs=2,
             join=True)
    for r in (0, 1):
        assert out[r][0] == np.asarray(want.shot_values).astype(np.int64).tolist()
    assert sorted(out[0][1] + out[1][1]) == [(b, chunk) for b in range(0, shots, chunk)]


def test_run_balanced_single_process_edges():
    """Without a process group every chunk runs locally; empty runs, chunks
    larger than the run and a wrong chunk length are handled."""
    vals, mine = run_balanced(lambda b, n: np.arange(b, b + n) * 3, 10, 4)
    assert vals.tolist() == [3 * i for i in range(10)] and mine == [(0, 4), (4, 4), (8, 2)]
    vals, mine = run_balanced(lambda b, n: np.zeros(n), 0, 4)
    assert vals.size == 0 and mine == []
    vals, mine = run_balanced(lambda b, n: np.ones(n), 3, 100)
    assert vals.tolist() == [1, 1, 1] and mine == [(0, 3)]
    with pytest.raises(ValueError):
        run_balanced(lambda b, n: np.ones(n + 1), 5, 2)
