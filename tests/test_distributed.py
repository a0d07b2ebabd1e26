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
from paper_2308_03399_b200.distributed import gather_counts, shard_range, weak_range


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
