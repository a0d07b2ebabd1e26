"""Multi-GPU shot sharding and the end-of-run gather.

Shots are independent and keyed by id (rng.cpp:36-46), so a run over S shots
on W ranks is W runs over contiguous id ranges with no data-path exchange
(communication "only needed to collect results"). The only
collective is the gather of the result — the reference's ``merge_counts``
(result.cpp:15-21) of per-worker ``Counts``:

* ``num_clbits <= 24``: a dense uint64 histogram of the register values,
  summed with one all-reduce (NCCL over NVLink on GPUs, gloo on CPU);
* otherwise: an all-gather of the per-shot values (8 B per shot).

One process per GPU, ``torch.distributed`` for the plumbing; the histogram
itself is built on the device by ``ssb_histogram_device``.

Cross-GPU load balancing ("migrate ... waiting lists
between GPUs"): instead of one static contiguous range per rank,
``run_balanced`` cuts the run into shot-id chunks that the ranks pull from one
atomic counter in the job's rendezvous store (``Store.add``). A rank whose
chunks branch less, hit fewer guard replays or simply run on a less loaded GPU
takes over the chunks still waiting; since every shot is keyed by its id the
values never depend on where a chunk ran. The per-shot values are then merged
with one all-reduce (each shot is written by exactly one rank).
"""

from __future__ import annotations

from typing import Dict, Optional, Tuple

import numpy as np

from .api import bitstring

DENSE_MAX_CLBITS = 24


def shard_range(rank: int, world: int, total: int) -> Tuple[int, int]:
    """Contiguous shot-id range [begin, begin + count) of `rank` for a run of
    `total` shots over `world` ranks (strong scaling: the split is balanced to
    within one shot)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if total < 0:
        raise ValueError("shots must be >= 0")
    begin = total * rank // world
    return begin, total * (rank + 1) // world - begin


def weak_range(rank: int, per_rank: int) -> Tuple[int, int]:
    """Weak scaling: every rank runs `per_rank` shots, rank r ids [r*S, (r+1)*S)."""
    return rank * per_rank, per_rank


def histogram_of(values, num_clbits: int):
    """Dense histogram (torch int64, 2^num_clbits bins) of register values on
    the values' device — CPU reference of what ssb_histogram_device builds."""
    import torch
    if num_clbits > DENSE_MAX_CLBITS:
        raise ValueError("dense histogram limited to 24 clbits")
    v = torch.as_tensor(np.asarray(values, dtype=np.int64) if not torch.is_tensor(values) else values)
    mask = (1 << num_clbits) - 1
    return torch.bincount(v & mask, minlength=1 << num_clbits).to(torch.int64)


def allreduce_histogram(hist, group=None):
    """Sums the ranks' histograms in place (merge_counts is a sum, so the
    gathered result is independent of how shots were sharded)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, group=group)
    return hist


def allgather_values(values, group=None):
    """Concatenates every rank's per-shot values in rank order (for registers
    wider than the dense histogram)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return values
    world = dist.get_world_size(group)
    n = torch.tensor([values.numel()], dtype=torch.int64, device=values.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    cap = int(max(int(s.item()) for s in sizes))
    padded = torch.zeros(cap, dtype=values.dtype, device=values.device)
    padded[: values.numel()] = values
    parts = [torch.zeros_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)])


def counts_from_histogram(hist, width: int, has_measure: bool) -> Dict[str, int]:
    """counts_from_values (result.cpp:40-48) from a dense histogram."""
    h = np.asarray(hist.cpu() if hasattr(hist, "cpu") else hist, dtype=np.int64)
    total = int(h.sum())
    if not has_measure:
        return {"": total} if total else {}
    nz = np.nonzero(h)[0]
    return {bitstring(int(v), width): int(h[v]) for v in nz}


def gather_counts(values, num_clbits: int, has_measure: bool, group=None) -> Dict[str, int]:
    """The whole gather: dense all-reduce for <= 24 clbits, else all-gather."""
    if num_clbits <= DENSE_MAX_CLBITS:
        return counts_from_histogram(allreduce_histogram(histogram_of(values, num_clbits), group), num_clbits,
                                     has_measure)
    import torch
    allv = allgather_values(torch.as_tensor(np.asarray(values, dtype=np.int64)), group)
    uniq, cnt = np.unique(allv.cpu().numpy().astype(np.uint64), return_counts=True)
    if not has_measure:
        return {"": int(cnt.sum())}
    return {bitstring(int(u), num_clbits): int(c) for u, c in zip(uniq, cnt)}


class ChunkQueue:
    """Shot-id chunks [i * chunk, min((i + 1) * chunk, total)) handed out to
    whichever rank asks next: ``Store.add(key, 1)`` is atomic across ranks, so
    every chunk goes to exactly one rank. `key` must be fresh per run (the
    counter is never reset)."""

    def __init__(self, store, total: int, chunk: int, key: str):
        if chunk < 1:
            raise ValueError("chunk must be >= 1")
        if total < 0:
            raise ValueError("shots must be >= 0")
        self.store, self.total, self.chunk, self.key = store, total, chunk, key

    @property
    def num_chunks(self) -> int:
        return -(-self.total // self.chunk)

    def next(self) -> Optional[Tuple[int, int]]:
        i = int(self.store.add(self.key, 1)) - 1
        begin = i * self.chunk
        if begin >= self.total:
            return None
        return begin, min(self.chunk, self.total - begin)


def default_store():
    """The default process group's rendezvous store (the one torchrun or
    init_process_group created)."""
    import torch.distributed as dist
    return dist.distributed_c10d._get_default_store()


_RUN_SEQ = [0]


def run_balanced(run_chunk, total: int, chunk: int, store=None, key: Optional[str] = None, group=None):
    """Runs `total` shots in chunks pulled dynamically by the ranks.
    ``run_chunk(begin, count)`` returns the chunk's per-shot values (array-like
    of non-negative ints). Returns ``(values, mine)``: every shot's value on
    every rank (int64 numpy, shot-id order) and the chunks this rank ran.
    Single process (no process group): all chunks run locally."""
    import torch
    import torch.distributed as dist
    distributed = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    if key is None:  # the same sequence number on every rank: runs are collective
        _RUN_SEQ[0] += 1
        key = f"ssb_balanced_{_RUN_SEQ[0]}"
    if distributed:
        q = ChunkQueue(store if store is not None else default_store(), total, chunk, key)
    else:
        q = ChunkQueue(_LocalStore(), total, chunk, key)
    vals = np.zeros(total, dtype=np.int64)
    seen = np.zeros(total, dtype=np.int32)
    mine = []
    while True:
        c = q.next()
        if c is None:
            break
        b, n = c
        v = np.asarray(run_chunk(b, n), dtype=np.int64)
        if v.shape != (n,):
            raise ValueError("run_chunk returned the wrong number of values")
        vals[b:b + n] = v
        seen[b:b + n] += 1
        mine.append(c)
    if distributed:
        tv, ts = torch.from_numpy(vals), torch.from_numpy(seen)
        dist.all_reduce(tv, group=group)
        dist.all_reduce(ts, group=group)
        vals, seen = tv.numpy(), ts.numpy()
    if total and not (seen == 1).all():
        raise RuntimeError("chunk schedule did not cover every shot exactly once")
    return vals, mine


class _LocalStore:
    """Counter with Store.add semantics for the single-process case."""

    def __init__(self):
        self._v = {}

    def add(self, key, n):
        self._v[key] = self._v.get(key, 0) + n
        return self._v[key]
