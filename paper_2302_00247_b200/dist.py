"""Multi-GPU search: candidate ranges sharded over ranks, exact key exchange.

Each rank (one process per GPU) scores its contiguous slice of every block's
index range -- the split search_subgraph hands its worker pool
(search.py:331-336).  Per block the ranks then exchange one record
(has_best, total bits, num_split, index, valid) with a single all_gather
over NCCL and reduce it to the lexicographic (total, num_split, index)
minimum and the summed valid count (search.py:337-343).  A single 64-bit
allreduce-min cannot carry this key losslessly, so the record
is gathered whole; it is 40 bytes per block.
"""

from __future__ import annotations

import struct
from typing import Callable

import numpy as np

from ._abi import SpScoreOut


def _key(s: SpScoreOut):
    return (s.best_total, s.best_num_split, s.best_index)


def merge_scores(parts: list) -> list:
    """Merge per-shard result lists (same block order) exactly."""
    out = []
    for recs in zip(*parts):
        acc = SpScoreOut()
        acc.candidates = recs[0].candidates
        for r in recs:
            acc.valid += r.valid
            if r.has_best and (not acc.has_best or _key(r) < _key(acc)):
                acc.has_best = 1
                acc.best_total = r.best_total
                acc.best_num_split = r.best_num_split
                acc.best_index = r.best_index
        out.append(acc)
    return out


def pack(scores: list) -> np.ndarray:
    """[nb, 6] int64 records (fp64 total carried as its bit pattern)."""
    a = np.zeros((len(scores), 6), np.int64)
    for i, s in enumerate(scores):
        bits = struct.unpack("<q", struct.pack("<d", s.best_total))[0]
        a[i] = (s.has_best, bits, s.best_num_split, np.uint64(s.best_index).view(np.int64),
                np.uint64(s.valid).view(np.int64), np.uint64(s.candidates).view(np.int64))
    return a


def unpack(a: np.ndarray) -> list:
    out = []
    for row in a:
        s = SpScoreOut()
        s.has_best = int(row[0])
        s.best_total = struct.unpack("<d", struct.pack("<q", int(row[1])))[0]
        s.best_num_split = int(row[2])
        s.best_index = int(np.int64(row[3]).view(np.uint64))
        s.valid = int(np.int64(row[4]).view(np.uint64))
        s.candidates = int(np.int64(row[5]).view(np.uint64))
        out.append(s)
    return out


def allgather_exchange(group=None, device=None) -> Callable:
    """exchange(scores) -> merged scores over all ranks of `group`.

    Uses torch.distributed only as plumbing: one all_gather of the packed
    records (NCCL when the group's backend is nccl, on `device`)."""
    import torch
    import torch.distributed as dist

    def exchange(scores: list) -> list:
        world = dist.get_world_size(group)
        if world == 1:
            return scores
        local = torch.from_numpy(pack(scores))
        if dist.get_backend(group) == "nccl":
            local = local.to(device or torch.device("cuda", torch.cuda.current_device()))
        bufs = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(bufs, local, group=group)
        parts = [unpack(b.cpu().numpy()) for b in bufs]
        return merge_scores(parts)

    return exchange
