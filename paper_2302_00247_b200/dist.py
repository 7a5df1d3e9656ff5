"""Multi-GPU search: candidate ranges sharded over ranks, exact key exchange.

Each rank (one process per GPU) scores its share of every block's index
range: the work items of all blocks are dealt round-robin over the ranks
(search_subgraph hands its worker pool contiguous slices, search.py:331-336;
early-exit cost varies along a range, so contiguous slices load one rank
with the expensive end).  Per block the ranks then exchange one record
(candidates, valid, index, total bits, num_split, has_best) with a single
all_gather over NCCL and reduce it, vectorised over blocks, to the
lexicographic (total, num_split, index) minimum and the summed valid count
(search.py:337-343).  A single 64-bit allreduce-min cannot carry this key
losslessly, so the record is gathered whole; it is 40 bytes
per block.
"""

from __future__ import annotations

import ctypes as C
from typing import Callable

import numpy as np

from ._abi import SpScoreOut


#: numpy view of sp_score_out (include/shardsearch.h): 40-byte records
REC = np.dtype([("candidates", "<u8"), ("valid", "<u8"), ("best_index", "<u8"), ("best_total", "<f8"),
                ("best_num_split", "<i4"), ("has_best", "<i4")])
assert REC.itemsize == C.sizeof(SpScoreOut)


def to_records(scores: list) -> np.ndarray:
    """SpScoreOut list -> structured array (one copy of the raw records)."""
    return np.frombuffer(b"".join(map(bytes, scores)), dtype=REC) if scores else np.zeros(0, REC)


def from_records(rec: np.ndarray) -> list:
    from ._native import RawList

    arr = (SpScoreOut * max(1, len(rec))).from_buffer_copy(np.ascontiguousarray(rec, REC).tobytes() or bytes(40))
    return RawList(arr, len(rec))


def merge_records(parts: np.ndarray) -> np.ndarray:
    """[world, nb] records -> [nb]: lexicographic (total, num_split, index) min over the
    ranks that have a winner (search.py:337-343), valid counts summed.  Totals are
    non-negative doubles, so their bit patterns order like the values."""
    world, nb = parts.shape
    if world == 1:
        return parts[0].copy()
    tb = parts["best_total"].view("<u8")
    no = (parts["has_best"] == 0).astype(np.uint8)
    # lexsort: last key is primary; per block (column) over the ranks (rows)
    order = np.lexsort((parts["best_index"], parts["best_num_split"], tb, no), axis=0)
    win = order[0]
    out = parts[win, np.arange(nb)].copy()
    out["valid"] = parts["valid"].sum(axis=0)
    out["candidates"] = parts["candidates"][0]
    none = out["has_best"] == 0  # no rank routed a candidate of this block
    for f in ("best_index", "best_total", "best_num_split"):
        out[f][none] = 0
    return out


def merge_scores(parts: list) -> list:
    """Merge per-shard result lists (same block order) exactly."""
    if not parts:
        return []
    return from_records(merge_records(np.stack([to_records(p) for p in parts])))


def pack(scores: list) -> np.ndarray:
    """[nb, 5] int64 view of the records (fp64 total carried as its bit pattern)."""
    return to_records(scores).view(np.int64).reshape(-1, 5)


def unpack(a: np.ndarray) -> list:
    return from_records(np.ascontiguousarray(a, np.int64).reshape(-1).view(REC))


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
        local = torch.from_numpy(pack(scores).copy())
        if dist.get_backend(group) == "nccl":
            local = local.to(device or torch.device("cuda", torch.cuda.current_device()))
            out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
            dist.all_gather_into_tensor(out, local, group=group)
        else:  # gloo: list form
            bufs = [torch.empty_like(local) for _ in range(world)]
            dist.all_gather(bufs, local, group=group)
            out = torch.stack(bufs)
        parts = out.cpu().numpy().reshape(world, -1).view(REC)
        return from_records(merge_records(parts))

    return exchange


def init_comm(backend, rank: int, world: int, store=None) -> dict:
    """Join `world` processes (one GPU each) in the library's own NCCL
    communicator (sp_ctx_comm_init): afterwards every derive_plan on `backend`
    scores this rank's share and merges the per-block records on the device
    with one ncclAllGather -- no host exchange, no torch on the data path.

    Only the 128-byte NCCL unique id has to travel, rank 0 -> the others, through
    `store` (anything with set(key, bytes) / get(key) -> bytes, e.g. a
    torch.distributed TCPStore); by default the store of the initialised
    torch.distributed process group, else a TCPStore client of the launcher's
    MASTER_ADDR/MASTER_PORT (torchrun's agent store)."""
    if world <= 1:
        return backend.comm
    if store is None:
        import torch.distributed as tdist

        if tdist.is_available() and tdist.is_initialized():
            store = tdist.distributed_c10d._get_default_store()
        else:
            import datetime
            import os

            agent = os.environ.get("TORCHELASTIC_USE_AGENT_STORE", "").lower() == "true"
            store = tdist.TCPStore(os.environ.get("MASTER_ADDR", "127.0.0.1"), int(os.environ["MASTER_PORT"]),
                                   world, is_master=(rank == 0 and not agent),
                                   timeout=datetime.timedelta(seconds=300))
    key = "shardsearch/nccl_unique_id"
    if rank == 0:
        uid = backend.comm_unique_id()
        store.set(key, uid)
    else:
        uid = bytes(store.get(key))
    backend.comm_init(world, rank, uid)
    return backend.comm
