"""World-size-2 test of the multi-GPU key exchange on CPU (gloo).

Each rank scores its contiguous slice of every block's candidate range (the
split search_subgraph gives its pool, search.py:331-336) -- here with the CPU
oracle standing in for the GPU scorer -- and the ranks merge with
paper_2302_00247_b200.dist.allgather_exchange, the exact code the NCCL path
runs.  The merged per-block (valid, argmin) must equal the unsharded search.
"""

from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = ("c2_1x8", "tiny_2x2", "chain6_2x4_mu")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_scores(name: str, rank: int, world: int):
    from golden_io import case, lowered, mesh
    from oracle import oracle
    from paper_2302_00247_b200._abi import SpScoreOut
    from paper_2302_00247_b200.blocks import BlockArrays

    c = case(name)
    low = lowered(c["graph"])
    ba = BlockArrays.from_dict(oracle.prune(low, c["min_dup"]))
    m = mesh(c["mesh"])
    out = []
    for b in range(ba.n_blocks):
        tn = ba.template_nodes(b)
        total, _ = oracle.score(low, tn, m, mu=c["mu"], chunk=c["chunk_size"], hi=0)
        C = total.candidates
        step = -(-C // world)
        lo, hi = min(C, rank * step), min(C, (rank + 1) * step)
        if lo < hi:
            res, _ = oracle.score(low, tn, m, mu=c["mu"], chunk=c["chunk_size"], lo=lo, hi=hi,
                                  threads=2)
        else:
            res = SpScoreOut()
            res.candidates = C
        out.append(res)
    return out


def _worker(rank: int, world: int, port: int, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2302_00247_b200.dist import allgather_exchange

        ex = allgather_exchange()
        result = {}
        for name in CASES:
            merged = ex(_shard_scores(name, rank, world))
            result[name] = [(r.valid, r.has_best, r.best_index, r.best_num_split, r.best_total)
                            for r in merged]
        q.put((rank, result))
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_two_rank_exchange_matches_single_process():
    from golden_io import case

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0] == results[1]  # every rank ends with the same plan keys
    single = {name: [(r.valid, r.has_best, r.best_index, r.best_num_split, r.best_total)
                     for r in _shard_scores(name, 0, 1)] for name in CASES}
    assert results[0] == single
    for name in CASES:  # and with the reference's goldens
        exp = case(name)["best"]
        assert [(v, i, repr(t)) for v, _, i, _, t in results[0][name]] == [
            (e["valid"], e["index"], e["total"]) for e in exp]


# -- the same exchange behind the real device scorer (two ranks share cuda:0) -------------

def _gpu_worker(rank: int, world: int, port: int, q, names):
    import hashlib
    import json
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from golden_io import case, graph, mesh
        from paper_2302_00247_b200._native import Backend
        from paper_2302_00247_b200.dist import allgather_exchange
        from paper_2302_00247_b200.search import derive_plan

        be = Backend(0)
        ex = allgather_exchange()
        out = {}
        for name in names:
            c = case(name)
            for mode in ("skip", "walk"):
                be.set_mode(mode)
                rep = derive_plan(graph(c["graph"]), mesh(c["mesh"]), min_duplicates=c["min_dup"], mu=c["mu"],
                                  chunk_size=c["chunk_size"], backend=be, shard=rank, n_shards=world, exchange=ex)
                doc = json.dumps(rep.to_json(), sort_keys=True, separators=(",", ":"))
                out[(name, mode)] = hashlib.sha256(doc.encode()).hexdigest()
        q.put((rank, out))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_device_search_byte_identical():
    """derive_plan sharded over 2 ranks (device scoring of each rank's slice +
    the all_gather key exchange) gives the reference's plan JSON, byte for byte."""
    import hashlib

    from golden_io import case

    names = ("c2_1x8", "chain6_2x4_mu", "c1_1x8")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, names)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert results[0] == results[1]
    for name in names:
        exp = hashlib.sha256(case(name)["plan_json"].encode()).hexdigest()
        for mode in ("skip", "walk"):
            assert results[0][(name, mode)] == exp, (name, mode)


class _StubTables:
    nbytes = 0
    overflow = False

    def close(self):
        pass


class _StubBackend:
    """Just enough of Backend for _plan_searches: tables are stubs, no device."""

    def __init__(self, rank, nranks):
        self.comm = {"nranks": nranks, "rank": rank, "devices": 1, "transport": "nccl", "nccl_version": 0}
        self.launched = []
        self.smem_limit = 1 << 30

    is_root = property(lambda self: self.comm["rank"] == 0)
    sharded_in_library = property(lambda self: self.comm["nranks"] > 1)

    def tables(self, *a):
        return _StubTables()

    def block_info(self, t):
        import numpy as np
        return np.zeros(0, np.int64), np.zeros(0, np.int64), None


@pytest.mark.parametrize("rank", [0, 1, 3])
def test_cheap_group_root_local(monkeypatch, rank):
    """Multi-rank derive_plan: the cheap group of a two-group split is a local
    search on rank 0 (SP_SCORE_LOCAL) and is not built on any other rank; the
    expensive group is a collective on every rank."""
    import numpy as np

    from paper_2302_00247_b200 import search as S

    csr = (np.array([0, 1, 2, 3], np.int64), np.arange(3, dtype=np.int32))
    monkeypatch.setattr(S, "_route_mask", lambda low, c: np.zeros(3, bool))
    monkeypatch.setattr(S, "_block_groups", lambda low, c: [([0, 1], c), ([2], c)])
    be = _StubBackend(rank, 4)
    ses = S.Session(be, None, None)
    got = S._plan_searches(ses, csr, None, 1, 1 << 20, 0, 1, None, root_local=True)
    if rank == 0:
        assert [(ids, s.local) for s, ids in got] == [([0, 1], True), ([2], False)]
    else:
        assert [(ids, s.local) for s, ids in got] == [([2], False)]
    # without the root-local rule every rank builds both groups
    got = S._plan_searches(ses, csr, None, 1, 1 << 20, 0, 1, None, root_local=False)
    assert [(ids, s.local) for s, ids in got] == [([0, 1], False), ([2], False)]
