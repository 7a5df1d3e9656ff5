"""Host utilities of the reference API (rows F7, R3, R6, R8) against the reference."""

from __future__ import annotations

import os
import random
import sys

import pytest

from golden_io import graph
from paper_2302_00247_b200 import reference_api as api
from paper_2302_00247_b200.ir import TensorSpec

REF = "/root/reference/pkg/src"


def test_pack_gradients_anchor():
    # acceptance criterion 6 (test_acceptance.py:165-192): 15 full + 1 partial bucket
    buckets, unfused = api.pack_gradients([TensorSpec((16,), "f32", True)] * 1000, mu=1024,
                                          chunk_size=4096)
    assert not unfused
    assert [b.total_bytes for b in buckets] == [4096] * 15 + [2560]
    assert [len(b.members) for b in buckets] == [64] * 15 + [40]


def test_node_tree_and_signatures_on_fixture():
    g = graph("graphs/tf24.json.gz")
    tree = api.build_node_tree(g)
    sigs = api.find_similar_blocks(tree, 2, g)
    assert max(c for _, c in sigs) == 24  # test_pruning.py:30-35


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_helpers_match_reference():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import shardplan
    from shardplan import patterns as P
    from shardplan.costmodel import collective_call_cost, collective_cost_bytes
    from shardplan.pruning import build_node_tree, find_similar_blocks
    from shardplan.rewrite import pack_gradients
    from randgraph import random_graph, to_reference

    from paper_2302_00247_b200.api_types import ClusterSpec, Collective, CollectiveKind, ShardSpec

    # node tree / signatures on random graphs
    for seed in range(6):
        g = random_graph(seed)
        rg = to_reference(g)
        t1, t2 = api.build_node_tree(g), build_node_tree(rg)
        assert t1.max_depth == t2.max_depth
        for d in range(1, t1.max_depth + 1):
            assert [(x.prefix, x.members) for x in t1.level(d)] == [(x.prefix, x.members)
                                                                  for x in t2.level(d)]
            assert api.find_similar_blocks(t1, d, g) == find_similar_blocks(t2, d, rg)
    # conversions and costs over every state pair, several meshes
    specs = [("replica", None), ("partial", None), ("split", 0), ("split", 1), ("split", -1)]
    for m, n, kw in ((1, 8, {}), (2, 4, {"inter_bw": 1e9}), (1, 1, {}), (2, 3, {})):
        mine, ref = ClusterSpec(m=m, n=n, **kw), shardplan.ClusterSpec(m=m, n=n, **kw)
        for kind in ("allreduce", "allgather", "reducescatter", "alltoall", "identity"):
            for nbytes in (1, 4096, 123456789):
                assert api.collective_cost_bytes(CollectiveKind(kind), nbytes, mine) == \
                    collective_cost_bytes(P.CollectiveKind(kind), nbytes, ref)
                assert api.collective_call_cost(Collective(CollectiveKind(kind)), nbytes, mine) == \
                    collective_call_cost(P.Collective(P.CollectiveKind(kind)), nbytes, ref)
    t = TensorSpec((8, 16, 32))
    rt = shardplan.TensorSpec((8, 16, 32))
    from shardplan.patterns import ShardKind as RK, ShardSpec as RS
    for a in specs:
        for b in specs:
            mine_a = ShardSpec(__import__("paper_2302_00247_b200.api_types", fromlist=["x"]).ShardKind(a[0]), a[1])
            mine_b = ShardSpec(type(mine_a.kind)(b[0]), b[1])
            try:
                exp = P.conversion_collective(RS(RK(a[0]), a[1]), RS(RK(b[0]), b[1]), rt)
                got = api.conversion_collective(mine_a, mine_b, t)
                assert (got.kind.value, got.axis) == (exp.kind.value, exp.axis)
            except shardplan.ShardplanError as exc:
                with pytest.raises(Exception) as info:
                    api.conversion_collective(mine_a, mine_b, t)
                assert type(info.value).__name__ == type(exc).__name__
    # gradient packing on random lists (criterion 6 style)
    rng = random.Random(0)
    for _ in range(200):
        sizes = [4 * rng.randint(1, 750) for _ in range(rng.randint(0, 40))]
        mu = rng.randint(1, 2048)
        chunk = mu * rng.randint(1, 8)
        gb, gu = api.pack_gradients([TensorSpec((s // 4,), "f32", True) for s in sizes], mu, chunk)
        rb, ru = pack_gradients([shardplan.TensorSpec((s // 4,), trainable=True) for s in sizes],
                                mu, chunk)
        assert [b.total_bytes for b in gb] == [b.total_bytes for b in rb]
        assert [u.byte_size for u in gu] == [u.byte_size for u in ru]
