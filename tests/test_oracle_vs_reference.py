"""Pin the oracle against the live reference on seeded random graphs.

Runs only where the reference is importable (the build container); the
committed goldens (test_oracle.py) pin the same functions everywhere else.
"""

from __future__ import annotations

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import shardplan  # noqa: F401
    from shardplan import ClusterSpec, prune_graph
    from shardplan.search import _eval_range, count_candidates

    return ClusterSpec, prune_graph, _eval_range, count_candidates


MESHES = [("1x4", {}), ("2x4", {}), ("1x2", {"intra_bw": float("inf"), "setup_latency_s": 0.0}),
          ("1x1", {}), ("2x3", {"inter_bw": 1e9})]


@pytest.mark.parametrize("seed", range(24))
def test_random_graph_prune_and_score(ref, seed):
    from oracle import oracle
    from paper_2302_00247_b200.api_types import ClusterSpec as MyCS
    from paper_2302_00247_b200.blocks import BlockArrays, to_prune_doc
    from paper_2302_00247_b200.lowering import lower
    from randgraph import random_graph, to_reference

    ClusterSpec, prune_graph, _eval_range, count_candidates = ref
    g = random_graph(seed)
    rg = to_reference(g)
    assert list(rg.topo_order) == list(g.topo_order)
    low = lower(g)
    for md in (1, 2, 3):
        try:
            subs = prune_graph(rg, md)
        except TypeError:  # divergence trap D2 (pruning.py:165)
            continue
        doc = [[s.template_prefix, list(s.template), [[p, list(m)] for p, m in s.instances]]
               for s in subs]
        ba = BlockArrays.from_dict(oracle.prune(low, md))
        assert to_prune_doc(low, ba) == doc
    subs = prune_graph(rg, 2)
    ba = BlockArrays.from_dict(oracle.prune(low, 2))
    mname, kw = MESHES[seed % len(MESHES)]
    rm, mm = ClusterSpec.from_mesh(mname, **kw), MyCS.from_mesh(mname, **kw)
    for b, s in enumerate(subs):
        C = count_candidates(rg, s)
        if C > 800:
            continue
        _, key, valid, table = _eval_range((rg, s, rm, 1 << 20, 4 << 20, 0, C, True))
        out, totals = oracle.score(low, ba.template_nodes(b), mm, hi=C, want_totals=True)
        assert out.valid == valid
        assert [None if t != t else t for t in totals.tolist()] == [r[2] for r in table]
        if key is None:
            assert not out.has_best
        else:
            assert key == (out.best_total, out.best_num_split, out.best_index)
