"""Blocks beyond the routing-table limits (template > 256 nodes, a node with
> 6 internal producers, tables larger than a CTA's shared memory) are searched
by the route search (sp_route_search): the plan must equal the oracle's, block
by block (the oracle is pinned to the reference on these graphs by
tests/test_limits_oracle.py), and replaying the plan must reproduce it."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["big_template", "wide_fanin", "heavy_tables"])
@pytest.mark.parametrize("mesh_name", ["1x8", "2x4"])
def test_route_search_matches_oracle(name, mesh_name):
    from limitgraphs import LIMIT_GRAPHS
    from oracle import oracle
    from paper_2302_00247_b200._native import default_backend
    from paper_2302_00247_b200.api_types import ClusterSpec
    from paper_2302_00247_b200.blocks import BlockArrays
    from paper_2302_00247_b200.search import (Session, _route_mask, derive_plan, fold_blocks,
                                              routed_plan_for_assignments)

    g = LIMIT_GRAPHS[name]()
    be = default_backend()
    ses = Session.open(g, be)
    m = ClusterSpec.from_mesh(mesh_name) if mesh_name == "1x8" else ClusterSpec(m=2, n=4, inter_bw=2e11 / 32)
    rep = derive_plan(g, m, session=ses)
    low = ses.low
    ba = fold_blocks(low, 2, session=ses)
    ob = BlockArrays.from_dict(oracle.prune(low, 2))
    assert ob.n_blocks == len(rep.results) == ba.n_blocks
    for b, res in enumerate(rep.results):
        exp, _ = oracle.score(low, ob.template_nodes(b), m, threads=8)
        assert (res.valid, res.best.plan.index, res.best.cost.total) == (exp.valid, exp.best_index, exp.best_total)
        assert res.candidates == exp.candidates
    if name != "heavy_tables":  # the smem overflow is found only once the tables exist
        assert _route_mask(low, ba.templates_csr()).any()
    rp = routed_plan_for_assignments(g, m, rep.assignments, session=ses)
    assert rp.total_cost == rep.total_cost
    for a, b in zip(rp.results, rep.results):
        assert a.best.routings == b.best.routings and a.best.cost == b.best.cost
