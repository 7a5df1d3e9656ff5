"""The CPU oracle on graphs beyond the table path's limits, against the live
reference (here, where /root/reference exists): it is the checker of the
route search in tests/test_gpu_limits.py."""

from __future__ import annotations

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.mark.parametrize("name", ["big_template", "wide_fanin", "heavy_tables"])
def test_oracle_matches_reference_beyond_table_limits(name):
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    from shardplan import ClusterSpec, derive_plan

    from golden_io import mesh as mesh_of
    from limitgraphs import LIMIT_GRAPHS
    from oracle import oracle
    from paper_2302_00247_b200.blocks import BlockArrays
    from paper_2302_00247_b200.lowering import lower
    from randgraph import to_reference

    g = LIMIT_GRAPHS[name]()
    low = lower(g)
    m = ClusterSpec.from_mesh("1x8")
    rep = derive_plan(to_reference(g), m)
    ob = BlockArrays.from_dict(oracle.prune(low, 2))
    assert ob.n_blocks == len(rep.results)
    om = mesh_of(m.to_json())
    for b, res in enumerate(rep.results):
        exp, _ = oracle.score(low, ob.template_nodes(b), om, threads=4)
        assert (exp.valid, exp.best_index, exp.best_total) == (res.valid, res.best.plan.index, res.best.cost.total)
