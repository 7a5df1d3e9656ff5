"""Weight specs outside the plain search options, on the device, vs the reference.

Goldens from tests/golden/make_spec_golden.py (the reference's pattern_routing,
plan_cost and routed_plan_for_assignments on edited labels: negative split
axes that normalise to an option, axes out of range, partial, split axes
beyond the options).  A negative axis must route exactly like its normalised
form (ShardSpec.normalized, patterns.py:44-50); a spec no weight pattern can
match must fail at the first failing node in topological order with the
reference's reason (search.py:156-199); the replay must keep the stored specs
and raise the reference's message (search.py:431-434).
"""

from __future__ import annotations

import functools
import hashlib
import json
import os

import pytest

from golden_io import GOLDEN, graph, mesh

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=1)
def _doc():
    with open(os.path.join(GOLDEN, "spec_cases.json")) as fh:
        return json.load(fh)["cases"]


def _graph(c):
    if c["graph"]:
        return graph(c["graph"])
    from randgraph import random_graph

    return random_graph(c["random_seed"])


def canon(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


@pytest.mark.parametrize("name", ["c1_1x8", "rand3", "rand11"])
def test_pattern_routing_edited_specs(name):
    from paper_2302_00247_b200._native import default_backend
    from paper_2302_00247_b200.api_types import CandidatePlan, RoutingFailure, ShardSpec
    from paper_2302_00247_b200.search import Session, pattern_routing, plan_cost, prune_graph

    c = next(x for x in _doc() if x["name"] == name)
    g, m = _graph(c), mesh(c["mesh"])
    ses = Session.open(g, default_backend())
    subs = prune_graph(g, 2, session=ses)
    for r in c["routes"]:
        sub = subs[r["block"]]
        plan = CandidatePlan(sub, tuple((s, ShardSpec.from_label(lab)) for s, lab in sorted(r["labels"].items())), -1)
        routed = pattern_routing(g, plan, m, session=ses)
        if "fail" in r:
            assert isinstance(routed, RoutingFailure), r["labels"]
            assert [routed.node, routed.reason] == r["fail"], r["labels"]
            continue
        assert not isinstance(routed, RoutingFailure), (r["labels"], routed)
        assert routed.plan is plan
        assert [[x.scope, x.pattern, x.state.label] for x in routed.routings] == r["routes"]
        assert [[s, coll.kind.value] for s, coll, _ in routed.exit_conversions] == r["exits"]
        assert canon(plan_cost(routed, g, m, session=ses).to_json()) == canon(r["cost"])


@pytest.mark.parametrize("name", ["c1_1x8", "rand3", "rand11"])
def test_replay_edited_labels(name):
    from paper_2302_00247_b200._native import default_backend
    from paper_2302_00247_b200.errors import ShardplanError
    from paper_2302_00247_b200.search import Session, routed_plan_for_assignments

    c = next(x for x in _doc() if x["name"] == name)
    g, m = _graph(c), mesh(c["mesh"])
    ses = Session.open(g, default_backend())
    for r in c["replays"]:
        if "error" in r:
            with pytest.raises(ShardplanError) as ei:
                routed_plan_for_assignments(g, m, r["assignments"], session=ses)
            assert [type(ei.value).__name__, str(ei.value)] == r["error"]
        else:
            rp = routed_plan_for_assignments(g, m, r["assignments"], session=ses)
            assert hashlib.sha256(canon(rp.to_json()).encode()).hexdigest() == r["plan_sha"]
            assert repr(rp.total_cost) == r["total_cost"]
