"""Goldens for weight specs that are not plain search options, from the reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_spec_golden.py

pattern_routing normalises a weight's assigned spec (ShardSpec.normalized,
patterns.py:44-50: a negative split axis counts from the weight's rank) and
skips every pattern whose spec cannot match (search.py:156-166), and
routed_plan_for_assignments replays stored labels such as "split-1"
(search.py:411-444).  For the c1 graph and two random graphs this records,
for plans built from edited labels: the reference's RoutingFailure (node,
reason) or the routed plan's (pattern, state) per node plus its plan_cost
JSON; and for the replay, the error (class, message) or the report JSON hash.
Written to tests/golden/spec_cases.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), f"{REF}/src"]
sys.dont_write_bytecode = True

from shardplan import derive_plan, prune_graph  # noqa: E402
from shardplan.costmodel import plan_cost  # noqa: E402
from shardplan.errors import ShardplanError  # noqa: E402
from shardplan.patterns import ShardSpec  # noqa: E402
from shardplan.search import (  # noqa: E402
    CandidatePlan,
    RoutingFailure,
    pattern_routing,
    routed_plan_for_assignments,
    weight_nodes,
)

from golden_io import case  # noqa: E402
from randgraph import random_graph, to_reference  # noqa: E402

EDITS = ("split-1", "split-1", "split-1", "split-2", "split-2", "split-3", "split2", "split5", "partial", "replica",
         "split0", "split1")


def canon(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def ref_graph(src):
    if isinstance(src, str):
        from golden_io import graph

        return to_reference(graph(src))
    return to_reference(src)


def routed_doc(routed) -> dict:
    if isinstance(routed, RoutingFailure):
        return {"fail": [routed.node, routed.reason]}
    return {"routes": [[r.scope, r.pattern, r.state.label] for r in routed.routings],
            "exits": [[s, c.kind.value] for s, c, _ in routed.exit_conversions]}


def main() -> None:
    from shardplan import ClusterSpec

    out = []
    c1 = case("c1_1x8")
    sources = [("c1_1x8", c1["graph"], c1["mesh"]), ("rand3", random_graph(3), c1["mesh"]),
               ("rand11", random_graph(11), c1["mesh"])]
    for name, src, mdoc in sources:
        g = ref_graph(src)
        m = ClusterSpec.from_json(mdoc)
        rng = random.Random(name)
        rep = derive_plan(g, m)
        subs = prune_graph(g, 2)
        routes = []
        for b, sub in enumerate(subs):
            scopes = weight_nodes(g, sub)
            if not scopes:
                continue
            best = dict(rep.results[b].best.plan.assignments)
            for _ in range(6):
                labels = {s: best[s].label for s in scopes}
                for s in rng.sample(scopes, min(len(scopes), rng.randint(1, 2))):
                    labels[s] = rng.choice(EDITS)
                plan = CandidatePlan(sub, tuple((s, ShardSpec.from_label(labels[s])) for s in scopes), -1)
                routed = pattern_routing(g, plan, m)
                doc = {"block": b, "labels": labels, **routed_doc(routed)}
                if not isinstance(routed, RoutingFailure):
                    doc["cost"] = plan_cost(routed, g, m).to_json()
                routes.append(doc)
        replays = []
        for k in range(16):
            asg = dict(rep.assignments)
            # the same edit on every instance of a block (replay requires it)
            for res in rep.results:
                sub = res.subgraph
                for scope, spec in res.best.plan.assignments:
                    if rng.random() < 0.06:
                        lab = rng.choice(EDITS)
                        for prefix, _ in sub.instances:
                            asg[sub.instance_node(prefix, scope)] = lab
            try:
                rp = routed_plan_for_assignments(g, m, asg)
                replays.append({"assignments": asg, "plan_sha": hashlib.sha256(canon(rp.to_json()).encode()).hexdigest(),
                                "total_cost": repr(rp.total_cost)})
            except ShardplanError as exc:
                replays.append({"assignments": asg, "error": [type(exc).__name__, str(exc)]})
        out.append({"name": name, "graph": src if isinstance(src, str) else None,
                    "random_seed": None if isinstance(src, str) else int(name[4:]), "mesh": mdoc,
                    "routes": routes, "replays": replays})
    with open(os.path.join(HERE, "spec_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_spec_golden.py", "reference": "shardplan 0.1.0",
                   "cases": out}, fh, indent=0, sort_keys=True)
        fh.write("\n")
    n_fail = sum("fail" in r for c in out for r in c["routes"])
    n_err = sum("error" in r for c in out for r in c["replays"])
    print(f"{sum(len(c['routes']) for c in out)} routes ({n_fail} failures), "
          f"{sum(len(c['replays']) for c in out)} replays ({n_err} errors)")


if __name__ == "__main__":
    main()
