"""Whole-plan golden for the BENCH config (c5 throughput tier), from the reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_c5_full.py

The c5 throughput tier (motif_dag(0, "throughput"): 1018 blocks, 3,918,656,938
candidates) is what bench.py times.  Its three big blocks (43,046,721,
387,420,489 and 3,486,784,401 candidates) are out of reach of the reference's
Python search (~5e3 candidates/s/core), so the whole-plan golden is built in
two halves:

* every block with <= 2e6 candidates (1015 blocks, 1.4M candidates) is searched
  by the reference itself: shardplan.search.search_subgraph (search.py:317-345,
  the ProcessPool range split with jobs=cores);
* the three big blocks are searched by the CPU oracle (oracle/oracle.c, a plain-C
  restatement of _eval_range, search.py:289-310, parity-pinned to the reference
  by tests/test_oracle*.py), brute force on every candidate.  The oracle's
  winning index is then handed back to the REFERENCE, which rebuilds the
  winner with its own candidate_by_index + pattern_routing + plan_cost
  (search.py:103-116, 134-224, costmodel.py:193-267) and checks the oracle's
  total and num_split against it.  The oracle also re-searches every small
  block, and must agree with the reference there.

The report is then assembled exactly like derive_plan does (search.py:362-379)
from reference SubgraphResults, and the sha256 of its to_json() is recorded.
Written to tests/golden/c5_full.json.  Takes ~4 min on 8 cores.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), f"{REF}/src"]
sys.dont_write_bytecode = True

from shardplan import ClusterSpec, prune_graph  # noqa: E402
from shardplan.costmodel import plan_cost  # noqa: E402
from shardplan.search import (  # noqa: E402
    BestPlanReport,
    RoutedPlan,
    RoutingFailure,
    SubgraphResult,
    candidate_by_index,
    count_candidates,
    pattern_routing,
    search_subgraph,
)

from oracle import oracle  # noqa: E402
from paper_2302_00247_b200.blocks import BlockArrays, to_prune_doc  # noqa: E402
from paper_2302_00247_b200.lowering import lower  # noqa: E402
from paper_2302_00247_b200.workloads import motif_dag  # noqa: E402
from randgraph import to_reference  # noqa: E402

BIG = 2_000_000


def canon(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def sha(obj) -> str:
    return hashlib.sha256(canon(obj).encode()).hexdigest()


def prune_doc(subs) -> list:
    return [[s.template_prefix, list(s.template), [[p, list(m)] for p, m in s.instances]]
            for s in subs]


def main() -> None:
    threads = os.cpu_count() or 8
    mesh = ClusterSpec.from_mesh("1x8")
    from golden_io import mesh as mesh_of

    omesh = mesh_of(mesh.to_json())
    g = motif_dag(0, "throughput")
    rg = to_reference(g)
    t0 = time.perf_counter()
    subs = prune_graph(rg, 2)
    low = lower(g)
    ob = BlockArrays.from_dict(oracle.prune(low, 2))
    assert to_prune_doc(low, ob) == prune_doc(subs), "oracle fold != reference fold"
    print(f"prune {time.perf_counter() - t0:.1f}s, {len(subs)} blocks", flush=True)

    results, blocks = [], []
    for b, sub in enumerate(subs):
        C = count_candidates(rg, sub)
        t1 = time.perf_counter()
        exp, _ = oracle.score(low, ob.template_nodes(b), omesh, threads=threads)
        t_oracle = time.perf_counter() - t1
        if C <= BIG:
            res = search_subgraph(rg, sub, mesh, jobs=threads if C >= 4096 else 1)
            by = "reference"
        else:
            plan = candidate_by_index(rg, sub, exp.best_index)
            routed = pattern_routing(rg, plan, mesh)
            assert not isinstance(routed, RoutingFailure), f"block {b}: oracle winner does not route"
            cost = plan_cost(routed, rg, mesh, mu=1 << 20, chunk_size=4 << 20)
            best = RoutedPlan(routed.plan, routed.routings, routed.exit_conversions, cost)
            res = SubgraphResult(sub, best, C, exp.valid, [])
            by = "oracle argmin, rebuilt by the reference"
            print(f"  block {b}: {C} candidates, oracle {t_oracle:.1f}s on {threads} threads, "
                  f"best {exp.best_index} valid {exp.valid}", flush=True)
        key = (res.best.cost.total, res.best.plan.num_split, res.best.plan.index)
        assert (exp.valid, exp.best_total, exp.best_num_split, exp.best_index) == (
            res.valid, *key), f"block {b}: oracle {exp} != reference {key}"
        results.append(res)
        blocks.append([res.best.plan.index, res.best.plan.num_split, repr(res.best.cost.total),
                       res.valid, C, by])

    # derive_plan's assembly (search.py:362-379), on the reference's own objects
    assignments, total_cost, candidates, valid = {}, 0.0, 0, 0
    for res in results:
        sub = res.subgraph
        candidates += res.candidates
        valid += res.valid
        total_cost += res.best.cost.total * sub.multiplicity
        for prefix, _ in sub.instances:
            for scope, spec in res.best.plan.assignments:
                assignments[sub.instance_node(prefix, scope)] = spec.label
    rep = BestPlanReport(mesh, 2, results, assignments, total_cost, candidates, valid)
    doc = {
        "generator": "tests/golden/make_golden_c5_full.py",
        "reference": "shardplan 0.1.0",
        "workload": "motif_dag(0, 'throughput'), mesh 1x8, min_dup 2, mu 1 MiB, chunk 4 MiB",
        "plan_sha": sha(rep.to_json()),
        "total_cost": repr(total_cost),
        "candidates": candidates,
        "valid": valid,
        "blocks": blocks,
        "seconds": round(time.perf_counter() - t0, 1),
        "threads": threads,
    }
    with open(os.path.join(HERE, "c5_full.json"), "w") as fh:
        json.dump(doc, fh, indent=0, sort_keys=True)
        fh.write("\n")
    print(f"done in {doc['seconds']}s: plan {doc['plan_sha'][:16]} total {total_cost!r} valid {valid}")


if __name__ == "__main__":
    main()
