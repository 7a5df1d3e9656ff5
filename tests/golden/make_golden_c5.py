"""Config-5 goldens (10^5-op motif DAG) from the reference itself.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_c5.py

The graph is produced by paper_2302_00247_b200.workloads.motif_dag (the
reference has no such generator); it is handed to the reference
as a ModelGraph of its own GraphNodes, and every expectation below comes from
the reference's prune_graph / derive_plan / _eval_range.  Only hashes,
per-block summaries and per-candidate slices are committed (tests/golden/c5.json).
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

from shardplan import ClusterSpec, derive_plan, prune_graph  # noqa: E402
from shardplan.search import _eval_range, count_candidates  # noqa: E402

from paper_2302_00247_b200.ir import dump_grouped  # noqa: E402
from paper_2302_00247_b200.workloads import motif_dag  # noqa: E402
from randgraph import to_reference  # noqa: E402


def canon(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def sha(obj) -> str:
    return hashlib.sha256(canon(obj).encode()).hexdigest()


def prune_doc(subs) -> list:
    return [[s.template_prefix, list(s.template), [[p, list(m)] for p, m in s.instances]]
            for s in subs]


def main() -> None:
    out = []
    mesh = ClusterSpec.from_mesh("1x8")
    for seed, tier in ((0, "parity"), (0, "throughput"), (1, "parity"), (2, "parity")):
        t0 = time.perf_counter()
        g = motif_dag(seed, tier)
        rg = to_reference(g)
        subs = prune_graph(rg, 2)
        entry = {"tier": tier, "seed": seed, "nodes": len(g.nodes), "graph_sha": sha(dump_grouped(g)),
                 "prune_sha": sha(prune_doc(subs)), "blocks": len(subs),
                 "candidates": [count_candidates(rg, s) for s in subs], "mesh": mesh.to_json()}
        print(f"{tier} seed {seed}: {len(g.nodes)} nodes, {len(subs)} blocks, prune {time.perf_counter() - t0:.1f}s",
              flush=True)
        if tier == "parity":
            t1 = time.perf_counter()
            rep = derive_plan(rg, mesh, jobs=os.cpu_count() or 8)
            entry["plan_sha"] = sha(rep.to_json())
            entry["total_cost"] = repr(rep.total_cost)
            entry["valid"] = rep.valid
            entry["best"] = [[r.best.plan.index, r.best.plan.num_split, repr(r.best.cost.total), r.valid]
                             for r in rep.results]
            entry["ref_search_seconds"] = round(time.perf_counter() - t1, 1)
            print(f"  derive_plan {time.perf_counter() - t1:.1f}s", flush=True)
        slices = []
        big = sorted(range(len(subs)), key=lambda i: -entry["candidates"][i])[:3]
        for b in big:
            C = entry["candidates"][b]
            for k in range(8):
                lo = k * C // 8
                hi = min(C, lo + 256)
                _, _, valid, table = _eval_range((rg, subs[b], mesh, 1 << 20, 4 << 20, lo, hi, True))
                slices.append({"block": b, "lo": lo, "hi": hi, "totals": [r[2] for r in table]})
        entry["slices"] = slices
        out.append(entry)
        print(f"  {tier} done in {time.perf_counter() - t0:.1f}s", flush=True)
    with open(os.path.join(HERE, "c5.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_c5.py", "reference": "shardplan 0.1.0",
                   "c5": out}, fh, indent=1, sort_keys=True)
        fh.write("\n")


if __name__ == "__main__":
    main()
