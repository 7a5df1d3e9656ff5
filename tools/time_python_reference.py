"""Time the REFERENCE itself (shardplan, pure Python) on this host: the second
CPU baseline of bench.py.

    python tools/time_python_reference.py [--budget-s 40]

Imports the unmodified reference from baseline/_ref (tools/install_reference.sh;
it travels to the GPU box with the repo, /root/reference does not) and times,
on the configs BASELINE.json names:
  * derive_plan(graph, mesh, jobs=1) and jobs=os.cpu_count() (the reference's
    own ProcessPool range split, search.py:327-343) on c1, c3 (2x4, slow inter
    link) and c4 -- whole searches;
  * the c5 throughput tier's largest block (3,486,784,401 candidates; the
    reference would need days) on fixed slices [k*C/8, k*C/8 + W), k = 0..7,
    with _eval_range (search.py:289-310): sequentially (1 core) and as one
    ProcessPool map over the slices (all cores);
and prints one JSON object.  The graphs are handed to the reference as its
own ModelGraph of GraphNodes (tests/randgraph.to_reference).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path[:0] = [REF, ROOT, os.path.join(ROOT, "tests")]
sys.dont_write_bytecode = True

_G = {}


def _slice(args):
    from shardplan.search import _eval_range

    lo, hi = args
    g, sub, mesh = _G["c5"]
    t0 = time.perf_counter()
    _, key, valid, _ = _eval_range((g, sub, mesh, 1 << 20, 4 << 20, lo, hi, False))
    return hi - lo, valid, time.perf_counter() - t0


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--slice", type=int, default=2048, help="candidates per c5 slice")
    args = ap.parse_args()
    if not os.path.isdir(os.path.join(REF, "shardplan")):
        print(json.dumps({"unavailable": "baseline/_ref not installed (tools/install_reference.sh)"}))
        return
    import shardplan
    from shardplan import ClusterSpec, derive_plan, prune_graph
    from shardplan.search import count_candidates

    from paper_2302_00247_b200.ir import load_grouped
    from paper_2302_00247_b200.workloads import motif_dag
    from randgraph import to_reference

    cores = os.cpu_count() or 1
    gold = os.path.join(ROOT, "tests", "golden", "graphs")
    out = {"reference": f"shardplan {shardplan.__version__} (baseline/_ref, unmodified)", "cores": cores,
           "python": sys.version.split()[0], "configs": {}}
    for name, path, mesh in (("c1", "c1.json.gz", ClusterSpec.from_mesh("1x8")),
                             ("c3_slow", "c3.json.gz", ClusterSpec(m=2, n=4, inter_bw=2e11 / 32)),
                             ("c4", "c4.json.gz", ClusterSpec.from_mesh("1x8"))):
        g = to_reference(load_grouped(os.path.join(gold, path)))
        row = {}
        for jobs in (1, cores):
            derive_plan(g, mesh, jobs=jobs)  # warm (imports, pool start-up paths)
            reps, t0 = 0, time.perf_counter()
            while reps < 3 or time.perf_counter() - t0 < 0.5:
                rep = derive_plan(g, mesh, jobs=jobs)
                reps += 1
                if reps >= 20:
                    break
            dt = (time.perf_counter() - t0) / reps
            row[f"jobs{jobs}"] = {"ms_per_search": dt * 1e3, "candidates": rep.candidates,
                                  "candidates_per_s": rep.candidates / dt, "total_cost": repr(rep.total_cost)}
        out["configs"][name] = row
    # c5: slices of the largest block
    g = to_reference(motif_dag(0, "throughput"))
    mesh = ClusterSpec.from_mesh("1x8")
    t0 = time.perf_counter()
    subs = prune_graph(g, 2)
    prune_s = time.perf_counter() - t0
    big = max(subs, key=lambda s: count_candidates(g, s))
    C = count_candidates(g, big)
    _G["c5"] = (g, big, mesh)
    tasks = [(k * C // 8, k * C // 8 + args.slice) for k in range(8)]
    t0 = time.perf_counter()
    seq = [_slice(t) for t in tasks]
    t_seq = time.perf_counter() - t0
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=min(cores, len(tasks))) as pool:  # fork: _G is inherited
        par = list(pool.map(_slice, tasks))
    t_par = time.perf_counter() - t0
    walked = sum(x[0] for x in seq)
    assert [x[1] for x in seq] == [x[1] for x in par]
    out["c5_slices"] = {"block_candidates": C, "slices": f"8 x {args.slice} candidates at k*C/8",
                        "prune_graph_s": prune_s, "walked": walked, "valid": sum(x[1] for x in seq),
                        "jobs1_candidates_per_s": walked / t_seq,
                        f"jobs{min(cores, len(tasks))}_candidates_per_s": walked / t_par,
                        "extrapolated_full_block_hours_jobs1": C / (walked / t_seq) / 3600}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
