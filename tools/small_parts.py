import os, sys, time
ROOT="/root/repo"; sys.path[:0]=[ROOT, os.path.join(ROOT,"tests")]
import numpy as np
import bench
from paper_2302_00247_b200 import search as S
from paper_2302_00247_b200._native import Backend
from paper_2302_00247_b200.api_types import DEFAULT_TYPES as types
wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
g, mesh = bench.load_workload(wl)
be = Backend(0)
ses = S.Session.open(g, be)
for _ in range(50): S.derive_plan(g, mesh, session=ses)
N=2000
acc = {}
def tick(k, t): acc[k] = acc.get(k, 0.0) + t
for _ in range(N):
    t0=time.perf_counter()
    ba, csr, scores, detail = ses.backend.plan(ses.dgraph, 2, mesh, 1<<20, 4<<20)
    t1=time.perf_counter(); tick("plan", t1-t0)
    low = ses.low
    subs = S.subgraphs_from_blocks(low, ba, types); t2=time.perf_counter(); tick("subgraphs", t2-t1)
    slots = S.Slots.of(low, csr); t3=time.perf_counter(); tick("slots", t3-t2)
    mult = np.diff(np.asarray(ba.block_inst_off, np.int64))
    native = S._native_results(ses, subs, scores, detail, csr, slots, mult, mesh, types); t4=time.perf_counter(); tick("native_results", t4-t3)
    results, terms, labs = native
    off = slots.off
    slot_labels = [lab for b, ls in enumerate(labs) if off[b + 1] > off[b] for lab in ls]
    lk = S._label_keys(ba, subs, slots); t5=time.perf_counter(); tick("label_keys", t5-t4)
    assignments = S._assignments(low.names, lk, slot_labels); t6=time.perf_counter(); tick("assignments", t6-t5)
    rep = types.BestPlanReport(mesh, 2, results, assignments, 0.0, 0, 0); t7=time.perf_counter(); tick("report", t7-t6)
print(wl, {k: round(v/N*1e6,1) for k,v in acc.items()}, "us")
t0=time.perf_counter()
for _ in range(N): S.derive_plan(g, mesh, session=ses)
print("derive_plan", round((time.perf_counter()-t0)/N*1e6,1), "us")
