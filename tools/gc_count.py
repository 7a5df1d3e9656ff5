import gc, os, sys, time, collections
ROOT = "/root/repo"
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench
from paper_2302_00247_b200 import search as S
from paper_2302_00247_b200._native import Backend
g, mesh = bench.load_workload("c5")
be = Backend(0); be.set_mode("walk")
ses = S.Session.open(g, be)
rep = S.derive_plan(g, mesh, session=ses)
rep = None
gc.collect()
before = set(id(o) for o in gc.get_objects())
gc.disable()
rep = S.derive_plan(g, mesh, session=ses)
objs = [o for o in gc.get_objects() if id(o) not in before]
cnt = collections.Counter(type(o).__name__ for o in objs)
print("new tracked objects", len(objs), cnt.most_common(15))
t0 = time.perf_counter(); gc.collect(0); print("gen0 collect ms", (time.perf_counter()-t0)*1e3)
before = None
refs = [(len(gc.get_referents(o)), type(o).__name__) for o in objs]
byt = collections.Counter()
for r, t in refs:
    byt[t] += r
print("referents by type", byt.most_common(8))
sub = rep.results[0].subgraph
print("subgraph fields", {k: (type(v).__name__, len(v) if hasattr(v, '__len__') else None) for k, v in vars(sub).items()} if hasattr(sub, '__dict__') else type(sub))
rp = rep.results[0].best
print("routed fields", {k: (type(v).__name__, len(v) if hasattr(v, '__len__') else None) for k, v in vars(rp).items()} if hasattr(rp, '__dict__') else type(rp))
refs.sort(reverse=True)
print("total referents", sum(r for r, _ in refs), "largest", refs[:8])
print("assignments type", type(rep.assignments), len(rep.assignments), gc.is_tracked(rep.assignments),
      type(next(iter(rep.assignments.values()))))
gc.disable()
rep = None
rep = S.derive_plan(g, mesh, session=ses)
a = rep.assignments
t0 = time.perf_counter(); gc.collect(0); print("gen0 collect again ms", (time.perf_counter()-t0)*1e3)
