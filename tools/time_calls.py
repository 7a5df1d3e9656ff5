"""Per-call host time of the backend entry points on a small config (c1/c3/c4).

    python tools/time_calls.py c1 [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402
from paper_2302_00247_b200.search import Session, derive_plan  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g, mesh = bench.load_workload(w)
be = Backend(0)
be.set_mode("walk")
ses = Session.open(g, be)
acc = {}


def tick(name, t0):
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0


for i in range(reps + 20):
    if i == 20:
        acc.clear()
    t0 = time.perf_counter()
    ba = be.fold(ses.dgraph, 2)
    tick("fold", t0)
    t0 = time.perf_counter()
    off, nodes = ba.templates_csr()
    tick("templates_csr", t0)
    t0 = time.perf_counter()
    t = be.tables(ses.dgraph, off, nodes, mesh, 1 << 20, 4 << 20)
    tick("tables", t0)
    t0 = time.perf_counter()
    be.score_launch(t, 0, 1, explain=True)
    tick("score_launch", t0)
    t0 = time.perf_counter()
    be.score_wait(t)
    tick("score_wait", t0)
    t0 = time.perf_counter()
    t.close()
    tick("close", t0)
    t0 = time.perf_counter()
    derive_plan(g, mesh, session=ses)
    tick("derive_plan", t0)
print(w, {k: round(v / reps * 1e3, 4) for k, v in acc.items()}, "ms per call")
