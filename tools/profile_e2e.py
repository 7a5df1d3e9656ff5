"""cProfile of the c5 end-to-end step (derive_plan from host objects, cache=False)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
from paper_2302_00247_b200 import search as S  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
g, mesh = bench.load_workload(wl)
be = Backend(0)
be.set_mode("walk")
rep = None
for _ in range(3):
    rep = None
    rep = S.derive_plan(g, mesh, backend=be, cache=False)
ts = []
for _ in range(5):
    rep = None
    t0 = time.perf_counter()
    rep = S.derive_plan(g, mesh, backend=be, cache=False)
    ts.append((time.perf_counter() - t0) * 1e3)
print("e2e ms", [round(t, 2) for t in ts], S.LAST_PHASES)
pr = cProfile.Profile()
rep = None
pr.enable()
rep = S.derive_plan(g, mesh, backend=be, cache=False)
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(25)
