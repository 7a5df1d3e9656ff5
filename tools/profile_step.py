"""Host-side profile of one derive_plan step (cProfile + per-phase wall times).

    python tools/profile_step.py [c5|c2] [steps]
"""
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

workload = sys.argv[1] if len(sys.argv) > 1 else "c5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mode = sys.argv[3] if len(sys.argv) > 3 else "walk"
g, mesh = bench.load_workload(workload)
be = Backend(0)
be.set_mode(mode)
ses = S.Session.open(g, be)
for _ in range(3):
    S.derive_plan(g, mesh, session=ses)
t0 = time.perf_counter()
for _ in range(N):
    S.derive_plan(g, mesh, session=ses)
print(f"resident step: {(time.perf_counter() - t0) / N * 1e3:.3f} ms", S.LAST_PHASES, be.timings())
t0 = time.perf_counter()
for _ in range(N):
    S.derive_plan(g, mesh, backend=be, cache=False)
print(f"e2e step: {(time.perf_counter() - t0) / N * 1e3:.3f} ms", S.LAST_PHASES)
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    S.derive_plan(g, mesh, session=ses)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    S.derive_plan(g, mesh, backend=be, cache=False)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
