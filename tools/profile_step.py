"""Host-side profile of one c2 derive_plan step (cProfile + per-phase wall times)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from paper_2302_00247_b200._native import Backend  # noqa: E402
from paper_2302_00247_b200.api_types import ClusterSpec  # noqa: E402
from paper_2302_00247_b200.ir import load_grouped  # noqa: E402
from paper_2302_00247_b200.search import Session, derive_plan  # noqa: E402

g = load_grouped(os.path.join(ROOT, "tests/golden/graphs/c2_t5.json.gz"))
mesh = ClusterSpec.from_mesh("1x8")
be = Backend(0)
ses = Session.open(g, be)
for _ in range(10):
    derive_plan(g, mesh, session=ses)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
t0 = time.perf_counter()
for _ in range(N):
    derive_plan(g, mesh, session=ses)
print(f"resident step: {(time.perf_counter() - t0) / N * 1e3:.3f} ms")
t0 = time.perf_counter()
for _ in range(N):
    derive_plan(g, mesh, backend=be, cache=False)
print(f"e2e step: {(time.perf_counter() - t0) / N * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    derive_plan(g, mesh, session=ses)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    derive_plan(g, mesh, backend=be, cache=False)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
