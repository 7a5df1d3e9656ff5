"""c5 prefix-skip search: median k_score_skip time (backend timings) over 10 steps."""
import os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench
from paper_2302_00247_b200 import search as S
from paper_2302_00247_b200._native import Backend
g, mesh = bench.load_workload("c5")
be = Backend(0)
be.set_mode("skip")
ses = S.Session.open(g, be)
ks = []
for i in range(13):
    rep = None
    rep = S.derive_plan(g, mesh, session=ses)
    if i >= 3:
        ks.append(be.timings()["score_kernel_ms"])
print(os.environ.get("SP_SKIP_TAIL", "0"), round(statistics.median(ks), 3), rep.valid, rep.total_cost)
