"""Minimal process for ncu captures: N derive_plan calls on a workload."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402
from paper_2302_00247_b200.search import Session, derive_plan  # noqa: E402

workload = sys.argv[1] if len(sys.argv) > 1 else "c5"
mode = sys.argv[2] if len(sys.argv) > 2 else "memo"
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2
be = Backend(0)
be.set_mode(mode)
g, mesh = bench.load_workload(workload)
ses = Session.open(g, be)
for _ in range(calls):
    rep = derive_plan(g, mesh, session=ses)
print(workload, mode, rep.candidates, rep.valid, be.timings())
