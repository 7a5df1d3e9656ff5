import os, sys
sys.path[:0]=["/root/repo", "/root/repo/tests"]
import bench
from paper_2302_00247_b200 import search as S
from paper_2302_00247_b200._native import Backend
wl = sys.argv[1]
g, mesh = bench.load_workload(wl)
be = Backend(0)
ses = S.Session.open(g, be)
for _ in range(30): S.derive_plan(g, mesh, session=ses)
sys.stderr.write("=== steady\n"); sys.stderr.flush()
for _ in range(3): S.derive_plan(g, mesh, session=ses)
