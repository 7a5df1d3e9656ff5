"""Kernel-only timing of c5 scoring in each mode (development A/B helper).
usage: SP_LIB=path/to/lib.so python tools/kbench.py [modes...]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402
from paper_2302_00247_b200.search import Session, fold_blocks  # noqa: E402

modes = sys.argv[1:] or ["walk", "skip"]
be = Backend(0)
g, mesh = bench.load_workload("c5")
ses = Session.open(g, be)
ba = fold_blocks(ses.low, 2, session=ses)
off, nodes = ba.templates_csr()
t = be.tables(ses.dgraph, off, nodes, mesh, 1 << 20, 4 << 20)
for mode in modes:
    be.set_mode(mode)
    ks = []
    for _ in range(5):
        res = be.score(t)
        ks.append(be.timings()["score_kernel_ms"])
    print(os.environ.get("SP_LIB", "default"), mode, "kernel ms", sorted(ks)[len(ks) // 2],
          "valid", sum(r.valid for r in res), flush=True)
