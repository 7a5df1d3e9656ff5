"""Fold the c5 workload (motif_dag(0, "throughput"), 99,658 GraphNodes) `reps` times.

    python tools/fold_c5.py [reps]        (for ncu launch lists of the medium-size fold)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_00247_b200._native import Backend  # noqa: E402
from paper_2302_00247_b200.lowering import lower  # noqa: E402
from paper_2302_00247_b200.search import Session  # noqa: E402
from paper_2302_00247_b200.workloads import motif_dag  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
be = Backend(0)
ses = Session.open(lower(motif_dag(0, "throughput")), be)
be.fold(ses.dgraph, 2)
t0 = time.perf_counter()
for _ in range(reps):
    ba = be.fold(ses.dgraph, 2)
print(f"fold {((time.perf_counter() - t0) / reps) * 1e3:.3f} ms wall, {ba.n_blocks} blocks", be.timings())
