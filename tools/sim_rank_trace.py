"""One simulated rank of an N-rank c5 search with the library's traces on
(SP_TRACE host phases, SP_SCORE_TRACE device phases per search).

    SP_TRACE=1 SP_SCORE_TRACE=1 python tools/sim_rank_trace.py RANK N
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import bench  # noqa: E402
from paper_2302_00247_b200 import search as S  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402

r, n = int(sys.argv[1]), int(sys.argv[2])
g, mesh = bench.load_workload("c5")
be = Backend(0)
be.set_mode("walk")
ses = S.Session.open(g, be)
be.comm = dict(be.comm_info(), nranks=n, rank=r)
be.set_sim_shard(r, n)
kept = []
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
for i in range(steps):
    if i == steps - 1:
        print("---- traced step", file=sys.stderr, flush=True)
    rep = None
    t0 = time.perf_counter()
    rep = S.derive_plan(g, mesh, session=ses)
    dt = (time.perf_counter() - t0) * 1e3
    if not os.environ.get("SP_TRACE"):
        print(f"step {i}: {dt:.2f} ms", S.LAST_PHASES.get("groups_at_ms"), round(be.timings()["score_kernel_ms"], 3),
              file=sys.stderr)
print(f"rank {r}/{n}: step {dt:.2f} ms", S.LAST_PHASES, be.timings(), file=sys.stderr)
