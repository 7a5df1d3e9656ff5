"""Per-rank step time of a strong-scaled c5 search, simulated on one GPU.

Every rank's share of an N-rank run (`shard=r, n_shards=N`, one after the
other) with the exchange replaced by a replay of the merged scores, i.e. everything
a rank does except the NCCL all_gather of the 40-byte block records; the step is the
slowest rank's.  As in the in-library multi-process form, only rank 0 assembles
the report (the others return once their share is scored and exchanged).  Shows
the kernel balance over ranks and where the fixed per-step host work caps
strong scaling.

    python tools/shard_sim.py [steps]
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import bench  # noqa: E402
from paper_2302_00247_b200 import search as S  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
g, mesh = bench.load_workload("c5")
be = Backend(0)
be.set_mode("walk")
ses = S.Session.open(g, be)
# the exchange returns what the all_gather + merge would: the global scores of
# each search (recorded once from an unsharded run, in call order)
recorded, calls = [], [0]


def record(scores):
    recorded.append(scores)
    return scores


def replay(scores):
    out = recorded[calls[0] % len(recorded)]
    calls[0] += 1
    return out


S.derive_plan(g, mesh, session=ses, exchange=record)
base = None
for n in (1, 2, 4, 8):
    ex = replay if n > 1 else None
    per = []
    for r in range(n):
        # ranks other than 0 skip the report (derive_plan's root_only, Backend.is_root)
        be.comm = dict(be.comm_info(), nranks=n, rank=r)
        for _ in range(2):
            S.derive_plan(g, mesh, session=ses, shard=r, n_shards=n, exchange=ex)
        ts, ks = [], []
        for _ in range(steps):
            t0 = time.perf_counter()
            S.derive_plan(g, mesh, session=ses, shard=r, n_shards=n, exchange=ex)
            ts.append((time.perf_counter() - t0) * 1e3)
            ks.append(be.timings()["score_kernel_ms"])
        per.append((statistics.median(ts), statistics.median(ks)))
    be.comm = be.comm_info()
    t = max(p[0] for p in per)
    base = base or t
    ks = [round(p[1], 2) for p in per]
    print(f"n_shards {n}: slowest rank step {t:.2f} ms (rank 0 {per[0][0]:.2f}, others "
          f"{max([p[0] for p in per[1:]] or [0]):.2f}), kernel per rank {ks}, "
          f"speed-up {base / t:.2f}x, phases {({k: (round(v, 2) if isinstance(v, float) else v) for k, v in S.LAST_PHASES.items()})}",
          flush=True)
