"""Per-rank step time of a strong-scaled c5 search, simulated on one GPU.

The in-library multi-process form (one process per GPU, NCCL inside
libshardsearch): every rank folds, builds the tables and scores its
round-robin share of every block's work items; one ncclAllGather of the
40-byte block records and k_merge_ranks follow on the device, and the winner
detail is chained behind the merge, so the Python flow is the one-GPU flow.
Here each rank's share runs in turn on one GPU (SP_OPT_SIM_SHARD: the share's
winners stand in for the merged ones, the same kernels on the same sizes) and
only rank 0 assembles the report (derive_plan's root_only).  Not modelled:
the all-gather itself (40 B x 1018 blocks per rank over NVLink, ~10-30 us).

Rank 0 cannot finish before the slowest rank's kernel has ended (its merge
waits for every rank's records), so the step is
    max over ranks of (time to the end of its kernel) + rank 0's time after its own kernel.

    python tools/shard_sim.py [steps] [--host-exchange]

--host-exchange: the older host form (shard/n_shards/exchange arguments; the
cheap group's winners are merged on the host before the expensive launch).
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

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = int(args[0]) if args else 10
host_exchange = "--host-exchange" in sys.argv
g, mesh = bench.load_workload("c5")
be = Backend(0)
be.set_mode("walk")
ses = S.Session.open(g, be)
recorded, calls = [], [0]


def record(scores):
    recorded.append(scores)
    return scores


def replay(scores):
    out = recorded[calls[0] % len(recorded)]
    calls[0] += 1
    return out


if host_exchange:
    S.derive_plan(g, mesh, session=ses, exchange=record)
real_comm = be.comm_info()
base = None
for n in (1, 2, 4, 8):
    per = []
    for r in range(n):
        be.comm = dict(real_comm, nranks=n, rank=r)  # is_root: only rank 0 assembles
        if host_exchange:
            kw = dict(shard=r, n_shards=n, exchange=replay if n > 1 else None)
        else:
            be.set_sim_shard(r, n)
            kw = {}
        for _ in range(2):
            S.derive_plan(g, mesh, session=ses, **kw)
        ts, ks, tails, kept = [], [], [], []
        for _ in range(steps):
            rep = None  # the previous report is freed outside the timed region (as bench.py)
            t0 = time.perf_counter()
            rep = S.derive_plan(g, mesh, session=ses, **kw)
            ts.append((time.perf_counter() - t0) * 1e3)
            ks.append(be.timings()["score_kernel_ms"])
            ph = S.LAST_PHASES
            # host time after the expensive group's results landed (rank 0's report)
            tails.append(ph.get("assemble_ms", 0.0) + ph.get("routes_ms", 0.0) if r == 0 else 0.0)
        per.append((statistics.median(ts), statistics.median(ks), statistics.median(tails), dict(S.LAST_PHASES)))
    be.set_sim_shard(0, 1)
    be.comm = real_comm
    t_other = max([p[0] for p in per[1:]] or [0.0])
    r0, tail0 = per[0][0], per[0][2]
    t = max(r0, t_other + tail0)
    base = base or t
    ks = [round(p[1], 2) for p in per]
    print(f"n_ranks {n}: step {t:.2f} ms (rank 0 {r0:.2f} of which {tail0:.2f} after its results; slowest "
          f"other rank {t_other:.2f}), kernel per rank {ks}, speed-up {base / t:.2f}x, rank-0 phases "
          f"{({k: (round(v, 2) if isinstance(v, float) else v) for k, v in per[0][3].items()})}"
          + (f", rank-1 phases {({k: (round(v, 2) if isinstance(v, float) else v) for k, v in per[1][3].items()})}"
             if n > 1 else ""), flush=True)
