"""A/B of how the previous step's report is released around a timed c5 step:
A  rebinding `rep = step()` (the old report is freed inside the timed region)
B  `rep = None` before the timed region
C  `rep = None; gc.collect()` before the timed region
Modes interleaved on one box; CUDA-event step times, median of each."""
import gc
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2302_00247_b200 import search as S  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
g, mesh = bench.load_workload(wl)
be = Backend(0)
be.set_mode("walk")
ses = S.Session.open(g, be)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {"A": [], "B": [], "C": []}
rep = S.derive_plan(g, mesh, session=ses)
for it in range(8):
    for m in ("A", "B", "C"):
        if m != "A":
            rep = None
        if m == "C":
            gc.collect()
        flush.zero_()
        torch.cuda.synchronize()
        be.timer_start()
        rep = S.derive_plan(g, mesh, session=ses)
        res[m].append(be.timer_stop())
print(wl, {m: round(statistics.median(v[2:]), 3) for m, v in res.items()})
