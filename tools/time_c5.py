"""Time c5 derive_plan phases on the GPU (development helper)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_2302_00247_b200._native import Backend
from paper_2302_00247_b200.api_types import ClusterSpec
from paper_2302_00247_b200 import search as S
from paper_2302_00247_b200.workloads import motif_dag
be = Backend(0)
mesh = ClusterSpec.from_mesh("1x8")
for tier, mode in (("parity", "skip"), ("throughput", "skip"), ("throughput", "memo"),
                   ("throughput", "walk")):
    be.set_mode(mode)
    g = motif_dag(0, tier)
    ses = S.Session.open(g, be)
    for it in range(3):
        t0 = time.perf_counter()
        rep = S.derive_plan(g, mesh, session=ses)
        dt = time.perf_counter() - t0
        print(tier, mode, f"{dt*1e3:.1f} ms", rep.candidates, rep.valid, f"{rep.candidates/dt:.3e} cand/s",
              {k: round(v, 2) for k, v in S.LAST_PHASES.items()}, be.timings(), flush=True)
