"""Diagnose: score the c5 throughput tables in one mode sequence (one process per run).

    python tools/diag_c5_modes.py <seq>      seq: comma list of slices|skip|memo|walk
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from golden_io import c5, mesh  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402
from paper_2302_00247_b200.lowering import lower  # noqa: E402
from paper_2302_00247_b200.search import Session, fold_blocks  # noqa: E402
from paper_2302_00247_b200.workloads import motif_dag  # noqa: E402

seq = []
for tok in sys.argv[1].split(","):
    name, _, rep = tok.partition("*")
    seq += [name] * int(rep or 1)
gold = c5()["throughput"]
be = Backend(0)
ses = Session.open(lower(motif_dag(0, "throughput")), be)
ba = fold_blocks(ses.low, 2, session=ses)
off, nodes = ba.templates_csr()
t = be.tables(ses.dgraph, off, nodes, mesh(gold["mesh"]), 1 << 20, 4 << 20)
ref = None
for step in seq:
    t0 = time.perf_counter()
    if step == "slices":
        for sl in gold["slices"]:
            be.score_range(t, sl["block"], sl["lo"], sl["hi"], want_totals=True)
        print("slices ok", flush=True)
        continue
    be.set_mode(step)
    res = be.score(t)
    key = [(r.valid, r.best_index, r.best_total) for r in res]
    print(step, "ok", f"{(time.perf_counter() - t0) * 1e3:.1f} ms", "same" if ref is None or key == ref else "DIFF",
          flush=True)
    ref = ref or key
t.close()
