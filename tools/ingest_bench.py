"""Native ingest vs the reference's load_graph + trim_and_group on one raw document.

    python tools/ingest_bench.py [layers]      (needs /root/reference for the reference arm)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"
sys.path[:0] = [ROOT, REF]

from shardplan.generators import gen_transformer_stack  # noqa: E402
from shardplan.ir import load_graph, save_graph, trim_and_group  # noqa: E402

from paper_2302_00247_b200.ingest import load_lowered  # noqa: E402
from paper_2302_00247_b200.lowering import lower  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 7000
text = save_graph(gen_transformer_stack(layers, d_model=64, heads=4))
best = 1e9
for _ in range(3):
    t0 = time.perf_counter()
    g = load_lowered(text)
    best = min(best, time.perf_counter() - t0)
t0 = time.perf_counter()
ref = trim_and_group(load_graph(text))
t1 = time.perf_counter()
low = lower(ref)
t2 = time.perf_counter()
same = all((getattr(g.low, k) == getattr(low, k)).all() for k in ("name_off", "op", "act_bytes", "w_bytes", "in_idx"))
print(f"{len(text) / 1e6:.1f} MB, {g.n_raw} raw -> {len(g.names)} GraphNodes: native ingest {best * 1e3:.0f} ms; "
      f"reference load_graph+trim_and_group {(t1 - t0) * 1e3:.0f} ms (+ lowering {(t2 - t1) * 1e3:.0f} ms); "
      f"speed-up {(t2 - t0) / best:.1f}x; identical arrays: {same}")
