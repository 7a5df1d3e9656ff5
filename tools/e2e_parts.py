"""Host-side parts of the c5 e2e step: lowering from objects, the sp_graph
view, and the upload call (SP_LOWER_TRACE / SP_UPLOAD_TRACE for detail)."""
import gc
import sys
import time

sys.path[:0] = ['/root/repo', '/root/repo/tests']
from paper_2302_00247_b200._abi import make_sp_graph  # noqa: E402
from paper_2302_00247_b200._native import Backend  # noqa: E402
from paper_2302_00247_b200.lowering import lower  # noqa: E402
from paper_2302_00247_b200.search import _Uncached  # noqa: E402
from paper_2302_00247_b200.workloads import motif_dag  # noqa: E402

g = motif_dag(0, 'throughput')
be = Backend(0)
gc.disable()
for i in range(5):
    t0 = time.perf_counter()
    low = lower(_Uncached(g))
    t1 = time.perf_counter()
    make_sp_graph(low)
    t2 = time.perf_counter()
    d = be.upload(low)
    t3 = time.perf_counter()
    print(f"lower {1e3*(t1-t0):.2f} ms  sp_graph view {1e3*(t2-t1):.2f} ms  upload {1e3*(t3-t2):.2f} ms  "
          f"bytes {low.nbytes()/1e6:.1f} MB", flush=True)
