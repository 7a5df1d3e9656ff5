import os, sys, time
sys.path[:0]=['/root/repo','/root/repo/tests']
import gc
import numpy as np
from paper_2302_00247_b200.workloads import motif_dag
from paper_2302_00247_b200.lowering import lower
from paper_2302_00247_b200.search import _Uncached
from paper_2302_00247_b200._native import Backend
g = motif_dag(0, 'throughput')
be = Backend(0)
gc.disable()
for i in range(5):
    t0=time.perf_counter(); low = lower(_Uncached(g)); t1=time.perf_counter()
    d = be.upload(low); t2=time.perf_counter()
    print(f"lower {1e3*(t1-t0):.2f} ms  upload {1e3*(t2-t1):.2f} ms  bytes {low.nbytes()/1e6:.1f} MB")
