#!/bin/bash
# Same-box A/B of two builds of the _lower extension on the c5 resident step:
#   tools/ab_lower_so.sh A.so B.so
EXT=$(python -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
DST=paper_2302_00247_b200/_lower$EXT
cp "$DST" /tmp/_lower_keep.so
for r in 1 2 3; do for v in "$@"; do
  cp "$v" "$DST"
  python - <<'PY' | sed "s|^|$v |"
import sys, time, statistics
sys.path[:0] = ['.', 'tests']
import bench
from paper_2302_00247_b200 import search as S
from paper_2302_00247_b200._native import Backend
g, mesh = bench.load_workload('c5')
be = Backend(0); be.set_mode('walk')
ses = S.Session.open(g, be)
for _ in range(3): S.derive_plan(g, mesh, session=ses)
ts, asm = [], []
for _ in range(10):
    t0 = time.perf_counter(); S.derive_plan(g, mesh, session=ses); ts.append((time.perf_counter() - t0) * 1e3)
    asm.append(S.LAST_PHASES['assemble_ms'])
print(f"step {statistics.median(ts):.3f} ms assemble {statistics.median(asm):.3f} ms")
PY
done; done
cp /tmp/_lower_keep.so "$DST"
