"""Same-box A/B of host-side switches: resident c5 step wall time, interleaved.

    python tools/ab_step.py ENV=VAL [steps]
Runs the step with and without the environment switch (read at import, so
each side is a fresh process) several times, alternating."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
kv = sys.argv[1]
steps = sys.argv[2] if len(sys.argv) > 2 else "10"
code = f"""
import sys, time, statistics
sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, 'tests')!r}]
import bench
from paper_2302_00247_b200 import search as S
from paper_2302_00247_b200._native import Backend
g, mesh = bench.load_workload('c5')
be = Backend(0); be.set_mode('walk')
ses = S.Session.open(g, be)
for _ in range(3): S.derive_plan(g, mesh, session=ses)
ts = []
for _ in range({steps}):
    t0 = time.perf_counter(); S.derive_plan(g, mesh, session=ses); ts.append((time.perf_counter() - t0) * 1e3)
print(f"{{statistics.median(ts):.3f}}")
"""
k, v = kv.split("=", 1)
for rep in range(3):
    for on in (False, True):
        env = dict(os.environ)
        if on:
            env[k] = v
        else:
            env.pop(k, None)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(f"{kv if on else 'base':>20}: {out.stdout.strip()} ms {out.stderr.strip()[-200:] if out.returncode else ''}",
              flush=True)
