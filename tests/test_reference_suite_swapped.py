"""The reference's own 182-test suite, run with this backend swapped in, on the GPU.

SURVEY 4(iv) / 7 step 9: the drop-in claim is proven on the reference's own
tests (e.g. test_acceptance.py:217-233, criterion 8: the CLI's plan JSON is
byte-identical across runs; test_plan_search.py:159-192).  The reference and
its tests are installed unmodified into the git-ignored baseline/_ref/ by
tools/install_reference.sh (they travel to the GPU box; /root/reference does
not).  tests/ref_swap_plugin.py installs the swap before the reference's test
modules are imported and counts the calls that went through the backend.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


def test_reference_suite_passes_with_backend_swapped_in(tmp_path):
    if not os.path.isdir(os.path.join(REF, "tests")):
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    counts = tmp_path / "counts.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests")]),
               SP_SWAP_COUNTS=str(counts), PYTHONDONTWRITEBYTECODE="1")
    proc = subprocess.run([sys.executable, "-m", "pytest", "-p", "ref_swap_plugin", "-p", "no:cacheprovider",
                           "tests"], cwd=REF, env=env, capture_output=True, text=True, timeout=1200)
    tail = proc.stdout[-4000:] + proc.stderr[-2000:]
    assert proc.returncode == 0, tail
    assert "182 passed" in proc.stdout, tail
    n = json.loads(counts.read_text())
    # the suite's searches, folds and replays really ran on the device
    assert n.get("derive_plan", 0) >= 20 and n.get("prune_graph", 0) >= 10, n
    print(proc.stdout.strip().splitlines()[-1], n)
