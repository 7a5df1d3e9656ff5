"""The drop-in swap: rebinding the reference's entry points (CPU-side checks).

GPU execution of the swapped reference needs both the reference and a GPU;
the GPU tests cover the same code path through the stand-in types and the
committed reference JSON, byte for byte.
"""

from __future__ import annotations

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture()
def shardplan():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import shardplan as sp

    return sp


def test_install_rebinds_every_name_binding(shardplan):
    import shardplan.cli
    import shardplan.search

    from paper_2302_00247_b200 import swap

    orig = shardplan.search.derive_plan
    h = swap.install(shardplan)
    try:
        for mod in (shardplan, shardplan.search, shardplan.cli):
            assert mod.derive_plan is not orig
            assert mod.derive_plan.__wrapped__.__module__ == "paper_2302_00247_b200.search"
        assert shardplan.search.prune_graph.__wrapped__.__module__ == "paper_2302_00247_b200.search"
        assert shardplan.search.search_subgraph.__wrapped__.__module__ == "paper_2302_00247_b200.search"
    finally:
        h.uninstall()
    assert shardplan.search.derive_plan is orig


def test_reference_types_cover_registry(shardplan):
    from paper_2302_00247_b200.api_types import PATTERN_ROWS
    from paper_2302_00247_b200.swap import reference_types

    t = reference_types(shardplan)
    assert t.BestPlanReport is shardplan.BestPlanReport
    # the stand-in registry rows are the reference's, name for name
    assert {op: tuple(r[0] for r in rows) for op, rows in PATTERN_ROWS.items()} == t.pattern_names
    assert {op: tuple(r[4].kind.value for r in rows) for op, rows in PATTERN_ROWS.items()} == \
        t.pattern_collectives


def test_swapped_call_without_gpu_fails_loudly(shardplan):
    import torch

    from paper_2302_00247_b200 import swap
    from paper_2302_00247_b200.errors import BackendError

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = shardplan.trim_and_group(shardplan.gen_transformer_stack(2, d_model=8))
    h = swap.install(shardplan)
    try:
        with pytest.raises(BackendError):
            shardplan.derive_plan(g, shardplan.ClusterSpec.from_mesh("1x2"))
    finally:
        h.uninstall()


def test_errors_translate_to_reference_classes(shardplan):
    from paper_2302_00247_b200 import errors, swap

    exc = swap._translate(shardplan, errors.BadConfig("min_duplicates must be >= 1"))
    assert isinstance(exc, shardplan.BadConfig)
    exc = swap._translate(shardplan, errors.CycleError("a", "b"))
    assert isinstance(exc, shardplan.CycleError) and exc.src == "a"


def test_backend_only_errors_become_reference_planner_errors(shardplan):
    """UnsupportedSearch has no reference class: under the swap it surfaces as the
    reference's ShardplanError, so the reference CLI's `except ShardplanError`
    (cli.py:471) reports it; a CUDA failure (BackendError) stays a RuntimeError."""
    from paper_2302_00247_b200 import errors, swap

    exc = swap._translate(shardplan, errors.UnsupportedSearch("a block has more than 2**64 candidates"))
    assert type(exc) is shardplan.ShardplanError and "2**64" in str(exc)
    exc = swap._translate(shardplan, errors.SpecMismatch("x"))
    assert isinstance(exc, shardplan.SpecMismatch)


def test_install_forwards_backend_to_search_subgraph(shardplan, monkeypatch):
    from paper_2302_00247_b200 import search, swap

    seen = {}

    def fake(graph, subgraph, mesh, *a, backend=None, **k):
        seen["backend"] = backend
        return "ok"

    monkeypatch.setattr(search, "search_subgraph", fake)
    sentinel = object()
    h = swap.install(shardplan, backend=sentinel)
    try:
        assert shardplan.search.search_subgraph(None, None, None) == "ok"
    finally:
        h.uninstall()
    assert seen["backend"] is sentinel
