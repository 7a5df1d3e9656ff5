"""Swap the B200 backend into the reference package (the drop-in boundary).

    import shardplan
    from paper_2302_00247_b200 import swap
    handle = swap.install()          # shardplan now searches on the GPU
    ...
    handle.uninstall()

The reference binds its search entry points by name in three places
(SURVEY 8(b)): ``shardplan.search`` (derive_plan, search_subgraph, and the
prune_graph used by routed_plan_for_assignments, search.py:32, 424),
``shardplan.cli`` (cli.py:25-31) and the package namespace
(``shardplan/__init__.py:64, 72-82``).  ``install`` rebinds all of them to
wrappers that call this package with the reference's own result classes, so
BestPlanReport / Subgraph / RoutedPlan objects flowing into rewrite_graph,
broadcast_routing and the CLI are the reference's types, and errors are the
reference's exception classes.  The JSON graph writer (`save_graph`,
ir.py:358-367) is rebound to the native one too.
"""

from __future__ import annotations

import functools
import importlib
from dataclasses import dataclass, field

from . import errors as our_errors
from . import search as ours
from .api_types import TypeSet

_ENTRY_POINTS = ("derive_plan", "prune_graph", "search_subgraph", "routed_plan_for_assignments")


def reference_types(shardplan) -> TypeSet:
    """TypeSet built from the reference's classes (patterns.py, costmodel.py,
    pruning.py, search.py)."""
    patterns = importlib.import_module(shardplan.__name__ + ".patterns")
    costmodel = importlib.import_module(shardplan.__name__ + ".costmodel")
    pruning = importlib.import_module(shardplan.__name__ + ".pruning")
    search = importlib.import_module(shardplan.__name__ + ".search")
    reg = patterns.PATTERN_REGISTRY
    return TypeSet(
        ShardSpec=patterns.ShardSpec,
        ShardKind=patterns.ShardKind,
        Collective=patterns.Collective,
        CollectiveKind=patterns.CollectiveKind,
        CostReport=costmodel.CostReport,
        Subgraph=pruning.Subgraph,
        CandidatePlan=search.CandidatePlan,
        NodeRouting=search.NodeRouting,
        RoutedPlan=search.RoutedPlan,
        RoutingFailure=search.RoutingFailure,
        SubgraphResult=search.SubgraphResult,
        BestPlanReport=search.BestPlanReport,
        pattern_names={op.value: tuple(p.name for p in pats) for op, pats in reg.items()},
        pattern_collectives={op.value: tuple(p.collective.kind.value for p in pats)
                             for op, pats in reg.items()},
    )


def _translate(shardplan, exc: Exception) -> Exception:
    """Our error classes -> the reference's same-named classes.  Planner errors
    the reference has no class for (UnsupportedSearch: a search space outside
    the backend's limits) become the reference's ShardplanError, so its CLI
    (`except ShardplanError`, cli.py:471) reports them as planner errors.
    BackendError (a CUDA failure, RuntimeError) is not a planner error and is
    left as it is."""
    ref_errors = importlib.import_module(shardplan.__name__ + ".errors")
    if isinstance(exc, AssertionError):
        return exc
    cls = getattr(ref_errors, type(exc).__name__, None)
    if cls is None:
        return ref_errors.ShardplanError(f"{type(exc).__name__}: {exc}")
    if type(exc).__name__ == "CycleError":
        return cls(exc.src, exc.dst)
    return cls(str(exc))


@dataclass
class Installed:
    shardplan: object
    saved: list = field(default_factory=list)

    def uninstall(self) -> None:
        for module, name, fn in reversed(self.saved):
            setattr(module, name, fn)
        self.saved.clear()


def install(shardplan=None, backend=None) -> Installed:
    if shardplan is None:
        shardplan = importlib.import_module("shardplan")
    types = reference_types(shardplan)

    def wrap(fn):
        @functools.wraps(fn)
        def inner(*args, **kwargs):
            kwargs.setdefault("types", types)
            if backend is not None:
                kwargs.setdefault("backend", backend)
            try:
                return fn(*args, **kwargs)
            except our_errors.ShardplanError as exc:
                raise _translate(shardplan, exc) from exc

        return inner

    replacements = {
        "derive_plan": wrap(ours.derive_plan),
        "prune_graph": wrap(ours.prune_graph),
        "search_subgraph": wrap(ours.search_subgraph),
        "routed_plan_for_assignments": wrap(ours.routed_plan_for_assignments),
    }
    handle = Installed(shardplan)
    # save_graph (ir.py:358-367; bound by name in shardplan.ir, .cli and the package)
    from . import ingest as our_ingest

    @functools.wraps(our_ingest.save_graph)
    def save_graph(graph, version: int = 1) -> bytes:
        return our_ingest.save_graph(graph, version)

    for modname in ("ir", "cli", ""):
        module = importlib.import_module(f"{shardplan.__name__}.{modname}") if modname else shardplan
        if hasattr(module, "save_graph"):
            handle.saved.append((module, "save_graph", getattr(module, "save_graph")))
            setattr(module, "save_graph", save_graph)
    for modname in ("search", "cli", ""):
        module = (importlib.import_module(f"{shardplan.__name__}.{modname}") if modname
                  else shardplan)
        for name in _ENTRY_POINTS:
            if hasattr(module, name):
                handle.saved.append((module, name, getattr(module, name)))
                setattr(module, name, replacements[name])
    return handle
