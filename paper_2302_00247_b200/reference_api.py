"""The rest of the reference's search-side API, for drop-in completeness.

Small host utilities of the reference that sit beside the hot path (SURVEY 8(a)
rows F7, R3, R6, R8): the name-prefix tree (`build_node_tree`,
`find_similar_blocks`, pruning.py:16-30, 62-120), the pattern registry helpers
(`patterns_for`, `apply_collective`, `conversion_collective`,
patterns.py:166-221), the ring cost closed forms (`collective_cost_bytes`,
`collective_call_cost`, costmodel.py:122-145) and greedy gradient fusion
(`pack_gradients`, rewrite.py:78-111).  They are O(graph) or O(1) bookkeeping
the reference exposes to callers and tests; the search itself never calls
them -- it runs on the device (search.py in this package).
"""

from __future__ import annotations

from dataclasses import dataclass

from .api_types import (
    IDENTITY,
    PATTERN_REGISTRY,
    REPLICA,
    Collective,
    CollectiveKind,
    ShardKind,
    ShardSpec,
    split,
)
from .errors import BadConfig, NoRouteError, SpecMismatch

# ---------------------------------------------------------------------------
# name-prefix tree (pruning.py:16-30, 62-76, 79-94, 114-120)


@dataclass(frozen=True)
class PrefixGroup:
    prefix: str
    members: tuple


@dataclass(frozen=True)
class NodeTree:
    levels: tuple
    max_depth: int

    def level(self, depth: int) -> tuple:
        return dict(self.levels).get(depth, ())


def _prefix(scope: str, depth: int) -> str:
    return "/".join(scope.split("/")[:depth])


def build_node_tree(graph) -> NodeTree:
    """Prefix clusters at every depth from the deepest scope up."""
    names = sorted(graph.nodes)
    depth_of = {n: n.count("/") + 1 for n in names}
    max_depth = max(depth_of.values())
    levels = []
    for depth in range(max_depth, 0, -1):
        buckets: dict = {}
        for n in names:
            if depth_of[n] >= depth:
                buckets.setdefault(_prefix(n, depth), []).append(n)
        levels.append((depth, tuple(PrefixGroup(p, tuple(m)) for p, m in sorted(buckets.items()))))
    return NodeTree(tuple(levels), max_depth)


def signature(graph, members: tuple):
    """(sorted op labels, sorted weight shapes, internal edge count)."""
    member_set = set(members)
    ops = sorted(_op_label(graph.nodes[m].op) for m in members)
    shapes = sorted(tuple(graph.nodes[m].weight.shape) for m in members
                    if graph.nodes[m].weight is not None)
    edges = sum(1 for m in members for r in graph.nodes[m].inputs if r in member_set)
    return (tuple(ops), tuple(shapes), edges)


def find_similar_blocks(tree: NodeTree, depth: int, graph) -> list:
    counts: dict = {}
    for grp in tree.level(depth):
        sig = signature(graph, grp.members)
        counts[sig] = counts.get(sig, 0) + 1
    return sorted(counts.items(), key=lambda kv: kv[0])


def _op_label(op) -> str:
    return op if isinstance(op, str) else op.value


# ---------------------------------------------------------------------------
# pattern registry helpers (patterns.py:166-221)


def patterns_for(op) -> tuple:
    label = _op_label(op)
    if label not in PATTERN_REGISTRY:
        raise SpecMismatch(f"{label} is not a shardable compute kind")
    return PATTERN_REGISTRY[label]


def apply_collective(state: ShardSpec, coll: Collective) -> ShardSpec:
    if coll.kind is CollectiveKind.IDENTITY:
        return state
    if coll.kind in (CollectiveKind.ALL_REDUCE_SUM, CollectiveKind.ALL_GATHER):
        return REPLICA
    return split(coll.axis)


def conversion_collective(frm: ShardSpec, to: ShardSpec, tensor) -> Collective:
    a, b = frm.normalized(tensor.rank), to.normalized(tensor.rank)
    if a == b:
        return IDENTITY
    if b.kind is ShardKind.REPLICA:
        if a.kind is ShardKind.SPLIT:
            return Collective(CollectiveKind.ALL_GATHER, a.axis)
        if a.kind is ShardKind.PARTIAL:
            return Collective(CollectiveKind.ALL_REDUCE_SUM)
    if a.kind is ShardKind.SPLIT and b.kind is ShardKind.SPLIT and a.axis != b.axis:
        return Collective(CollectiveKind.ALL_TO_ALL, b.axis)
    if a.kind is ShardKind.PARTIAL and b.kind is ShardKind.SPLIT:
        return Collective(CollectiveKind.REDUCE_SCATTER, b.axis)
    raise NoRouteError(f"no single collective converts {a.label} -> {b.label}")


# ---------------------------------------------------------------------------
# cost closed forms (costmodel.py:122-145)


def collective_cost_bytes(kind, nbytes: int, mesh) -> float:
    kind = CollectiveKind(_op_label(kind)) if not isinstance(kind, CollectiveKind) else kind
    if kind is CollectiveKind.IDENTITY:
        return 0.0
    d = mesh.m * mesh.n
    if d == 1:
        return 0.0
    bw = mesh.inter_bw if mesh.m > 1 else mesh.intra_bw
    if kind is CollectiveKind.ALL_REDUCE_SUM:
        volume = 2.0 * (d - 1) / d * nbytes
    else:
        volume = (d - 1) / d * nbytes
    eff = {k.value if hasattr(k, "value") else k: v for k, v in mesh.efficiency}
    return volume / bw * eff.get(kind.value, 1.0)


def collective_call_cost(coll: Collective, nbytes: int, mesh) -> float:
    kind = coll.kind.value if hasattr(coll.kind, "value") else coll.kind
    if kind == "identity" or mesh.m * mesh.n == 1:
        return 0.0
    return mesh.setup_latency_s + collective_cost_bytes(CollectiveKind(kind), nbytes, mesh)


# ---------------------------------------------------------------------------
# gradient fusion (rewrite.py:71-111)


@dataclass(frozen=True)
class FusionBucket:
    members: tuple
    total_bytes: int
    chunk_index: int


def pack_gradients(gradients: list, mu: int, chunk_size: int) -> tuple:
    if mu > chunk_size:
        raise BadConfig(f"fusion threshold {mu} exceeds chunk size {chunk_size}")
    buckets, unfused, cur, cur_bytes = [], [], [], 0
    for grad in gradients:
        size = grad.byte_size
        if size >= mu:
            unfused.append(grad)
            continue
        if cur_bytes + size > chunk_size and cur:
            buckets.append(FusionBucket(tuple(cur), cur_bytes, len(buckets)))
            cur, cur_bytes = [], 0
        cur.append(grad)
        cur_bytes += size
    if cur:
        buckets.append(FusionBucket(tuple(cur), cur_bytes, len(buckets)))
    return buckets, unfused
