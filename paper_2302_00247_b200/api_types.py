"""Result and configuration types of the drop-in API.

Field-for-field stand-ins for the reference types the search path returns
(patterns.py:26-111 ShardSpec/Collective/ShardingPattern, costmodel.py:36-182
ClusterSpec/CostReport, pruning.py:33-55 Subgraph, search.py:39-82 and
236-281 CandidatePlan/NodeRouting/RoutedPlan/SubgraphResult/BestPlanReport),
so ``BestPlanReport.to_json()`` is byte-identical to the reference's for the
same search.  When the backend is installed into the reference package
(``swap.install``) the reference's own classes are used instead; see
``TypeSet``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional

from .errors import BadConfig, SpecMismatch

LAST = -1


class ShardKind(Enum):
    REPLICA = "replica"
    SPLIT = "split"
    PARTIAL = "partial"


@dataclass(frozen=True)
class ShardSpec:
    kind: ShardKind
    axis: Optional[int] = None

    def normalized(self, rank: int) -> "ShardSpec":
        if self.kind is not ShardKind.SPLIT:
            return self
        a = self.axis if self.axis >= 0 else rank + self.axis
        if not 0 <= a < rank:
            raise SpecMismatch(f"split axis {self.axis} out of range for rank {rank}")
        return ShardSpec(ShardKind.SPLIT, a)

    @property
    def label(self) -> str:
        return f"split{self.axis}" if self.kind is ShardKind.SPLIT else self.kind.value

    @classmethod
    def from_label(cls, label: str) -> "ShardSpec":
        if label in ("replica", "partial"):
            return cls(ShardKind(label))
        if label.startswith("split"):
            return cls(ShardKind.SPLIT, int(label[5:]))
        raise SpecMismatch(f"unknown shard spec label {label!r}")


REPLICA = ShardSpec(ShardKind.REPLICA)
PARTIAL = ShardSpec(ShardKind.PARTIAL)


def split(axis: int) -> ShardSpec:
    return ShardSpec(ShardKind.SPLIT, axis)


class CollectiveKind(Enum):
    IDENTITY = "identity"
    ALL_REDUCE_SUM = "allreduce"
    ALL_GATHER = "allgather"
    REDUCE_SCATTER = "reducescatter"
    ALL_TO_ALL = "alltoall"


@dataclass(frozen=True)
class Collective:
    kind: CollectiveKind
    axis: Optional[int] = None

    @property
    def label(self) -> str:
        return self.kind.value if self.axis is None else f"{self.kind.value}({self.axis})"


IDENTITY = Collective(CollectiveKind.IDENTITY)


@dataclass(frozen=True)
class ShardingPattern:
    name: str
    op: str
    input_spec: ShardSpec
    weight_spec: Optional[ShardSpec]
    output_spec: ShardSpec
    collective: Collective


_AR = Collective(CollectiveKind.ALL_REDUCE_SUM)

#: (name, input, weight, output, collective) per op label, in registry order.
#: Same closed table as the reference (patterns.py:118-159); the device tables
#: (csrc/tables.cuh) encode the identical rows.
PATTERN_ROWS = {
    "matmul": (
        ("matmul.replicate", REPLICA, REPLICA, REPLICA, IDENTITY),
        ("matmul.col", REPLICA, split(1), split(LAST), IDENTITY),
        ("matmul.row.allreduce", split(LAST), split(0), PARTIAL, _AR),
        ("matmul.data_parallel", split(0), REPLICA, split(0), IDENTITY),
    ),
    "elementwise": (
        ("elementwise.replicate", REPLICA, REPLICA, REPLICA, IDENTITY),
        ("elementwise.split0", split(0), REPLICA, split(0), IDENTITY),
        ("elementwise.split_last", split(LAST), split(0), split(LAST), IDENTITY),
    ),
    "layernorm": (
        ("layernorm.replicate", REPLICA, None, REPLICA, IDENTITY),
        ("layernorm.split0", split(0), None, split(0), IDENTITY),
    ),
    "softmax": (
        ("softmax.replicate", REPLICA, None, REPLICA, IDENTITY),
        ("softmax.split0", split(0), None, split(0), IDENTITY),
    ),
    "embedding": (
        ("embedding.replicate", REPLICA, REPLICA, REPLICA, IDENTITY),
        ("embedding.col", REPLICA, split(1), split(LAST), IDENTITY),
        ("embedding.data_parallel", split(0), REPLICA, split(0), IDENTITY),
    ),
    "reshape": (("reshape.replicate", REPLICA, None, REPLICA, IDENTITY),),
    "input": (("input.replicate", REPLICA, None, REPLICA, IDENTITY),),
    "output": (("output.replicate", REPLICA, None, REPLICA, IDENTITY),),
}

PATTERN_REGISTRY = {
    op: tuple(ShardingPattern(n, op, i, w, o, c) for n, i, w, o, c in rows)
    for op, rows in PATTERN_ROWS.items()
}

_EFF_LABELS = ("allgather", "allreduce", "alltoall", "reducescatter")
DEFAULT_EFFICIENCY = {
    CollectiveKind.ALL_REDUCE_SUM: 1.0,
    CollectiveKind.ALL_GATHER: 1.2,
    CollectiveKind.REDUCE_SCATTER: 1.2,
    CollectiveKind.ALL_TO_ALL: 1.5,
}


@dataclass(frozen=True)
class ClusterSpec:
    """m worker nodes x n accelerators (costmodel.py:36-119)."""

    m: int
    n: int
    intra_bw: float = 2.0e11
    inter_bw: float = 2.0e11
    efficiency: tuple = tuple(sorted(DEFAULT_EFFICIENCY.items(), key=lambda kv: kv[0].value))
    overlap_fraction: float = 0.5
    setup_latency_s: float = 3.0e-5

    def __post_init__(self):
        if self.m < 1 or self.n < 1:
            raise BadConfig(f"mesh must be at least 1x1, got {self.m}x{self.n}")
        if self.intra_bw <= 0 or self.inter_bw <= 0:
            raise BadConfig("bandwidths must be positive")
        if not 0.0 <= self.overlap_fraction <= 1.0:
            raise BadConfig("overlap_fraction must lie in [0, 1]")
        eff = dict(self.efficiency)
        if any(v < 1.0 for v in eff.values()):
            raise BadConfig("efficiency factors must be >= 1")
        if eff.get(CollectiveKind.ALL_REDUCE_SUM, 1.0) != 1.0:
            raise BadConfig("allreduce efficiency is the reference and must be 1.0")

    @property
    def device_count(self) -> int:
        return self.m * self.n

    @property
    def bandwidth(self) -> float:
        return self.inter_bw if self.m > 1 else self.intra_bw

    def eff(self, kind) -> float:
        return dict(self.efficiency).get(kind, 1.0)

    @classmethod
    def from_mesh(cls, mesh: str, **kw) -> "ClusterSpec":
        try:
            m, n = (int(p) for p in mesh.lower().split("x"))
        except ValueError as exc:
            raise BadConfig(f"mesh must look like 'MxN', got {mesh!r}") from exc
        return cls(m=m, n=n, **kw)

    def to_json(self) -> dict:
        return {
            "m": self.m,
            "n": self.n,
            "intra_bw": self.intra_bw,
            "inter_bw": self.inter_bw,
            "efficiency": {k.value: v for k, v in self.efficiency},
            "overlap_fraction": self.overlap_fraction,
            "setup_latency_s": self.setup_latency_s,
        }

    @classmethod
    def from_json(cls, doc) -> "ClusterSpec":
        if hasattr(doc, "read"):
            doc = doc.read()
        if isinstance(doc, (str, bytes)):
            doc = json.loads(doc)
        eff = dict(DEFAULT_EFFICIENCY)
        for key, val in (doc.get("efficiency") or {}).items():
            if key not in _EFF_LABELS:
                raise BadConfig(f"unknown efficiency key {key!r}")
            eff[CollectiveKind(key)] = float(val)
        try:
            return cls(
                m=int(doc["m"]), n=int(doc["n"]),
                intra_bw=float(doc.get("intra_bw", 2.0e11)),
                inter_bw=float(doc.get("inter_bw", 2.0e11)),
                efficiency=tuple(sorted(eff.items(), key=lambda kv: kv[0].value)),
                overlap_fraction=float(doc.get("overlap_fraction", 0.5)),
                setup_latency_s=float(doc.get("setup_latency_s", 3.0e-5)),
            )
        except KeyError as exc:
            raise BadConfig(f"cluster config missing key {exc}") from exc


@dataclass
class CostReport:
    forward_comm: float = 0.0
    backward_comm: float = 0.0
    overlap_fraction: float = 0.5
    bytes_by_collective: dict = field(default_factory=dict)
    collective_calls: int = 0
    flops: int = 0

    @property
    def effective_backward(self) -> float:
        return self.backward_comm * (1.0 - self.overlap_fraction)

    @property
    def total(self) -> float:
        return self.forward_comm + self.effective_backward

    def to_json(self) -> dict:
        return {
            "forward_comm_s": self.forward_comm,
            "backward_comm_s": self.backward_comm,
            "effective_backward_s": self.effective_backward,
            "total_s": self.total,
            "overlap_fraction": self.overlap_fraction,
            "bytes_by_collective": dict(sorted(self.bytes_by_collective.items())),
            "collective_calls": self.collective_calls,
            "flops": self.flops,
        }


@dataclass(frozen=True)
class Subgraph:
    template_prefix: str
    template: tuple
    instances: tuple

    @property
    def multiplicity(self) -> int:
        return len(self.instances)

    def instance_node(self, instance_prefix: str, template_scope: str) -> str:
        if instance_prefix == self.template_prefix:
            return template_scope
        return instance_prefix + template_scope[len(self.template_prefix):]


@dataclass(frozen=True)
class CandidatePlan:
    subgraph: Subgraph
    assignments: tuple
    index: int

    @property
    def assignment_map(self) -> dict:
        return dict(self.assignments)

    @property
    def num_split(self) -> int:
        return sum(1 for _, s in self.assignments if s.kind.value == "split")


@dataclass(frozen=True)
class NodeRouting:
    scope: str
    pattern: str
    input_conversions: tuple
    output_collective: Collective
    output_bytes: int
    state: ShardSpec
    exit_conversion: Optional[Collective] = None


@dataclass(frozen=True)
class RoutedPlan:
    plan: CandidatePlan
    routings: tuple
    exit_conversions: tuple
    cost: CostReport

    @property
    def routing_map(self) -> dict:
        return {r.scope: r for r in self.routings}


@dataclass(frozen=True)
class RoutingFailure:
    node: str
    reason: str


@dataclass
class SubgraphResult:
    subgraph: Subgraph
    best: Optional[RoutedPlan]
    candidates: int
    valid: int
    table: list = field(default_factory=list)


@dataclass
class BestPlanReport:
    mesh: ClusterSpec
    min_duplicates: int
    results: list
    assignments: dict
    total_cost: float
    candidates: int
    valid: int

    def to_json(self, with_table: bool = False) -> dict:
        subs = []
        for res in self.results:
            entry = {
                "template_prefix": res.subgraph.template_prefix,
                "multiplicity": res.subgraph.multiplicity,
                "nodes": len(res.subgraph.template),
                "candidates": res.candidates,
                "valid": res.valid,
                "best": {s: spec.label for s, spec in (res.best.plan.assignments if res.best else ())},
                "cost": res.best.cost.to_json() if res.best else None,
            }
            if with_table and res.table:
                entry["cost_table"] = res.table
            subs.append(entry)
        return {
            "mesh": self.mesh.to_json(),
            "min_duplicates": self.min_duplicates,
            "subgraphs": subs,
            "assignments": dict(sorted(self.assignments.items())),
            "total_cost_s": self.total_cost,
            "candidates_enumerated": self.candidates,
            "valid_plans": self.valid,
        }


@dataclass(frozen=True)
class TypeSet:
    """The classes results are built from: these stand-ins, or the reference's
    own when the backend is swapped into shardplan (swap.install)."""

    ShardSpec: type = ShardSpec
    ShardKind: type = ShardKind
    Collective: type = Collective
    CollectiveKind: type = CollectiveKind
    CostReport: type = CostReport
    Subgraph: type = Subgraph
    CandidatePlan: type = CandidatePlan
    NodeRouting: type = NodeRouting
    RoutedPlan: type = RoutedPlan
    RoutingFailure: type = RoutingFailure
    SubgraphResult: type = SubgraphResult
    BestPlanReport: type = BestPlanReport
    pattern_names: dict = field(default_factory=lambda: {
        op: tuple(r[0] for r in rows) for op, rows in PATTERN_ROWS.items()})
    pattern_collectives: dict = field(default_factory=lambda: {
        op: tuple(r[4].kind.value for r in rows) for op, rows in PATTERN_ROWS.items()})


DEFAULT_TYPES = TypeSet()
