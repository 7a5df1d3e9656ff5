"""Minimal grouped-graph container with the reference ModelGraph's read API.

The backend itself only needs the lowered arrays (``lowering.LoweredGraph``);
this container exists so the drop-in API can be exercised where the reference
package is not importable (the GPU box).  It mirrors the attributes the
search path reads from a grouped ``ModelGraph`` (ir.py:214-292) and
``GraphNode`` (ir.py:164-202): ``nodes``, ``topo_order`` (lexicographic-heap
Kahn order, ir.py:250-274), ``consumers`` (ir.py:243-248), ``depth`` and, per
node, ``op``/``weight``/``activation``/``inputs``/``depth``.
"""

from __future__ import annotations

import gzip
import heapq
import json
import math
from dataclasses import dataclass
from enum import Enum
from typing import Optional

from .errors import CycleError, DanglingRef, EmptyGraph, ParseError


class OpKind(Enum):
    MATMUL = "matmul"
    ELEMENTWISE = "elementwise"
    LAYERNORM = "layernorm"
    SOFTMAX = "softmax"
    EMBEDDING = "embedding"
    RESHAPE = "reshape"
    INPUT = "input"
    OUTPUT = "output"
    AUXILIARY = "auxiliary"
    COLLECTIVE = "collective"


#: op label -> sp_op code (include/shardsearch.h)
OP_CODE = {k.value: i for i, k in enumerate(OpKind)}

DTYPE_WIDTH = {"f32": 4, "f64": 8}


@dataclass(frozen=True, slots=True)
class TensorSpec:
    shape: tuple
    dtype: str = "f32"
    trainable: bool = False

    @property
    def rank(self) -> int:
        return len(self.shape)

    @property
    def num_elements(self) -> int:
        return math.prod(self.shape)

    @property
    def byte_size(self) -> int:
        return self.num_elements * DTYPE_WIDTH[self.dtype]


@dataclass(frozen=True, slots=True)
class GraphNode:
    scope: str
    op: OpKind
    inputs: tuple
    activation: TensorSpec
    weight: Optional[TensorSpec] = None

    @property
    def name(self) -> str:
        return self.scope

    @property
    def depth(self) -> int:
        return self.scope.count("/") + 1


class GroupedGraph:
    """Read-only grouped DAG (the shape of a trimmed ModelGraph)."""

    def __init__(self, nodes):
        self.nodes: dict[str, GraphNode] = {}
        for nd in nodes:
            if nd.scope in self.nodes:
                raise ParseError(f"duplicate node name {nd.scope!r}")
            self.nodes[nd.scope] = nd
        if not self.nodes:
            raise EmptyGraph("graph has no nodes")
        for nd in self.nodes.values():
            for ref in nd.inputs:
                if ref not in self.nodes:
                    raise DanglingRef(f"node {nd.scope!r} references unknown input {ref!r}")
        cons: dict[str, list] = {n: [] for n in self.nodes}
        for name in sorted(self.nodes):
            for ref in self.nodes[name].inputs:
                cons[ref].append(name)
        self.consumers = {n: tuple(v) for n, v in cons.items()}
        self.topo_order = self._toposort()
        self.depth = max(nd.depth for nd in self.nodes.values())

    def _toposort(self) -> tuple:
        # ready nodes leave in lexicographic order (same rule as ir.py:250-274)
        indeg = {n: len(set(nd.inputs)) for n, nd in self.nodes.items()}
        ready = [n for n, d in indeg.items() if d == 0]
        heapq.heapify(ready)
        order = []
        while ready:
            name = heapq.heappop(ready)
            order.append(name)
            for c in dict.fromkeys(self.consumers[name]):
                indeg[c] -= 1
                if indeg[c] == 0:
                    heapq.heappush(ready, c)
        if len(order) != len(self.nodes):
            left = [n for n in self.nodes if n not in set(order)]
            raise CycleError(left[0], left[0])
        return tuple(order)

    def __len__(self) -> int:
        return len(self.nodes)


def _spec(shape, dtype, trainable=False):
    return TensorSpec(tuple(int(d) for d in shape), dtype or "f32", bool(trainable))


def grouped_from_doc(doc: dict) -> GroupedGraph:
    """Build a GroupedGraph from the compact ``sp-grouped/1`` document."""
    if doc.get("format") != "sp-grouped/1":
        raise ParseError("not an sp-grouped/1 document")
    nodes = []
    for nd in doc["nodes"]:
        w = nd.get("w")
        nodes.append(
            GraphNode(
                nd["s"],
                OpKind(nd["op"]),
                tuple(nd["in"]),
                _spec(nd["a"], nd.get("ad")),
                _spec(w, nd.get("wd"), nd.get("wt")) if w else None,
            )
        )
    return GroupedGraph(nodes)


def load_grouped(path: str) -> GroupedGraph:
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt") as fh:
        return grouped_from_doc(json.load(fh))


def dump_grouped(graph) -> dict:
    """Inverse of grouped_from_doc for any ModelGraph-like object."""
    out = []
    for name in graph.topo_order:
        nd = graph.nodes[name]
        w, a = nd.weight, nd.activation
        out.append({
            "s": name, "op": nd.op.value, "in": list(nd.inputs),
            "a": list(a.shape), "ad": _dtype_label(a),
            "w": list(w.shape) if w else None, "wd": _dtype_label(w) if w else None,
            "wt": bool(w.trainable) if w else False,
        })
    return {"format": "sp-grouped/1", "nodes": out}


def _dtype_label(spec) -> str:
    d = spec.dtype
    return d if isinstance(d, str) else d.label
