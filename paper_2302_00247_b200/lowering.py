"""Lower a grouped ModelGraph to the flat arrays of ``sp_graph``.

Works on the reference's ``ModelGraph`` of ``GraphNode`` (ir.py:164-292) or on
``paper_2302_00247_b200.ir.GroupedGraph`` -- both expose ``topo_order``,
``nodes[name].{op, inputs, activation, weight}``.  Nodes are laid out in
``topo_order`` so a node's index IS its topological rank (the only use the
backend makes of the reference's lexicographic-heap order, ir.py:250-274).
The arrays are built once per graph and uploaded once (``sp_graph_upload``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import UnsupportedSearch
from .ir import OP_CODE

MAX_RANK = 8  # SP_MAX_RANK


@dataclass
class LoweredGraph:
    names: list
    index: dict
    name_bytes: np.ndarray   # uint8
    name_off: np.ndarray     # int64 [n+1]
    topo_rank: np.ndarray    # int64 [n]
    op: np.ndarray           # uint8 [n]
    act_rank: np.ndarray     # uint8 [n]
    act_shape: np.ndarray    # int64 [n, 8]
    act_bytes: np.ndarray    # int64 [n]
    w_rank: np.ndarray       # uint8 [n]
    w_shape: np.ndarray      # int64 [n, 8]
    w_bytes: np.ndarray      # int64 [n]
    w_trainable: np.ndarray  # uint8 [n]
    in_off: np.ndarray       # int64 [n+1]
    in_idx: np.ndarray       # int32 [E]
    source: object = None    # the graph object this was lowered from

    @property
    def n_nodes(self) -> int:
        return len(self.names)

    def nbytes(self) -> int:
        return sum(
            a.nbytes for a in (self.name_bytes, self.name_off, self.topo_rank, self.op,
                               self.act_rank, self.act_shape, self.act_bytes, self.w_rank,
                               self.w_shape, self.w_bytes, self.w_trainable, self.in_off,
                               self.in_idx)
        )


def _op_label(op) -> str:
    return op if isinstance(op, str) else op.value


def lower(graph) -> LoweredGraph:
    """Flatten a grouped graph; cached on the graph object when possible."""
    cached = getattr(graph, "_sp_lowered", None)
    if isinstance(cached, LoweredGraph) and cached.source is graph:
        return cached
    names = list(graph.topo_order)
    n = len(names)
    index = {nm: i for i, nm in enumerate(names)}
    nodes = graph.nodes
    op = np.empty(n, np.uint8)
    act_rank = np.empty(n, np.uint8)
    act_shape = np.zeros((n, MAX_RANK), np.int64)
    act_bytes = np.empty(n, np.int64)
    w_rank = np.zeros(n, np.uint8)
    w_shape = np.zeros((n, MAX_RANK), np.int64)
    w_bytes = np.zeros(n, np.int64)
    w_train = np.zeros(n, np.uint8)
    in_off = np.empty(n + 1, np.int64)
    in_idx = []
    in_off[0] = 0
    encoded = [nm.encode("utf-8") for nm in names]
    for i, nm in enumerate(names):
        nd = nodes[nm]
        op[i] = OP_CODE[_op_label(nd.op)]
        a = nd.activation
        shp = tuple(a.shape)
        if len(shp) > MAX_RANK:
            raise UnsupportedSearch(f"activation rank {len(shp)} of {nm!r} exceeds {MAX_RANK}")
        act_rank[i] = len(shp)
        act_shape[i, : len(shp)] = shp
        act_bytes[i] = a.byte_size
        w = nd.weight
        if w is not None:
            ws = tuple(w.shape)
            if len(ws) > MAX_RANK:
                raise UnsupportedSearch(f"weight rank {len(ws)} of {nm!r} exceeds {MAX_RANK}")
            w_rank[i] = len(ws)
            w_shape[i, : len(ws)] = ws
            w_bytes[i] = w.byte_size
            w_train[i] = 1 if w.trainable else 0
        ins = nd.inputs
        in_idx.extend(index[r] for r in ins)
        in_off[i + 1] = in_off[i] + len(ins)
    lens = np.fromiter((len(b) for b in encoded), np.int64, count=n)
    name_off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=name_off[1:])
    name_bytes = np.frombuffer(b"".join(encoded), np.uint8).copy()
    low = LoweredGraph(
        names=names, index=index, name_bytes=name_bytes, name_off=name_off,
        topo_rank=np.arange(n, dtype=np.int64), op=op, act_rank=act_rank,
        act_shape=act_shape, act_bytes=act_bytes, w_rank=w_rank, w_shape=w_shape,
        w_bytes=w_bytes, w_trainable=w_train, in_off=in_off,
        in_idx=np.asarray(in_idx, dtype=np.int32), source=graph,
    )
    try:
        graph._sp_lowered = low
    except AttributeError:  # pragma: no cover - slotted graph types
        pass
    return low
