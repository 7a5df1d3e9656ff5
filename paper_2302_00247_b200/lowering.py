"""Lower a grouped ModelGraph to the flat arrays of ``sp_graph``.

Works on the reference's ``ModelGraph`` of ``GraphNode`` (ir.py:164-292) or on
``paper_2302_00247_b200.ir.GroupedGraph`` -- both expose ``topo_order``,
``nodes[name].{op, inputs, activation, weight}``.  Nodes are laid out in
``topo_order`` so a node's index IS its topological rank (the only use the
backend makes of the reference's lexicographic-heap order, ir.py:250-274).
The arrays are built once per graph and uploaded once (``sp_graph_upload``).
"""

from __future__ import annotations

import itertools
import sys
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import UnsupportedSearch
from .ir import DTYPE_WIDTH, OP_CODE

MAX_RANK = 8  # SP_MAX_RANK


@dataclass
class LoweredGraph:
    names: list
    index_: Optional[dict]   # name -> row; built on first use of .index when None
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
    def index(self) -> dict:
        if self.index_ is None:
            self.index_ = dict(zip(self.names, range(len(self.names))))
        return self.index_

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


_OP_BY_ID: dict = {}
_WIDTH_BY_ID: dict = {}


def _codes(objs: list, cache: dict, fn, dtype) -> np.ndarray:
    """Map enum members / dtype objects to small ints through an id() cache
    (enum __hash__ is a Python-level call; members are singletons)."""
    ids = list(map(id, objs))
    missing = set(ids).difference(cache)
    if missing:
        first = dict(zip(ids, objs))
        for i in missing:
            cache[i] = fn(first[i])
    return np.fromiter(map(cache.__getitem__, ids), dtype, count=len(ids))


def _op_code(op) -> int:
    return OP_CODE[op if isinstance(op, str) else op.value]


def _width(dtype) -> int:
    return DTYPE_WIDTH[dtype] if isinstance(dtype, str) else int(dtype.width)


def _shapes(shapes: list, n: int, what: str):
    """(rank uint8 [n], shape int64 [n, 8], element count int64 [n]) from tuples."""
    rank = np.fromiter(map(len, shapes), np.int64, count=n)
    if n and rank.max() > MAX_RANK:
        raise UnsupportedSearch(f"{what} rank {int(rank.max())} exceeds {MAX_RANK}")
    out = np.ones((n, MAX_RANK), np.int64)
    if n and rank.min() == rank.max():  # uniform rank: one reshape, no scatter
        r = int(rank[0])
        out[:, :r] = np.fromiter(itertools.chain.from_iterable(shapes), np.int64,
                                 count=n * r).reshape(n, r)
    else:
        flat = np.fromiter(itertools.chain.from_iterable(shapes), np.int64, count=int(rank.sum()))
        starts = np.zeros(n, np.int64)
        np.cumsum(rank[:-1], out=starts[1:])
        rows = np.repeat(np.arange(n), rank)
        out[rows, np.arange(flat.size) - np.repeat(starts, rank)] = flat
    elems = out.prod(axis=1)
    if n and float(out.astype(np.float64).prod(axis=1).max()) * 8 >= 2.0 ** 63:
        raise UnsupportedSearch(f"{what} byte size beyond int64")
    out[np.arange(MAX_RANK)[None, :] >= rank[:, None]] = 0
    return rank.astype(np.uint8), out, elems


try:  # native walker of the object graph (csrc/lower_ext.c), built by `make`
    from . import _lower as _native_lower
except ImportError:  # pragma: no cover - unbuilt tree: the numpy restatement below
    _native_lower = None
# the walker reads this interpreter's object layouts in place: only under the
# minor version it was compiled for (the extension suffix already pins it)
if _native_lower is not None and (getattr(_native_lower, "built_for_hexversion", 0) >> 16) != (sys.hexversion >> 16):
    _native_lower = None  # pragma: no cover


def _lower_native(graph):
    """lower() through csrc/lower_ext.c: one C pass over the GraphNode objects."""
    (names, ascii_names, max_ar, max_wr, overflow, name_bytes, name_off, op, act_rank,
     act_shape, act_bytes, w_rank, w_shape, w_bytes, w_train, in_off, in_idx) = \
        _native_lower.lower_arrays(graph.topo_order, graph.nodes, _op_code, _width)
    n = len(names)
    if max_ar > MAX_RANK:
        raise UnsupportedSearch(f"activation rank {max_ar} exceeds {MAX_RANK}")
    if max_wr > MAX_RANK:
        raise UnsupportedSearch(f"weight rank {max_wr} exceeds {MAX_RANK}")
    if overflow:
        raise UnsupportedSearch(f"{overflow} byte size beyond int64")
    low = LoweredGraph(
        names=names, index_=None, name_bytes=np.frombuffer(name_bytes, np.uint8),
        name_off=np.frombuffer(name_off, np.int64), topo_rank=np.arange(n, dtype=np.int64),
        op=np.frombuffer(op, np.uint8), act_rank=np.frombuffer(act_rank, np.uint8),
        act_shape=np.frombuffer(act_shape, np.int64).reshape(n, MAX_RANK),
        act_bytes=np.frombuffer(act_bytes, np.int64), w_rank=np.frombuffer(w_rank, np.uint8),
        w_shape=np.frombuffer(w_shape, np.int64).reshape(n, MAX_RANK),
        w_bytes=np.frombuffer(w_bytes, np.int64), w_trainable=np.frombuffer(w_train, np.uint8),
        in_off=np.frombuffer(in_off, np.int64), in_idx=np.frombuffer(in_idx, np.int32), source=graph,
    )
    low.ascii = bool(ascii_names)
    return low


def lower(graph, native: bool = True) -> LoweredGraph:
    """Flatten a grouped graph (cached on the graph object when possible).  The
    native walker is used when built and the node table is a dict; the numpy
    path below is its restatement (tests check both give identical arrays)."""
    cached = getattr(graph, "_sp_lowered", None)
    if isinstance(cached, LoweredGraph) and cached.source is graph:
        return cached
    if native and _native_lower is not None and isinstance(graph.nodes, dict):
        low = _lower_native(graph)
        try:
            graph._sp_lowered = low
        except AttributeError:  # pragma: no cover - slotted graph types
            pass
        return low
    names = list(graph.topo_order)
    n = len(names)
    index = dict(zip(names, range(n)))
    nl = [graph.nodes[nm] for nm in names]
    op = _codes([nd.op for nd in nl], _OP_BY_ID, _op_code, np.uint8)
    acts = [nd.activation for nd in nl]
    act_rank, act_shape, act_el = _shapes([a.shape for a in acts], n, "activation")
    act_bytes = act_el * _codes([a.dtype for a in acts], _WIDTH_BY_ID, _width, np.int64)
    ws = [nd.weight for nd in nl]
    widx = np.fromiter((i for i, w in enumerate(ws) if w is not None), np.int64)
    w_rank = np.zeros(n, np.uint8)
    w_shape = np.zeros((n, MAX_RANK), np.int64)
    w_bytes = np.zeros(n, np.int64)
    w_train = np.zeros(n, np.uint8)
    if widx.size:
        wl = [ws[i] for i in widx.tolist()]
        r, shp, el = _shapes([w.shape for w in wl], len(wl), "weight")
        w_rank[widx] = r
        w_shape[widx] = shp
        w_bytes[widx] = el * _codes([w.dtype for w in wl], _WIDTH_BY_ID, _width, np.int64)
        w_train[widx] = np.fromiter((1 if w.trainable else 0 for w in wl), np.uint8, count=len(wl))
    ins = [nd.inputs for nd in nl]
    deg = np.fromiter(map(len, ins), np.int64, count=n)
    in_off = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=in_off[1:])
    in_idx = np.fromiter(map(index.__getitem__, itertools.chain.from_iterable(ins)), np.int32,
                         count=int(in_off[-1]))
    joined = "".join(names)
    name_off = np.zeros(n + 1, np.int64)
    if joined.isascii():
        np.cumsum(np.fromiter(map(len, names), np.int64, count=n), out=name_off[1:])
        name_bytes = np.frombuffer(joined.encode("ascii"), np.uint8).copy()
    else:
        encoded = [nm.encode("utf-8") for nm in names]
        np.cumsum(np.fromiter(map(len, encoded), np.int64, count=n), out=name_off[1:])
        name_bytes = np.frombuffer(b"".join(encoded), np.uint8).copy()
    low = LoweredGraph(
        names=names, index_=index, name_bytes=name_bytes, name_off=name_off,
        topo_rank=np.arange(n, dtype=np.int64), op=op, act_rank=act_rank,
        act_shape=act_shape, act_bytes=act_bytes, w_rank=w_rank, w_shape=w_shape,
        w_bytes=w_bytes, w_trainable=w_train, in_off=in_off, in_idx=in_idx, source=graph,
    )
    try:
        graph._sp_lowered = low
    except AttributeError:  # pragma: no cover - slotted graph types
        pass
    return low
