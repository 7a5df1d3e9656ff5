"""Native graph ingest: the JSON graph document straight to the search's flat arrays.

``load_lowered(source)`` replaces the reference's ``load_graph`` +
``trim_and_group`` (ir.py:302-338, 374-461) in front of ``derive_plan``: the
C++ ingest (csrc/ingest.cpp, ``sp_ingest_json``) parses the document,
validates and toposorts the raw DAG, trims auxiliary operators, groups by
name scope and lowers the grouped graph, with no Python node objects in
between.  ``plan_from_json`` is the CLI's ``shardplan plan --graph`` path
(cli.py:189-198) on top of it.  Errors are the reference's kinds
(ParseError, CycleError, DanglingRef, EmptyGraph).
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Union

import numpy as np

from ._abi import SpGraph
from ._native import load_library
from .errors import CycleError, DanglingRef, EmptyGraph, ParseError, UnsupportedSearch
from .ir import DTYPE_WIDTH, OpKind, TensorSpec
from .lowering import MAX_RANK, LoweredGraph

SP_ERR_UNSUPPORTED, SP_ERR_PARSE, SP_ERR_CYCLE, SP_ERR_DANGLING, SP_ERR_EMPTY = 2, 5, 6, 7, 8
_OPS = list(OpKind)
_WIDTH_LABEL = {w: d for d, w in DTYPE_WIDTH.items()}
_declared = False


def _lib():
    global _declared
    L = load_library()
    if not _declared:
        vp = C.c_void_p
        L.sp_ingest_json.argtypes = [C.c_char_p, C.c_int64, C.POINTER(vp)]
        L.sp_ingest_json.restype = C.c_int
        L.sp_ingest_error.argtypes = [C.c_int32]
        L.sp_ingest_error.restype = C.c_char_p
        L.sp_ingest_view.argtypes = [vp, C.POINTER(SpGraph), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.sp_ingest_view.restype = C.c_int
        L.sp_ingest_free.argtypes = [vp]
        L.sp_ingest_free.restype = None
        _declared = True
    return L


def _read(source) -> bytes:
    if hasattr(source, "read"):
        source = source.read()
    if isinstance(source, str):
        if os.path.exists(source):
            import gzip

            opener = gzip.open if source.endswith(".gz") else open
            with opener(source, "rb") as fh:
                return fh.read()
        return source.encode("utf-8")
    return bytes(source)


def _raise(L, rc: int):
    msg = (L.sp_ingest_error(0) or b"").decode("utf-8", "replace")
    if rc == SP_ERR_CYCLE:
        raise CycleError(L.sp_ingest_error(1).decode("utf-8", "replace"),
                         L.sp_ingest_error(2).decode("utf-8", "replace"))
    if rc == SP_ERR_DANGLING:
        raise DanglingRef(msg)
    if rc == SP_ERR_EMPTY:
        raise EmptyGraph(msg)
    if rc == SP_ERR_UNSUPPORTED:
        raise UnsupportedSearch(msg)
    raise ParseError(msg)


class _Node:
    """Read-only GraphNode view over one lowered row (op/inputs/activation/weight)."""

    __slots__ = ("_g", "_i")

    def __init__(self, g: "IngestedGraph", i: int):
        self._g, self._i = g, i

    @property
    def scope(self) -> str:
        return self._g.names[self._i]

    name = scope

    @property
    def op(self) -> OpKind:
        return _OPS[int(self._g.low.op[self._i])]

    @property
    def inputs(self) -> tuple:
        lo, hi = int(self._g.low.in_off[self._i]), int(self._g.low.in_off[self._i + 1])
        return tuple(self._g.names[j] for j in self._g.low.in_idx[lo:hi].tolist())

    def _spec(self, rank, shape, nbytes, trainable=False):
        r = int(rank[self._i])
        dims = tuple(int(x) for x in shape[self._i, :r])
        el = 1
        for d in dims:
            el *= d
        return TensorSpec(dims, _WIDTH_LABEL[int(nbytes[self._i]) // el], bool(trainable))

    @property
    def activation(self) -> TensorSpec:
        low = self._g.low
        return self._spec(low.act_rank, low.act_shape, low.act_bytes)

    @property
    def weight(self):
        low = self._g.low
        if not low.w_rank[self._i]:
            return None
        return self._spec(low.w_rank, low.w_shape, low.w_bytes, low.w_trainable[self._i])

    @property
    def depth(self) -> int:
        return self.scope.count("/") + 1


class _Nodes(dict):
    """name -> _Node, built lazily (the search itself only needs the arrays)."""

    def __init__(self, g: "IngestedGraph"):
        super().__init__()
        self._g = g

    def __missing__(self, name):
        node = _Node(self._g, self._g.low.index[name])
        self[name] = node
        return node

    def __contains__(self, name):
        return name in self._g.low.index

    def __len__(self):
        return len(self._g.names)

    def __iter__(self):
        return iter(self._g.names)


class IngestedGraph:
    """A grouped graph produced by the native ingest: the ModelGraph read API
    (``nodes``, ``topo_order``) over the lowered arrays it already carries."""

    def __init__(self, low: LoweredGraph, n_raw: int, n_aux: int):
        self.low = low
        self.names = low.names
        self.topo_order = tuple(low.names)
        self.nodes = _Nodes(self)
        self.n_raw, self.n_aux = n_raw, n_aux
        low.source = self
        self._sp_lowered = low

    def __len__(self) -> int:
        return len(self.names)


def load_lowered(source: Union[bytes, str, "os.PathLike"]) -> IngestedGraph:
    """Parse + trim + group + lower a JSON graph document natively (schema 1/2)."""
    L = _lib()
    text = _read(source)
    h = C.c_void_p()
    rc = L.sp_ingest_json(text, len(text), C.byref(h))
    if rc:
        _raise(L, rc)
    try:
        v = SpGraph()
        n_raw, n_aux = C.c_int64(), C.c_int64()
        L.sp_ingest_view(h, C.byref(v), C.byref(n_raw), C.byref(n_aux))
        n = int(v.n_nodes)

        def arr(p, count, dtype, shape=None):
            a = np.ctypeslib.as_array(p, shape=(max(count, 1),))[:count].copy()
            return a.astype(dtype, copy=False) if shape is None else a.reshape(shape)

        name_off = arr(v.name_off, n + 1, np.int64)
        nb = int(name_off[-1])
        name_bytes = np.ctypeslib.as_array(v.name_bytes, shape=(max(nb, 1),))[:nb].copy()
        E = int(arr(v.in_off, n + 1, np.int64)[-1])
        raw = name_bytes.tobytes()
        ascii_names = raw.isascii()
        text_names = raw.decode("ascii" if ascii_names else "utf-8")
        if ascii_names:
            offs = name_off.tolist()
            names = [text_names[a:b] for a, b in zip(offs[:-1], offs[1:])]
        else:
            offs = name_off.tolist()
            names = [raw[a:b].decode("utf-8") for a, b in zip(offs[:-1], offs[1:])]
        low = LoweredGraph(
            names=names, index_=None, name_bytes=name_bytes, name_off=name_off,
            topo_rank=arr(v.topo_rank, n, np.int64), op=arr(v.op, n, np.uint8),
            act_rank=arr(v.act_rank, n, np.uint8), act_shape=arr(v.act_shape, n * MAX_RANK, np.int64,
                                                                 (n, MAX_RANK)),
            act_bytes=arr(v.act_bytes, n, np.int64), w_rank=arr(v.w_rank, n, np.uint8),
            w_shape=arr(v.w_shape, n * MAX_RANK, np.int64, (n, MAX_RANK)), w_bytes=arr(v.w_bytes, n, np.int64),
            w_trainable=arr(v.w_trainable, n, np.uint8), in_off=arr(v.in_off, n + 1, np.int64),
            in_idx=arr(v.in_idx, E, np.int32) if E else np.zeros(0, np.int32),
        )
        low.ascii = ascii_names
        return IngestedGraph(low, int(n_raw.value), int(n_aux.value))
    finally:
        L.sp_ingest_free(h)


def plan_from_json(source, mesh, min_duplicates: int = 2, mu: int = 1 << 20, chunk_size: int = 4 << 20,
                   **kw):
    """`shardplan plan --graph FILE` (cli.py:189-198): native ingest + device search."""
    from .search import derive_plan

    return derive_plan(load_lowered(source), mesh, min_duplicates, mu, chunk_size, **kw)
