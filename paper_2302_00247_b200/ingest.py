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
        return _graph_from_handle(L, h)
    finally:
        L.sp_ingest_free(h)


def _graph_from_handle(L, h) -> IngestedGraph:
    """IngestedGraph copied out of an sp_ingest handle (the caller frees it)."""
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


def plan_from_json(source, mesh, min_duplicates: int = 2, mu: int = 1 << 20, chunk_size: int = 4 << 20,
                   **kw):
    """`shardplan plan --graph FILE` (cli.py:189-198): native ingest + device search."""
    from .search import derive_plan

    return derive_plan(load_lowered(source), mesh, min_duplicates, mu, chunk_size, **kw)


# ---------------------------------------------------------------------------
# ONNX (onnx_ingest: wire.py / model.py / convert.py)

SP_ERR_ONNX_PARSE, SP_ERR_ONNX_UNSUPPORTED = 9, 10


class ModelParseError(ValueError):
    """File is not a readable ONNX model (onnx_ingest/model.py:21-22)."""


class UnsupportedModel(ValueError):
    """Dynamic shapes, control flow or an unconvertible idiom (onnx_ingest/convert.py:37-38)."""


class ConversionReport:
    """Field-for-field ConversionReport (convert.py:41-47)."""

    def __init__(self, trainable_elements=0, skipped_elements=0, skipped=None, warnings=None,
                 initializer_elements=0):
        self.trainable_elements = trainable_elements
        self.skipped_elements = skipped_elements
        self.skipped = list(skipped or [])
        self.warnings = list(warnings or [])
        self.initializer_elements = initializer_elements

    def __eq__(self, other):
        return vars(self) == vars(other)

    def __repr__(self):
        return f"ConversionReport({vars(self)!r})"


def _onnx_lib():
    L = _lib()
    if not hasattr(L, "_sp_onnx_declared"):
        vp = C.c_void_p
        L.sp_ingest_onnx.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.c_int64, C.c_int32, C.POINTER(vp)]
        L.sp_ingest_onnx.restype = C.c_int
        L.sp_ingest_report.argtypes = [vp, C.POINTER(C.c_int64)]
        L.sp_ingest_report.restype = C.c_int
        L.sp_ingest_text.argtypes = [vp, C.c_int32, C.c_int64]
        L.sp_ingest_text.restype = C.c_void_p
        L._sp_onnx_declared = True
    return L


def _onnx_call(data: bytes, batch, export_only: bool):
    L = _onnx_lib()
    h = C.c_void_p()
    rc = L.sp_ingest_onnx(data, len(data), 0 if batch is None else 1, int(batch or 0), 1 if export_only else 0,
                          C.byref(h))
    if rc == SP_ERR_ONNX_PARSE:
        raise ModelParseError((L.sp_ingest_error(0) or b"").decode("utf-8", "replace"))
    if rc == SP_ERR_ONNX_UNSUPPORTED:
        raise UnsupportedModel((L.sp_ingest_error(0) or b"").decode("utf-8", "replace"))
    if rc:
        _raise(L, rc)
    counts = (C.c_int64 * 6)()
    L.sp_ingest_report(h, counts)

    def text(kind, i=0, size=None):
        p = L.sp_ingest_text(h, kind, i)
        return C.string_at(p, size).decode("utf-8") if size is not None else C.string_at(p).decode("utf-8")

    report = ConversionReport(int(counts[0]), int(counts[1]), [text(2, i) for i in range(counts[4])],
                              [text(1, i) for i in range(counts[3])], int(counts[2]))
    return h, report, (text(0, 0, int(counts[5])) if export_only else None)


def export_graph(data: bytes, batch=None):
    """ONNX model bytes -> (schema-1 JSON document, ConversionReport), natively
    (onnx_ingest.export_graph, convert.py:272-274)."""
    import json

    h, report, text = _onnx_call(bytes(data), batch, True)
    _lib().sp_ingest_free(h)
    return json.loads(text), report


def export_graph_json(data: bytes, batch=None) -> tuple:
    """As export_graph, with the document as the exact `json.dumps` text."""
    h, report, text = _onnx_call(bytes(data), batch, True)
    _lib().sp_ingest_free(h)
    return text, report


def load_onnx(data: bytes, batch=None) -> IngestedGraph:
    """ONNX bytes -> grouped graph arrays, natively: export_graph + load_graph +
    trim_and_group without the intermediate document or Python objects."""
    h, report, _ = _onnx_call(bytes(data), batch, False)
    try:
        g = _graph_from_handle(_lib(), h)
    finally:
        _lib().sp_ingest_free(h)
    g.report = report
    return g


def plan_from_onnx(data: bytes, mesh, batch=None, min_duplicates: int = 2, mu: int = 1 << 20,
                   chunk_size: int = 4 << 20, **kw):
    """ONNX model -> plan (onnx_ingest export_graph | shardplan plan), natively + device search."""
    from .search import derive_plan

    return derive_plan(load_onnx(data, batch), mesh, min_duplicates, mu, chunk_size, **kw)


def save_graph(graph, version: int = 1) -> bytes:
    """The reference's save_graph (ir.py:358-367) natively: every node of a
    ModelGraph in topo_order (a grouped node contributes its member RawNode) as
    the schema-1/2 JSON document, byte-identical to
    json.dumps(doc, sort_keys=True, separators=(",", ":")) + a newline
    (csrc/lower_ext.c save_graph_json; attribute values, arbitrary JSON, go
    through json.dumps)."""
    import functools
    import json

    from .lowering import _native_lower

    if _native_lower is None or not hasattr(_native_lower, "save_graph_json"):
        raise RuntimeError("native lowering extension (_lower) not built")
    dumps = functools.partial(json.dumps, sort_keys=True, separators=(",", ":"))
    nodes = graph.nodes if isinstance(graph.nodes, dict) else dict(graph.nodes)
    return _native_lower.save_graph_json(list(graph.topo_order), nodes, int(version), _enum_value, _dtype_label, dumps)


def _enum_value(op):
    return op.value if hasattr(op, "value") else str(op)


def _dtype_label(dt):
    return dt.label if hasattr(dt, "label") else str(dt)
