"""ctypes binding of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference arm.  The product package never
imports this module.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2302_00247_b200._abi import (
    SpBlocks,
    SpExplainOut,
    SpScoreOut,
    blocks_to_numpy,
    make_sp_graph,
    make_sp_mesh,
    ptr,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "liboracle.so")

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.oracle_prune.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]
        L.oracle_prune.restype = C.c_int
        L.oracle_blocks_view.argtypes = [C.c_void_p]
        L.oracle_blocks_view.restype = C.POINTER(SpBlocks)
        L.oracle_blocks_free.argtypes = [C.c_void_p]
        L.oracle_score.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64, C.c_void_p,
                                   C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_int32,
                                   C.POINTER(C.c_double), C.POINTER(SpScoreOut)]
        L.oracle_score.restype = C.c_int
        L.oracle_explain.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64, C.c_void_p,
                                     C.c_int64, C.c_int64, C.c_uint64, C.POINTER(SpExplainOut)]
        L.oracle_explain.restype = C.c_int
        L.oracle_slots.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64,
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.oracle_slots.restype = C.c_int
        L.oracle_graph_open.argtypes = [C.c_void_p]
        L.oracle_graph_open.restype = C.c_void_p
        L.oracle_graph_close.argtypes = [C.c_void_p]
        L.oracle_score_h.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64, C.c_void_p,
                                     C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_int32,
                                     C.POINTER(C.c_double), C.POINTER(SpScoreOut)]
        L.oracle_score_h.restype = C.c_int
        L.oracle_explain_h.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64, C.c_void_p,
                                       C.c_int64, C.c_int64, C.c_uint64, C.POINTER(SpExplainOut)]
        L.oracle_explain_h.restype = C.c_int
        _lib = L
    return _lib


def prune(low, min_dup: int) -> dict:
    g = make_sp_graph(low)
    h = C.c_void_p()
    rc = lib().oracle_prune(C.byref(g), min_dup, C.byref(h))
    if rc != 0:
        raise RuntimeError(f"oracle_prune rc={rc}")
    try:
        return blocks_to_numpy(lib().oracle_blocks_view(h).contents)
    finally:
        lib().oracle_blocks_free(h)


class _GraphHandle:
    """Per-graph oracle structures (name order, consumers), built once."""

    def __init__(self, low):
        self.keep = make_sp_graph(low)
        self.h = lib().oracle_graph_open(C.byref(self.keep))

    def __del__(self):  # pragma: no cover - GC timing
        try:
            lib().oracle_graph_close(self.h)
        except Exception:  # noqa: BLE001
            pass


def _handle(low):
    h = getattr(low, "_oracle_handle", None)
    if h is None:
        h = _GraphHandle(low)
        low._oracle_handle = h
    return h.h


def score(low, tmpl_nodes, mesh, mu=1 << 20, chunk=4 << 20, lo=0, hi=None, threads=1,
          want_totals=False):
    h = _handle(low)
    m = make_sp_mesh(mesh)
    tn = np.ascontiguousarray(tmpl_nodes, dtype=np.int32)
    out = SpScoreOut()
    if hi is None:
        hi = (1 << 64) - 1
    totals = None
    tp = None
    if want_totals:
        totals = np.empty(int(hi - lo), np.float64)
        tp = ptr(totals, C.c_double)
    rc = lib().oracle_score_h(h, ptr(tn, C.c_int32) if tn.size else None, tn.size,
                              C.byref(m), mu, chunk, lo, hi, threads, tp, C.byref(out))
    if rc != 0:
        raise RuntimeError(f"oracle_score rc={rc}")
    return out, totals


def explain(low, tmpl_nodes, mesh, index, mu=1 << 20, chunk=4 << 20) -> SpExplainOut:
    h = _handle(low)
    m = make_sp_mesh(mesh)
    tn = np.ascontiguousarray(tmpl_nodes, dtype=np.int32)
    out = SpExplainOut()
    rc = lib().oracle_explain_h(h, ptr(tn, C.c_int32), tn.size, C.byref(m), mu, chunk,
                                index, C.byref(out))
    if rc != 0:
        raise RuntimeError(f"oracle_explain rc={rc}")
    return out


def slots(low, tmpl_nodes) -> list:
    g = make_sp_graph(low)
    tn = np.ascontiguousarray(tmpl_nodes, dtype=np.int32)
    buf = np.zeros(max(1, tn.size), np.int32)
    n = C.c_int32()
    rc = lib().oracle_slots(C.byref(g), ptr(tn, C.c_int32), tn.size, ptr(buf, C.c_int32),
                            C.byref(n))
    if rc != 0:
        raise RuntimeError(f"oracle_slots rc={rc}")
    return buf[: n.value].tolist()
