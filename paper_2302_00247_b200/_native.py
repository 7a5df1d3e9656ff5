"""ctypes binding of lib/libshardsearch.so (include/shardsearch.h).

There is no fallback: if the library is missing or no CUDA device is usable,
every entry point raises ``BackendError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _abi
from ._abi import (
    SpBlocks,
    SpEdgeConv,
    SpExplainBlock,
    SpExplainOut,
    SpScoreOut,
    make_sp_graph,
    make_sp_mesh,
    ptr,
)
from .blocks import BlockArrays
from .errors import BackendError, BadConfig, SpecMismatch, UnsupportedSearch

HERE = os.path.dirname(os.path.abspath(__file__))
SP_SCORE_LOCAL = 2  # include/shardsearch.h
LIB_PATH = os.environ.get("SP_LIB") or os.path.join(HERE, "lib", "libshardsearch.so")

_lib = None
_lib_lock = threading.Lock()
#: SP_ABI_VERSION of include/shardsearch.h
ABI_VERSION = 2
#: SP_COMM_ID_BYTES
COMM_ID_BYTES = 128
TRANSPORTS = {0: "none", 1: "nccl", 2: "p2p"}


def _declare(L):
    vp = C.c_void_p
    L.sp_abi_version.restype = C.c_int
    L.sp_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(vp)]
    L.sp_comm_unique_id.argtypes = [C.POINTER(C.c_uint8)]
    L.sp_ctx_comm_init.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_uint8)]
    L.sp_ctx_comm_info.argtypes = [vp] + [C.POINTER(C.c_int32)] * 5
    L.sp_ctx_destroy.argtypes = [vp]
    L.sp_last_error.argtypes = [vp]
    L.sp_last_error.restype = C.c_char_p
    L.sp_graph_upload.argtypes = [vp, C.POINTER(_abi.SpGraph), C.POINTER(vp)]
    L.sp_graph_free.argtypes = [vp]
    L.sp_fold_run.argtypes = [vp, vp, C.c_int32, C.POINTER(vp)]
    L.sp_fold_view.argtypes = [vp, C.POINTER(SpBlocks)]
    L.sp_fold_free.argtypes = [vp]
    L.sp_tables_build.argtypes = [vp, vp, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                  C.POINTER(_abi.SpMesh), C.c_int64, C.c_int64, C.POINTER(vp)]
    L.sp_tables_free.argtypes = [vp]
    L.sp_tables_candidates.argtypes = [vp, C.POINTER(C.c_uint64)]
    L.sp_tables_slots.argtypes = [vp, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.sp_score.argtypes = [vp, vp, C.c_int32, C.c_int32, C.POINTER(SpScoreOut)]
    L.sp_score_range.argtypes = [vp, vp, C.c_int64, C.c_uint64, C.c_uint64, C.POINTER(C.c_double),
                                 C.POINTER(SpScoreOut)]
    L.sp_merge_keys.argtypes = [C.POINTER(SpScoreOut), C.POINTER(SpScoreOut)]
    L.sp_merge_keys.restype = None
    L.sp_explain.argtypes = [vp, vp, C.c_int64, C.c_uint64, C.POINTER(SpExplainOut),
                             C.POINTER(SpEdgeConv), C.c_int32, C.POINTER(C.c_int32)]
    L.sp_last_timings.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]
    L.sp_fold_stats.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    L.sp_timer_start.argtypes = [vp]
    L.sp_timer_stop.argtypes = [vp, C.POINTER(C.c_double)]
    L.sp_launch_counts.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.sp_tables_bytes.argtypes = [vp, C.POINTER(C.c_int64)]
    L.sp_set_option.argtypes = [vp, C.c_int32, C.c_int64]
    L.sp_search.argtypes = [vp, vp, C.POINTER(SpScoreOut), C.POINTER(SpExplainBlock),
                            C.POINTER(C.c_int8), C.POINTER(C.c_int8)]
    L.sp_score_launch.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_int32]
    L.sp_score_wait.argtypes = [vp, vp, C.POINTER(SpScoreOut), C.POINTER(SpExplainBlock),
                                C.POINTER(C.c_int8), C.POINTER(C.c_int8)]
    L.sp_tables_sizes.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.sp_tables_edge_offsets.argtypes = [vp, C.POINTER(C.c_int64)]
    L.sp_explain_all.argtypes = [vp, vp, C.POINTER(C.c_uint64), C.POINTER(SpExplainBlock),
                                 C.POINTER(C.c_int8), C.POINTER(C.c_int8)]
    L.sp_copy_bytes.argtypes = [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.sp_route_search.argtypes = [vp, vp, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int16), C.POINTER(C.c_uint8), C.POINTER(C.c_int64),
                                  C.POINTER(_abi.SpMesh), C.c_int64, C.c_int64, C.POINTER(C.c_uint64),
                                  C.POINTER(SpScoreOut), C.POINTER(SpExplainBlock), C.POINTER(C.c_int8),
                                  C.POINTER(C.c_int8)]
    L.sp_plan_run.argtypes = [vp, vp, C.c_int32, C.POINTER(_abi.SpMesh), C.c_int64, C.c_int64, C.POINTER(vp)]
    L.sp_plan_view_get.argtypes = [vp, C.POINTER(_abi.SpPlanView)]
    L.sp_plan_free.argtypes = [vp]
    L.sp_ctx_limits.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    L.sp_tables_block_info.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    for name in ("sp_plan_run", "sp_plan_view_get", "sp_route_search", "sp_ctx_limits", "sp_tables_block_info", "sp_comm_unique_id",
                 "sp_ctx_comm_init", "sp_ctx_comm_info", "sp_score_launch", "sp_score_wait", "sp_set_option", "sp_search", "sp_tables_sizes", "sp_tables_edge_offsets", "sp_explain_all", "sp_tables_bytes", "sp_copy_bytes", "sp_timer_start", "sp_timer_stop", "sp_launch_counts", "sp_ctx_create", "sp_graph_upload", "sp_fold_run", "sp_fold_view",
                 "sp_tables_build", "sp_tables_candidates", "sp_tables_slots", "sp_score",
                 "sp_score_range", "sp_explain", "sp_last_timings"):
        getattr(L, name).restype = C.c_int
    for name in ("sp_ctx_destroy", "sp_graph_free", "sp_fold_free", "sp_tables_free", "sp_plan_free"):
        getattr(L, name).restype = None


def load_library():
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendError(
                    f"native backend not built ({LIB_PATH} missing); run "
                    "`python -c 'import __graft_entry__ as g; g.build()'`")
            L = C.CDLL(LIB_PATH)
            _declare(L)
            if L.sp_abi_version() != ABI_VERSION:
                raise BackendError("libshardsearch ABI version mismatch")
            _lib = L
    return _lib


EXPORTED_SYMBOLS = (
    "sp_abi_version", "sp_ctx_create", "sp_ctx_destroy", "sp_last_error", "sp_graph_upload",
    "sp_graph_free", "sp_fold_run", "sp_fold_view", "sp_fold_free", "sp_tables_build",
    "sp_tables_free", "sp_tables_candidates", "sp_tables_slots", "sp_score", "sp_score_range",
    "sp_merge_keys", "sp_explain", "sp_last_timings", "sp_timer_start", "sp_timer_stop",
    "sp_launch_counts", "sp_copy_bytes", "sp_tables_bytes", "sp_tables_sizes",
    "sp_tables_edge_offsets", "sp_explain_all", "sp_search", "sp_set_option",
    "sp_fold_stats", "sp_score_launch", "sp_score_wait", "sp_ingest_json", "sp_ingest_error",
    "sp_ingest_view", "sp_ingest_free", "sp_ingest_onnx", "sp_ingest_report", "sp_ingest_text",
    "sp_comm_unique_id", "sp_ctx_comm_init", "sp_ctx_comm_info", "sp_route_search", "sp_ctx_limits",
    "sp_tables_block_info", "sp_plan_run", "sp_plan_view_get", "sp_plan_free",
)


class RawList(list):
    """The records of a ctypes array as a list, keeping the array as `.raw`
    (native consumers read the records without per-element objects)."""

    def __init__(self, arr, n: int):
        super().__init__(arr[i] for i in range(n))
        self.raw = arr


class _Handle:
    def __init__(self, backend, ptr_, free_fn):
        self.backend = backend
        self.ptr = ptr_
        self._free = free_fn

    def close(self):
        if self.ptr:
            # objects of a context that was already destroyed are gone with it
            # (their free would touch the context's stream and pools)
            if getattr(self.backend, "ctx", None):
                self._free(self.ptr)
            self.ptr = None

    def __del__(self):  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class Tables(_Handle):
    n_blocks: int
    candidates: np.ndarray
    overflow: bool


class Backend:
    """One library context (sp_ctx_create) over one device -- one process per
    GPU, joined to the other ranks with `comm_init` -- or over several devices
    of this process (`devices=[...]`): the library then fans every call out
    over them and a search deals each block's work items across the devices,
    merging on the first (search.py:327-343's pool split and min-merge)."""

    def __init__(self, device: int | None = None, devices=None):
        self.lib = load_library()
        if devices is None:
            if device is None:
                device = int(os.environ.get("SP_DEVICE", os.environ.get("LOCAL_RANK", "0")))
            devices = [device]
        devices = [int(d) for d in devices]
        self.devices = devices
        self.device = devices[0]
        h = C.c_void_p()
        arr = (C.c_int * len(devices))(*devices)
        rc = self.lib.sp_ctx_create(len(devices), arr, C.byref(h))
        if rc != 0:
            raise BackendError(f"sp_ctx_create(devices={devices}) failed with status {rc}")
        self.ctx = h
        self.comm = self.comm_info()
        self.smem_limit = self.limits()["smem_per_block"]

    # -- multi-GPU -----------------------------------------------------------------
    def comm_unique_id(self) -> bytes:
        """A fresh NCCL unique id (rank 0), to hand to every rank's comm_init."""
        buf = (C.c_uint8 * COMM_ID_BYTES)()
        self._check(self.lib.sp_comm_unique_id(buf), "sp_comm_unique_id")
        return bytes(buf)

    def comm_init(self, nranks: int, rank: int, uid: bytes) -> None:
        """Join `nranks` processes (one GPU each) in one NCCL communicator: from then
        on every search scores this rank's share and merges on the device."""
        if len(uid) != COMM_ID_BYTES:
            raise BadConfig(f"NCCL unique id must be {COMM_ID_BYTES} bytes")
        buf = (C.c_uint8 * COMM_ID_BYTES).from_buffer_copy(uid)
        self._check(self.lib.sp_ctx_comm_init(self.ctx, int(nranks), int(rank), buf), "sp_ctx_comm_init")
        self.comm = self.comm_info()

    def comm_info(self) -> dict:
        v = [C.c_int32() for _ in range(5)]
        self._check(self.lib.sp_ctx_comm_info(self.ctx, *[C.byref(x) for x in v]), "sp_ctx_comm_info")
        return {"nranks": v[0].value, "rank": v[1].value, "devices": v[2].value,
                "transport": TRANSPORTS.get(v[3].value, str(v[3].value)), "nccl_version": v[4].value}

    @property
    def sharded_in_library(self) -> bool:
        """True when searches are split and merged by the library itself (several
        devices in this context, or a multi-process communicator)."""
        return self.comm["nranks"] > 1

    @property
    def single_lane(self) -> bool:
        """One device and no communicator (sp_plan_run's contexts)."""
        return self.comm["devices"] == 1 and self.comm["transport"] == "none"

    @property
    def is_root(self) -> bool:
        """Rank 0 of a multi-process communicator (always true otherwise)."""
        return self.comm["devices"] > 1 or self.comm["rank"] == 0

    # -- errors --------------------------------------------------------------------
    def _check(self, rc: int, what: str):
        if rc == 0:
            return
        msg = (self.lib.sp_last_error(self.ctx) or b"").decode("utf-8", "replace")
        if rc == _abi.SP_ERR_CONFIG:
            raise BadConfig(msg or what)
        if rc == _abi.SP_ERR_UNSUPPORTED:
            raise UnsupportedSearch(msg or what)
        if rc == _abi.SP_ERR_SPEC:
            raise SpecMismatch(msg or what)
        raise BackendError(f"{what}: {msg}")

    # -- graph ---------------------------------------------------------------------
    def upload(self, low) -> _Handle:
        g = make_sp_graph(low)
        h = C.c_void_p()
        self._check(self.lib.sp_graph_upload(self.ctx, C.byref(g), C.byref(h)), "sp_graph_upload")
        return _Handle(self, h, self.lib.sp_graph_free)

    def fold(self, dgraph: _Handle, min_dup: int) -> BlockArrays:
        h = C.c_void_p()
        self._check(self.lib.sp_fold_run(self.ctx, dgraph.ptr, int(min_dup), C.byref(h)),
                    "sp_fold_run")
        owner = _Handle(self, h, self.lib.sp_fold_free)
        view = SpBlocks()
        self._check(self.lib.sp_fold_view(h, C.byref(view)), "sp_fold_view")
        # zero-copy: the arrays view the fold's own buffers, which stay alive
        # (owner) as long as any of them does (10^7-node folds: ~60 MB)
        return BlockArrays.from_dict(_abi.blocks_to_numpy(view, owner))

    def plan(self, dgraph: _Handle, min_dup: int, mesh, mu: int, chunk: int):
        """The device half of derive_plan in one call (sp_plan_run): (fold
        BlockArrays, template csr, scores, (blocks, node_detail, edge_detail,
        edge_off)) -- views into one library-owned result."""
        m = make_sp_mesh(mesh)
        h = C.c_void_p()
        self._check(self.lib.sp_plan_run(self.ctx, dgraph.ptr, int(min_dup), C.byref(m), int(mu), int(chunk),
                                         C.byref(h)), "sp_plan_run")
        owner = _Handle(self, h, self.lib.sp_plan_free)
        v = _abi.SpPlanView()
        self._check(self.lib.sp_plan_view_get(h, C.byref(v)), "sp_plan_view_get")
        bv = v.blocks
        nb, ni, nm, ne, nedge = bv.n_blocks, bv.n_instances, bv.n_members, v.n_entries, v.n_edges
        # the view's arrays are one contiguous block (16-byte aligned parts in
        # field order, include/shardsearch.h): one buffer, then numpy slices
        sizes = (8 * nb, 8 * (nb + 1), 8 * (nb + 1), 8 * ni, 8 * ni, 4 * nm, 8 * (nb + 1), 4 * ne,
                 C.sizeof(SpScoreOut) * max(nb, 1), C.sizeof(SpExplainBlock) * max(nb, 1), max(4 * ne, 1),
                 max(2 * nedge, 1), 8 * (nb + 1))
        offs, tot = [], 0
        for z in sizes:
            offs.append(tot)
            tot += (z + 15) & ~15
        base = C.addressof(bv.block_T.contents)
        buf = (C.c_char * tot).from_address(base)
        buf.owner = owner
        a = np.frombuffer(buf, np.uint8)
        a.flags.writeable = False
        part = lambda i, n, dt: a[offs[i]:offs[i] + n * np.dtype(dt).itemsize].view(dt)  # noqa: E731
        ba = BlockArrays.from_dict({
            "block_T": part(0, nb, np.int64), "block_inst_off": part(1, nb + 1, np.int64),
            "block_member_off": part(2, nb + 1, np.int64), "inst_prefix_node": part(3, ni, np.int64),
            "inst_prefix_len": part(4, ni, np.int64), "members": part(5, nm, np.int32)})
        toff = part(6, nb + 1, np.int64)
        tnodes = part(7, ne, np.int32)
        recs = (SpScoreOut * max(nb, 1)).from_address(base + offs[8])
        recs.owner = owner
        xb = (SpExplainBlock * max(nb, 1)).from_address(base + offs[9])
        xb.owner = owner
        node = part(10, 4 * ne, np.int8).reshape(ne, 4)
        edge = part(11, 2 * nedge, np.int8).reshape(nedge, 2)
        eoff = part(12, nb + 1, np.int64)
        return ba, (toff, tnodes), RawList(recs, nb), (RawList(xb, nb), node, edge, eoff)

    def tables(self, dgraph: _Handle, tmpl_off: np.ndarray, tmpl_nodes: np.ndarray, mesh,
               mu: int, chunk: int) -> Tables:
        off = np.ascontiguousarray(tmpl_off, dtype=np.int64)
        nodes = np.ascontiguousarray(tmpl_nodes, dtype=np.int32)
        if nodes.size == 0:
            nodes = np.zeros(1, np.int32)
        m = make_sp_mesh(mesh)
        h = C.c_void_p()
        nb = off.size - 1
        self._check(self.lib.sp_tables_build(self.ctx, dgraph.ptr, nb, ptr(off, C.c_int64),
                                              ptr(nodes, C.c_int32), C.byref(m), int(mu),
                                              int(chunk), C.byref(h)), "sp_tables_build")
        t = Tables(self, h, self.lib.sp_tables_free)
        t.n_blocks = nb
        cands = np.zeros(max(nb, 1), np.uint64)
        rc = self.lib.sp_tables_candidates(h, ptr(cands, C.c_uint64))
        t.overflow = rc == _abi.SP_ERR_UNSUPPORTED
        t.candidates = cands[:nb]
        nbytes = C.c_int64()
        self.lib.sp_tables_bytes(h, C.byref(nbytes))
        t.nbytes = nbytes.value
        return t

    def slots(self, t: Tables, block: int) -> list:
        n = C.c_int32()
        self._check(self.lib.sp_tables_slots(t.ptr, block, None, C.byref(n)), "sp_tables_slots")
        buf = np.zeros(max(1, n.value), np.int32)
        self._check(self.lib.sp_tables_slots(t.ptr, block, ptr(buf, C.c_int32), C.byref(n)),
                    "sp_tables_slots")
        return buf[: n.value].tolist()

    # -- scoring -------------------------------------------------------------------
    def score(self, t: Tables, shard: int = 0, n_shards: int = 1) -> list:
        outs = (SpScoreOut * max(1, t.n_blocks))()
        self._check(self.lib.sp_score(self.ctx, t.ptr, shard, n_shards, outs), "sp_score")
        return [outs[i] for i in range(t.n_blocks)]

    def score_range(self, t: Tables, block: int, lo: int, hi: int, want_totals: bool = False):
        out = SpScoreOut()
        totals = None
        tp = None
        if want_totals and hi > lo:
            totals = np.empty(hi - lo, np.float64)
            tp = ptr(totals, C.c_double)
        self._check(self.lib.sp_score_range(self.ctx, t.ptr, block, lo, hi, tp, C.byref(out)),
                    "sp_score_range")
        return out, totals

    def explain(self, t: Tables, block: int, index: int):
        out = SpExplainOut()
        cap = 4096
        edges = (SpEdgeConv * cap)()
        ne = C.c_int32()
        self._check(self.lib.sp_explain(self.ctx, t.ptr, block, index, C.byref(out), edges, cap,
                                        C.byref(ne)), "sp_explain")
        return out, [edges[i] for i in range(min(ne.value, cap))]

    def _detail_buffers(self, t: Tables):
        nb = t.n_blocks
        ne, nedge = C.c_int64(), C.c_int64()
        self.lib.sp_tables_sizes(t.ptr, C.byref(ne), C.byref(nedge))
        blocks = (SpExplainBlock * max(1, nb))()
        node = np.zeros((max(1, ne.value), 4), np.int8)
        edge = np.zeros((max(1, nedge.value), 2), np.int8)
        eoff = np.zeros(nb + 1, np.int64)
        self.lib.sp_tables_edge_offsets(t.ptr, ptr(eoff, C.c_int64))
        return blocks, node, edge, eoff

    def search(self, t: Tables) -> tuple:
        """Score every block and explain each block's argmin in one call (one sync).
        Returns (scores, (blocks, node_detail, edge_detail, edge_off))."""
        outs = (SpScoreOut * max(1, t.n_blocks))()
        blocks, node, edge, eoff = self._detail_buffers(t)
        self._check(self.lib.sp_search(self.ctx, t.ptr, outs, blocks, ptr(node, C.c_int8),
                                       ptr(edge, C.c_int8)), "sp_search")
        nb = t.n_blocks
        return [outs[i] for i in range(nb)], ([blocks[i] for i in range(nb)], node, edge, eoff)

    def score_launch(self, t: Tables, shard: int = 0, n_shards: int = 1, explain: bool = False,
                     local: bool = False) -> None:
        """Enqueue the search (sp_score_launch) and return at once; collect with score_wait.
        `local`: the whole search on this device with no exchange (SP_SCORE_LOCAL)."""
        flags = (1 if explain else 0) | (SP_SCORE_LOCAL if local else 0)
        self._check(self.lib.sp_score_launch(self.ctx, t.ptr, shard, n_shards, flags), "sp_score_launch")
        t.pending_explain = explain

    def score_wait(self, t: Tables) -> tuple:
        """(scores, detail) of the search in flight; detail is None unless it was
        launched with explain (then as explain_all returns it)."""
        nb = t.n_blocks
        outs = (SpScoreOut * max(1, nb))()
        if getattr(t, "pending_explain", False):
            blocks, node, edge, eoff = self._detail_buffers(t)
            self._check(self.lib.sp_score_wait(self.ctx, t.ptr, outs, blocks, ptr(node, C.c_int8),
                                               ptr(edge, C.c_int8)), "sp_score_wait")
            detail = (RawList(blocks, nb), node, edge, eoff)
        else:
            self._check(self.lib.sp_score_wait(self.ctx, t.ptr, outs, None, None, None),
                        "sp_score_wait")
            detail = None
        t.pending_explain = False
        return RawList(outs, nb), detail

    def explain_all(self, t: Tables, indices) -> tuple:
        """Winner detail of every block: (blocks, node_detail [ne,4], edge_detail [nedge,2],
        edge_off [nb+1])."""
        nb = t.n_blocks
        idx = np.ascontiguousarray(indices, dtype=np.uint64)
        blocks, node, edge, eoff = self._detail_buffers(t)
        self._check(self.lib.sp_explain_all(self.ctx, t.ptr, ptr(idx, C.c_uint64), blocks,
                                            ptr(node, C.c_int8), ptr(edge, C.c_int8)),
                    "sp_explain_all")
        return RawList(blocks, nb), node, edge, eoff

    def limits(self) -> dict:
        sm, nsm = C.c_int64(), C.c_int32()
        self._check(self.lib.sp_ctx_limits(self.ctx, C.byref(sm), C.byref(nsm)), "sp_ctx_limits")
        return {"smem_per_block": sm.value, "sm_count": nsm.value}

    def block_info(self, t: Tables) -> tuple:
        """(blob bytes, live-value pool slots, template nodes) per block of built tables."""
        nb = t.n_blocks
        by = np.zeros(max(1, nb), np.int64)
        pool = np.zeros(max(1, nb), np.int32)
        T = np.zeros(max(1, nb), np.int32)
        self._check(self.lib.sp_tables_block_info(t.ptr, ptr(by, C.c_int64), ptr(pool, C.c_int32),
                                                  ptr(T, C.c_int32)), "sp_tables_block_info")
        return by[:nb], pool[:nb], T[:nb]

    def route_search(self, dgraph: _Handle, tmpl_off, tmpl_nodes, ref_slot, radix, edge_off, mesh, mu: int,
                     chunk: int, indices=None) -> tuple:
        """Table-free search of blocks beyond the table limits (sp_route_search):
        (scores, (blocks, node_detail, edge_detail, edge_off)); with `indices`,
        the detail of those candidates only (scores None)."""
        off = np.ascontiguousarray(tmpl_off, dtype=np.int64)
        nodes = np.ascontiguousarray(tmpl_nodes, dtype=np.int32)
        rs = np.ascontiguousarray(ref_slot, dtype=np.int16)
        rx = np.ascontiguousarray(radix, dtype=np.uint8)
        eoff = np.ascontiguousarray(edge_off, dtype=np.int64)
        nb = len(off) - 1
        ne, nedge = int(off[-1]), int(eoff[-1])
        if nodes.size == 0:
            nodes, rs, rx = np.zeros(1, np.int32), np.zeros(1, np.int16), np.zeros(1, np.uint8)
        m = make_sp_mesh(mesh)
        blocks = (SpExplainBlock * max(1, nb))()
        node = np.zeros((max(1, ne), 4), np.int8)
        edge = np.zeros((max(1, nedge), 2), np.int8)
        outs = None if indices is not None else (SpScoreOut * max(1, nb))()
        idx = None if indices is None else np.ascontiguousarray(indices, dtype=np.uint64)
        self._check(self.lib.sp_route_search(self.ctx, dgraph.ptr, nb, ptr(off, C.c_int64), ptr(nodes, C.c_int32),
                                             ptr(rs, C.c_int16), ptr(rx, C.c_uint8), ptr(eoff, C.c_int64),
                                             C.byref(m), int(mu), int(chunk),
                                             ptr(idx, C.c_uint64) if idx is not None else None, outs, blocks,
                                             ptr(node, C.c_int8), ptr(edge, C.c_int8)), "sp_route_search")
        scores = RawList(outs, nb) if outs is not None else None
        return scores, (RawList(blocks, nb), node, edge, eoff)

    def timings(self) -> dict:
        f, s, k = C.c_double(), C.c_double(), C.c_double()
        self.lib.sp_last_timings(self.ctx, C.byref(f), C.byref(s), C.byref(k))
        d, lv = C.c_double(), C.c_int32()
        self.lib.sp_fold_stats(self.ctx, C.byref(d), C.byref(lv))
        return {"fold_ms": f.value, "score_ms": s.value, "score_kernel_ms": k.value,
                "fold_device_ms": d.value, "fold_levels": lv.value}

    def set_prefix_skip(self, on: bool) -> None:
        """Exact prefix-failure skipping in sp_score/sp_search (default on)."""
        self._check(self.lib.sp_set_option(self.ctx, 1, 1 if on else 0), "sp_set_option")

    def set_memo(self, on: bool) -> None:
        """Memoised brute force when skipping is off (default on)."""
        self._check(self.lib.sp_set_option(self.ctx, 2, 1 if on else 0), "sp_set_option")

    def set_host_layout(self, on: bool) -> None:
        """Table layout of small graphs on the host (default on); off: on the device."""
        self._check(self.lib.sp_set_option(self.ctx, 3, 1 if on else 0), "sp_set_option")

    def set_sim_shard(self, rank: int, nranks: int) -> None:
        """Measurement only (tools/shard_sim.py): every search scores rank `rank`'s
        share of an `nranks`-rank search, winner detail chained on the device as
        after the multi-GPU merge.  (0, 1) turns it off."""
        v = 0 if nranks <= 1 else (int(nranks) << 16) | int(rank)
        self._check(self.lib.sp_set_option(self.ctx, 4, v), "sp_set_option")
        self.sim_nranks = max(1, int(nranks))

    def set_mode(self, mode: str) -> None:
        """'skip' (default), 'memo' (every candidate visited, dirty nodes re-routed)
        or 'walk' (every node of every candidate)."""
        if mode not in ("skip", "memo", "walk"):
            raise ValueError(mode)
        self.set_prefix_skip(mode == "skip")
        self.set_memo(mode == "memo")

    def timer_start(self):
        self._check(self.lib.sp_timer_start(self.ctx), "sp_timer_start")

    def timer_stop(self) -> float:
        ms = C.c_double()
        self._check(self.lib.sp_timer_stop(self.ctx, C.byref(ms)), "sp_timer_stop")
        return ms.value

    def launch_counts(self) -> tuple:
        a, b = C.c_int64(), C.c_int64()
        self.lib.sp_launch_counts(self.ctx, C.byref(a), C.byref(b))
        return a.value, b.value

    def copy_bytes(self) -> tuple:
        a, b = C.c_int64(), C.c_int64()
        self.lib.sp_copy_bytes(C.byref(a), C.byref(b))
        return a.value, b.value

    def close(self):
        if self.ctx:
            self.lib.sp_ctx_destroy(self.ctx)
            self.ctx = None


_default: Backend | None = None


def default_backend() -> Backend:
    global _default
    if _default is None:
        _default = Backend()
    return _default
