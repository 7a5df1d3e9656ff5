"""ctypes mirror of include/shardsearch.h (structs and enums only)."""

from __future__ import annotations

import ctypes as C

import numpy as np

SP_MAX_RANK = 8
SP_EXPLAIN_MAX_T = 256

SP_OK = 0
SP_ERR_CONFIG = 1
SP_ERR_UNSUPPORTED = 2
SP_ERR_CUDA = 3
SP_ERR_SPEC = 4

c_i64p = C.POINTER(C.c_int64)
c_i32p = C.POINTER(C.c_int32)
c_u8p = C.POINTER(C.c_uint8)
c_u64p = C.POINTER(C.c_uint64)
c_f64p = C.POINTER(C.c_double)


class SpGraph(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64),
        ("name_bytes", c_u8p),
        ("name_off", c_i64p),
        ("topo_rank", c_i64p),
        ("op", c_u8p),
        ("act_rank", c_u8p),
        ("act_shape", c_i64p),
        ("act_bytes", c_i64p),
        ("w_rank", c_u8p),
        ("w_shape", c_i64p),
        ("w_bytes", c_i64p),
        ("w_trainable", c_u8p),
        ("in_off", c_i64p),
        ("in_idx", c_i32p),
    ]


class SpMesh(C.Structure):
    _fields_ = [
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("intra_bw", C.c_double),
        ("inter_bw", C.c_double),
        ("eff_allreduce", C.c_double),
        ("eff_allgather", C.c_double),
        ("eff_reducescatter", C.c_double),
        ("eff_alltoall", C.c_double),
        ("overlap_fraction", C.c_double),
        ("setup_latency_s", C.c_double),
    ]


class SpBlocks(C.Structure):
    _fields_ = [
        ("n_blocks", C.c_int64),
        ("n_instances", C.c_int64),
        ("n_members", C.c_int64),
        ("block_T", c_i64p),
        ("block_inst_off", c_i64p),
        ("block_member_off", c_i64p),
        ("inst_prefix_node", c_i64p),
        ("inst_prefix_len", c_i64p),
        ("members", c_i32p),
    ]


class SpScoreOut(C.Structure):
    _fields_ = [
        ("candidates", C.c_uint64),
        ("valid", C.c_uint64),
        ("best_index", C.c_uint64),
        ("best_total", C.c_double),
        ("best_num_split", C.c_int32),
        ("has_best", C.c_int32),
    ]


class SpExplainOut(C.Structure):
    _fields_ = [
        ("valid", C.c_int32),
        ("T", C.c_int32),
        ("fail_pos", C.c_int32),
        ("pattern", C.c_int32 * SP_EXPLAIN_MAX_T),
        ("state_axis", C.c_int32 * SP_EXPLAIN_MAX_T),
        ("exit_axis", C.c_int32 * SP_EXPLAIN_MAX_T),
        ("forward_comm", C.c_double),
        ("backward_comm", C.c_double),
        ("total", C.c_double),
        ("bytes_allreduce", C.c_int64),
        ("bytes_allgather", C.c_int64),
        ("bytes_reducescatter", C.c_int64),
        ("bytes_alltoall", C.c_int64),
        ("calls_allreduce", C.c_int64),
        ("calls_allgather", C.c_int64),
        ("calls_reducescatter", C.c_int64),
        ("calls_alltoall", C.c_int64),
        ("collective_calls", C.c_int64),
    ]


class SpExplainBlock(C.Structure):
    _fields_ = [
        ("valid", C.c_int32),
        ("fail_pos", C.c_int32),
        ("forward_comm", C.c_double),
        ("backward_comm", C.c_double),
        ("total", C.c_double),
        ("bytes", C.c_int64 * 4),
        ("calls", C.c_int64 * 4),
        ("collective_calls", C.c_int64),
    ]


class SpEdgeConv(C.Structure):
    _fields_ = [
        ("consumer_pos", C.c_int32),
        ("producer_pos", C.c_int32),
        ("kind", C.c_int32),
        ("axis", C.c_int32),
    ]


class SpPlanView(C.Structure):
    _fields_ = [
        ("blocks", SpBlocks),
        ("tmpl_off", c_i64p),
        ("tmpl_nodes", c_i32p),
        ("scores", C.POINTER(SpScoreOut)),
        ("detail", C.POINTER(SpExplainBlock)),
        ("node_detail", C.POINTER(C.c_int8)),
        ("edge_detail", C.POINTER(C.c_int8)),
        ("edge_off", c_i64p),
        ("n_entries", C.c_int64),
        ("n_edges", C.c_int64),
    ]


def ptr(arr: np.ndarray, ctype):
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(C.POINTER(ctype))


def make_sp_graph(low) -> SpGraph:
    """SpGraph view over a LoweredGraph (the arrays must outlive the struct)."""
    g = SpGraph()
    g.n_nodes = low.n_nodes
    g.name_bytes = ptr(low.name_bytes, C.c_uint8)
    g.name_off = ptr(low.name_off, C.c_int64)
    g.topo_rank = ptr(low.topo_rank, C.c_int64)
    g.op = ptr(low.op, C.c_uint8)
    g.act_rank = ptr(low.act_rank, C.c_uint8)
    g.act_shape = ptr(low.act_shape, C.c_int64)
    g.act_bytes = ptr(low.act_bytes, C.c_int64)
    g.w_rank = ptr(low.w_rank, C.c_uint8)
    g.w_shape = ptr(low.w_shape, C.c_int64)
    g.w_bytes = ptr(low.w_bytes, C.c_int64)
    g.w_trainable = ptr(low.w_trainable, C.c_uint8)
    g.in_off = ptr(low.in_off, C.c_int64)
    # ctypes needs a non-null pointer even for an edgeless graph
    idx = low.in_idx if low.in_idx.size else np.zeros(1, np.int32)
    g._keep = idx  # type: ignore[attr-defined]
    g.in_idx = ptr(idx, C.c_int32)
    return g


_MESH_CACHE: dict = {}


def make_sp_mesh(mesh) -> SpMesh:
    """SpMesh from a ClusterSpec-like object (costmodel.py:36-119); cached for
    hashable (frozen, value-hashed) specs."""
    try:
        hit = _MESH_CACHE.get(mesh)
    except TypeError:  # unhashable spec: built every call
        return _build_sp_mesh(mesh)
    if hit is None:
        if len(_MESH_CACHE) > 64:
            _MESH_CACHE.clear()
        hit = _MESH_CACHE[mesh] = _build_sp_mesh(mesh)
    return hit


def _build_sp_mesh(mesh) -> SpMesh:
    eff = {}
    for kind, val in mesh.efficiency:
        eff[kind.value if hasattr(kind, "value") else str(kind)] = float(val)
    m = SpMesh()
    m.m = int(mesh.m)
    m.n = int(mesh.n)
    m.intra_bw = float(mesh.intra_bw)
    m.inter_bw = float(mesh.inter_bw)
    m.eff_allreduce = eff.get("allreduce", 1.0)
    m.eff_allgather = eff.get("allgather", 1.0)
    m.eff_reducescatter = eff.get("reducescatter", 1.0)
    m.eff_alltoall = eff.get("alltoall", 1.0)
    m.overlap_fraction = float(mesh.overlap_fraction)
    m.setup_latency_s = float(mesh.setup_latency_s)
    return m


def view_array(p, n: int, dt, owner=None) -> np.ndarray:
    """n elements at ctypes pointer p as numpy: a copy, or (with `owner`, the
    object that frees the memory) a read-only view that keeps `owner` alive."""
    if n == 0:
        return np.zeros(0, dt)
    if owner is None:
        return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)
    buf = (p._type_ * n).from_address(C.addressof(p.contents))
    buf.owner = owner
    a = np.frombuffer(buf, dt)
    a.flags.writeable = False
    return a


def blocks_to_numpy(view: SpBlocks, owner=None) -> dict:
    """numpy arrays of an sp_fold view: copies, or (with `owner`, the object
    that frees the fold) read-only views that keep `owner` alive."""
    nb, ni, nm = view.n_blocks, view.n_instances, view.n_members

    arr = lambda p, n, dt: view_array(p, n, dt, owner)  # noqa: E731
    return {
        "block_T": arr(view.block_T, nb, np.int64),
        "block_inst_off": arr(view.block_inst_off, nb + 1, np.int64),
        "block_member_off": arr(view.block_member_off, nb + 1, np.int64),
        "inst_prefix_node": arr(view.inst_prefix_node, ni, np.int64),
        "inst_prefix_len": arr(view.inst_prefix_len, ni, np.int64),
        "members": arr(view.members, nm, np.int32),
    }
