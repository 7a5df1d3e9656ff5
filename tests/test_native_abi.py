"""CPU checks of the boundary: the library loads and exports every symbol the
header declares; host-side helpers (lowering, block assembly, shard merge)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shardsearch.h")


def declared_functions() -> list:
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(sp_\w+)\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for need in ("sp_ctx_create", "sp_graph_upload", "sp_fold_run", "sp_tables_build", "sp_score",
                 "sp_score_range", "sp_explain", "sp_merge_keys"):
        assert need in names


def test_library_exports_every_declared_symbol():
    from paper_2302_00247_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("backend not built")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(_native.EXPORTED_SYMBOLS)
    lib.sp_abi_version.restype = ctypes.c_int
    assert lib.sp_abi_version() == _native.ABI_VERSION == 2


def test_missing_device_fails_loudly():
    """No CPU fallback: without a usable GPU the backend raises."""
    import torch

    from paper_2302_00247_b200 import _native
    from paper_2302_00247_b200.errors import BackendError

    if torch.cuda.is_available() or not os.path.exists(_native.LIB_PATH):
        pytest.skip("needs the built library and no GPU")
    with pytest.raises(BackendError):
        _native.Backend(0)


def test_lowering_matches_graph():
    from golden_io import graph
    from paper_2302_00247_b200.lowering import lower

    g = graph("graphs/c1.json.gz")
    low = lower(g)
    assert low.n_nodes == len(g.nodes) == 172
    assert low.in_off[-1] == sum(len(n.inputs) for n in g.nodes.values()) == 219
    for i, name in enumerate(g.topo_order):
        nd = g.nodes[name]
        o = low.name_off
        assert bytes(low.name_bytes[o[i]:o[i + 1]]).decode() == name
        assert low.act_bytes[i] == nd.activation.byte_size
        assert [low.names[j] for j in low.in_idx[low.in_off[i]:low.in_off[i + 1]]] == list(nd.inputs)


def test_merge_scores_is_exact_lexicographic():
    from paper_2302_00247_b200._abi import SpScoreOut
    from paper_2302_00247_b200.dist import merge_scores, pack, unpack

    def rec(t, ns, idx, v, has=1):
        s = SpScoreOut()
        s.best_total, s.best_num_split, s.best_index, s.valid, s.has_best = t, ns, idx, v, has
        s.candidates = 100
        return s

    a = [rec(1.5, 3, 10, 4), rec(0.0, 0, 0, 1), rec(0.0, 0, 0, 0, has=0)]
    b = [rec(1.5, 2, 90, 2), rec(0.0, 0, 5, 3), rec(2.0, 1, 7, 1)]
    m = merge_scores([a, b])
    assert (m[0].best_num_split, m[0].best_index, m[0].valid) == (2, 90, 6)
    assert (m[1].best_index, m[1].valid) == (0, 4)
    assert (m[2].has_best, m[2].best_index, m[2].valid) == (1, 7, 1)
    rt = unpack(pack(m))
    assert [(r.best_total, r.best_index, r.valid) for r in rt] == [(x.best_total, x.best_index, x.valid)
                                                                     for x in m]
    big = rec(3.0, 1, (1 << 64) - 5, (1 << 63) + 1)
    assert unpack(pack([big]))[0].best_index == (1 << 64) - 5


def test_api_types_json_matches_reference_shape():
    from paper_2302_00247_b200.api_types import ClusterSpec, CostReport

    m = ClusterSpec.from_mesh("2x4")
    assert m.to_json()["efficiency"] == {"allgather": 1.2, "allreduce": 1.0, "alltoall": 1.5,
                                         "reducescatter": 1.2}
    c = CostReport(1.0, 2.0, 0.5, {"allreduce": 4}, 1, 0)
    assert c.total == 2.0 and c.to_json()["effective_backward_s"] == 1.0


def test_blocks_to_subgraphs_roundtrip():
    from golden_io import case, lowered
    from oracle import oracle
    from paper_2302_00247_b200.blocks import BlockArrays, to_prune_doc
    from paper_2302_00247_b200.search import subgraphs_from_blocks

    c = case("tiny_1x2")
    low = lowered(c["graph"])
    ba = BlockArrays.from_dict(oracle.prune(low, 2))
    subs = subgraphs_from_blocks(low, ba)
    assert [[s.template_prefix, list(s.template), [[p, list(m)] for p, m in s.instances]]
            for s in subs] == c["prune"] == to_prune_doc(low, ba)
    off, nodes = ba.templates_csr()
    assert off[-1] == nodes.size == sum(len(s.template) for s in subs)
    assert np.all(np.diff(off) >= 1)


def test_nccl_loads_on_demand_only():
    """The library has no link-time NCCL dependency (dlopen on first use), and
    the NCCL it would load exports what comm.cu resolves."""
    import subprocess

    from paper_2302_00247_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("backend not built")
    deps = subprocess.run(["ldd", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "nccl" not in deps
    nccl = ctypes.CDLL("libnccl.so.2")
    for sym in ("ncclGetUniqueId", "ncclCommInitRank", "ncclCommInitAll", "ncclCommDestroy", "ncclAllGather",
                "ncclGroupStart", "ncclGroupEnd", "ncclGetErrorString", "ncclGetVersion"):
        assert hasattr(nccl, sym), sym


def test_comm_unique_id_without_gpu():
    """sp_comm_unique_id needs no device (rank 0 makes it before any context)."""
    from paper_2302_00247_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("backend not built")
    L = _native.load_library()
    a = (ctypes.c_uint8 * _native.COMM_ID_BYTES)()
    b = (ctypes.c_uint8 * _native.COMM_ID_BYTES)()
    assert L.sp_comm_unique_id(a) == 0 and L.sp_comm_unique_id(b) == 0
    assert bytes(a) != bytes(b)
