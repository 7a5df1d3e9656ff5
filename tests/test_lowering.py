"""Native lowering (csrc/lower_ext.c) == the numpy restatement (lowering.lower(native=False)).

Both walk the same grouped-graph objects (ir.py:164-292); every array the
device receives must be identical, for this package's graph types, for
JSON-loaded graphs (one str object per dtype) and -- when the reference is
importable here -- for the reference's own ModelGraph/GraphNode/TensorSpec.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from golden_io import graph
from paper_2302_00247_b200 import lowering
from paper_2302_00247_b200.errors import UnsupportedSearch
from paper_2302_00247_b200.ir import GraphNode, GroupedGraph, OpKind, TensorSpec
from paper_2302_00247_b200.search import _Uncached
from paper_2302_00247_b200.workloads import motif_dag

ARRAYS = ("name_bytes", "name_off", "topo_rank", "op", "act_rank", "act_shape", "act_bytes", "w_rank",
          "w_shape", "w_bytes", "w_trainable", "in_off", "in_idx")
REF = "/root/reference/pkg/src"

pytestmark = pytest.mark.skipif(lowering._native_lower is None, reason="native lowering not built")


def _same(g):
    a = lowering.lower(_Uncached(g), native=False)
    b = lowering.lower(_Uncached(g), native=True)
    for k in ARRAYS:
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and x.shape == y.shape and np.array_equal(x, y), k
    assert a.names == b.names
    assert a.index == b.index
    return b


@pytest.mark.parametrize("path", ["graphs/c1.json.gz", "graphs/c2_t5.json.gz", "graphs/c3.json.gz",
                                  "graphs/tiny_transformer_f64.json.gz", "graphs/weighted_layernorm.json.gz",
                                  "graphs/zero_weight.json.gz", "graphs/wide150.json.gz"])
def test_native_equals_numpy_on_golden_graphs(path):
    _same(graph(path))


def test_native_equals_numpy_on_motif_dag():
    low = _same(motif_dag(1, "parity"))
    assert low.ascii


def test_native_rejects_rank_overflow_and_unknown_inputs():
    nodes = {"a": GraphNode("a", OpKind.INPUT, (), TensorSpec(tuple([2] * 9)))}
    g = GroupedGraph.__new__(GroupedGraph)
    g.nodes, g.topo_order = nodes, ["a"]
    with pytest.raises(UnsupportedSearch):
        lowering.lower(_Uncached(g))
    nodes = {"a": GraphNode("a", OpKind.INPUT, ("ghost",), TensorSpec((2,)))}
    g.nodes = nodes
    with pytest.raises(KeyError):
        lowering.lower(_Uncached(g))


def test_native_non_ascii_names():
    nodes = {"é/a": GraphNode("é/a", OpKind.INPUT, (), TensorSpec((4, 4))),
             "é/b": GraphNode("é/b", OpKind.MATMUL, ("é/a",), TensorSpec((4, 4)), TensorSpec((4, 4), "f64", True))}
    g = GroupedGraph.__new__(GroupedGraph)
    g.nodes, g.topo_order = nodes, ["é/a", "é/b"]
    low = _same(g)
    assert not low.ascii
    assert bytes(low.name_bytes).decode() == "é/aé/b"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_native_equals_numpy_on_reference_types():
    sys.path.insert(0, REF)
    try:
        from shardplan.generators import gen_transformer_stack
        from shardplan.ir import trim_and_group
    finally:
        sys.path.remove(REF)
    _same(trim_and_group(gen_transformer_stack(3, d_model=64, heads=4)))


def _chain(n=6000, bad=None, copies=False):
    """n-node chain of matmuls (above the parallel walker's size threshold),
    with one node perturbed to fall outside the walker's envelope.  `copies`:
    inputs and dict keys are equal but distinct str objects (as a JSON-loaded
    graph has), so every lookup goes by content, not by object."""
    nodes = {}
    prev = None
    for i in range(n):
        nm = f"net/l{i}/MatMul" if i else "net/in"
        ins = ("".join(list(prev)),) if prev and copies else (prev,) if prev else ()
        w = TensorSpec((8, 8), "f32", bool(i % 2)) if i else None
        nodes[nm] = GraphNode(nm, OpKind.MATMUL if i else OpKind.INPUT, ins, TensorSpec((4, 8)), w)
        prev = nm
    names = list(nodes)
    if bad == "non_ascii":
        old = names[n // 2]
        new = old.replace("net", "nét")
        nodes = {(new if k == old else k): v for k, v in nodes.items()}
        names[n // 2] = new
        nx = names[n // 2 + 1]
        nodes[nx] = GraphNode(nx, OpKind.MATMUL, (new,), TensorSpec((4, 8)), TensorSpec((8, 8)))
    elif bad == "list_inputs":
        k = names[n - 3]
        nodes[k] = GraphNode(k, OpKind.MATMUL, list(nodes[k].inputs), TensorSpec((4, 8)), TensorSpec((8, 8)))
    elif bad == "big_int":
        k = names[n - 2]
        nodes[k] = GraphNode(k, OpKind.MATMUL, nodes[k].inputs, TensorSpec((4, 2 ** 40)), None)
    elif bad == "ghost":
        k = names[n - 1]
        nodes[k] = GraphNode(k, OpKind.MATMUL, ("ghost",), TensorSpec((4, 8)), None)
    elif bad == "rank9":
        k = names[17]
        nodes[k] = GraphNode(k, OpKind.MATMUL, nodes[k].inputs, TensorSpec(tuple([2] * 9)), None)
    if copies:
        nodes = {"".join(list(k)): v for k, v in nodes.items()}
    g = GroupedGraph.__new__(GroupedGraph)
    g.nodes, g.topo_order = nodes, names
    return g


@pytest.mark.parametrize("threads", ["2", "3", "7", "16"])
def test_parallel_walker_equals_numpy(monkeypatch, threads):
    monkeypatch.setenv("SP_LOWER_THREADS", threads)
    low = _same(motif_dag(1, "parity"))
    assert low.ascii
    _same(_chain())
    _same(_chain(copies=True))


def test_parallel_walker_equals_serial(monkeypatch):
    g = motif_dag(2, "parity")
    par = lowering.lower(_Uncached(g))
    monkeypatch.setenv("SP_LOWER_SERIAL", "1")
    ser = lowering.lower(_Uncached(g))
    for k in ARRAYS:
        assert np.array_equal(getattr(par, k), getattr(ser, k)), k


@pytest.mark.parametrize("bad", ["non_ascii", "list_inputs", "big_int"])
def test_parallel_walker_declines_outside_envelope(bad):
    low = _same(_chain(bad=bad))
    assert low.ascii == (bad != "non_ascii")


def test_parallel_walker_errors_match_serial():
    with pytest.raises(KeyError):
        lowering.lower(_Uncached(_chain(bad="ghost")))
    with pytest.raises(UnsupportedSearch):
        lowering.lower(_Uncached(_chain(bad="rank9")))


def test_native_walker_version_guard():
    """csrc/lower_ext.c reads CPython object layouts in place (compact str and
    int): the module records the interpreter it was built for, and lowering
    uses it only under that minor version; both search modules bind the same
    extension (or none)."""
    import sys

    from paper_2302_00247_b200 import lowering, search

    lw = lowering._native_lower
    if lw is None:
        import pytest

        pytest.skip("native walker not built")
    assert lw.built_for_hexversion >> 16 == sys.hexversion >> 16
    assert (3, 12) <= sys.version_info[:2] < (3, 14)
    assert search._native_lower is None or search._native_lower is lw
