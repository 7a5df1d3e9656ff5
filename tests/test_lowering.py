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
