"""Native graph ingest (csrc/ingest.cpp) vs the reference's load_graph + trim_and_group.

Pinned by tests/golden/ingest (made by make_ingest_golden.py from the
reference itself): the grouped graph every raw document lowers to and the
exception class every malformed document raises.  When the reference is
importable (this container) the same comparison also runs on seeded random
raw graphs with auxiliary chains, scope collisions and duplicate edges.
Host-only code: no GPU needed.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

import numpy as np
import pytest

from paper_2302_00247_b200 import errors as E
from paper_2302_00247_b200.ingest import load_lowered
from paper_2302_00247_b200.ir import grouped_from_doc
from paper_2302_00247_b200.lowering import lower

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ingest")
REF = "/root/reference/pkg/src"
ARRAYS = ("name_bytes", "name_off", "topo_rank", "op", "act_rank", "act_shape", "act_bytes", "w_rank",
          "w_shape", "w_bytes", "w_trainable", "in_off", "in_idx")
FIXTURES = sorted(f[: -len(".raw.json.gz")] for f in os.listdir(GOLD) if f.endswith(".raw.json.gz"))


def _same(got, exp):
    for k in ARRAYS:
        x, y = getattr(got, k), getattr(exp, k)
        assert x.dtype == y.dtype and x.shape == y.shape and np.array_equal(x, y), k
    assert got.names == exp.names


@pytest.mark.parametrize("name", FIXTURES)
def test_ingest_matches_reference_grouping(name):
    raw = gzip.open(os.path.join(GOLD, f"{name}.raw.json.gz")).read()
    exp = grouped_from_doc(json.load(gzip.open(os.path.join(GOLD, f"{name}.grouped.json.gz"), "rt")))
    g = load_lowered(raw)
    _same(g.low, lower(exp))
    # the ModelGraph read API over the ingested arrays
    assert list(g.topo_order) == list(exp.topo_order)
    for s in exp.topo_order[:50]:
        a, b = g.nodes[s], exp.nodes[s]
        assert (a.op, a.inputs, a.activation, a.weight) == (b.op, b.inputs, b.activation, b.weight)


ERRORS = json.load(open(os.path.join(GOLD, "errors.json")))


@pytest.mark.parametrize("case", ERRORS, ids=[c["name"] for c in ERRORS])
def test_ingest_errors_like_reference(case):
    cls = getattr(E, case["error"])
    with pytest.raises(cls) as info:
        load_lowered(case["doc"].encode())
    if case["error"] == "CycleError":
        assert (info.value.src, info.value.dst) == (case["src"], case["dst"])


def test_ingest_path_and_gzip(tmp_path):
    raw = gzip.open(os.path.join(GOLD, "tiny_transformer.raw.json.gz")).read()
    p = tmp_path / "g.json"
    p.write_bytes(raw)
    a = load_lowered(str(p))
    b = load_lowered(os.path.join(GOLD, "tiny_transformer.raw.json.gz"))
    _same(a.low, b.low)
    assert a.n_raw > len(a.names) and a.n_aux > 0


def test_ingest_escapes_and_unicode_names():
    doc = {"nodes": [
        {"name": "iné/x", "op": "input", "output": {"shape": [2, 2]}},
        {"name": 'b"q/中', "op": "matmul", "inputs": ["iné/x"], "output": {"shape": [2, 4]},
         "weight": {"shape": [2, 4], "trainable": True, "dtype": "f64"}},
    ]}
    g = load_lowered(json.dumps(doc).encode())  # json.dumps escapes non-ASCII as \\uXXXX
    assert g.names == ["iné", 'b"q']  # single compute node per scope: grouped to the scope
    assert not g.low.ascii
    assert g.nodes['b"q'].weight.dtype == "f64"
    assert g.nodes['b"q'].inputs == ("iné",)


def _random_raw(rng: random.Random):
    """Raw DAG with nested scopes, aux chains, duplicate edges and scope/name collisions."""
    sys.path.insert(0, REF)
    try:
        from shardplan.ir import DType, ModelGraph, OpKind, RawNode, TensorSpec
    finally:
        sys.path.remove(REF)
    kinds = [OpKind.MATMUL, OpKind.ELEMENTWISE, OpKind.LAYERNORM, OpKind.SOFTMAX, OpKind.RESHAPE,
             OpKind.AUXILIARY, OpKind.AUXILIARY]
    nodes = [RawNode("input", OpKind.INPUT, (), TensorSpec((4, 8)))]
    scopes = ["a", "a/b", "a/b/c", "d", "d/e", ""]
    used = {"input"}
    for i in range(rng.randint(5, 60)):
        sc = rng.choice(scopes)
        nm = f"{sc}/n{i}" if sc else f"n{i}"
        if rng.random() < 0.1 and sc and sc not in used:
            nm = sc  # a node sitting on a scope other nodes extend
        if nm in used:
            nm = f"{nm}_{i}"
        used.add(nm)
        k = rng.choice(kinds)
        srcs = [rng.choice(nodes).name for _ in range(rng.choice((1, 1, 2, 3)))]
        w = None
        if k in (OpKind.MATMUL, OpKind.ELEMENTWISE) and rng.random() < 0.6:
            w = TensorSpec((8, rng.choice((8, 16))), rng.choice((DType.F32, DType.F64)), rng.random() < 0.8)
        nodes.append(RawNode(nm, k, tuple(srcs), TensorSpec((4, rng.choice((8, 16)))), w))
    nodes.append(RawNode("output", OpKind.OUTPUT, (nodes[-1].name,), TensorSpec((4, 8))))
    return ModelGraph(nodes)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
@pytest.mark.parametrize("seed", range(25))
def test_ingest_random_graphs_vs_live_reference(seed):
    sys.path.insert(0, REF)
    try:
        from shardplan.errors import ShardplanError
        from shardplan.ir import load_graph, save_graph, trim_and_group
    finally:
        sys.path.remove(REF)
    raw = save_graph(_random_raw(random.Random(seed)))
    try:
        exp = trim_and_group(load_graph(raw))
    except ShardplanError as exc:
        with pytest.raises(getattr(E, type(exc).__name__)):
            load_lowered(raw)
        return
    _same(load_lowered(raw).low, lower(exp))
