"""Native save_graph (ir.py:358-367) byte-identical to the reference's, on its
generators, the ingest fixtures (schema 1 and 2, attrs, device/collective
extras), grouped graphs and documents with escaped / non-ASCII names and nested
attribute values."""

from __future__ import annotations

import gzip
import json
import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def sp():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import shardplan

    return shardplan


def _docs():
    d = os.path.join(HERE, "golden", "ingest")
    return sorted(f for f in os.listdir(d) if f.endswith(".raw.json.gz"))


@pytest.mark.parametrize("name", _docs())
def test_fixture_documents(sp, name):
    from paper_2302_00247_b200.ingest import save_graph

    with gzip.open(os.path.join(HERE, "golden", "ingest", name), "rb") as fh:
        doc = fh.read()
    g = sp.load_graph(doc)
    for version in (1, 2):
        assert save_graph(g, version) == sp.save_graph(g, version)
    # grouped graphs contribute their members
    gg = sp.trim_and_group(g)
    assert save_graph(gg) == sp.save_graph(gg)


def test_generators(sp):
    from paper_2302_00247_b200.ingest import save_graph

    for g in (sp.gen_transformer_stack(3), sp.gen_wide_classifier(64, 16), sp.gen_encoder_decoder(2, 2),
              sp.gen_transformer_stack(2, d_model=8, dtype=sp.DType.F64)):
        assert save_graph(g) == sp.save_graph(g)


def test_strings_and_attrs(sp):
    """Names needing JSON escapes (quote, backslash, control characters,
    non-ASCII incl. an astral character), attrs with nested values, floats,
    booleans, None, and schema-2 device / collective extras."""
    from paper_2302_00247_b200.ingest import save_graph

    a = "in" + chr(0xE9) + '/"q"'
    b = "blk" + chr(92) + "a/" + chr(0x3BB) + chr(0x1F600) + chr(9) + "x"
    c = "out" + chr(10) + chr(1)
    nodes = [
        {"name": a, "op": "input", "inputs": [], "output": {"shape": [2, 4], "dtype": "f32"}},
        {"name": b, "op": "matmul", "inputs": [a], "output": {"shape": [2, 4], "dtype": "f64"},
         "weight": {"shape": [4, 4], "trainable": True},
         "attrs": {"z": [1, 2.5, None, True, {"b": 1, "a": chr(0xFC)}], "a": 1e-7, "m": 1e300},
         "device": 3, "collective": "allreduce"},
        {"name": c, "op": "output", "inputs": [b], "output": {"shape": [2, 4]}, "attrs": {"note": "xy", "k": -0.0}},
    ]
    g = sp.load_graph(json.dumps({"version": 2, "nodes": nodes}))
    for version in (1, 2):
        assert save_graph(g, version) == sp.save_graph(g, version)


def test_native_is_faster_than_the_reference_on_98k_nodes(sp):
    """A 10^5-node document (the c4 fold-stress size): same bytes, and the native
    writer takes a fraction of the reference's time."""
    import time

    from paper_2302_00247_b200.ingest import save_graph

    g = sp.gen_transformer_stack(2000)
    t0 = time.perf_counter()
    ref = sp.save_graph(g)
    t1 = time.perf_counter()
    got = save_graph(g)
    t2 = time.perf_counter()
    assert got == ref
    assert (t2 - t1) < (t1 - t0)


def test_swap_binds_the_native_writer(sp):
    import shardplan.cli
    import shardplan.ir

    from paper_2302_00247_b200 import swap

    orig = shardplan.ir.save_graph
    g = sp.gen_transformer_stack(2, d_model=8)
    h = swap.install(sp)
    try:
        for mod in (sp, shardplan.ir, shardplan.cli):
            assert mod.save_graph is not orig
            assert mod.save_graph.__wrapped__.__module__ == "paper_2302_00247_b200.ingest"
        assert sp.save_graph(g) == orig(g)
    finally:
        h.uninstall()
    assert shardplan.ir.save_graph is orig
