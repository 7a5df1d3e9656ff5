"""Native ONNX ingest (csrc/ingest.cpp sp_ingest_onnx) vs the reference's onnx_ingest.

Pinned by tests/golden/onnx/cases.json.gz (made by make_onnx_golden.py from
the reference's own wire codec, fixture builders and export_graph): the
converted document byte for byte as `json.dumps` text, the ConversionReport,
the exception class and message for unconvertible models, and the grouped
graph load_graph + trim_and_group make of the document.  Host-only: no GPU.
"""

from __future__ import annotations

import base64
import gzip
import json
import os

import numpy as np
import pytest

from paper_2302_00247_b200 import ingest
from paper_2302_00247_b200.ir import grouped_from_doc
from paper_2302_00247_b200.lowering import lower

CASES = json.loads(gzip.decompress(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "onnx",
                                                     "cases.json.gz"), "rb").read()))
ARRAYS = ("name_bytes", "name_off", "op", "act_rank", "act_shape", "act_bytes", "w_rank", "w_shape", "w_bytes",
          "w_trainable", "in_off", "in_idx")


def _data(case):
    return base64.b64decode(case["data"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_export_graph_matches_reference(case):
    if "error" in case:
        cls = getattr(ingest, case["error"])
        with pytest.raises(cls) as info:
            ingest.export_graph_json(_data(case), case["batch"])
        msg = str(info.value)
        if case["error"] == "ModelParseError":  # codec detail after the colon is Python's wording
            assert msg.split(":")[0] == case["message"].split(":")[0]
        else:
            assert msg == case["message"]
        return
    text, report = ingest.export_graph_json(_data(case), case["batch"])
    assert text == case["json"]  # json.dumps(doc), byte for byte
    assert vars(report) == case["report"]
    doc, report2 = ingest.export_graph(_data(case), case["batch"])
    assert doc == json.loads(case["json"]) and report2 == report


@pytest.mark.parametrize("case", [c for c in CASES if "grouped" in c], ids=lambda c: c["name"])
def test_load_onnx_matches_reference_grouping(case):
    g = ingest.load_onnx(_data(case), case["batch"])
    exp = lower(grouped_from_doc(case["grouped"]))
    for k in ARRAYS:
        x, y = getattr(g.low, k), getattr(exp, k)
        assert x.dtype == y.dtype and x.shape == y.shape and np.array_equal(x, y), k
    assert g.names == exp.names
    assert vars(g.report) == case["report"]


def test_load_onnx_error_kinds():
    for case in CASES:
        if "error" in case:
            with pytest.raises(getattr(ingest, case["error"])):
                ingest.load_onnx(_data(case), case["batch"])


REF = "/root/reference/pkg"


def _random_model(seed: int):
    """Random ONNX models over the converter's whole op table (and a few it lacks),
    with shared / surplus / unused initializers, empty and duplicate node names,
    value infos that override shapes, and models that must be rejected."""
    import random
    import sys

    sys.path[:0] = [f"{REF}/src", f"{REF}/onnx_ingest/src", REF]
    try:
        from tests.test_onnx_ingest import model, node, tensor, vi
    finally:
        del sys.path[:3]
    rng = random.Random(seed)
    F, D, I64 = 1, 11, 7
    d = rng.choice((4, 8))
    inits, nodes, vis = [], [], []
    values = ["x"]
    ops = ["MatMul", "Gemm", "Add", "Mul", "Relu", "LayerNormalization", "Softmax", "Gather", "Reshape",
           "Transpose", "Constant", "Identity", "Erf"]
    for i in range(rng.randint(1, 12)):
        op = rng.choice(ops)
        src = rng.choice(values)
        ins = [src]
        attrs = {}
        if op in ("MatMul", "Gemm") and rng.random() < 0.9:
            inits.append(tensor(f"W{i}", rng.choice((F, F, D, I64)), (d, d)))
            ins.append(f"W{i}")
            if op == "Gemm" and rng.random() < 0.5:
                attrs["transB"] = 1
            if rng.random() < 0.4:
                inits.append(tensor(f"b{i}", F, (d,)))
                ins.append(f"b{i}")
        elif op in ("Add", "Mul", "LayerNormalization") and rng.random() < 0.5:
            inits.append(tensor(f"s{i}", F, (d,)))
            ins.append(f"s{i}")
            if rng.random() < 0.3:
                ins.append(f"s{i}")
        elif op == "Gather":
            if rng.random() < 0.7:
                inits.append(tensor(f"E{i}", F, (16, d)))
                ins = [f"E{i}", src]
            if rng.random() < 0.2:
                attrs["axis"] = 1
        elif op == "Reshape":
            inits.append(tensor(f"sh{i}", I64, (2,), int64_values=[rng.choice((2, -1)), 2 * d]))
            ins.append(f"sh{i}")
        elif op == "Constant":
            ins = []
        elif op == "Add" and len(values) > 1:
            ins.append(rng.choice(values))
        name = rng.choice(("", f"/blk{i % 3}/{op}", f"blk{i % 2}/{op}", f"/dup/{op}"))
        out = f"v{i}"
        nodes.append(node(op, name, ins, [out], attrs))
        if rng.random() < 0.3:
            vis.append(vi(out, F, (2, rng.choice((d, 2 * d)))))
        values.append(out)
    if rng.random() < 0.2:
        inits.append(tensor("unused", F, (3,)))
    outs = [vi(values[-1], F, (2, d))]
    if rng.random() < 0.2:
        outs.append(vi(values[1] if len(values) > 1 else "x", F, (2, d)))
    batch_in = ("N", d) if rng.random() < 0.15 else (2, d)
    return model(nodes, inits, [vi("x", F, batch_in)], outs, vis), (3 if rng.random() < 0.5 else None)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
@pytest.mark.parametrize("seed", range(60))
def test_export_graph_random_models_vs_live_reference(seed):
    import sys

    data, batch = _random_model(seed)
    sys.path[:0] = [f"{REF}/onnx_ingest/src"]
    try:
        from onnx_ingest import export_graph as ref_export
    finally:
        del sys.path[0]
    try:
        doc, rep = ref_export(data, batch=batch)
    except Exception as exc:  # noqa: BLE001
        with pytest.raises(getattr(ingest, type(exc).__name__, Exception)) as info:
            ingest.export_graph_json(data, batch)
        assert type(info.value).__name__ == type(exc).__name__
        return
    text, report = ingest.export_graph_json(data, batch)
    assert text == json.dumps(doc)
    assert vars(report) == vars(rep)
