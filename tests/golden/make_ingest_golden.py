"""Golden fixtures for the native graph ingest (csrc/ingest.cpp).

Run HERE, where the reference is importable from the read-only tree:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ingest_golden.py

For every raw graph document (schema 1, the reference's own `save_graph` /
`export_graph` output) it records what the reference's
`trim_and_group(load_graph(doc))` (ir.py:319-338, 378-461) produces, in the
compact grouped format `paper_2302_00247_b200.ir.grouped_from_doc` reads, and
for malformed documents the exception class the reference raises.

Outputs (tests/golden/ingest/):
  <name>.raw.json.gz       the raw document
  <name>.grouped.json.gz   the reference's grouped graph
  errors.json              [{name, doc, error, src?, dst?}]
"""

from __future__ import annotations

import gzip
import json
import os
import sys

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [f"{REF}/src", f"{REF}/onnx_ingest/src", REF, os.path.dirname(os.path.dirname(HERE))]
sys.dont_write_bytecode = True

from shardplan import (  # noqa: E402
    DType,
    ModelGraph,
    OpKind,
    RawNode,
    TensorSpec,
    gen_encoder_decoder,
    gen_transformer_stack,
    gen_wide_classifier,
    load_graph,
    trim_and_group,
)
from shardplan.ir import save_graph  # noqa: E402

from paper_2302_00247_b200.ir import dump_grouped  # noqa: E402

OUT = os.path.join(HERE, "ingest")


def aux_chain_graph() -> ModelGraph:
    """Chains of auxiliary nodes between compute nodes, a duplicate direct edge
    (x*x), an aux node with two producers, root-level names and a scope name
    that collides with a node name (trim_and_group's `claimed` fallback)."""
    t = TensorSpec((4, 8))
    w = TensorSpec((8, 8), DType.F64, True)
    n = [
        RawNode("input", OpKind.INPUT, (), t),
        RawNode("blk/a/mm", OpKind.MATMUL, ("input",), t, w),
        RawNode("blk/a/aux0", OpKind.AUXILIARY, ("blk/a/mm",), TensorSpec((1,))),
        RawNode("blk/a/aux1", OpKind.AUXILIARY, ("blk/a/aux0", "input"), TensorSpec((1,))),
        RawNode("blk/b/sq", OpKind.ELEMENTWISE, ("blk/a/aux1", "blk/a/mm", "blk/a/mm"), t),
        RawNode("blk/b/ln", OpKind.LAYERNORM, ("blk/b/sq",), t),
        RawNode("blk/b", OpKind.SOFTMAX, ("blk/b/ln",), t),
        RawNode("blk/c/x", OpKind.RESHAPE, ("blk/b",), TensorSpec((32,))),
        RawNode("blk/c/aux", OpKind.AUXILIARY, ("blk/c/x",), TensorSpec((1,))),
        RawNode("tail", OpKind.ELEMENTWISE, ("blk/c/aux",), TensorSpec((32,)), TensorSpec((32,), trainable=True)),
        RawNode("output", OpKind.OUTPUT, ("tail",), TensorSpec((32,))),
    ]
    return ModelGraph(n)


def t5_raw_doc() -> bytes:
    """The export_graph document of the c2 T5-base ONNX fixture (make_golden.py)."""
    sys.path.insert(0, HERE)
    import make_golden
    import onnx_ingest

    captured = {}
    real = onnx_ingest.export_graph

    def spy(data):
        doc, rep = real(data)
        captured["doc"] = doc
        return doc, rep

    onnx_ingest.export_graph = spy
    try:
        make_golden.t5_base_onnx_graph()
    finally:
        onnx_ingest.export_graph = real
    return json.dumps(captured["doc"]).encode()


def _gz(path: str, data: bytes) -> None:
    with open(path, "wb") as fh:  # mtime 0: byte-stable fixtures
        fh.write(gzip.compress(data, mtime=0))


def write(name: str, raw: bytes) -> None:
    g = trim_and_group(load_graph(raw))
    _gz(os.path.join(OUT, f"{name}.raw.json.gz"), raw)
    _gz(os.path.join(OUT, f"{name}.grouped.json.gz"),
        json.dumps(dump_grouped(g), sort_keys=True, separators=(",", ":")).encode())
    print(name, len(raw), "bytes ->", len(g.nodes), "GraphNodes")


def errors() -> list:
    from shardplan.errors import ShardplanError

    def node(name, inputs=(), op="matmul", out=None, **kw):
        d = {"name": name, "op": op, "inputs": list(inputs), "output": out or {"shape": [2, 2]}}
        d.update(kw)
        return d

    cases = {
        "malformed": '{"nodes": [',
        "not_object": "[1, 2]",
        "no_nodes": '{"version": 1}',
        "bad_version": json.dumps({"version": 3, "nodes": [node("a")]}),
        "missing_name": json.dumps({"nodes": [{"op": "input", "output": {"shape": [1]}}]}),
        "missing_output": json.dumps({"nodes": [{"name": "a", "op": "input"}]}),
        "null_output": json.dumps({"nodes": [node("a", out=None) | {"output": None}]}),
        "bad_dtype": json.dumps({"nodes": [node("a", out={"shape": [2], "dtype": "f16"})]}),
        "empty_shape": json.dumps({"nodes": [node("a", out={"shape": []})]}),
        "zero_dim": json.dumps({"nodes": [node("a", out={"shape": [2, 0]})]}),
        "no_shape": json.dumps({"nodes": [node("a", out={"dtype": "f32"})]}),
        "duplicate": json.dumps({"nodes": [node("a", op="input"), node("a", op="input")]}),
        "dangling": json.dumps({"nodes": [node("a", ["ghost"])]}),
        "self_loop": json.dumps({"nodes": [node("a", ["a"])]}),
        "two_cycle": json.dumps({"nodes": [node("x", op="input"), node("a", ["b", "x"]), node("b", ["a"])]}),
        "empty_list": json.dumps({"nodes": []}),
        "all_aux": json.dumps({"nodes": [node("a", op="auxiliary"), node("b", ["a"], op="auxiliary")]}),
        "bad_weight": json.dumps({"nodes": [node("a", weight={"dtype": "f32"})]}),
    }
    out = []
    for name, doc in cases.items():
        rec = {"name": name, "doc": doc}
        try:
            trim_and_group(load_graph(doc))
            rec["error"] = None
        except ShardplanError as exc:
            rec["error"] = type(exc).__name__
            if hasattr(exc, "src"):
                rec["src"], rec["dst"] = exc.src, exc.dst
        out.append(rec)
        print(name, rec["error"])
    return out


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    write("tiny_transformer", save_graph(gen_transformer_stack(2, d_model=8, heads=2)))
    write("transformer_l3_f64", save_graph(gen_transformer_stack(3, d_model=16, heads=2, dtype=DType.F64)))
    write("encdec", save_graph(gen_encoder_decoder(2, 2, d_model=8, heads=2)))
    write("wide_classifier", save_graph(gen_wide_classifier(1000, 64, blocks=6)))
    write("aux_chain", save_graph(aux_chain_graph()))
    write("t5_onnx", t5_raw_doc())
    # unknown op labels map to elementwise; extra keys, attrs and schema 2 fields are ignored
    doc = json.loads(save_graph(gen_transformer_stack(1, d_model=8, heads=2)))
    doc["version"] = 2
    doc["nodes"][1]["op"] = "fancy_op"
    doc["nodes"][2]["attrs"] = {"k": [1, {"x": None}]}
    doc["nodes"][3]["device"] = 3
    doc["extra"] = {"anything": [True, False, None, 1.5e3, "\\u00e9"]}
    write("schema2_extras", json.dumps(doc).encode())
    with open(os.path.join(OUT, "errors.json"), "w") as fh:
        json.dump(errors(), fh, indent=1)


if __name__ == "__main__":
    main()
