"""Golden fixtures for the native ONNX ingest (csrc/ingest.cpp, sp_ingest_onnx).

Run HERE, where the reference (with its onnx_ingest package and test helpers)
is importable from the read-only tree:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_onnx_golden.py

Models are hand-encoded with the reference's own wire codec and fixture
builders (pkg/tests/test_onnx_ingest.py:27-110) plus the c2 T5-base model of
make_golden.py.  For each model it records what the reference's
`export_graph` (convert.py:272-274) returns -- the document, its exact
`json.dumps` text and the ConversionReport -- or the exception it raises, and
what `trim_and_group(load_graph(document))` makes of the document.

Output: tests/golden/onnx/cases.json.gz
"""

from __future__ import annotations

import base64
import gzip
import json
import os
import sys

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [f"{REF}/src", f"{REF}/onnx_ingest/src", REF, os.path.dirname(os.path.dirname(HERE)), HERE]
sys.dont_write_bytecode = True

from onnx_ingest import export_graph  # noqa: E402
from onnx_ingest import wire as W  # noqa: E402
from shardplan import load_graph, trim_and_group  # noqa: E402
from shardplan.errors import ShardplanError  # noqa: E402
from tests.test_onnx_ingest import DOUBLE, INT64, encoder_model, mlp_model, model, node, tensor, vi  # noqa: E402

from paper_2302_00247_b200.ir import dump_grouped  # noqa: E402

FLOAT = 1


def t5_model() -> bytes:
    import make_golden
    import onnx_ingest

    captured = {}
    real = onnx_ingest.export_graph

    def spy(data, batch=None):
        captured["data"] = data
        return real(data, batch)

    onnx_ingest.export_graph = spy
    try:
        make_golden.t5_base_onnx_graph()
    finally:
        onnx_ingest.export_graph = real
    return captured["data"]


def raw_int64_tensor(name, dims, values):
    body = b"".join(W.field_varint(1, d) for d in dims)
    body += W.field_varint(2, INT64) + W.field_string(8, name)
    body += W.field_bytes(9, b"".join(int(v).to_bytes(8, "little", signed=True) for v in values))
    return body


def cases() -> dict:
    x = vi("x", FLOAT, (4, 16))
    c = {
        "mlp": (mlp_model(), None),
        "encoder": (encoder_model(), None),
        "t5_base": (t5_model(), None),
        "dynamic": (model([node("MatMul", "/l/MatMul", ["x", "W"], ["y"])], [tensor("W", DOUBLE, (16, 8))],
                          [vi("x", DOUBLE, ("N", 16))], [vi("y", DOUBLE, ("N", 8))]), None),
        "dynamic_batch6": (model([node("MatMul", "/l/MatMul", ["x", "W"], ["y"])], [tensor("W", DOUBLE, (16, 8))],
                                 [vi("x", DOUBLE, ("N", 16))], [vi("y", DOUBLE, ("N", 8))]), 6),
        "loop": (model([node("Loop", "/loop", ["x"], ["y"])], inputs=[vi("x", DOUBLE, (2,))],
                       outputs=[vi("y", DOUBLE, (2,))]), None),
        "unknown_op": (model([node("Erf", "/odd/Erf", ["x"], ["y"])], inputs=[vi("x", DOUBLE, (2, 3))],
                             outputs=[vi("y", DOUBLE, (2, 3))]), None),
        "reshape_operand": (model([node("Reshape", "/r/Reshape", ["x", "shape"], ["y"])],
                                  [tensor("shape", INT64, (2,), int64_values=[3, 8])], [vi("x", DOUBLE, (4, 6))],
                                  [vi("y", DOUBLE, (3, 8))]), None),
        "reshape_raw_data": (model([node("Reshape", "/r/Reshape", ["x", "shape"], ["y"])],
                                   [raw_int64_tensor("shape", (2,), [2, 12])], [vi("x", DOUBLE, (4, 6))],
                                   [vi("y", DOUBLE, (2, 12))], ), None),
        "reshape_undetermined": (model([node("Reshape", "/r/Reshape", ["x", "shape"], ["y"])],
                                       [tensor("shape", INT64, (2,), int64_values=[-1, 8])],
                                       [vi("x", DOUBLE, (4, 6))], [vi("z", DOUBLE, (3, 8))]), None),
        "gather_embedding": (model([node("Gather", "/emb/Gather", ["E", "x"], ["y"])], [tensor("E", DOUBLE, (16, 8))],
                                   [vi("x", DOUBLE, (2, 4))], [vi("y", DOUBLE, (2, 4, 8))]), None),
        "gather_axis1": (model([node("Gather", "/g/Gather", ["E", "x"], ["y"], {"axis": 1})],
                               [tensor("E", DOUBLE, (16, 8))], [vi("x", DOUBLE, (2, 4))], [vi("y", DOUBLE, (2, 4))]),
                         None),
        "unnamed": (model([node("Relu", "", ["x"], ["y"]), node("Relu", "", ["y"], ["z"])],
                          inputs=[vi("x", DOUBLE, (2,))], outputs=[vi("z", DOUBLE, (2,))]), None),
        "gemm_transb_bias": (model([node("Gemm", "/fc/Gemm", ["x", "W", "b"], ["y"], {"transB": 1})],
                                   [tensor("W", FLOAT, (8, 16)), tensor("b", FLOAT, (8,))], [x],
                                   [vi("y", FLOAT, (4, 8))]), None),
        "layernorm_scale_bias": (model([node("LayerNormalization", "/ln/LN", ["x", "s", "b"], ["y"]),
                                        node("MatMul", "/fc/MatMul", ["y", "W"], ["z"])],
                                       [tensor("s", FLOAT, (16,)), tensor("b", FLOAT, (16,)),
                                        tensor("W", FLOAT, (16, 4))], [x], [vi("z", FLOAT, (4, 4))]), None),
        "transpose_aux_dupnames": (model([node("Transpose", "/t/Transpose", ["x"], ["t"]),
                                          node("Identity", "/t/Transpose", ["t"], ["i"]),
                                          node("Constant", "/c/Constant", [], ["k"]),
                                          node("Add", "/t/Transpose", ["i", "k", "W", "W2"], ["y"])],
                                         [tensor("W", FLOAT, (16, 4)), tensor("W2", FLOAT, (16, 4)),
                                          tensor("unused", FLOAT, (3, 3))],
                                         [x], [vi("y", FLOAT, (16, 4))]), None),
        "two_outputs_value_info": (model([node("Softmax", "/s/Softmax", ["x"], ["a"]),
                                          node("Mul", "/m/Mul", ["a", "x"], ["b"])],
                                         inputs=[x], outputs=[vi("a", FLOAT, (4, 16)), vi("b", FLOAT, (4, 16))],
                                         value_infos=[vi("a", FLOAT, (4, 16)), vi("b", DOUBLE, (2, 32))]), None),
        "undeclared_value": (model([node("Relu", "/r/Relu", ["ghost"], ["y"])], inputs=[x],
                                   outputs=[vi("y", FLOAT, (4, 16))]), None),
        "output_never_produced": (model([node("Relu", "/r/Relu", ["x"], ["y"])], inputs=[x],
                                        outputs=[vi("zz", FLOAT, (4, 16))]), None),
        "int_weight": (model([node("MatMul", "/l/MatMul", ["x", "W"], ["y"])], [tensor("W", INT64, (16, 8))],
                             [x], [vi("y", FLOAT, (4, 8))]), None),
        "matmul_no_weight": (model([node("MatMul", "/l/MatMul", ["x", "x"], ["y"])], [], [x],
                                   [vi("y", FLOAT, (4, 16))]), None),
        "garbage": (b"\xff\xfe not a protobuf", None),
        "no_graph": (W.field_varint(1, 8), None),
        "nameless_initializer": (W.field_bytes(7, W.field_bytes(5, W.field_varint(1, 2) + W.field_varint(2, 1))),
                                 None),
        "bad_utf8": (W.field_bytes(7, W.field_bytes(1, W.field_bytes(3, b"\xc3\x28"))), None),
    }
    return c


def main() -> None:
    out = []
    for name, (data, batch) in cases().items():
        rec = {"name": name, "data": base64.b64encode(data).decode(), "batch": batch}
        try:
            doc, rep = export_graph(data, batch=batch)
        except Exception as exc:  # noqa: BLE001 - recorded, the native path must match
            rec["error"] = type(exc).__name__
            rec["message"] = str(exc)
            out.append(rec)
            print(name, "->", rec["error"], rec["message"][:60])
            continue
        rec["json"] = json.dumps(doc)
        rec["report"] = vars(rep)
        try:
            rec["grouped"] = dump_grouped(trim_and_group(load_graph(json.dumps(doc))))
        except ShardplanError as exc:
            rec["graph_error"] = type(exc).__name__
        out.append(rec)
        print(name, "->", len(doc["nodes"]), "nodes", rec.get("graph_error", ""))
    os.makedirs(os.path.join(HERE, "onnx"), exist_ok=True)
    with open(os.path.join(HERE, "onnx", "cases.json.gz"), "wb") as fh:
        fh.write(gzip.compress(json.dumps(out, sort_keys=True).encode(), mtime=0))


if __name__ == "__main__":
    main()
