"""Grouped benchmark graphs generated directly in GraphNode form.

`transformer_stack` yields exactly trim_and_group(gen_transformer_stack(...))
of the reference (generators.py:27-172, ir.py:378-461): auxiliary operators
are dropped at generation time and every remaining operator already sits
alone in its parent scope, so the grouped scopes are the parent scopes.
Pinned against the reference-generated fixtures by tests/test_workloads.py.
Used for the fold-stress sizes (L = 480 .. 7000 layers, up to ~10^5
GraphNodes) where committing the reference's output is impractical.
"""

from __future__ import annotations

from .ir import GraphNode, GroupedGraph, OpKind, TensorSpec


def transformer_stack(layers: int, d_model: int = 64, heads: int = 4, batch: int = 8,
                      seq: int = 16, vocab: int = 32, ffn_mult: int = 4, dtype: str = "f32",
                      stack_name: str = "encoder") -> GroupedGraph:
    if layers < 1 or d_model < 1 or heads < 1 or d_model % heads:
        raise ValueError("bad transformer configuration")
    act = TensorSpec((batch, seq, d_model), dtype)
    inter = TensorSpec((batch, seq, ffn_mult * d_model), dtype)

    def w(r, c):
        return TensorSpec((r, c), dtype, trainable=True)

    nodes = [
        GraphNode("input", OpKind.INPUT, (), TensorSpec((batch, seq), dtype)),
        GraphNode("embedding", OpKind.EMBEDDING, ("input",), act, w(vocab, d_model)),
    ]
    prev = "embedding"
    for i in range(layers):
        p = f"{stack_name}/layer_{i}"
        nodes += [
            GraphNode(f"{p}/ln1", OpKind.LAYERNORM, (prev,), act),
            GraphNode(f"{p}/gate", OpKind.SOFTMAX, (f"{p}/ln1",), act),
            GraphNode(f"{p}/attention/q", OpKind.MATMUL, (f"{p}/gate",), act, w(d_model, d_model)),
            GraphNode(f"{p}/attention/k", OpKind.MATMUL, (f"{p}/gate",), act, w(d_model, d_model)),
            GraphNode(f"{p}/attention/v", OpKind.MATMUL, (f"{p}/gate",), act, w(d_model, d_model)),
            GraphNode(f"{p}/attention/scores", OpKind.ELEMENTWISE,
                      (f"{p}/attention/q", f"{p}/attention/k"), act),
            GraphNode(f"{p}/attention/context", OpKind.ELEMENTWISE,
                      (f"{p}/attention/scores", f"{p}/attention/v"), act),
            GraphNode(f"{p}/attention/out", OpKind.MATMUL, (f"{p}/attention/context",), act,
                      w(d_model, d_model)),
            GraphNode(f"{p}/residual1", OpKind.ELEMENTWISE, (prev, f"{p}/attention/out"), act),
            GraphNode(f"{p}/ln2", OpKind.LAYERNORM, (f"{p}/residual1",), act),
            GraphNode(f"{p}/ffn/intermediate", OpKind.MATMUL, (f"{p}/ln2",), inter,
                      w(d_model, ffn_mult * d_model)),
            GraphNode(f"{p}/ffn/act", OpKind.ELEMENTWISE, (f"{p}/ffn/intermediate",), inter),
            GraphNode(f"{p}/ffn/output", OpKind.MATMUL, (f"{p}/ffn/act",), act,
                      w(ffn_mult * d_model, d_model)),
            GraphNode(f"{p}/residual2", OpKind.ELEMENTWISE, (f"{p}/residual1", f"{p}/ffn/output"),
                      act),
        ]
        prev = f"{p}/residual2"
    nodes += [
        GraphNode("head/proj", OpKind.MATMUL, (prev,), TensorSpec((batch, seq, vocab), dtype),
                  w(d_model, vocab)),
        GraphNode("output", OpKind.OUTPUT, ("head/proj",), TensorSpec((batch, seq, vocab), dtype)),
    ]
    return GroupedGraph(nodes)


def wide_classifier(num_classes: int, feature_dim: int, blocks: int = 4, batch: int = 32,
                    dtype: str = "f32") -> GroupedGraph:
    """trim_and_group(gen_wide_classifier(...)) (generators.py:233-284)."""
    feat = TensorSpec((batch, feature_dim), dtype)
    nodes = [GraphNode("input", OpKind.INPUT, (), feat)]
    prev = "input"
    for i in range(blocks):
        p = f"backbone/block_{i}"
        nodes += [
            GraphNode(f"{p}/proj", OpKind.MATMUL, (prev,), feat,
                      TensorSpec((feature_dim, feature_dim), dtype, trainable=True)),
            GraphNode(f"{p}/act", OpKind.ELEMENTWISE, (f"{p}/proj",), feat),
        ]
        prev = f"{p}/act"
    nodes += [
        GraphNode("backbone/flatten", OpKind.RESHAPE, (prev,), feat),
        GraphNode("classifier/fc", OpKind.MATMUL, ("backbone/flatten",),
                  TensorSpec((batch, num_classes), dtype),
                  TensorSpec((feature_dim, num_classes), dtype, trainable=True)),
        GraphNode("output", OpKind.OUTPUT, ("classifier/fc",), TensorSpec((batch, num_classes), dtype)),
    ]
    return GroupedGraph(nodes)
