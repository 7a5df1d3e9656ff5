"""Seeded random grouped graphs with repeated motifs (test inputs).

Exercises the folding and routing corners the reference's own fixtures touch
only lightly: nested scopes, a node whose scope is the prefix of other nodes
(T5's `.../SelfAttention` softmax next to `.../SelfAttention/k`), classes that
split because one instance differs, fan-in up to 3, rank-1/2/3 activations,
dimensions that do or do not divide the device count, and names containing
characters that sort before '/' ('.', '-').
"""

from __future__ import annotations

import random

from paper_2302_00247_b200.ir import GraphNode, GroupedGraph, OpKind, TensorSpec

OPS_W = (OpKind.MATMUL, OpKind.ELEMENTWISE, OpKind.EMBEDDING)
OPS_NW = (OpKind.ELEMENTWISE, OpKind.LAYERNORM, OpKind.SOFTMAX, OpKind.RESHAPE)


def _motif(rng: random.Random, k: int, n_ops: int, dims: list):
    """Abstract motif: list of (rel name, op, n_inputs_from, weight shape, act shape)."""
    ops = []
    subs = ["a", "b.1", "b-2", "c"]
    for i in range(n_ops):
        weighted = rng.random() < 0.55
        op = rng.choice(OPS_W if weighted else OPS_NW)
        if op in (OpKind.LAYERNORM, OpKind.SOFTMAX, OpKind.RESHAPE):
            weighted = False
        w = None
        if weighted:
            if op == OpKind.ELEMENTWISE and rng.random() < 0.5:
                w = (rng.choice(dims),)
            else:
                w = (rng.choice(dims), rng.choice(dims))
        rank = rng.choice((1, 2, 3, 3, 3))
        act = tuple(rng.choice(dims) for _ in range(rank))
        # nested scopes; sometimes a node sits exactly on a scope other nodes extend
        scope = rng.choice(subs)
        if rng.random() < 0.3:
            rel = f"{scope}/t{k}_{i}/op"
        elif rng.random() < 0.2 and i > 0:
            rel = f"{scope}"
        else:
            rel = f"{scope}/t{k}o{i}"
        fan = 1 if i == 0 else rng.choice((1, 1, 2, 2, 3))
        srcs = sorted(set(rng.randrange(-1, i) for _ in range(fan)))
        ops.append([rel, op, srcs, w, act])
    # de-duplicate relative names (GraphNode scopes are unique)
    seen = set()
    for o in ops:
        base = o[0]
        j = 0
        while o[0] in seen:
            j += 1
            o[0] = f"{base}{j}"
        seen.add(o[0])
    return ops


def random_graph(seed: int, n_types: int = 3, reps=(2, 5), ops=(3, 9), residuals: int = 4,
                 dims=(2, 3, 4, 6, 8, 12, 16), variant_p: float = 0.2) -> GroupedGraph:
    rng = random.Random(seed)
    nodes = []
    nodes.append(GraphNode("input", OpKind.INPUT, (), TensorSpec((8, 4, 16))))
    prev = "input"
    for k in range(n_types):
        motif = _motif(rng, k, rng.randint(*ops), list(dims))
        outer = rng.choice(("net", "net/stack"))
        for j in range(rng.randint(*reps)):
            pre = f"{outer}/m{k}_{j}"
            variant = rng.random() < variant_p
            names = []
            for i, (rel, op, srcs, w, act) in enumerate(motif):
                name = f"{pre}/{rel}"
                ins = tuple(dict.fromkeys(prev if s < 0 else names[s] for s in srcs))
                wt = None
                if w is not None:
                    shape = w
                    if variant and i == 0:
                        shape = tuple(x * 2 for x in w)
                    wt = TensorSpec(shape, "f32", trainable=rng.random() < 0.9)
                nodes.append(GraphNode(name, op, ins, TensorSpec(act), wt))
                names.append(name)
            prev = names[-1]
    for r in range(residuals):
        name = f"tail/r{r}" if r % 2 else f"tail.x/r{r}"
        w = TensorSpec((rng.choice(dims), rng.choice(dims)), trainable=True) if r % 3 else None
        nodes.append(GraphNode(name, OpKind.MATMUL if w else OpKind.ELEMENTWISE, (prev,),
                               TensorSpec((8, 4, rng.choice(dims))), w))
        prev = name
    nodes.append(GraphNode("output", OpKind.OUTPUT, (prev,), TensorSpec((8, 4, 16))))
    return GroupedGraph(nodes)


def to_reference(graph: GroupedGraph):
    """Same graph as a reference ModelGraph of GraphNodes (requires shardplan)."""
    from shardplan.ir import DType, GraphNode as RGN, ModelGraph, OpKind as ROp, RawNode
    from shardplan.ir import TensorSpec as RTS

    def ts(t):
        return RTS(tuple(t.shape), DType.F32 if t.dtype == "f32" else DType.F64, t.trainable)

    out = []
    for name in graph.topo_order:
        nd = graph.nodes[name]
        raw = RawNode(name, ROp(nd.op.value), nd.inputs, ts(nd.activation),
                      ts(nd.weight) if nd.weight else None)
        out.append(RGN(name, raw, nd.inputs))
    return ModelGraph(out)
