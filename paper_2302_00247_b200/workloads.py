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


def motif_dag(seed: int = 0, tier: str = "parity", n_target: int = 100_000, motif_types: int = 16,
              residuals: int = 1000, d: int = 768, batch: int = 8, seq: int = 128) -> GroupedGraph:
    """Config 5: ~10^5-op DAG of repeated random motifs.

    `motif_types` motif kinds, each a random DAG of M in [16, 48] ops over
    matmul ((d,d)/(d,4d)/(4d,d) weights), elementwise add/mul with an optional
    (d,) bias, layernorm and softmax (never weighted: divergence trap D1);
    fan-in 1-2 from earlier motif ops or the motif entry.  Instances
    `net/m{k}_{j}` are chained entry <- previous exit, so all are siblings
    under `net`; scopes `net/m{k}_{j}/k{k}o{i}` make every type's first
    relative name distinct (divergence trap D2).  `residuals` unique ops under
    `tail/` never fold.  Tiers: "parity" motifs carry 6..12 two-dim weights
    (every block searchable by the CPU reference); "throughput" swaps the
    first three types for motifs with 16 / 18 / 20 two-dim weights
    (4.3e7 .. 3.5e9 candidates).
    """
    import random

    if tier not in ("parity", "throughput"):
        raise ValueError("tier must be 'parity' or 'throughput'")
    rng = random.Random(seed)
    wide = 4 * d
    motifs = []
    for k in range(motif_types):
        if tier == "throughput" and k < 3:
            v2, v1 = (16, 18, 20)[k], 0
        else:
            v2, v1 = rng.randint(6, 12), rng.randint(0, 1)
        m = rng.randint(max(16, v2 + v1 + 4), 48)
        kinds = ["mm"] * v2 + ["bias"] * v1 + [rng.choice(("ew", "ew", "ln", "sm")) for _ in range(m - v2 - v1)]
        rng.shuffle(kinds)
        ops = []  # (kind, inputs as motif positions (-1 entry), weight shape, width)
        widths = []
        for i, kind in enumerate(kinds):
            cands = list(range(-1, i))
            a = rng.choice(cands[-6:])  # mostly local structure
            win = d if a < 0 else widths[a]
            if kind == "mm":
                if win == wide:
                    w, wout = (wide, d), d
                else:
                    w, wout = rng.choice((((d, d), d), ((d, wide), wide)))
                ins = (a,)
            else:
                w = (d,) if kind == "bias" else None
                wout = win
                ins = (a,)
                if kind in ("ew", "bias") and rng.random() < 0.5:
                    same = [c for c in cands if (d if c < 0 else widths[c]) == win and c != a]
                    if same:
                        ins = (a, rng.choice(same[-6:]))
            widths.append(wout)
            ops.append((kind, ins, w, wout))
        motifs.append(ops)
    op_kind = {"mm": OpKind.MATMUL, "bias": OpKind.ELEMENTWISE, "ew": OpKind.ELEMENTWISE,
               "ln": OpKind.LAYERNORM, "sm": OpKind.SOFTMAX}
    budget = n_target - residuals - 2
    nodes = [GraphNode("input", OpKind.INPUT, (), TensorSpec((batch, seq, d)))]
    prev = "input"
    for k, ops in enumerate(motifs):
        reps = max(2, budget // (motif_types * len(ops)))
        for j in range(reps):
            pre = f"net/m{k}_{j}"
            names = [f"{pre}/k{k}o{i}" for i in range(len(ops))]
            for i, (kind, ins, w, wout) in enumerate(ops):
                src = tuple(dict.fromkeys(prev if a < 0 else names[a] for a in ins))
                wt = TensorSpec(w, trainable=True) if w is not None else None
                nodes.append(GraphNode(names[i], op_kind[kind], src, TensorSpec((batch, seq, wout)), wt))
            prev = names[-1]
    for r in range(residuals):
        name = f"tail/r{r}/u{r}"
        w = TensorSpec((d, d), trainable=True) if r % 2 else None
        nodes.append(GraphNode(name, OpKind.MATMUL if w else OpKind.ELEMENTWISE, (prev,),
                               TensorSpec((batch, seq, d)), w))
        prev = name
    nodes.append(GraphNode("output", OpKind.OUTPUT, (prev,), TensorSpec((batch, seq, d))))
    return GroupedGraph(nodes)


def transformer_stack_lowered(layers: int, **kw):
    """`lower(transformer_stack(layers, **kw))` built directly as arrays, for the
    fold scale-up (10^6 .. 10^7 GraphNodes) where per-node Python objects would
    dominate.  Layers repeat with period 14 in the reference's topological order
    (each layer only consumes the previous layer's residual2), so the layer rows
    are tiled and the producer indices shifted; checked against the object path
    by tests/test_workloads.py."""
    import numpy as np

    from .lowering import LoweredGraph, lower

    if layers < 2:
        return lower(transformer_stack(layers, **kw))
    base = lower(transformer_stack(2, **kw))
    P = 14
    head, l0, l1, tail = slice(0, 2), slice(2, 2 + P), slice(2 + P, 2 + 2 * P), slice(2 + 2 * P, None)
    n = 2 + P * layers + 2

    def tile(a):
        return np.concatenate([a[head], np.tile(a[l0], (layers,) + (1,) * (a.ndim - 1)), a[tail]])

    suffixes = [nm.split("/", 2)[2] for nm in base.names[l0]]
    stack = base.names[2].split("/")[0]
    names = (base.names[:2] + [f"{stack}/layer_{i}/{s}" for i in range(layers) for s in suffixes]
             + base.names[-2:])
    # producer CSR: layer 0 as generated, layers >= 1 shifted copies of layer 1
    def rows(lo, hi):
        return [base.in_idx[base.in_off[i]:base.in_off[i + 1]] for i in range(lo, hi)]
    l0_rows, l1_rows = rows(2, 2 + P), rows(2 + P, 2 + 2 * P)
    deg = np.array([len(r) for r in l1_rows], np.int64)
    flat1 = np.concatenate(l1_rows)
    shifts = (np.arange(1, layers, dtype=np.int64) - 1) * P
    body = (flat1[None, :] + shifts[:, None]).ravel() if layers > 1 else np.zeros(0, np.int64)
    last_res2 = 2 + P * layers - 1
    in_idx = np.concatenate([base.in_idx[base.in_off[0]:base.in_off[2]],
                             np.concatenate(l0_rows), body,
                             np.array([last_res2, last_res2 + 1], np.int64)]).astype(np.int32)
    degs = np.concatenate([np.diff(base.in_off)[:2], np.array([len(r) for r in l0_rows]),
                           np.tile(deg, layers - 1), np.array([1, 1])])
    in_off = np.zeros(n + 1, np.int64)
    np.cumsum(degs, out=in_off[1:])
    lens = np.fromiter(map(len, names), np.int64, count=n)
    name_off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=name_off[1:])
    return LoweredGraph(
        names=names, index_=None, name_bytes=np.frombuffer("".join(names).encode("ascii"), np.uint8).copy(),
        name_off=name_off, topo_rank=np.arange(n, dtype=np.int64), op=tile(base.op),
        act_rank=tile(base.act_rank), act_shape=tile(base.act_shape), act_bytes=tile(base.act_bytes),
        w_rank=tile(base.w_rank), w_shape=tile(base.w_shape), w_bytes=tile(base.w_bytes),
        w_trainable=tile(base.w_trainable), in_off=in_off, in_idx=in_idx, source=None)
