"""Graphs beyond the routing-table limits of the table path (test inputs).

* big_template: two sibling instances of a 300-node motif (one block of T = 300
  > 256 template nodes);
* wide_fanin: a motif whose join node has 8 internal producers (> 6);
* heavy_tables: a motif of 120 nodes with 6 internal producers each (routing
  tables of 4 x 3^6 bytes per node: more than a CTA's shared memory).
Few weighted nodes keep every block's candidate count small enough for the
CPU oracle to search exhaustively.
"""

from __future__ import annotations

from paper_2302_00247_b200.ir import GraphNode, GroupedGraph, OpKind, TensorSpec


def _weight(i: int, every: int):
    if i % every == 0:
        return TensorSpec((16, 16), trainable=True)
    return None


def _instances(body, reps: int = 2):
    nodes = [GraphNode("input", OpKind.INPUT, (), TensorSpec((8, 16)))]
    prev = "input"
    for j in range(reps):
        pre = f"net/inst_{j}"
        names = body(pre, prev, nodes)
        prev = names[-1]
    nodes.append(GraphNode("output", OpKind.OUTPUT, (prev,), TensorSpec((8, 16))))
    return GroupedGraph(nodes)


def big_template(T: int = 300, weighted_every: int = 50, reps: int = 2) -> GroupedGraph:
    def body(pre, prev, nodes):
        names = []
        for i in range(T):
            sc = f"{pre}/op{i:04d}"
            ins = (prev,) if i == 0 else tuple(dict.fromkeys([names[i - 1]] + ([names[i - 3]] if i >= 3 and i % 7 == 0 else [])))
            w = _weight(i, weighted_every)
            nodes.append(GraphNode(sc, OpKind.MATMUL if w else OpKind.ELEMENTWISE, ins, TensorSpec((8, 16)), w))
            names.append(sc)
        return names

    return _instances(body, reps)


def wide_fanin(k: int = 8, reps: int = 2) -> GroupedGraph:
    def body(pre, prev, nodes):
        names = []
        src = f"{pre}/src"
        nodes.append(GraphNode(src, OpKind.ELEMENTWISE, (prev,), TensorSpec((8, 16))))
        names.append(src)
        branches = []
        for i in range(k):
            sc = f"{pre}/b{i}"
            w = TensorSpec((16, 16), trainable=True) if i < 5 else None
            nodes.append(GraphNode(sc, OpKind.MATMUL if w else OpKind.ELEMENTWISE, (src,), TensorSpec((8, 16)), w))
            branches.append(sc)
        join = f"{pre}/join"
        nodes.append(GraphNode(join, OpKind.ELEMENTWISE, tuple(branches), TensorSpec((8, 16)),
                               TensorSpec((16,), trainable=True)))
        names += branches + [join]
        return names

    return _instances(body, reps)


def heavy_tables(T: int = 120, fan: int = 6, reps: int = 2) -> GroupedGraph:
    def body(pre, prev, nodes):
        names = []
        for i in range(T):
            sc = f"{pre}/n{i:04d}"
            ins = (prev,) if i == 0 else tuple(names[max(0, i - fan):i])
            w = TensorSpec((16, 16), trainable=True) if i % 30 == 0 else None
            nodes.append(GraphNode(sc, OpKind.MATMUL if w else OpKind.ELEMENTWISE, ins, TensorSpec((8, 16)), w))
            names.append(sc)
        return names

    return _instances(body, reps)


LIMIT_GRAPHS = {"big_template": big_template, "wide_fanin": wide_fanin, "heavy_tables": heavy_tables}
