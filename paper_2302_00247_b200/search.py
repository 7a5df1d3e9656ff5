"""Drop-in ``prune_graph`` / ``search_subgraph`` / ``derive_plan`` on the B200 backend.

Same names, arguments and results as the reference (pruning.py:123-201,
search.py:85-116, 317-379); the work runs in the sm_100a kernels behind
``include/shardsearch.h``:

* folding          -> ``sp_fold_run``   (device hashing / radix sort / verify)
* candidate search -> ``sp_tables_build`` + ``sp_score`` (batched over all
  blocks in one launch; exact (total, num_split, index) argmin + valid count)
* winner detail    -> ``sp_explain`` (device re-route of the argmin only), from
  which RoutedPlan / CostReport are assembled exactly as the reference's.

``jobs`` is accepted for signature compatibility; the GPU is the parallel
resource (multi-GPU sharding lives in ``paper_2302_00247_b200.dist``).
"""

from __future__ import annotations

import dataclasses
import gc
import math
import os
import time
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from ._native import Backend, default_backend
from .api_types import DEFAULT_TYPES, TypeSet
from .blocks import BlockArrays, prefix_of
from .errors import BackendError, BadConfig, SpecMismatch, UnsupportedSearch
from .lowering import LoweredGraph, _native_lower, lower

_KIND_LABEL = {1: "allreduce", 2: "allgather", 3: "reducescatter", 4: "alltoall"}

#: wall-clock phases (ms) of the last derive_plan call in this process
LAST_PHASES: dict = {}


@dataclass
class Session:
    """A graph resident on one device: lowered arrays + device handle."""

    backend: Backend
    low: LoweredGraph
    dgraph: object

    @classmethod
    def open(cls, graph, backend: Optional[Backend] = None, cache: bool = True) -> "Session":
        backend = backend or default_backend()
        if isinstance(graph, LoweredGraph):
            low = graph
        else:
            low = lower(graph) if cache else lower(_Uncached(graph))
        if cache:
            d = getattr(low, "_sp_dgraph", None)
            if d is not None and d.backend is backend and d.ptr:
                return cls(backend, low, d)
        d = backend.upload(low)
        if cache:
            low._sp_dgraph = d  # type: ignore[attr-defined]
        return cls(backend, low, d)


class _Uncached:
    """Wrapper that hides a graph's cached lowering (forces a fresh lower())."""

    def __init__(self, g):
        self.nodes = g.nodes
        self.topo_order = g.topo_order


# ---------------------------------------------------------------------------
# folding


def subgraphs_from_blocks(low: LoweredGraph, ba: BlockArrays, types: TypeSet = DEFAULT_TYPES) -> list:
    """Subgraph objects (pruning.py:33-55) of a folding result."""
    ascii_names = getattr(low, "ascii", None)
    if ascii_names is None:
        ascii_names = low.ascii = len(low.name_bytes) == sum(map(len, low.names))
    if _native_lower is not None and isinstance(low.names, list):
        # instance tuples built in C (csrc/lower_ext.c) straight from the fold arrays
        per_block = _native_lower.block_instances(
            low.names, np.ascontiguousarray(ba.members, np.int32), np.ascontiguousarray(ba.inst_prefix_node, np.int64),
            np.ascontiguousarray(ba.inst_prefix_len, np.int64), np.ascontiguousarray(ba.block_inst_off, np.int64),
            np.ascontiguousarray(ba.block_T, np.int64), ascii_names)
        subgraph = _ctor(types.Subgraph, 3)
        return [subgraph(insts[0][0], insts[0][1], insts) for insts in per_block]
    names = low.names
    member_names = list(map(names.__getitem__, ba.members.tolist()))
    pnode, plen = ba.inst_prefix_node.tolist(), ba.inst_prefix_len.tolist()
    ioff, moff, Ts = ba.block_inst_off.tolist(), ba.block_member_off.tolist(), ba.block_T.tolist()
    subgraph = types.Subgraph
    subs = []
    for b in range(len(Ts)):
        T, m = Ts[b], moff[b]
        insts = []
        for j in range(ioff[b], ioff[b + 1]):
            nm = names[pnode[j]]
            pre = nm[: plen[j]] if ascii_names else prefix_of(low, pnode[j], plen[j])
            insts.append((pre, tuple(member_names[m: m + T])))
            m += T
        subs.append(subgraph(insts[0][0], insts[0][1], tuple(insts)))
    return subs


def prune_graph(graph, min_duplicates: int, *, backend: Optional[Backend] = None,
                types: TypeSet = DEFAULT_TYPES, session: Optional[Session] = None) -> list:
    """Partition GraphNodes into shared subgraphs plus residuals (pruning.py:123-201)."""
    if min_duplicates < 1:
        raise BadConfig("min_duplicates must be >= 1")
    ses = session or Session.open(graph, backend)
    ba = ses.backend.fold(ses.dgraph, int(min_duplicates))
    return subgraphs_from_blocks(ses.low, ba, types)


def fold_blocks(graph, min_duplicates: int, session: Optional[Session] = None) -> BlockArrays:
    """Folding result as flat arrays (no Python Subgraph objects)."""
    if min_duplicates < 1:
        raise BadConfig("min_duplicates must be >= 1")
    ses = session or Session.open(graph)
    return ses.backend.fold(ses.dgraph, int(min_duplicates))


# ---------------------------------------------------------------------------
# enumeration helpers (search.py:85-116) -- host metadata only


def weight_nodes(graph, subgraph) -> tuple:
    return tuple(s for s in sorted(subgraph.template) if graph.nodes[s].weight is not None)


def count_candidates(graph, subgraph) -> int:
    total = 1
    for s in weight_nodes(graph, subgraph):
        total *= 3 if graph.nodes[s].weight.rank >= 2 else 2
    return total


def _digits(index: int, radices: list) -> list:
    out = [0] * len(radices)
    for i in range(len(radices) - 1, -1, -1):
        index, out[i] = divmod(index, radices[i])
    return out


def _spec_for_digit(types: TypeSet, digit: int):
    if digit == 0:
        return types.ShardSpec(types.ShardKind.REPLICA)
    return types.ShardSpec(types.ShardKind.SPLIT, digit - 1)


def candidate_by_index(graph, subgraph, index: int, types: TypeSet = DEFAULT_TYPES):
    scopes = weight_nodes(graph, subgraph)
    radices = [3 if graph.nodes[s].weight.rank >= 2 else 2 for s in scopes]
    digits = _digits(index, radices)
    return types.CandidatePlan(
        subgraph, tuple((s, _spec_for_digit(types, d)) for s, d in zip(scopes, digits)), index)


def enumerate_all_plans(graph, subgraph, types: TypeSet = DEFAULT_TYPES):
    """Lazily yield the full product of weight decisions (search.py:119-125)."""
    import itertools

    scopes = weight_nodes(graph, subgraph)
    opts = [range(3 if graph.nodes[s].weight.rank >= 2 else 2) for s in scopes]
    for index, digits in enumerate(itertools.product(*opts)):
        yield types.CandidatePlan(
            subgraph, tuple((s, _spec_for_digit(types, d)) for s, d in zip(scopes, digits)), index)


def _spec_digit(spec, w_rank: int, radix: int) -> Optional[int]:
    """Search digit of a weight spec after the reference's normalisation
    (ShardSpec.normalized, patterns.py:44-50: a negative split axis counts from
    the weight's rank), or None when no weight pattern can match it (axis out of
    range, partial, or a split axis beyond the options): pattern_routing then
    skips every pattern of that node (search.py:156-166), a RoutingFailure."""
    kind = spec.kind.value if hasattr(spec.kind, "value") else spec.kind
    if kind == "replica":
        return 0
    if kind == "split":
        axis = spec.axis if spec.axis >= 0 else w_rank + spec.axis
        if 0 <= axis < w_rank and axis + 1 < radix:
            return axis + 1
    return None


def _plan_index(graph, plan):
    """Reference index of a plan's assignments (inverse of candidate_by_index),
    plus the template position of the first node whose spec is not a search
    option (None if every spec is one).  Such nodes get digit 0: the routing of
    every node before them does not depend on their digit."""
    amap = dict(plan.assignments)
    index = 0
    bad = None
    template = plan.subgraph.template
    for s in weight_nodes(graph, plan.subgraph):
        w = graph.nodes[s].weight
        r = 3 if w.rank >= 2 else 2
        d = _spec_digit(amap[s], w.rank, r)
        if d is None:
            q = template.index(s)
            bad = q if bad is None else min(bad, q)
            d = 0
        index = index * r + d
    return index, bad


# ---------------------------------------------------------------------------
# search


def _templates_csr(low: LoweredGraph, subgraphs: list):
    idx = low.index
    off = np.zeros(len(subgraphs) + 1, np.int64)
    nodes = []
    for b, sub in enumerate(subgraphs):
        nodes.extend(idx[s] for s in sub.template)
        off[b + 1] = len(nodes)
    return off, np.asarray(nodes, dtype=np.int32)


def _flops(low: LoweredGraph, tnodes) -> int:
    total = 0
    for v in tnodes:
        if low.op[v] == 0 and low.w_rank[v]:  # matmul with weight (costmodel.py:185-190)
            r = int(low.act_rank[v])
            total += 2 * math.prod(int(x) for x in low.act_shape[v, :r]) * int(low.w_shape[v, 0])
    return total


def _block_flops(low: LoweredGraph, csr) -> list:
    """_flops of every template of `csr` at once (costmodel.py:185-190: 2 x the
    activation's elements x the weight's first dim, summed over matmuls with a
    weight); blocks whose sum may exceed int64 fall back to Python integers."""
    off, tn = csr
    nb = len(off) - 1
    if nb == 0:
        return []
    tn = np.asarray(tn, np.int64)
    mm = (low.op[tn] == 0) & (low.w_rank[tn] > 0)
    r = low.act_rank[tn].astype(np.int64)
    shp = np.where(np.arange(low.act_shape.shape[1])[None, :] < r[:, None], low.act_shape[tn], 1)
    fl = np.where(mm, 2.0 * shp.astype(np.float64).prod(axis=1) * low.w_shape[tn, 0].astype(np.float64), 0.0)
    iv = np.where(mm, 2 * shp.prod(axis=1) * low.w_shape[tn, 0], 0)
    off = np.asarray(off, np.int64)
    nonempty = off[1:] > off[:-1]
    sums = np.zeros(nb, np.int64)
    fsum = np.zeros(nb, np.float64)
    if len(tn):
        idx = off[:-1][nonempty]
        sums[nonempty] = np.add.reduceat(iv, idx)
        fsum[nonempty] = np.add.reduceat(fl, idx)
    out = sums.tolist()
    for b in np.nonzero(fsum >= 2.0 ** 62)[0].tolist():
        out[b] = _flops(low, tn[off[b]:off[b + 1]].tolist())
    return out


def _collective(types: TypeSet, kind: int, axis: int):
    ck = types.CollectiveKind(_KIND_LABEL[kind])
    return types.Collective(ck, None if kind == 1 else int(axis))


def routed_plan(ses: Session, tables, b: int, sub, index: int, mesh, types: TypeSet = DEFAULT_TYPES,
                expect_total: Optional[float] = None):
    """RoutedPlan + CostReport of candidate `index` of block `b`, from sp_explain."""
    low = ses.low
    ex, edges = ses.backend.explain(tables, b, index)
    if not ex.valid:
        return None
    tnodes = [low.index[s] for s in sub.template]
    T = len(tnodes)
    slot_pos = ses.backend.slots(tables, b)
    radices = [3 if low.w_rank[tnodes[p]] >= 2 else 2 for p in slot_pos]
    digits = _digits(index, radices)
    assignments = tuple((sub.template[p], _spec_for_digit(types, d)) for p, d in zip(slot_pos, digits))
    plan = types.CandidatePlan(sub, assignments, index)
    by_consumer: dict = {}
    for e in edges:
        by_consumer.setdefault(e.consumer_pos, []).append(e)
    replica = types.ShardSpec(types.ShardKind.REPLICA)
    identity = types.Collective(types.CollectiveKind.IDENTITY)
    routings = []
    exits = []
    for i in range(T):
        v = tnodes[i]
        op_label = _OP_LABELS[int(low.op[v])]
        pidx = int(ex.pattern[i])
        convs = tuple(
            (sub.template[e.producer_pos], _collective(types, e.kind, e.axis),
             int(low.act_bytes[tnodes[e.producer_pos]]))
            for e in by_consumer.get(i, ()))
        out_coll = (types.Collective(types.CollectiveKind.ALL_REDUCE_SUM)
                    if types.pattern_collectives[op_label][pidx] == "allreduce" else identity)
        ax = int(ex.state_axis[i])
        state = replica if ax < 0 else types.ShardSpec(types.ShardKind.SPLIT, ax)
        routings.append(types.NodeRouting(sub.template[i], types.pattern_names[op_label][pidx], convs,
                                          out_coll, int(low.act_bytes[v]), state))
        if ex.exit_axis[i] >= 0:
            exits.append((sub.template[i], _collective(types, 2, ex.exit_axis[i]),
                          int(low.act_bytes[v])))
    bbc = {}
    for kind, b_, c_ in ((1, ex.bytes_allreduce, ex.calls_allreduce),
                         (2, ex.bytes_allgather, ex.calls_allgather),
                         (3, ex.bytes_reducescatter, ex.calls_reducescatter),
                         (4, ex.bytes_alltoall, ex.calls_alltoall)):
        if c_:
            bbc[_KIND_LABEL[kind]] = int(b_)
    cost = types.CostReport(forward_comm=ex.forward_comm, backward_comm=ex.backward_comm,
                            overlap_fraction=mesh.overlap_fraction, bytes_by_collective=bbc,
                            collective_calls=int(ex.collective_calls), flops=_flops(low, tnodes))
    if expect_total is not None and cost.total != expect_total:
        raise BackendError(
            f"explain/score disagree on block {b} index {index}: {cost.total!r} != {expect_total!r}")
    return types.RoutedPlan(plan, tuple(routings), tuple(exits), cost)


_OP_LABELS = ("matmul", "elementwise", "layernorm", "softmax", "embedding", "reshape", "input",
              "output", "auxiliary", "collective")


def route_prep(ses: Session, subgraphs: list, types: TypeSet = DEFAULT_TYPES, csr=None) -> list:
    """Winner-independent part of every block's RoutedPlan (computed while the
    device searches): template node indices, weight slots in weight_nodes order
    (names sorted, search.py:85-88) with their radices, and per template node
    (scope, op label, pattern names, pattern collectives, output bytes,
    internal producers as (scope, bytes) in GraphNode.inputs order)."""
    low = ses.low
    names = low.names
    in_off, in_idx = low.in_off, low.in_idx
    op, w_rank, act_bytes = low.op, low.w_rank, low.act_bytes
    pnames, pcolls = types.pattern_names, types.pattern_collectives
    if csr is None:
        csr = _templates_csr(low, subgraphs)
    toff, tnl = csr[0].tolist(), csr[1].tolist()
    # per template node scalars as Python lists (one conversion, no per-node numpy indexing)
    tn = csr[1]
    t_op, t_w = op[tn].tolist(), w_rank[tn].tolist()
    t_bytes = act_bytes[tn].tolist()
    b_flops = _block_flops(low, csr)
    out = []
    for b, sub in enumerate(subgraphs):
        template = sub.template
        e0 = toff[b]
        if toff[b + 1] - e0 == 1:
            # singleton block (residual op): no internal producers
            v = tnl[e0]
            lab = _OP_LABELS[t_op[e0]]
            node = (template[0], lab, pnames[lab], pcolls[lab], t_bytes[e0], [])
            if t_w[e0]:
                out.append(([0], [3 if t_w[e0] >= 2 else 2], [node], b_flops[b]))
            else:
                out.append(([], [], [node], 0))
            continue
        tnodes = tnl[toff[b]:toff[b + 1]]
        members = set(tnodes)
        wpos = [i for i, v in enumerate(tnodes) if w_rank[v]]
        slot_pos = sorted(wpos, key=template.__getitem__)
        radices = [3 if w_rank[tnodes[q]] >= 2 else 2 for q in slot_pos]
        nodes = []
        for i, v in enumerate(tnodes):
            lab = _OP_LABELS[int(op[v])]
            prods = [(names[r], int(act_bytes[r]))
                     for r in in_idx[in_off[v]:in_off[v + 1]].tolist() if r in members]
            nodes.append((template[i], lab, pnames[lab], pcolls[lab], int(act_bytes[v]), prods))
        out.append((slot_pos, radices, nodes, b_flops[b]))
    return out


def routed_plans_all(ses: Session, tables, subgraphs: list, scores: list, mesh,
                     types: TypeSet = DEFAULT_TYPES, detail=None, prep=None, only=None) -> list:
    """RoutedPlan of every block's argmin from ONE sp_explain_all launch (or the
    detail the search itself returned), on top of route_prep.  With `only`
    (block positions), just those blocks, in that order."""
    if detail is None:
        idx = [int(sc.best_index) if sc.has_best else (1 << 64) - 1 for sc in scores]
        detail = ses.backend.explain_all(tables, idx)
    if prep is None:
        prep = route_prep(ses, subgraphs, types)
    blocks, node, edge, eoff = detail
    node_l = node.tolist()
    edge_l = edge.tolist()
    replica = types.ShardSpec(types.ShardKind.REPLICA)
    splits = [types.ShardSpec(types.ShardKind.SPLIT, a) for a in range(8)]
    specs = [replica] + splits
    identity = types.Collective(types.CollectiveKind.IDENTITY)
    allreduce = types.Collective(types.CollectiveKind.ALL_REDUCE_SUM)
    colls = {}
    NodeRouting, CandidatePlan = _ctor(types.NodeRouting, 6), _ctor(types.CandidatePlan, 3)
    RoutedPlan, CostReport = _ctor(types.RoutedPlan, 4), _ctor(types.CostReport, 6)
    overlap = mesh.overlap_fraction
    out = []
    starts = [0]
    for pb in prep:
        starts.append(starts[-1] + len(pb[2]))
    for b in (range(len(subgraphs)) if only is None else only):
        sub, sc, X, pb = subgraphs[b], scores[b], blocks[b], prep[b]
        slot_pos, radices, nodes, flops = pb
        T = len(nodes)
        e0 = starts[b]
        if not sc.has_best or not X.valid:
            out.append(types.RoutingFailure(sub.template[X.fail_pos],
                                            "no pattern chains from producer states")
                       if sc.has_best and X.fail_pos >= 0 else None)
            continue
        template = sub.template
        digits = _digits(int(sc.best_index), radices)
        assignments = tuple((template[q], specs[d]) for q, d in zip(slot_pos, digits))
        plan = CandidatePlan(sub, assignments, int(sc.best_index))
        routings, exits = [], []
        k = int(eoff[b])
        for i in range(T):
            scope, lab, pn, pc, obytes, prods = nodes[i]
            pidx, sax, xax, _ = node_l[e0 + i]
            convs = []
            for pname, pbytes in prods:
                kind, axis = edge_l[k]
                k += 1
                if kind:
                    key = (kind, axis)
                    c = colls.get(key)
                    if c is None:
                        c = colls[key] = _collective(types, kind, axis)
                    convs.append((pname, c, pbytes))
            out_coll = allreduce if pc[pidx] == "allreduce" else identity
            state = replica if sax < 0 else splits[sax]
            routings.append(NodeRouting(scope, pn[pidx], tuple(convs), out_coll, obytes, state))
            if xax >= 0:
                key = (2, xax)
                c = colls.get(key)
                if c is None:
                    c = colls[key] = _collective(types, 2, xax)
                exits.append((scope, c, obytes))
        bbc = {_KIND_LABEL[j + 1]: int(X.bytes[j]) for j in range(4) if X.calls[j]}
        cost = CostReport(X.forward_comm, X.backward_comm, overlap, bbc, int(X.collective_calls), flops)
        if sc.best_total == sc.best_total and cost.total != sc.best_total:  # NaN: no score to check
            raise BackendError(f"explain/score disagree on block {b}: {cost.total!r} != "
                               f"{sc.best_total!r}")
        out.append(RoutedPlan(plan, tuple(routings), tuple(exits), cost))
    return out


_CTORS: dict = {}


def _ctor(cls, n_pos: int):
    """Constructor of dataclass `cls` from its first `n_pos` fields, positionally.
    The native one (csrc/lower_ext.c make_ctor) skips the generated __init__,
    which for frozen classes costs one object.__setattr__ per field; it is
    used only where that __init__ would do nothing else (no __post_init__,
    every field init=True, the remaining fields with plain defaults)."""
    key = (cls, n_pos)
    f = _CTORS.get(key)
    if f is None:
        f = cls
        if _native_lower is not None and dataclasses.is_dataclass(cls) and not hasattr(cls, "__post_init__"):
            fs = dataclasses.fields(cls)
            rest = fs[n_pos:]
            if (len(fs) >= n_pos and all(x.init for x in fs)
                    and all(x.default is not dataclasses.MISSING for x in rest)):
                f = _native_lower.make_ctor(cls, tuple(x.name for x in fs[:n_pos]),
                                            tuple(x.name for x in rest), tuple(x.default for x in rest))
        _CTORS[key] = f
    return f


def _singleton_results(ses: Session, subgraphs: list, scores, detail, prep, csr, mesh, types: TypeSet) -> list:
    """SubgraphResult of every one-node block with a routed winner, built in C
    (csrc/lower_ext.c singleton_results) from the raw score / explain records;
    None elsewhere (the Python path builds those)."""
    nb = len(subgraphs)
    blocks, node = detail[0], detail[1]
    raw_s, raw_x = getattr(scores, "raw", None), getattr(blocks, "raw", None)
    if _native_lower is None or raw_s is None or raw_x is None or nb == 0:
        return [None] * nb
    sel = np.fromiter((b for b in range(nb) if len(prep[b][2]) == 1), np.int64)
    if sel.size == 0:
        return [None] * nb
    low = ses.low
    toff = np.ascontiguousarray(csr[0], np.int64)
    first = csr[1][toff[:-1]] if len(csr[1]) else np.zeros(0, np.int32)
    op = np.ascontiguousarray(low.op[first], np.uint8)
    wr = low.w_rank[first]
    radix = np.where(wr >= 2, 3, np.where(wr == 1, 2, 0)).astype(np.uint8)
    obytes = np.ascontiguousarray(low.act_bytes[first], np.int64)
    flops = np.zeros(nb, np.int64)
    for b in sel.tolist():
        flops[b] = prep[b][3]
    pn, pc = types.pattern_names, types.pattern_collectives
    pnames = tuple(tuple(pn.get(lab, ())) for lab in _OP_LABELS)
    pallred = tuple(tuple(c == "allreduce" for c in pc.get(lab, ())) for lab in _OP_LABELS)
    specs = (types.ShardSpec(types.ShardKind.REPLICA),) + tuple(
        types.ShardSpec(types.ShardKind.SPLIT, a) for a in range(8))
    gather = tuple(_collective(types, 2, a) for a in range(8))
    ctors = (_ctor(types.CandidatePlan, 3), _ctor(types.NodeRouting, 6), _ctor(types.RoutedPlan, 4),
             _ctor(types.CostReport, 6), _ctor(types.SubgraphResult, 5))
    got = _native_lower.singleton_results(
        ctors, subgraphs if isinstance(subgraphs, list) else list(subgraphs), sel, raw_s, raw_x,
        np.ascontiguousarray(node, np.int8), toff, op, radix, obytes, flops, pnames, pallred, specs,
        types.Collective(types.CollectiveKind.IDENTITY), types.Collective(types.CollectiveKind.ALL_REDUCE_SUM),
        gather, tuple(_KIND_LABEL[k] for k in (1, 2, 3, 4)), float(mesh.overlap_fraction))
    out = [None] * nb
    for b, r in zip(sel.tolist(), got):
        out[b] = r
    return out


class Slots:
    """Weight slots of every block of a template CSR: `off` int64 [nb + 1],
    `pos` int32 [S] (template positions in weight_nodes order: names sorted,
    search.py:85-88), `radix` uint8 [S] (_options, search.py:91-93)."""

    __slots__ = ("off", "pos", "radix")

    def __init__(self, off, pos, radix):
        self.off, self.pos, self.radix = off, pos, radix

    @classmethod
    def of(cls, low: LoweredGraph, csr) -> Optional["Slots"]:
        if _native_lower is None or not hasattr(_native_lower, "slot_positions") or not isinstance(low.names, list):
            return None
        o, p, r = _native_lower.slot_positions(low.names, np.ascontiguousarray(csr[0], np.int64),
                                               np.ascontiguousarray(csr[1], np.int32),
                                               np.ascontiguousarray(low.w_rank, np.uint8))
        return cls(np.frombuffer(o, np.int64), np.frombuffer(p, np.int32), np.frombuffer(r, np.uint8))

    @classmethod
    def from_prep(cls, prep: list) -> "Slots":
        off = np.zeros(len(prep) + 1, np.int64)
        np.cumsum([len(pb[0]) for pb in prep], out=off[1:])
        pos = np.fromiter((q for pb in prep for q in pb[0]), np.int32, count=int(off[-1]))
        radix = np.fromiter((r for pb in prep for r in pb[1]), np.uint8, count=int(off[-1]))
        return cls(off, pos, radix)

    def subset(self, ids) -> "Slots":
        ids = np.asarray(ids, np.int64)
        S = self.off[ids + 1] - self.off[ids]
        off = np.zeros(len(ids) + 1, np.int64)
        np.cumsum(S, out=off[1:])
        gather = np.repeat(self.off[ids] - off[:-1], S) + np.arange(off[-1])
        return Slots(off, self.pos[gather], self.radix[gather])


def _native_results(ses: Session, subgraphs: list, scores, detail, csr, slots: Optional[Slots], mult, mesh,
                    types: TypeSet):
    """(results, terms, labels) of every block from the raw score / winner-detail
    records, built in C (csrc/lower_ext.c block_results); None entries where
    the Python path must build (or raise for) the block; None overall when the
    native builder does not apply."""
    blocks, node, edge, eoff = detail
    raw_s, raw_x = getattr(scores, "raw", None), getattr(blocks, "raw", None)
    nb = len(subgraphs)
    if (_native_lower is None or not hasattr(_native_lower, "block_results") or raw_s is None or raw_x is None
            or slots is None or nb == 0 or not isinstance(ses.low.names, list)):
        return None
    low = ses.low
    c = _RESULT_CONSTS.get(id(types))
    if c is None or c[0] is not types:
        specs = (types.ShardSpec(types.ShardKind.REPLICA),) + tuple(
            types.ShardSpec(types.ShardKind.SPLIT, a) for a in range(8))
        pn, pc = types.pattern_names, types.pattern_collectives
        c = _RESULT_CONSTS[id(types)] = (types, (
            (_ctor(types.CandidatePlan, 3), _ctor(types.NodeRouting, 6), _ctor(types.RoutedPlan, 4),
             _ctor(types.CostReport, 6), _ctor(types.SubgraphResult, 5)),
            tuple(tuple(pn.get(lab, ())) for lab in _OP_LABELS),
            tuple(tuple(x == "allreduce" for x in pc.get(lab, ())) for lab in _OP_LABELS),
            specs, tuple(sp.label for sp in specs),
            types.Collective(types.CollectiveKind.IDENTITY), types.Collective(types.CollectiveKind.ALL_REDUCE_SUM),
            tuple(tuple(_collective(types, k, a) for a in range(8)) for k in (1, 2, 3, 4)),
            tuple(_KIND_LABEL[k] for k in (1, 2, 3, 4))))
    ctors, pnames, pallred, specs, labels, identity, allreduce, colls, kinds = c[1]
    g = getattr(low, "_sp_result_arrays", None)
    if g is None:
        g = (np.ascontiguousarray(low.op, np.uint8), np.ascontiguousarray(low.act_rank, np.uint8),
             np.ascontiguousarray(low.act_shape, np.int64), int(low.act_shape.shape[1]),
             np.ascontiguousarray(low.w_rank, np.uint8), np.ascontiguousarray(low.w_shape, np.int64),
             int(low.w_shape.shape[1]), np.ascontiguousarray(low.act_bytes, np.int64),
             np.ascontiguousarray(low.in_off, np.int64),
             np.ascontiguousarray(low.in_idx if len(low.in_idx) else np.zeros(1, np.int32), np.int32))
        try:
            low._sp_result_arrays = g
        except AttributeError:
            pass
    io = np.zeros(nb + 1, np.int64)
    np.cumsum(mult, out=io[1:])
    tn = csr[1] if len(csr[1]) else np.zeros(1, np.int32)
    bl = (np.ascontiguousarray(csr[0], np.int64), np.ascontiguousarray(tn, np.int32), slots.off,
          slots.pos if len(slots.pos) else np.zeros(1, np.int32),
          slots.radix if len(slots.radix) else np.zeros(1, np.uint8), io)
    return _native_lower.block_results(
        ctors, subgraphs if isinstance(subgraphs, list) else list(subgraphs), low.names, g, bl, raw_s, raw_x,
        np.ascontiguousarray(node, np.int8), np.ascontiguousarray(edge, np.int8),
        np.ascontiguousarray(eoff, np.int64), pnames, pallred, specs, labels, identity, allreduce, colls, kinds,
        float(mesh.overlap_fraction))


_RESULT_CONSTS: dict = {}


def _label_keys(ba: BlockArrays, subs: list, prep: list):
    """(member row, slot) of every entry of derive_plan's assignment map, in its
    order: block by block, instance by instance, the block's weight slots in
    weight_nodes order (search.py:374-376).  Slots are numbered over all blocks
    with weights; vectorised over the fold's member matrix."""
    sl = prep if isinstance(prep, Slots) else Slots.from_prep(prep)
    if _native_lower is not None and hasattr(_native_lower, "label_rows"):
        r, q = _native_lower.label_rows(
            np.ascontiguousarray(ba.members, np.int32), np.ascontiguousarray(ba.block_T, np.int64),
            np.ascontiguousarray(ba.block_inst_off, np.int64), np.ascontiguousarray(ba.block_member_off, np.int64),
            np.ascontiguousarray(sl.off, np.int64),
            np.ascontiguousarray(sl.pos if len(sl.pos) else np.zeros(1, np.int32), np.int32))
        return np.frombuffer(r, np.int32), np.frombuffer(q, np.int32)
    cnt = np.diff(sl.off)
    wb = np.nonzero(cnt)[0]
    if not len(wb):
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    S = cnt[wb]
    soff = np.zeros(len(wb) + 1, np.int64)
    np.cumsum(S, out=soff[1:])
    q_flat = sl.pos[np.repeat(sl.off[wb] - soff[:-1], S) + np.arange(soff[-1])].astype(np.int64)
    T = np.asarray(ba.block_T, np.int64)[wb]
    mo = np.asarray(ba.block_member_off, np.int64)[wb]
    R = np.diff(np.asarray(ba.block_inst_off, np.int64))[wb]
    # (block, instance) pairs, then each pair's slots
    pb_ = np.repeat(np.arange(len(wb)), R)
    pstart = np.zeros(len(wb), np.int64)
    np.cumsum(R[:-1], out=pstart[1:])
    pr = np.arange(len(pb_)) - np.repeat(pstart, R)
    base = mo[pb_] + pr * T[pb_]
    Sp = S[pb_]
    kstart = np.zeros(len(pb_), np.int64)
    np.cumsum(Sp[:-1], out=kstart[1:])
    within = np.arange(int(Sp.sum())) - np.repeat(kstart, Sp)
    slot = np.repeat(soff[:-1][pb_], Sp) + within
    rows = np.asarray(ba.members, np.int64)[np.repeat(base, Sp) + q_flat[slot]]
    return rows.astype(np.int32), slot.astype(np.int32)


def _assignments(names: list, label_keys, slot_labels: list) -> dict:
    """{names[row]: slot_labels[slot]} over label_keys = (rows, slots), in order."""
    rows, slots = label_keys
    if _native_lower is not None and isinstance(names, list):
        return _native_lower.assignments_dict(names, np.ascontiguousarray(rows, np.int32),
                                              np.ascontiguousarray(slots, np.int32), slot_labels)
    return dict(zip(map(names.__getitem__, rows.tolist()), map(slot_labels.__getitem__, slots.tolist())))


def _labels(assignments) -> dict:
    return {s: spec.label for s, spec in assignments}


class _Search:
    """A search in flight: routing tables built and the scoring launched on the
    device (sp_score_launch); `collect` waits and assembles SubgraphResults.
    Host work placed between the two overlaps the device search."""

    def __init__(self, ses: Session, csr, mesh, mu: int, chunk_size: int, shard: int, n_shards: int,
                 exchange: Optional[Callable], launch: bool = True, local: bool = False):
        self.ses, self.mesh, self.mu, self.chunk_size = ses, mesh, mu, chunk_size
        self.local = local
        self.exchange = exchange
        self._fetched = None
        # pack_gradients raises BadConfig for mu > chunk only once a candidate is
        # costed; build with a legal chunk to learn which error the reference hits first
        self.bad_mu = mu > chunk_size
        ta = time.perf_counter()
        off, nodes = csr
        self.csr = csr
        self.tables = ses.backend.tables(ses.dgraph, off, nodes, mesh, mu,
                                         chunk_size if not self.bad_mu else mu)
        ses.last_table_bytes = self.tables.nbytes
        self.tables_ms = (time.perf_counter() - ta) * 1e3
        self.shard, self.n_shards = shard, n_shards
        self.explain = exchange is None and n_shards == 1
        if launch:
            self.launch()

    def over_smem(self) -> list:
        """Blocks (positions in this search) whose staged tables + live-value pool
        exceed the shared memory of a CTA."""
        by, pool, _ = self.ses.backend.block_info(self.tables)
        if len(by) == 0:
            return []
        need = ((by + 15) // 16) * 16 + pool.astype(np.int64) * SCORE_THREADS * 18 + 16
        return np.nonzero(need > self.ses.backend.smem_limit)[0].tolist()

    def launch(self) -> None:
        """Queue the scoring (and the copy of its results to the host) on the stream."""
        try:
            if self.tables.overflow:
                raise UnsupportedSearch("a block has more than 2**64 candidates (reference: big-int index)")
            self.t_launch = time.perf_counter()
            self.ses.backend.score_launch(self.tables, self.shard, self.n_shards, explain=self.explain,
                                          local=self.local)
        except BaseException:
            self.tables.close()
            raise

    def fetch(self, explain_now: bool = False) -> None:
        """Wait for the device results (and exchange them across ranks).  With
        `explain_now`, also re-route the merged winners at once (sharded runs
        cannot chain that on the device: the winners are known only after the
        exchange)."""
        if self._fetched is not None:
            return
        try:
            scores, detail = self.ses.backend.score_wait(self.tables)
            if self.exchange is not None:
                scores = self.exchange(scores)
            if explain_now and detail is None:
                idx = [int(sc.best_index) if sc.has_best else (1 << 64) - 1 for sc in scores]
                detail = self.ses.backend.explain_all(self.tables, idx)
        except BaseException:
            self.tables.close()
            raise
        self._fetched = (scores, detail, time.perf_counter())

    def collect(self, graph, subgraphs: list, want_table: bool, types: TypeSet, prep=None,
                slots: Optional[Slots] = None, mult=None) -> list:
        """SubgraphResult per block.  Also sets `self.extra` = (terms, labels)
        per block (cost x multiplicity, weight labels in weight_nodes order) when
        the native builder produced them (None entries elsewhere), else None."""
        ses, tables = self.ses, self.tables
        self.extra = None
        try:
            self.fetch()
            scores, detail, tc = self._fetched
            t_routes = time.perf_counter()
            for sc in scores:
                if not sc.has_best:
                    raise AssertionError("all-replica fallback must always route")
                if self.bad_mu:
                    raise BadConfig(f"fusion threshold {self.mu} exceeds chunk size {self.chunk_size}")
            if detail is None:
                idx = [int(sc.best_index) if sc.has_best else (1 << 64) - 1 for sc in scores]
                detail = ses.backend.explain_all(tables, idx)
            nb = len(subgraphs)
            native = None
            if not want_table:
                if slots is None:
                    slots = Slots.of(ses.low, self.csr)
                if mult is None:
                    mult = [len(sub.instances) for sub in subgraphs]
                native = _native_results(ses, subgraphs, scores, detail, self.csr, slots, mult, self.mesh, types)
            if native is not None:
                bests, terms, labs = native
                rest = [b for b, r in enumerate(bests) if r is None]
                self.extra = (terms, labs)
            else:
                bests = [None] * nb
                rest = list(range(nb))
            if rest:
                if prep is None:
                    prep = route_prep(ses, subgraphs, types, self.csr)
                # one-node blocks (c5: ~1000 residual ops) straight from the raw
                # records in C; the rest (and any block the C path declines) here
                if native is None and not want_table:
                    fast = _singleton_results(ses, subgraphs, scores, detail, prep, self.csr, self.mesh, types)
                    for b, r in enumerate(fast):
                        bests[b] = r
                    rest = [b for b, r in enumerate(fast) if r is None]
                routed = dict(zip(rest, routed_plans_all(ses, tables, subgraphs, scores, self.mesh, types, detail,
                                                         prep, only=rest)))
            else:
                routed = {}
            LAST_PHASES.update(tables_ms=self.tables_ms, score_call_ms=(tc - self.t_launch) * 1e3,
                               routes_ms=(time.perf_counter() - t_routes) * 1e3)
            if not routed and not want_table:
                return bests
            results = []
            SubgraphResult = _ctor(types.SubgraphResult, 5)
            for b, (sub, sc) in enumerate(zip(subgraphs, scores)):
                if b not in routed:
                    results.append(bests[b])
                    continue
                best = routed[b]
                table = []
                if want_table:
                    C = int(sc.candidates)
                    _, totals = ses.backend.score_range(tables, b, 0, C, want_totals=True)
                    for i in range(C):
                        t = float(totals[i])
                        plan = candidate_by_index(graph, sub, i, types)
                        table.append([i, _labels(plan.assignments), None if math.isnan(t) else t])
                results.append(SubgraphResult(sub, best, int(sc.candidates), int(sc.valid), table))
            return results
        finally:
            tables.close()


def search_blocks(graph, subgraphs: list, mesh, mu: int = 1 << 20, chunk_size: int = 4 << 20,
                  want_table: bool = False, *, session: Optional[Session] = None,
                  types: TypeSet = DEFAULT_TYPES, shard: int = 0, n_shards: int = 1,
                  exchange: Optional[Callable] = None, csr=None,
                  backend: Optional[Backend] = None) -> list:
    """Score every candidate of every block in one batched launch; returns
    SubgraphResult per block (search_subgraph semantics, search.py:317-345).
    `csr` = (offsets, node indices) of the templates when already known."""
    ses = session or Session.open(graph, backend)
    if not subgraphs:
        return []
    if csr is None:
        csr = _templates_csr(ses.low, subgraphs)
    searches = _plan_searches(ses, csr, mesh, mu, chunk_size, shard, n_shards, exchange)
    try:
        for srch, _ in searches:
            srch.launch()
    except BaseException:
        for srch, _ in searches:
            srch.tables.close()
        raise
    prep = route_prep(ses, subgraphs, types, csr)  # overlaps the device search
    results = [None] * len(subgraphs)
    try:
        for srch, ids in searches:
            got = srch.collect(graph, [subgraphs[i] for i in ids], want_table, types, [prep[i] for i in ids])
            for i, r in zip(ids, got):
                results[i] = r
    finally:
        for srch, _ in searches:
            srch.tables.close()
    return results


def search_subgraph(graph, subgraph, mesh, mu: int = 1 << 20, chunk_size: int = 4 << 20,
                    jobs: int = 1, want_table: bool = False, *, types: TypeSet = DEFAULT_TYPES,
                    session: Optional[Session] = None, backend: Optional[Backend] = None):
    """Exhaustive argmin over one block's candidates (search.py:317-345)."""
    del jobs
    return search_blocks(graph, [subgraph], mesh, mu, chunk_size, want_table, session=session,
                         types=types, backend=backend)[0]


def derive_plan(graph, mesh, min_duplicates: int = 2, mu: int = 1 << 20,
                chunk_size: int = 4 << 20, jobs: int = 1, want_table: bool = False, *,
                types: TypeSet = DEFAULT_TYPES, backend: Optional[Backend] = None,
                session: Optional[Session] = None, cache: bool = True,
                shard: int = 0, n_shards: int = 1, exchange: Optional[Callable] = None,
                root_only: bool = True):
    """Prune, search every unique block, assemble the whole-graph plan (search.py:348-379).

    Multi-GPU: with a backend over several devices, or one joined to other
    processes (Backend.comm_init), the library splits every block's work items
    across the GPUs and merges the per-block argmin on the device (one NCCL
    all-gather).  Every rank takes part in the search; with `root_only` only
    rank 0 assembles the report and the other ranks return None.  (`shard`,
    `n_shards`, `exchange`: the host-exchange form, kept for callers that
    bring their own transport.)"""
    del jobs
    gc_was = gc.isenabled()
    gc.disable()  # the result is ~10^5 small objects: no collector pauses mid-search
    try:
        return _derive_plan(graph, mesh, min_duplicates, mu, chunk_size, want_table, types,
                            backend, session, cache, shard, n_shards, exchange, root_only)
    finally:
        if gc_was:
            gc.enable()


#: blocks with fewer candidates than this are scored in a first, separate
#: launch (when there are at least SPLIT_MIN_SMALL_BLOCKS of them and the
#: remaining blocks hold at least SPLIT_MIN_BIG_CANDIDATES candidates).  The
#: group then runs as the library's one-kernel small search (one CTA per block):
#: c5's 1002 blocks of <= 64 candidates in one k_search_small launch instead of
#: the item scorer + k_reduce + k_explain_fast; its 10 blocks of 1.5e3-5.9e4
#: candidates join the expensive group (at 8192, one CTA walking a 6561-candidate
#: block made the launch 0.23 ms)
SMALL_BLOCK_CANDIDATES = 1024
SPLIT_MIN_SMALL_BLOCKS = 64
SPLIT_MIN_BIG_CANDIDATES = float(1 << 26)


def _block_groups(low: LoweredGraph, csr) -> list:
    """[(block ids, template csr)] in launch order: cheap blocks first, then the
    rest; a single group when either side is empty."""
    off, nodes = csr
    nb = len(off) - 1
    if nb == 0:
        return []
    wr = low.w_rank[nodes]
    bits = np.where(wr >= 2, math.log2(3), np.where(wr == 1, 1.0, 0.0))
    lg = np.add.reduceat(bits, off[:-1]) if len(nodes) else np.zeros(nb)
    lg[off[1:] == off[:-1]] = 0.0
    small = lg < math.log2(SMALL_BLOCK_CANDIDATES)
    # a second launch pays off only when there are many cheap blocks to
    # explain and enough expensive work to hide them behind
    big_work = float(np.sum(np.exp2(np.minimum(lg[~small], 62.0))))
    if small.sum() < SPLIT_MIN_SMALL_BLOCKS or big_work < SPLIT_MIN_BIG_CANDIDATES:
        return [(list(range(nb)), csr)]
    out = []
    for mask in (small, ~small):
        ids = np.nonzero(mask)[0]
        T = off[ids + 1] - off[ids]
        goff = np.zeros(len(ids) + 1, np.int64)
        np.cumsum(T, out=goff[1:])
        gather = np.repeat(off[ids] - goff[:-1], T) + np.arange(goff[-1])
        out.append((ids.tolist(), (goff, np.ascontiguousarray(nodes[gather]))))
    return out


#: limits of the table path (csrc/search.cu MAXT, KMAX; smem per CTA): blocks
#: beyond them are searched by sp_route_search (no routing tables)
TABLE_MAX_T = 256
TABLE_MAX_FANIN = 6
SCORE_THREADS = 256


def _subset_csr(csr, ids):
    off, nodes = csr
    ids = np.asarray(ids, np.int64)
    T = off[ids + 1] - off[ids]
    goff = np.zeros(len(ids) + 1, np.int64)
    np.cumsum(T, out=goff[1:])
    gather = np.repeat(off[ids] - goff[:-1], T) + np.arange(goff[-1])
    return goff, np.ascontiguousarray(nodes[gather])


def _route_mask(low: LoweredGraph, csr) -> np.ndarray:
    """Blocks the routing tables cannot hold: more than TABLE_MAX_T template
    nodes, or a node with more than TABLE_MAX_FANIN internal producers."""
    off, nodes = csr
    nb = len(off) - 1
    T = np.diff(off)
    mask = T > TABLE_MAX_T
    if len(nodes) == 0:
        return mask
    fan_all = getattr(low, "_max_fanin", None)
    if fan_all is None:  # the graph's largest in-degree, once per lowered graph
        fan_all = int(np.diff(low.in_off).max(initial=0))
        try:
            low._max_fanin = fan_all
        except AttributeError:
            pass
    if fan_all <= TABLE_MAX_FANIN:
        return mask
    nodes = np.asarray(nodes, np.int64)
    blk = np.full(low.n_nodes, -1, np.int64)
    blk[nodes] = np.repeat(np.arange(nb), T)
    cnt = (low.in_off[nodes + 1] - low.in_off[nodes]).astype(np.int64)
    if cnt.sum() == 0:
        return mask
    coff = np.zeros(len(nodes) + 1, np.int64)
    np.cumsum(cnt, out=coff[1:])
    prod = low.in_idx[np.repeat(low.in_off[nodes] - coff[:-1], cnt) + np.arange(coff[-1])]
    internal = blk[prod] == np.repeat(blk[nodes], cnt)
    fan = np.bincount(np.repeat(np.arange(len(nodes)), cnt), weights=internal, minlength=len(nodes))
    if fan.max(initial=0) <= TABLE_MAX_FANIN:
        return mask
    nonempty = T > 0
    bmax = np.zeros(nb)
    bmax[nonempty] = np.maximum.reduceat(fan, off[:-1][nonempty])
    return mask | (bmax > TABLE_MAX_FANIN)


class _RouteSearch:
    """The blocks beyond the table limits, searched by sp_route_search (every
    candidate routed node by node on the device, no tables).  Same interface as
    _Search; every rank searches them whole (no exchange: results are equal)."""

    explain = True

    class _NoTables:
        def close(self):
            pass

    def __init__(self, ses: Session, csr, mesh, mu: int, chunk_size: int):
        self.ses, self.csr, self.mesh, self.mu, self.chunk_size = ses, csr, mesh, mu, chunk_size
        self.tables = self._NoTables()

    def launch(self) -> None:
        pass

    def fetch(self, explain_now: bool = False) -> None:
        pass

    def run(self, prep, indices=None):
        """(scores or None, detail) of the blocks (indices: explain those candidates)."""
        off, nodes = self.csr
        ref_slot = np.full(len(nodes), -1, np.int16)
        radix = np.ones(len(nodes), np.uint8)
        eoff = np.zeros(len(off), np.int64)
        for b, (slot_pos, radices, tnodes, _) in enumerate(prep):
            e0 = int(off[b])
            for k, (q, r) in enumerate(zip(slot_pos, radices)):
                ref_slot[e0 + q] = k
                radix[e0 + q] = r
            eoff[b + 1] = eoff[b] + sum(len(x[5]) for x in tnodes)
        # mu > chunk: pack_gradients' BadConfig comes from the first costed
        # candidate (rewrite.py:88); search with a legal chunk, collect raises
        return self.ses.backend.route_search(self.ses.dgraph, off, nodes, ref_slot, radix, eoff, self.mesh,
                                             self.mu, max(self.mu, self.chunk_size), indices)

    def collect(self, graph, subgraphs: list, want_table: bool, types: TypeSet, prep=None, slots=None,
                mult=None) -> list:
        self.extra = None
        if want_table:
            raise UnsupportedSearch("want_table for blocks beyond the routing-table limits "
                                    f"(> {TABLE_MAX_T} nodes or > {TABLE_MAX_FANIN} internal producers)")
        ses = self.ses
        low = ses.low
        bad = np.isin(low.op[self.csr[1]], (8, 9)) if len(self.csr[1]) else np.zeros(0, bool)
        if bad.any():  # patterns_for raises on routing such a node (patterns.py:166-170)
            raise SpecMismatch(f"{_OP_LABELS[int(low.op[self.csr[1][np.argmax(bad)]])]} is not a shardable compute kind")
        if prep is None:
            prep = route_prep(ses, subgraphs, types, self.csr)
        scores, detail = self.run(prep)
        for sc in scores:
            if not sc.has_best:
                raise AssertionError("all-replica fallback must always route")
            if self.mu > self.chunk_size:
                raise BadConfig(f"fusion threshold {self.mu} exceeds chunk size {self.chunk_size}")
        bests = routed_plans_all(ses, None, subgraphs, scores, self.mesh, types, detail, prep)
        SubgraphResult = _ctor(types.SubgraphResult, 5)
        return [SubgraphResult(sub, best, int(sc.candidates), int(sc.valid), [])
                for sub, sc, best in zip(subgraphs, scores, bests)]


class _NeedRoute(Exception):
    def __init__(self, ids):
        super().__init__(ids)
        self.ids = ids


def _explain_groups(ses: Session, csr, prep: list, indices: list, mesh, mu: int, chunk_size: int) -> list:
    """Detail of the given candidate of every block (the winner re-routing of
    pattern_routing / plan_cost / the replay): [(block ids, prep, indices,
    detail, tables or None)] -- explain_all on routing tables, the route search
    for the blocks beyond the table limits (including tables that turn out
    larger than a CTA's shared memory).  The caller closes the tables."""
    route = _route_mask(ses.low, csr)
    out = []
    try:
        tids = np.nonzero(~route)[0].tolist()
        if tids:
            gcsr = _subset_csr(csr, tids)
            tables = ses.backend.tables(ses.dgraph, gcsr[0], gcsr[1], mesh, mu, max(mu, chunk_size))
            by, _, _ = ses.backend.block_info(tables)
            over = np.nonzero(((by + 15) // 16) * 16 + 16 > ses.backend.smem_limit)[0]
            if len(over):
                tables.close()
                route[np.asarray(tids)[over]] = True
                tids = np.nonzero(~route)[0].tolist()
                gcsr = _subset_csr(csr, tids)
                tables = ses.backend.tables(ses.dgraph, gcsr[0], gcsr[1], mesh, mu, max(mu, chunk_size)) if tids else None
            if tids:
                gidx = [indices[i] for i in tids]
                out.append((tids, [prep[i] for i in tids], gidx, None, tables))
                out[-1] = (tids, out[-1][1], gidx, ses.backend.explain_all(tables, gidx), tables)
        rids = np.nonzero(route)[0].tolist()
        if rids:
            gprep = [prep[i] for i in rids]
            gidx = [indices[i] for i in rids]
            _, detail = _RouteSearch(ses, _subset_csr(csr, rids), mesh, mu, max(mu, chunk_size)).run(gprep, gidx)
            out.append((rids, gprep, gidx, detail, None))
    except BaseException:
        for *_, t in out:
            if t is not None:
                t.close()
        raise
    return out


def _plan_searches(ses: Session, csr, mesh, mu, chunk_size, shard, n_shards, exchange, root_local=False) -> list:
    """[(search, block ids)]: the route search of the blocks beyond the table
    limits (if any), then the table searches (cheap group first, _block_groups).
    A block whose tables turn out larger than shared memory moves to the route
    search (the tables are rebuilt without it).

    `root_local` (a multi-rank search inside the library where only rank 0
    assembles): the cheap group of a two-group split is scored whole on rank 0
    with no exchange (SP_SCORE_LOCAL) and not built at all on the other ranks --
    its results feed only the report, and every rank takes the same decision
    from the same fold."""
    nb = len(csr[0]) - 1
    route = _route_mask(ses.low, csr)
    while True:
        out = []
        rids = np.nonzero(route)[0]
        tids = np.nonzero(~route)[0]
        try:
            tcsr = csr if len(rids) == 0 else _subset_csr(csr, tids)
            groups = _block_groups(ses.low, tcsr)
            for k, (ids, gcsr) in enumerate(groups):
                gids = [int(tids[i]) for i in ids] if len(rids) else ids
                local = root_local and k == 0 and len(groups) > 1
                if local and not ses.backend.is_root:
                    continue
                srch = _Search(ses, gcsr, mesh, mu, chunk_size, shard, n_shards, exchange, launch=False,
                               local=local)
                out.append((srch, gids))
                over = srch.over_smem()
                if len(over):
                    raise _NeedRoute([gids[i] for i in over])
            if len(rids):  # last: the table groups keep their cheap-first order
                out.append((_RouteSearch(ses, _subset_csr(csr, rids), mesh, mu, chunk_size), rids.tolist()))
            return out
        except _NeedRoute as e:
            for srch, _ in out:
                srch.tables.close()
            route[e.ids] = True
        except BaseException:
            for srch, _ in out:
                srch.tables.close()
            raise


def _launch_all(searches: list) -> None:
    """Launch the searches of _plan_searches in order."""
    try:
        if len(searches) > 1 and not searches[0][0].explain:
            # sharded: the cheap group's winners are merged across ranks and
            # re-routed BEFORE the expensive launch -- once that persistent
            # kernel holds every SM, the re-routing kernel could not start
            searches[0][0].launch()
            searches[0][0].fetch(explain_now=True)
            for srch, _ in searches[1:]:
                srch.launch()
        else:
            for srch, _ in searches:
                srch.launch()
    except BaseException:
        for srch, _ in searches:
            srch.tables.close()
        raise


#: graphs up to this many GraphNodes (the one-CTA fold) take the one-call path
SMALL_PLAN_NODES = 8192


def _derive_small(ses: Session, mesh, min_duplicates: int, mu: int, chunk_size: int, types: TypeSet, t0: float,
                  t1: float):
    """derive_plan for a small graph: the device half in ONE library call
    (sp_plan_run: fold, templates, tables, search, winner detail), then the
    report from the raw records in C (block_results).  None when a block is
    beyond the table path (the caller's general path route-searches it)."""
    try:
        ba, csr, scores, detail = ses.backend.plan(ses.dgraph, int(min_duplicates), mesh, mu, chunk_size)
    except UnsupportedSearch:
        return None
    t2 = time.perf_counter()
    low = ses.low
    subs = subgraphs_from_blocks(low, ba, types)
    slots = Slots.of(low, csr)
    for sc in scores:
        if not sc.has_best:
            raise AssertionError("all-replica fallback must always route")
    nb = len(subs)
    mult = np.diff(np.asarray(ba.block_inst_off, np.int64))
    native = _native_results(ses, subs, scores, detail, csr, slots, mult, mesh, types)
    if native is None or any(r is None for r in native[0]):
        return None
    results, terms, labs = native
    t3 = time.perf_counter()
    total_cost = 0.0
    for x in terms:  # block order (search.py:373): the sum is not reassociated
        total_cost += x
    candidates = valid = 0
    for sc in scores:
        candidates += sc.candidates
        valid += sc.valid
    off = slots.off
    slot_labels = [lab for b, ls in enumerate(labs) if off[b + 1] > off[b] for lab in ls]
    assignments = _assignments(low.names, _label_keys(ba, subs, slots), slot_labels)
    LAST_PHASES.clear()
    LAST_PHASES.update(session_ms=(t1 - t0) * 1e3, plan_ms=(t2 - t1) * 1e3, results_ms=(t3 - t2) * 1e3,
                       assemble_ms=(time.perf_counter() - t3) * 1e3, path="one-call", blocks=nb)
    return types.BestPlanReport(mesh, min_duplicates, results, assignments, total_cost, candidates, valid)


def _derive_plan(graph, mesh, min_duplicates, mu, chunk_size, want_table, types, backend, session,
                 cache, shard, n_shards, exchange, root_only=True):
    t0 = time.perf_counter()
    ses = session or Session.open(graph, backend, cache=cache)
    t1 = time.perf_counter()
    if min_duplicates < 1:
        raise BadConfig("min_duplicates must be >= 1")
    if (ses.low.n_nodes <= SMALL_PLAN_NODES and not want_table and n_shards == 1 and exchange is None
            and mu <= chunk_size and ses.backend.single_lane and _native_lower is not None
            and isinstance(ses.low.names, list)):
        rep = _derive_small(ses, mesh, min_duplicates, mu, chunk_size, types, t0, t1)
        if rep is not None:
            return rep
    ba = ses.backend.fold(ses.dgraph, int(min_duplicates))
    t2 = time.perf_counter()
    n_blocks = ba.n_blocks
    csr = ba.templates_csr()
    # two launches when the blocks split into cheap and expensive ones: the
    # cheap group's results (typically hundreds of residual singletons) are
    # turned into RoutedPlans while the device still scores the expensive group
    # every group's tables first (each build syncs the stream once), then all
    # launches back to back: each search copies its results to the host behind
    # its own kernels, so the cheap group is collected while the expensive one
    # still scores
    if mu > chunk_size and n_blocks:
        # the reference fails in the first block (search.py:366): its first valid
        # candidate's plan_cost -> pack_gradients raises BadConfig (rewrite.py:88),
        # or, with no valid candidate, the all-replica assertion; score block 0 only
        off, nodes = csr
        c0 = (np.array([0, off[1] - off[0]], np.int64), nodes[off[0]:off[1]])
        first = (_RouteSearch(ses, c0, mesh, mu, chunk_size) if _route_mask(ses.low, c0)[0]
                 else _Search(ses, c0, mesh, mu, chunk_size, 0, 1, None))
        first.collect(graph, subgraphs_from_blocks(ses.low, ba, types)[:1], False, types)
        raise AssertionError("unreachable: block 0 raises BadConfig or the all-replica assertion")
    root_local = (root_only and exchange is None and n_shards == 1 and ses.backend.sharded_in_library
                  and not os.environ.get("SP_NO_ROOT_LOCAL"))
    searches = _plan_searches(ses, csr, mesh, mu, chunk_size, shard, n_shards, exchange, root_local)
    _launch_all(searches)
    if root_only and not ses.backend.is_root:
            # sharded: the cheap group's winners are merged across ranks and
            # re-routed BEFORE the expensive launch -- once that persistent
            # kernel holds every SM, the re-routing kernel could not start

        # a non-root rank of a multi-process search: its share is scored and
        # exchanged on the device; the report is rank 0's
        t3 = time.perf_counter()
        try:
            for srch, _ in searches:
                srch.fetch()
        finally:
            for srch, _ in searches:
                srch.tables.close()
        LAST_PHASES.clear()
        LAST_PHASES.update(path="general", session_ms=(t1 - t0) * 1e3, fold_ms=(t2 - t1) * 1e3,
                           launch_ms=(t3 - t2) * 1e3, collect_ms=(time.perf_counter() - t3) * 1e3)
        return None
    # host work that does not depend on the winners overlaps the device search:
    # Subgraph objects, the static part of every RoutedPlan, and the member
    # scopes that receive each block's weight labels (search.py:374-376)
    t3 = time.perf_counter()
    subs = subgraphs_from_blocks(ses.low, ba, types)
    t3a = time.perf_counter()
    slots = Slots.of(ses.low, csr)
    prep = None
    if slots is None:
        prep = route_prep(ses, subs, types, csr)
        slots = Slots.from_prep(prep)
    mult = np.diff(np.asarray(ba.block_inst_off, np.int64))
    t3b = time.perf_counter()
    label_keys = _label_keys(ba, subs, slots)
    # the assignment map's keys (scattered name objects) while the device searches
    akeys = None
    if _native_lower is not None and hasattr(_native_lower, "assignments_keys") and isinstance(ses.low.names, list):
        akeys = _native_lower.assignments_keys(ses.low.names, np.ascontiguousarray(label_keys[0], np.int32))
    t4 = time.perf_counter()
    # per block: the report's cost term and its weight labels, computed as each
    # group's results land (the cheap group's while the expensive one scores)
    results = [None] * n_blocks
    terms = [0.0] * n_blocks
    labs = [None] * n_blocks
    candidates = valid = 0
    marks = []
    try:
        for srch, ids in searches:
            if len(searches) == 1:
                got = srch.collect(graph, subs, want_table, types, prep, slots, mult)
            else:
                got = srch.collect(graph, [subs[i] for i in ids], want_table, types,
                                   None if prep is None else [prep[i] for i in ids], slots.subset(ids), mult[ids])
            extra = getattr(srch, "extra", None)
            for j, (i, res) in enumerate(zip(ids, got)):
                results[i] = res
                candidates += res.candidates
                valid += res.valid
                if extra is not None and extra[0][j] is not None:
                    terms[i] = extra[0][j]
                    if slots.off[i + 1] > slots.off[i]:
                        labs[i] = extra[1][j]
                else:
                    terms[i] = res.best.cost.total * subs[i].multiplicity
                    if slots.off[i + 1] > slots.off[i]:
                        labs[i] = [spec.label for _, spec in res.best.plan.assignments]
            fetched = getattr(srch, "_fetched", None)
            marks.append(round((fetched[2] - t0) * 1e3, 3) if fetched else None)
            marks.append(round((time.perf_counter() - t0) * 1e3, 3))
    finally:
        for srch, _ in searches:  # a group whose collect never ran (an earlier one raised)
            srch.tables.close()
    t5 = time.perf_counter()
    total_cost = 0.0
    for x in terms:  # block order (search.py:373): the sum is not reassociated
        total_cost += x
    slot_labels = [lab for ls in labs if ls is not None for lab in ls]
    # every instance takes the template's labels in weight_nodes order
    # (search.py:374-376); instance members come from the fold's member matrix
    if akeys is not None:
        assignments = _native_lower.assignments_fill(akeys[0], ses.low.names,
                                                     np.ascontiguousarray(label_keys[0], np.int32), akeys[1],
                                                     np.ascontiguousarray(label_keys[1], np.int32), slot_labels)
    else:
        assignments = _assignments(ses.low.names, label_keys, slot_labels)
    LAST_PHASES.clear()
    LAST_PHASES.update(path="general", session_ms=(t1 - t0) * 1e3, fold_ms=(t2 - t1) * 1e3,
                       launch_ms=(t3 - t2) * 1e3, overlap_host_ms=(t4 - t3) * 1e3,
                       subgraphs_ms=(t3a - t3) * 1e3, route_prep_ms=(t3b - t3a) * 1e3,
                       collect_ms=(t5 - t4) * 1e3, assemble_ms=(time.perf_counter() - t5) * 1e3,
                       groups_at_ms=marks)
    return types.BestPlanReport(mesh, min_duplicates, results, assignments, total_cost, candidates,
                                valid)


class _OneScore:
    """Score stand-in so routed_plans_all can explain an arbitrary candidate."""

    def __init__(self, index: int):
        self.best_index = index
        self.has_best = 1
        self.best_total = float("nan")


def _explain_plan(graph, plan, mesh, mu, chunk_size, types, session):
    ses = session or Session.open(graph)
    index, bad = _plan_index(graph, plan)
    csr = _templates_csr(ses.low, [plan.subgraph])
    prep = route_prep(ses, [plan.subgraph], types, csr)
    groups = _explain_groups(ses, csr, prep, [index], mesh, mu, chunk_size)
    try:
        _, gprep, _, detail, tables = groups[0]
        routed = routed_plans_all(ses, tables, [plan.subgraph], [_OneScore(index)], mesh, types, detail, gprep)[0]
    finally:
        for *_, t in groups:
            if t is not None:
                t.close()
    template = plan.subgraph.template
    if bad is not None and (not isinstance(routed, types.RoutingFailure)
                            or template.index(routed.node) > bad):
        # the first node (topological order) whose weight spec matches no pattern
        return types.RoutingFailure(template[bad], "no pattern chains from producer states")
    if isinstance(routed, types.RoutingFailure):
        return routed
    # the caller's plan object, as the reference returns it (search.py:224)
    return types.RoutedPlan(plan, routed.routings, routed.exit_conversions, routed.cost)


def pattern_routing(graph, plan, mesh, *, types: TypeSet = DEFAULT_TYPES,
                    session: Optional[Session] = None):
    """Route one candidate (search.py:134-224): RoutedPlan with an empty CostReport, or
    RoutingFailure (returned, not raised).  Evaluated on the device (sp_explain_all)."""
    routed = _explain_plan(graph, plan, mesh, 1 << 20, 4 << 20, types, session)
    if isinstance(routed, types.RoutingFailure):
        return routed
    return types.RoutedPlan(plan, routed.routings, routed.exit_conversions, types.CostReport())


def plan_cost(routed, graph, mesh, mu: int = 1 << 20, chunk_size: int = 4 << 20, *,
              types: TypeSet = DEFAULT_TYPES, session: Optional[Session] = None):
    """CostReport of a routed plan (costmodel.py:193-267), on the device."""
    if mu > chunk_size:
        raise BadConfig(f"fusion threshold {mu} exceeds chunk size {chunk_size}")
    full = _explain_plan(graph, routed.plan, mesh, mu, chunk_size, types, session)
    return full.cost


# ---------------------------------------------------------------------------
# plan replay (search.py:382-444): the "resume" path of a stored plan file


def routed_plan_for_assignments(graph, mesh, assignments: dict, min_duplicates: int = 2, mu: int = 1 << 20,
                                chunk_size: int = 4 << 20, *, types: TypeSet = DEFAULT_TYPES,
                                backend: Optional[Backend] = None, session: Optional[Session] = None):
    """Re-route a plan loaded from a report file (assignment labels only), on the
    device: the fold, then every block's stored assignment routed and costed in
    ONE explain launch (search.py:411-444 loops pattern_routing + plan_cost)."""
    from .errors import ShardplanError

    ses = session or Session.open(graph, backend)
    if min_duplicates < 1:
        raise BadConfig("min_duplicates must be >= 1")
    ba = ses.backend.fold(ses.dgraph, int(min_duplicates))
    subs = subgraphs_from_blocks(ses.low, ba, types)
    csr = ba.templates_csr()
    prep = route_prep(ses, subs, types, csr)
    # stored labels -> candidate index in the reference's enumeration order; a spec
    # that is not a search option gets digit 0 and fails at its node (see _plan_index)
    indices, bads, chosen = [], [], []
    for sub, (slot_pos, radices, _, _) in zip(subs, prep):
        index = 0
        bad = None
        specs = []
        for q, r in zip(slot_pos, radices):
            scope = sub.template[q]
            spec = types.ShardSpec.from_label(assignments[scope])
            specs.append((scope, spec))
            d = _spec_digit(spec, int(ses.low.w_rank[ses.low.index[scope]]), r)
            if d is None:
                bad = q if bad is None else min(bad, q)
                d = 0
            index = index * r + d
        indices.append(index)
        bads.append(bad)
        chosen.append(tuple(sorted(specs, key=lambda t: t[0])))
    # per block group (routing tables / route search beyond the table limits)
    groups = _explain_groups(ses, csr, prep, indices, mesh, mu, chunk_size)
    Xs = [None] * len(subs)
    for ids, _, _, detail, _ in groups:
        for i, X in zip(ids, detail[0]):
            Xs[i] = X
    try:
        for b, X in enumerate(Xs):
            fail = None if X.valid else int(X.fail_pos)
            if bads[b] is not None and (fail is None or fail > bads[b]):
                fail = bads[b]
            if fail is not None:
                raise ShardplanError(f"stored plan does not route at node {subs[b].template[fail]}: "
                                     "no pattern chains from producer states")
            if mu > chunk_size:
                raise BadConfig(f"fusion threshold {mu} exceeds chunk size {chunk_size}")
        bests = [None] * len(subs)
        for ids, gprep, gidx, detail, tables in groups:
            got = routed_plans_all(ses, tables, [subs[i] for i in ids], [_OneScore(i) for i in gidx], mesh, types,
                                   detail, gprep)
            for i, r in zip(ids, got):
                bests[i] = r
    finally:
        for *_, tables in groups:
            if tables is not None:
                tables.close()
    results = []
    total_cost = 0.0
    for sub, routed, specs in zip(subs, bests, chosen):
        plan = types.CandidatePlan(sub, specs, -1)  # the stored specs (search.py:427-430)
        routed = types.RoutedPlan(plan, routed.routings, routed.exit_conversions, routed.cost)
        results.append(types.SubgraphResult(sub, routed, 1, 1))
        total_cost += routed.cost.total * sub.multiplicity
    return types.BestPlanReport(mesh, min_duplicates, results, dict(assignments), total_cost, 0, 0)


def broadcast_routing(report, types: TypeSet = DEFAULT_TYPES) -> dict:
    """Whole-graph routing map: each winning template routing replayed on every
    instance with prefix-swapped producer scopes (search.py:382-408)."""
    out: dict = {}
    NodeRouting = types.NodeRouting
    for res in report.results:
        sub = res.subgraph
        tp = sub.template_prefix
        for prefix, _ in sub.instances:
            swap = (lambda s: s) if prefix == tp else (lambda s, p=prefix, n=len(tp): p + s[n:])
            for r in res.best.routings:
                scope = swap(r.scope)
                out[scope] = NodeRouting(scope, r.pattern, tuple((swap(p), c, b) for p, c, b in r.input_conversions),
                                         r.output_collective, r.output_bytes, r.state)
            for scope, coll, _ in res.best.exit_conversions:
                s = swap(scope)
                r = out[s]
                out[s] = NodeRouting(r.scope, r.pattern, r.input_conversions, r.output_collective, r.output_bytes,
                                     r.state, exit_conversion=coll)
    return out
