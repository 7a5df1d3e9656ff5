"""Native dataclass constructors (csrc/lower_ext.c make_ctor, search._ctor):
objects equal to the generated __init__'s, for this package's result types and
the reference's, and the generated __init__ kept wherever it does more."""

from __future__ import annotations

import copy
import dataclasses
import os
import pickle
import sys

import pytest

from paper_2302_00247_b200 import api_types as A
from paper_2302_00247_b200 import search
from paper_2302_00247_b200.lowering import _native_lower

pytestmark = pytest.mark.skipif(_native_lower is None, reason="native extension not built")
REF = "/root/reference/pkg/src"


def _samples(ns):
    sub = ns.Subgraph("net/a", ("net/a/x", "net/a/y"), (("net/a", ("net/a/x", "net/a/y")),))
    rep = ns.ShardSpec(ns.ShardKind.REPLICA)
    ident = ns.Collective(ns.CollectiveKind.IDENTITY)
    plan = ns.CandidatePlan(sub, (("net/a/x", rep),), 7)
    nr = ns.NodeRouting("net/a/x", "matmul.col", (), ident, 4096, rep)
    cost = ns.CostReport(1e-5, 2e-5, 0.5, {"allreduce": 64}, 3, 128)
    rp = ns.RoutedPlan(plan, (nr,), (), cost)
    res = ns.SubgraphResult(sub, rp, 9, 4, [])
    return [(ns.Subgraph, sub, 3), (ns.CandidatePlan, plan, 3), (ns.NodeRouting, nr, 6),
            (ns.CostReport, cost, 6), (ns.RoutedPlan, rp, 4), (ns.SubgraphResult, res, 5)]


def _check(ns):
    for cls, obj, n in _samples(ns):
        f = search._ctor(cls, n)
        assert f is not cls, cls  # native path taken
        names = [x.name for x in dataclasses.fields(cls)][:n]
        got = f(*[getattr(obj, k) for k in names])
        assert type(got) is cls and got == obj and repr(got) == repr(obj)
        assert vars(got) == vars(obj) and list(vars(got)) == list(vars(obj))
        assert pickle.loads(pickle.dumps(got)) == obj and copy.deepcopy(got) == obj
        try:
            h = hash(obj)
        except TypeError:  # e.g. a frozen class holding a CostReport
            h = None
        if h is not None:
            assert hash(got) == h
        if cls.__dataclass_params__.frozen:
            with pytest.raises(dataclasses.FrozenInstanceError):
                setattr(got, names[0], None)


def test_native_ctor_matches_generated_init():
    _check(A)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_native_ctor_on_reference_types():
    sys.path.insert(0, REF)
    try:
        from shardplan import costmodel, patterns, pruning
        from shardplan import search as rs
    finally:
        sys.path.remove(REF)

    class NS:
        Subgraph = pruning.Subgraph
        CandidatePlan, NodeRouting, RoutedPlan, SubgraphResult = (rs.CandidatePlan, rs.NodeRouting, rs.RoutedPlan,
                                                                  rs.SubgraphResult)
        CostReport = costmodel.CostReport
        ShardSpec, ShardKind = patterns.ShardSpec, patterns.ShardKind
        Collective, CollectiveKind = patterns.Collective, patterns.CollectiveKind

    _check(NS)


def test_generated_init_kept_where_it_does_more():
    @dataclasses.dataclass
    class Post:
        a: int

        def __post_init__(self):
            self.b = 2 * self.a

    @dataclasses.dataclass
    class Factory:
        a: int
        b: list = dataclasses.field(default_factory=list)

    @dataclasses.dataclass
    class NoInit:
        a: int
        b: int = dataclasses.field(default=0, init=False)

    assert search._ctor(Post, 1) is Post
    assert search._ctor(Factory, 1) is Factory  # a fresh list per instance
    assert search._ctor(Factory, 2) is not Factory
    assert search._ctor(NoInit, 1) is NoInit
    f = search._ctor(A.NodeRouting, 6)  # the seventh field takes its default
    r = f("s", "p", (), A.Collective(A.CollectiveKind.IDENTITY), 1, A.ShardSpec(A.ShardKind.REPLICA))
    assert r.exit_conversion is None
    with pytest.raises(TypeError):
        f("too", "few")


@pytest.mark.parametrize("seed", range(6))
def test_block_flops_vectorised_equals_reference_loop(seed):
    """search._block_flops (numpy over every template node) == _flops per block
    (costmodel.py:185-190), including blocks with huge shapes (Python ints)."""
    import dataclasses as dc

    import numpy as np

    from paper_2302_00247_b200.lowering import lower
    from randgraph import random_graph

    low = lower(random_graph(seed, n_types=4, reps=(2, 6), ops=(3, 11)))
    if seed % 2:  # a matmul whose flops pass 2**63
        mm = np.nonzero((low.op == 0) & (low.w_rank > 0))[0]
        if len(mm):
            shp = low.act_shape.copy()
            shp[mm[0], 0] = 1 << 40
            low = dc.replace(low, act_shape=shp)
    rng = np.random.default_rng(seed)
    n = low.n_nodes
    cuts = np.sort(rng.choice(np.arange(1, n), size=min(20, n - 1), replace=False))
    off = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    tn = rng.permutation(n).astype(np.int32)
    assert search._block_flops(low, (off, tn)) == [search._flops(low, tn[off[b]:off[b + 1]].tolist())
                                                    for b in range(len(off) - 1)]


@pytest.mark.parametrize("seed", range(0, 12, 2))
def test_assignment_map_vectorised_equals_block_loop(seed):
    """_label_keys + the native dict builder give the assignment map the
    per-block loop over the fold's member matrix gives (search.py:374-376):
    same keys, same order, same labels."""
    import numpy as np

    from oracle import oracle
    from paper_2302_00247_b200.blocks import BlockArrays
    from paper_2302_00247_b200.lowering import lower
    from randgraph import random_graph

    low = lower(random_graph(seed, n_types=4, reps=(2, 6), ops=(3, 11)))
    ba = BlockArrays.from_dict(oracle.prune(low, 1 + seed % 3))
    subs = search.subgraphs_from_blocks(low, ba)

    class Ses:
        pass

    ses = Ses()
    ses.low = low
    prep = search.route_prep(ses, subs, A.DEFAULT_TYPES if hasattr(A, "DEFAULT_TYPES") else search.DEFAULT_TYPES,
                             ba.templates_csr())
    labels, exp = [], {}
    for b, (sub, pb) in enumerate(zip(subs, prep)):
        if not pb[0]:
            continue
        mine = [f"L{b}.{q}" for q in range(len(pb[0]))]
        labels.extend(mine)
        T, mo, R = int(ba.block_T[b]), int(ba.block_member_off[b]), sub.multiplicity
        mat = ba.members[mo: mo + R * T].reshape(R, T)[:, pb[0]]
        for k, v in zip([low.names[i] for i in mat.ravel().tolist()], mine * R):
            exp[k] = v
    got = search._assignments(low.names, search._label_keys(ba, subs, prep), labels)
    assert list(got.items()) == list(exp.items())
    rows, slots = search._label_keys(ba, subs, prep)
    py = dict(zip(map(low.names.__getitem__, rows.tolist()), map(labels.__getitem__, slots.tolist())))
    assert list(py.items()) == list(exp.items())
    assert np.all(slots >= 0)


def _fake_search(types, seed):
    """A folded random graph with fabricated, self-consistent score and explain
    records (every block routed), as a search would return them."""
    import ctypes as C

    import numpy as np

    from oracle import oracle
    from paper_2302_00247_b200._abi import SpExplainBlock, SpScoreOut
    from paper_2302_00247_b200._native import RawList
    from paper_2302_00247_b200.api_types import ClusterSpec
    from paper_2302_00247_b200.blocks import BlockArrays
    from paper_2302_00247_b200.lowering import lower
    from randgraph import random_graph

    low = lower(random_graph(seed, n_types=3, reps=(2, 5), ops=(3, 9)))
    ba = BlockArrays.from_dict(oracle.prune(low, 2))
    subs = search.subgraphs_from_blocks(low, ba, types)
    csr = ba.templates_csr()

    class Ses:
        pass

    ses = Ses()
    ses.low = low
    prep = search.route_prep(ses, subs, types, csr)
    mesh = ClusterSpec.from_mesh("2x4")
    rng = np.random.default_rng(seed)
    nb = len(subs)
    sc = (SpScoreOut * nb)()
    xb = (SpExplainBlock * nb)()
    ne = int(csr[0][-1])
    node = np.zeros((max(1, ne), 4), np.int8)
    for b in range(nb):
        slot_pos, radices, nodes, _ = prep[b]
        npat = [len(types.pattern_names.get(n[1], ())) for n in nodes]
        routed = all(npat)
        fwd, bwd = float(rng.random()) * 1e-4, float(rng.random()) * 1e-4
        idx = int(rng.integers(0, int(np.prod(radices)) if radices else 1))
        sc[b].candidates, sc[b].valid, sc[b].best_index = 7 + b, 3, idx
        sc[b].best_total = fwd + bwd * (1.0 - mesh.overlap_fraction)
        sc[b].best_num_split, sc[b].has_best = 0, 1 if routed else 0
        x = xb[b]
        x.valid, x.fail_pos = (1, -1) if routed else (0, 0)
        x.forward_comm, x.backward_comm, x.total = fwd, bwd, sc[b].best_total
        for j in range(4):
            x.calls[j] = int(rng.integers(0, 3))
            x.bytes[j] = int(rng.integers(0, 1 << 40)) if x.calls[j] else 0
        x.collective_calls = sum(x.calls)
        for i, k in enumerate(npat):
            e = int(csr[0][b]) + i
            node[e] = (int(rng.integers(0, max(1, k))), int(rng.integers(-1, 2)), int(rng.integers(-1, 2)), 0)
    scores = RawList(sc, nb)
    blocks = RawList(xb, nb)
    eoff = np.zeros(nb + 1, np.int64)
    detail = (blocks, node, np.zeros((1, 2), np.int8), eoff)
    return ses, subs, scores, detail, prep, csr, mesh


def _check_singletons(types, seed):
    ses, subs, scores, detail, prep, csr, mesh = _fake_search(types, seed)
    fast = search._singleton_results(ses, subs, scores, detail, prep, csr, mesh, types)
    done = [b for b, r in enumerate(fast) if r is not None]
    assert done, "no one-node block took the native path"
    py = search.routed_plans_all(ses, None, subs, scores, mesh, types, detail, prep, only=done)
    for b, rp in zip(done, py):
        exp = types.SubgraphResult(subs[b], rp, int(scores[b].candidates), int(scores[b].valid), [])
        assert fast[b] == exp and repr(fast[b]) == repr(exp)
        assert type(fast[b].best.cost) is type(rp.cost) and fast[b].best.cost.total == scores[b].best_total


@pytest.mark.parametrize("seed", range(4))
def test_singleton_results_equal_python_path(seed):
    """csrc singleton_results builds the same SubgraphResult/RoutedPlan/CostReport
    objects routed_plans_all + collect build, from the same raw records."""
    _check_singletons(search.DEFAULT_TYPES, seed)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
@pytest.mark.parametrize("seed", range(2))
def test_singleton_results_with_reference_types(seed):
    sys.path.insert(0, REF)
    try:
        import shardplan

        from paper_2302_00247_b200.swap import reference_types
        types = reference_types(shardplan)
    finally:
        sys.path.remove(REF)
    _check_singletons(types, seed)
