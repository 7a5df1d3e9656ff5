"""Pin the in-package graph generators to the reference-generated fixtures."""

from __future__ import annotations

import pytest

from golden_io import graph
from paper_2302_00247_b200.ir import dump_grouped
from paper_2302_00247_b200.workloads import transformer_stack, wide_classifier


@pytest.mark.parametrize("path,kw", [
    ("graphs/tiny_transformer.json.gz", dict(layers=2, d_model=8)),
    ("graphs/tiny_transformer_f64.json.gz", dict(layers=2, d_model=8, dtype="f64")),
    ("graphs/c1.json.gz", dict(layers=12, d_model=768, heads=12)),
    ("graphs/c4.json.gz", dict(layers=48, d_model=6144, heads=48)),
    ("graphs/bench_L48.json.gz", dict(layers=48, d_model=8, heads=2)),
    ("graphs/crit5.json.gz", dict(layers=4, d_model=512, heads=8, batch=96, seq=16)),
    ("graphs/tf24.json.gz", dict(layers=24)),
])
def test_transformer_stack_matches_reference(path, kw):
    assert dump_grouped(transformer_stack(**kw)) == dump_grouped(graph(path))


@pytest.mark.parametrize("path,kw", [
    ("graphs/c3.json.gz", dict(num_classes=100000, feature_dim=2048, blocks=16, batch=32)),
    ("graphs/tiny_classifier_f64.json.gz", dict(num_classes=64, feature_dim=16, dtype="f64")),
    ("graphs/wide150.json.gz", dict(num_classes=64, feature_dim=16, blocks=150)),
])
def test_wide_classifier_matches_reference(path, kw):
    assert dump_grouped(wide_classifier(**kw)) == dump_grouped(graph(path))


def _sha(obj) -> str:
    import hashlib
    import json

    return hashlib.sha256(json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


@pytest.mark.parametrize("idx", range(4))
def test_fold_stress_graph_and_oracle_pinned(idx):
    """Config-4 fold stress (L=480 / 7000 layers): generator == reference graph and
    oracle prune == reference prune, by hash."""
    from golden_io import fold_stress
    from oracle import oracle
    from paper_2302_00247_b200.blocks import BlockArrays, to_prune_doc
    from paper_2302_00247_b200.lowering import lower

    fs = fold_stress()[idx]
    g = transformer_stack(fs["layers"])
    assert len(g.nodes) == fs["nodes"]
    assert _sha(dump_grouped(g)) == fs["graph_sha"]
    low = lower(g)
    ba = BlockArrays.from_dict(oracle.prune(low, fs["min_dup"]))
    assert _sha(to_prune_doc(low, ba)) == fs["prune_sha"]


C5_KEYS = [("parity", 0), ("throughput", 0), ("parity", 1), ("parity", 2)]


@pytest.mark.parametrize("tier,seed", C5_KEYS)
def test_c5_graph_and_oracle_fold_pinned(tier, seed):
    """Config 5: generator == the graph the reference was run on; oracle fold == reference."""
    from golden_io import c5
    from oracle import oracle
    from paper_2302_00247_b200.blocks import BlockArrays, to_prune_doc
    from paper_2302_00247_b200.lowering import lower
    from paper_2302_00247_b200.workloads import motif_dag

    gold = c5()[(tier, seed)]
    g = motif_dag(seed, tier)
    assert _sha(dump_grouped(g)) == gold["graph_sha"]
    low = lower(g)
    ba = BlockArrays.from_dict(oracle.prune(low, 2))
    assert _sha(to_prune_doc(low, ba)) == gold["prune_sha"]


@pytest.mark.parametrize("tier,seed", C5_KEYS)
def test_c5_oracle_slices_and_search(tier, seed):
    """Per-candidate totals on the golden slices; full parity-tier search == reference."""
    from golden_io import c5, mesh
    from oracle import oracle
    from paper_2302_00247_b200.blocks import BlockArrays
    from paper_2302_00247_b200.lowering import lower
    from paper_2302_00247_b200.workloads import motif_dag

    gold = c5()[(tier, seed)]
    low = lower(motif_dag(seed, tier))
    ba = BlockArrays.from_dict(oracle.prune(low, 2))
    m = mesh(gold["mesh"])
    for sl in gold["slices"]:
        _, tot = oracle.score(low, ba.template_nodes(sl["block"]), m, lo=sl["lo"], hi=sl["hi"],
                              want_totals=True)
        assert [None if t != t else t for t in tot.tolist()] == sl["totals"]
    if tier == "parity":
        total = 0.0
        for b, (idx, ns, tot, valid) in enumerate(gold["best"]):
            out, _ = oracle.score(low, ba.template_nodes(b), m, threads=8)
            assert (out.best_index, out.best_num_split, repr(out.best_total), out.valid) == (
                idx, ns, tot, valid)
            total += out.best_total * ba.multiplicity(b)
        assert repr(total) == gold["total_cost"]


@pytest.mark.parametrize("layers", [2, 3, 7, 40])
def test_transformer_stack_lowered_equals_object_path(layers):
    import numpy as np

    from paper_2302_00247_b200.lowering import lower
    from paper_2302_00247_b200.workloads import transformer_stack_lowered

    a = lower(transformer_stack(layers, d_model=64))
    b = transformer_stack_lowered(layers, d_model=64)
    assert a.names == b.names
    for f in ("name_bytes", "name_off", "topo_rank", "op", "act_rank", "act_shape", "act_bytes",
              "w_rank", "w_shape", "w_bytes", "w_trainable", "in_off", "in_idx"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
