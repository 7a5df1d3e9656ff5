"""Pin the CPU oracle (oracle/oracle.c) to the reference's golden vectors.

The goldens were produced by the reference itself (tests/golden/make_golden.py).
Once these pass, the oracle is a trusted checker for the GPU path on inputs
the reference was never run on (random graphs, larger sizes).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from golden_io import case, case_names, graph, lowered, mesh
from oracle import oracle
from paper_2302_00247_b200.blocks import BlockArrays, to_prune_doc

PRUNE_CASES = case_names(lambda c: "prune" in c)
PLAN_CASES = case_names(lambda c: "best" in c)


@pytest.mark.parametrize("name", PRUNE_CASES)
def test_oracle_prune_matches_reference(name):
    c = case(name)
    low = lowered(c["graph"])
    ba = BlockArrays.from_dict(oracle.prune(low, c["min_dup"]))
    assert to_prune_doc(low, ba) == c["prune"]


def _block_results(c, ba, low, threads=4):
    m = mesh(c["mesh"])
    out = []
    for b in range(ba.n_blocks):
        res, _ = oracle.score(low, ba.template_nodes(b), m, mu=c["mu"], chunk=c["chunk_size"],
                              threads=threads)
        out.append(res)
    return out


SMALL_PLAN_CASES = [n for n in PLAN_CASES if case(n)["candidates"] < 200000]


@pytest.mark.parametrize("name", SMALL_PLAN_CASES)
def test_oracle_search_matches_reference(name):
    c = case(name)
    low = lowered(c["graph"])
    ba = BlockArrays.from_dict(oracle.prune(low, c["min_dup"]))
    results = _block_results(c, ba, low)
    assert len(results) == len(c["best"])
    for res, exp in zip(results, c["best"]):
        assert res.valid == exp["valid"]
        assert res.has_best
        assert res.best_index == exp["index"]
        assert res.best_num_split == exp["num_split"]
        assert repr(res.best_total) == exp["total"]  # bit-exact fp64
    assert sum(r.candidates for r in results) == c["candidates"]
    total = 0.0
    for res, b in zip(results, range(ba.n_blocks)):
        total += res.best_total * ba.multiplicity(b)
    assert repr(total) == c["total_cost"]


@pytest.mark.slow
@pytest.mark.parametrize("name", [n for n in PLAN_CASES if n not in SMALL_PLAN_CASES])
def test_oracle_search_large(name):
    c = case(name)
    low = lowered(c["graph"])
    ba = BlockArrays.from_dict(oracle.prune(low, c["min_dup"]))
    results = _block_results(c, ba, low, threads=8)
    for res, exp in zip(results, c["best"]):
        assert (res.valid, res.best_index, repr(res.best_total)) == (
            exp["valid"], exp["index"], exp["total"])


TABLE_CASES = case_names(lambda c: "tables" in c)


@pytest.mark.parametrize("name", TABLE_CASES)
def test_oracle_per_candidate_totals(name):
    c = case(name)
    low = lowered(c["graph"])
    ba = BlockArrays.from_dict(oracle.prune(low, c["min_dup"]))
    m = mesh(c["mesh"])
    for tab in c["tables"]:
        _, totals = oracle.score(low, ba.template_nodes(tab["block"]), m, mu=c["mu"],
                                 chunk=c["chunk_size"], lo=tab["lo"], hi=tab["hi"],
                                 threads=2, want_totals=True)
        got = [None if math.isnan(t) else t for t in totals.tolist()]
        exp = [row[1] for row in tab["rows"]]
        assert [r[0] for r in tab["rows"]] == list(range(tab["lo"], tab["hi"]))
        assert got == exp  # exact (json floats round-trip)


def test_oracle_error_cases():
    c = case("weighted_layernorm")
    assert c["derive_error"].startswith("AssertionError")
    low = lowered(c["graph"])
    ba = BlockArrays.from_dict(oracle.prune(low, c["min_dup"]))
    zero_valid = []
    for b in range(ba.n_blocks):
        res, _ = oracle.score(low, ba.template_nodes(b), mesh(c["mesh"]))
        zero_valid.append(res.valid == 0)
    assert any(zero_valid)  # the weighted layernorm block never routes (D1)
