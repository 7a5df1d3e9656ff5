"""Shared loaders for the committed golden fixtures (tests/golden/)."""

from __future__ import annotations

import functools
import json
import os

from paper_2302_00247_b200.api_types import ClusterSpec, CollectiveKind
from paper_2302_00247_b200.ir import load_grouped
from paper_2302_00247_b200.lowering import lower

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def _doc() -> dict:
    with open(os.path.join(GOLDEN, "cases.json")) as fh:
        return json.load(fh)


def cases() -> list:
    return _doc()["cases"]


def fold_stress() -> list:
    return _doc()["fold_stress"]


def case(name: str) -> dict:
    for c in cases():
        if c["case"] == name:
            return c
    raise KeyError(name)


@functools.lru_cache(maxsize=None)
def graph(path: str):
    return load_grouped(os.path.join(GOLDEN, path))


@functools.lru_cache(maxsize=None)
def lowered(path: str):
    return lower(graph(path))


def mesh(doc: dict) -> ClusterSpec:
    eff = tuple(sorted(((CollectiveKind(k), float(v)) for k, v in doc["efficiency"].items()),
                       key=lambda kv: kv[0].value))
    return ClusterSpec(m=doc["m"], n=doc["n"], intra_bw=float(doc["intra_bw"]),
                       inter_bw=float(doc["inter_bw"]), efficiency=eff,
                       overlap_fraction=float(doc["overlap_fraction"]),
                       setup_latency_s=float(doc["setup_latency_s"]))


def case_names(pred=lambda c: True) -> list:
    return [c["case"] for c in cases() if pred(c)]


@functools.lru_cache(maxsize=1)
def c5() -> dict:
    with open(os.path.join(GOLDEN, "c5.json")) as fh:
        out = {}
        for e in json.load(fh)["c5"]:
            out[(e["tier"], e["seed"])] = e
            if e["seed"] == 0:
                out[e["tier"]] = e
        return out
