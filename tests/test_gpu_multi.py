"""Multi-GPU search inside the library, on one B200.

* A context over several devices of one process (sp_ctx_create(ngpu, ...)):
  here the same GPU listed 2 and 3 times, so the lanes exchange their per-block
  records by peer copies onto the primary (the NCCL transport needs distinct
  devices); every lane scores its round-robin share of each block's work items
  and k_merge_ranks merges them on the device.
* A process-per-GPU context joined to an NCCL communicator
  (sp_comm_unique_id + sp_ctx_comm_init, ncclCommInitRank) at nranks 1: the
  search goes through the real ncclAllGather + device merge + chained explain.

Both must give byte-identical derive_plan JSON to the single-device search
(the reference's pool split + exact min-merge, search.py:327-343), including
the bench workload's whole plan.
"""

from __future__ import annotations

import hashlib
import json
import os

import pytest

from golden_io import GOLDEN, case, graph, mesh

pytestmark = pytest.mark.gpu

CASES = ("c1_1x8", "c2_1x8", "chain6_2x4_mu", "tiny_2x2", "crit5_slow", "c3_2x4_slow", "encdec34")


def canon(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


@pytest.fixture(scope="module")
def single():
    from paper_2302_00247_b200._native import default_backend

    return default_backend()


@pytest.fixture(scope="module", params=[2, 3])
def lanes(request):
    from paper_2302_00247_b200._native import Backend

    be = Backend(devices=[0] * request.param)
    yield be
    be.close()


@pytest.fixture(scope="module")
def nccl1():
    from paper_2302_00247_b200._native import Backend
    from paper_2302_00247_b200.dist import init_comm

    be = Backend(0)

    class Store(dict):
        def set(self, k, v):
            self[k] = v

        def get(self, k):  # noqa: A003
            return self[k]

    be.comm_init(1, 0, be.comm_unique_id())
    assert init_comm(be, 0, 1, Store()) == be.comm
    yield be
    be.close()


def _plans(be, single, name):
    from paper_2302_00247_b200.search import derive_plan

    c = case(name)
    kw = dict(min_duplicates=c["min_dup"], mu=c["mu"], chunk_size=c["chunk_size"])
    g, m = graph(c["graph"]), mesh(c["mesh"])
    return derive_plan(g, m, backend=be, **kw), derive_plan(g, m, backend=single, **kw), c


@pytest.mark.parametrize("name", CASES)
def test_multi_lane_search_equals_single_device(lanes, single, name):
    info = lanes.comm_info()
    assert info["transport"] == "p2p" and info["devices"] == info["nranks"] >= 2
    got, ref, c = _plans(lanes, single, name)
    assert canon(got.to_json()) == canon(ref.to_json()) == c["plan_json"]


@pytest.mark.parametrize("name", CASES)
def test_nccl_communicator_search_equals_single_device(nccl1, single, name):
    info = nccl1.comm_info()
    assert info["transport"] == "nccl" and info["nranks"] == 1 and info["nccl_version"] >= 22000
    got, ref, c = _plans(nccl1, single, name)
    assert canon(got.to_json()) == canon(ref.to_json()) == c["plan_json"]


@pytest.mark.parametrize("mode", ["walk", "skip"])
def test_multi_lane_bench_workload_whole_plan(mode):
    """The bench workload (c5 throughput tier, 3.9e9 candidates) split over 2
    lanes == the reference's whole plan (tests/golden/c5_full.json)."""
    from paper_2302_00247_b200._native import Backend
    from paper_2302_00247_b200.api_types import ClusterSpec
    from paper_2302_00247_b200.search import derive_plan
    from paper_2302_00247_b200.workloads import motif_dag

    with open(os.path.join(GOLDEN, "c5_full.json")) as fh:
        gold = json.load(fh)
    be = Backend(devices=[0, 0])
    try:
        be.set_mode(mode)
        rep = derive_plan(motif_dag(0, "throughput"), ClusterSpec.from_mesh("1x8"), backend=be)
    finally:
        be.close()
    assert hashlib.sha256(canon(rep.to_json()).encode()).hexdigest() == gold["plan_sha"]


def test_lanes_split_the_work(lanes, single):
    """Each lane launches its own scoring kernel (launch counts grow with the lanes)."""
    from paper_2302_00247_b200.search import derive_plan

    c = case("c2_1x8")
    g, m = graph(c["graph"]), mesh(c["mesh"])
    derive_plan(g, m, backend=lanes)
    a0, _ = lanes.launch_counts()
    b0, _ = single.launch_counts()
    derive_plan(g, m, backend=lanes)
    derive_plan(g, m, backend=single)
    a1, _ = lanes.launch_counts()
    b1, _ = single.launch_counts()
    assert (a1 - a0) > (b1 - b0)
