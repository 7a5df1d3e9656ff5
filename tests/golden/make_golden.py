"""Generate the golden fixtures that pin the oracle and the CUDA path.

Run HERE (the build container), where the reference is importable from the
read-only tree; the outputs are committed so the GPU box never needs
/root/reference:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every expected value below is produced by the reference's own code
(shardplan 0.1.0): ``trim_and_group`` / ``prune_graph`` (pruning.py:123-201),
``derive_plan(...).to_json()`` (search.py:255-281, 348-379) and
``_eval_range(..., want_table=True)`` (search.py:289-310) for per-candidate
totals.  Graphs are written in the compact grouped format read by
``paper_2302_00247_b200.graph.load_grouped`` (nodes in the reference's
topological order, so topo rank == list position).

Outputs:
  tests/golden/graphs/<graph>.json.gz   grouped graphs
  tests/golden/cases.json               per-case expectations
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time

REF = "/root/reference/pkg"
sys.path[:0] = [f"{REF}/src", f"{REF}/onnx_ingest/src", REF]
sys.dont_write_bytecode = True

from shardplan import (  # noqa: E402
    ClusterSpec,
    DType,
    ModelGraph,
    OpKind,
    RawNode,
    TensorSpec,
    derive_plan,
    gen_encoder_decoder,
    gen_transformer_stack,
    gen_wide_classifier,
    load_graph,
    prune_graph,
    trim_and_group,
)
from shardplan.search import _eval_range, count_candidates, weight_nodes  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GRAPHS = os.path.join(HERE, "graphs")


# ---------------------------------------------------------------------------
# graph fixtures


def dump_graph(g) -> dict:
    """Compact grouped-graph document (nodes in topo order)."""
    nodes = []
    for name in g.topo_order:
        nd = g.nodes[name]
        w = nd.weight
        a = nd.activation
        nodes.append(
            {
                "s": name,
                "op": nd.op.value,
                "in": list(nd.inputs),
                "a": list(a.shape),
                "ad": a.dtype.label,
                "w": list(w.shape) if w else None,
                "wd": w.dtype.label if w else None,
                "wt": bool(w.trainable) if w else False,
            }
        )
    return {"format": "sp-grouped/1", "nodes": nodes}


def save_graph_fixture(name: str, g) -> str:
    os.makedirs(GRAPHS, exist_ok=True)
    path = os.path.join(GRAPHS, f"{name}.json.gz")
    data = json.dumps(dump_graph(g), separators=(",", ":"), sort_keys=True).encode()
    # mtime=0 keeps the gzip bytes reproducible
    with open(path, "wb") as fh:
        with gzip.GzipFile(fileobj=fh, mode="wb", mtime=0) as gz:
            gz.write(data)
    return f"graphs/{name}.json.gz"


def chain_graph(num_matmuls, dim=4, batch=2, dtype=DType.F64):
    # same construction as the reference fixture (pkg/tests/conftest.py:42-57)
    act = TensorSpec((batch, dim), dtype)
    nodes = [RawNode("input", OpKind.INPUT, (), act)]
    prev = "input"
    for i in range(num_matmuls):
        name = f"blk/m{i}/matmul"
        nodes.append(RawNode(name, OpKind.MATMUL, (prev,), act,
                             TensorSpec((dim, dim), dtype, trainable=True)))
        prev = name
    nodes.append(RawNode("output", OpKind.OUTPUT, (prev,), act))
    return trim_and_group(ModelGraph(nodes))


def weighted_layernorm_graph():
    # divergence trap D1: a weighted layernorm never routes (search.py:344)
    act = TensorSpec((4, 8))
    nodes = [
        RawNode("input", OpKind.INPUT, (), act),
        RawNode("blk/ln/norm", OpKind.LAYERNORM, ("input",), act,
                TensorSpec((8,), trainable=True)),
        RawNode("output", OpKind.OUTPUT, ("blk/ln/norm",), act),
    ]
    return trim_and_group(ModelGraph(nodes))


def zero_weight_graph():
    nodes = [
        RawNode("input", OpKind.INPUT, (), TensorSpec((2, 2))),
        RawNode("output", OpKind.OUTPUT, ("input",), TensorSpec((2, 2))),
    ]
    return trim_and_group(ModelGraph(nodes))


def t5_base_onnx_graph():
    """Config 2: T5-base-structured ONNX built with the reference's wire codec
    (helpers from pkg/tests/test_onnx_ingest.py:27-62), converted by
    onnx_ingest.export_graph (convert.py:272).  RMSNorm scale is a Mul by a
    (d,) initializer and attention products are Mul."""
    from tests.test_onnx_ingest import model, node, tensor, vi
    from onnx_ingest import export_graph

    F = 1
    D, FF, V, B, S, NL = 768, 3072, 32128, 8, 128, 12
    nodes, inits = [], []

    def W(name, dims):
        inits.append(tensor(name, F, dims))
        return name

    def attn(p, x, kv, tag):
        nodes.append(node("MatMul", f"{p}/q/MatMul", [x, W(f"{tag}.q", (D, D))], [f"{tag}.qo"]))
        nodes.append(node("MatMul", f"{p}/k/MatMul", [kv, W(f"{tag}.k", (D, D))], [f"{tag}.ko"]))
        nodes.append(node("MatMul", f"{p}/v/MatMul", [kv, W(f"{tag}.v", (D, D))], [f"{tag}.vo"]))
        nodes.append(node("Mul", f"{p}/scores/Mul", [f"{tag}.qo", f"{tag}.ko"], [f"{tag}.s"]))
        nodes.append(node("Softmax", f"{p}/Softmax", [f"{tag}.s"], [f"{tag}.p"]))
        nodes.append(node("Mul", f"{p}/ctx/Mul", [f"{tag}.p", f"{tag}.vo"], [f"{tag}.c"]))
        nodes.append(node("MatMul", f"{p}/o/MatMul", [f"{tag}.c", W(f"{tag}.o", (D, D))], [f"{tag}.out"]))
        return f"{tag}.out"

    def sub(p, x, tag, body):
        nodes.append(node("Mul", f"{p}/layer_norm/Mul", [x, W(f"{tag}.ln", (D,))], [f"{tag}.n"]))
        y = body(f"{tag}.n")
        nodes.append(node("Add", f"{p}/Add", [x, y], [f"{tag}.r"]))
        return f"{tag}.r"

    def ffn(p, tag):
        def body(x):
            nodes.append(node("MatMul", f"{p}/DenseReluDense/wi/MatMul", [x, W(f"{tag}.wi", (D, FF))], [f"{tag}.h"]))
            nodes.append(node("Relu", f"{p}/DenseReluDense/Relu", [f"{tag}.h"], [f"{tag}.ha"]))
            nodes.append(node("MatMul", f"{p}/DenseReluDense/wo/MatMul", [f"{tag}.ha", W(f"{tag}.wo", (FF, D))], [f"{tag}.f"]))
            return f"{tag}.f"
        return body

    nodes.append(node("Gather", "/shared/Gather", [W("shared", (V, D)), "ids"], ["e"]))
    x = "e"
    for i in range(NL):
        p = f"/encoder/block.{i}"
        x = sub(f"{p}/layer.0", x, f"e{i}l0",
                lambda h, p=p, i=i: attn(f"{p}/layer.0/SelfAttention", h, h, f"e{i}sa"))
        x = sub(f"{p}/layer.1", x, f"e{i}l1", ffn(f"{p}/layer.1", f"e{i}l1"))
    nodes.append(node("Mul", "/encoder/final_layer_norm/Mul", [x, W("enc.fln", (D,))], ["enc_out"]))
    y = "e"
    for i in range(NL):
        p = f"/decoder/block.{i}"
        y = sub(f"{p}/layer.0", y, f"d{i}l0",
                lambda h, p=p, i=i: attn(f"{p}/layer.0/SelfAttention", h, h, f"d{i}sa"))
        y = sub(f"{p}/layer.1", y, f"d{i}l1",
                lambda h, p=p, i=i: attn(f"{p}/layer.1/EncDecAttention", h, "enc_out", f"d{i}ca"))
        y = sub(f"{p}/layer.2", y, f"d{i}l2", ffn(f"{p}/layer.2", f"d{i}l2"))
    nodes.append(node("Mul", "/decoder/final_layer_norm/Mul", [y, W("dec.fln", (D,))], ["dec_n"]))
    nodes.append(node("MatMul", "/lm_head/MatMul", ["dec_n", W("lm_head", (D, V))], ["logits"]))
    data = model(nodes, inits, [vi("ids", F, (B, S))], [vi("logits", F, (B, S, V))])
    doc, _ = export_graph(data)
    return trim_and_group(load_graph(json.dumps(doc)))


# ---------------------------------------------------------------------------
# expectations


def prune_doc(subs) -> list:
    return [
        [s.template_prefix, list(s.template), [[p, list(m)] for p, m in s.instances]]
        for s in subs
    ]


def canon(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def sha(obj) -> str:
    return hashlib.sha256(canon(obj).encode()).hexdigest()


def mesh_doc(mesh: ClusterSpec) -> dict:
    return mesh.to_json()


def table_rows(g, sub, mesh, lo, hi, mu=1 << 20, chunk=4 << 20):
    _, _, _, table = _eval_range((g, sub, mesh, mu, chunk, lo, hi, True))
    return [[row[0], row[2]] for row in table]


def main() -> None:
    t_start = time.perf_counter()
    cases = []
    graph_files = {}

    def graph(name, g):
        if name not in graph_files:
            graph_files[name] = save_graph_fixture(name, g)
        return graph_files[name]

    def plan_case(case, gname, g, mesh, min_dup=2, jobs=8, full_prune=True,
                  tables=(), slices=(), mu=1 << 20, chunk=4 << 20):
        t0 = time.perf_counter()
        entry = {"case": case, "graph": graph(gname, g), "mesh": mesh_doc(mesh),
                 "min_dup": min_dup, "mu": mu, "chunk_size": chunk}
        try:
            subs = prune_graph(g, min_dup)
        except Exception as exc:  # noqa: BLE001 - record the reference's failure
            entry["prune_error"] = f"{type(exc).__name__}: {exc}"
            cases.append(entry)
            return
        entry["prune_sha"] = sha(prune_doc(subs))
        if full_prune:
            entry["prune"] = prune_doc(subs)
        entry["blocks"] = [
            {"prefix": s.template_prefix, "mult": s.multiplicity,
             "T": len(s.template), "V": len(weight_nodes(g, s)),
             "C": count_candidates(g, s)}
            for s in subs
        ]
        try:
            rep = derive_plan(g, mesh, min_duplicates=min_dup, mu=mu,
                              chunk_size=chunk, jobs=jobs)
        except AssertionError as exc:
            entry["derive_error"] = f"AssertionError: {exc}"
            cases.append(entry)
            return
        except Exception as exc:  # noqa: BLE001
            entry["derive_error"] = f"{type(exc).__name__}: {exc}"
            cases.append(entry)
            return
        doc = rep.to_json()
        entry["plan_json"] = canon(doc)
        entry["total_cost"] = repr(rep.total_cost)
        entry["candidates"] = rep.candidates
        entry["valid"] = rep.valid
        entry["best"] = [
            {"prefix": r.subgraph.template_prefix, "index": r.best.plan.index,
             "num_split": r.best.plan.num_split, "total": repr(r.best.cost.total),
             "valid": r.valid, "routing_steps": len(r.best.routings)}
            for r in rep.results
        ]
        def resolve(bi):
            if bi == "max":
                return max(range(len(subs)), key=lambda i: count_candidates(g, subs[i]))
            return bi

        tabs = []
        for bi in map(resolve, tables):
            s = subs[bi]
            C = count_candidates(g, s)
            tabs.append({"block": bi, "lo": 0, "hi": C,
                         "rows": table_rows(g, s, mesh, 0, C, mu, chunk)})
        for bi, width in slices:
            bi = resolve(bi)
            s = subs[bi]
            C = count_candidates(g, s)
            for k in range(8):
                lo = k * C // 8
                hi = min(C, lo + width)
                tabs.append({"block": bi, "lo": lo, "hi": hi,
                             "rows": table_rows(g, s, mesh, lo, hi, mu, chunk)})
        if tabs:
            entry["tables"] = tabs
        entry["ref_seconds"] = round(time.perf_counter() - t0, 3)
        cases.append(entry)
        print(f"  {case}: {entry.get('candidates')} cands, {time.perf_counter() - t0:.2f}s",
              flush=True)

    m12 = ClusterSpec(m=1, n=2)
    m22 = ClusterSpec(m=2, n=2)
    m11 = ClusterSpec(m=1, n=1)
    m18 = ClusterSpec.from_mesh("1x8")
    m24 = ClusterSpec.from_mesh("2x4")
    m24_slow = ClusterSpec(m=2, n=4, inter_bw=2e11 / 32)

    # --- reference-test derived cases (pkg/tests/test_plan_search.py, test_pruning.py,
    #     test_acceptance.py) ---------------------------------------------------------
    tiny = trim_and_group(gen_transformer_stack(2, d_model=8))
    plan_case("tiny_1x2", "tiny_transformer", tiny, m12, tables=["max"])
    plan_case("tiny_2x2", "tiny_transformer", tiny, m22, tables=["max"])
    plan_case("tiny_1x1", "tiny_transformer", tiny, m11)
    plan_case("tiny_min99", "tiny_transformer", tiny, m22, min_dup=99)
    plan_case("tiny_min1_2x2", "tiny_transformer", tiny, m22, min_dup=1, slices=[("max", 256)])
    tiny64 = trim_and_group(gen_transformer_stack(2, d_model=8, dtype=DType.F64))
    plan_case("tiny_f64_2x2", "tiny_transformer_f64", tiny64, m22)
    cls64 = trim_and_group(gen_wide_classifier(64, 16, dtype=DType.F64))
    plan_case("tiny_classifier_1x2", "tiny_classifier_f64", cls64, m12)
    plan_case("tiny_classifier_2x2", "tiny_classifier_f64", cls64, m22)
    for v in range(1, 7):
        plan_case(f"chain{v}_1x2", f"chain{v}", chain_graph(v), m12, min_dup=1,
                  tables=["max"])
    plan_case("chain1_dim6_1x4", "chain1_dim6", chain_graph(1, dim=6), ClusterSpec(m=1, n=4),
              min_dup=1, tables=["max"])
    plan_case("chain2_tie_inf", "chain2", chain_graph(2),
              ClusterSpec(m=1, n=2, intra_bw=float("inf"), setup_latency_s=0.0), min_dup=1,
              tables=["max"])
    plan_case("chain6_2x4_mu", "chain6_d8b8", chain_graph(6, dim=8, batch=8), m24, min_dup=1,
              mu=64, chunk=512, tables=["max"])
    plan_case("weighted_layernorm", "weighted_layernorm", weighted_layernorm_graph(), m12,
              min_dup=1)
    plan_case("zero_weight", "zero_weight", zero_weight_graph(), m12, min_dup=1)
    crit5 = trim_and_group(gen_transformer_stack(4, d_model=512, heads=8, batch=96, seq=16))
    plan_case("crit5_fast", "crit5", crit5, ClusterSpec(m=2, n=8))
    plan_case("crit5_slow", "crit5", crit5, ClusterSpec(m=2, n=8, inter_bw=2e11 / 32))
    for L in (2, 48):
        plan_case(f"bench_L{L}", f"bench_L{L}",
                  trim_and_group(gen_transformer_stack(L, d_model=8, heads=2)), m12)
    plan_case("wide150", "wide150", trim_and_group(gen_wide_classifier(64, 16, blocks=150)), m12)
    plan_case("encdec34", "encdec34", trim_and_group(gen_encoder_decoder(3, 4)), m22)
    plan_case("encdec33_min3", "encdec33", trim_and_group(gen_encoder_decoder(3, 3)), m22,
              min_dup=3)
    tf24 = trim_and_group(gen_transformer_stack(24))
    for k in (2, 5, 8):
        plan_case(f"tf24_min{k}", "tf24", tf24, m12, min_dup=k)

    # --- BASELINE.json configs ----------------------------------------------------------
    c1 = trim_and_group(gen_transformer_stack(12, d_model=768, heads=12))
    plan_case("c1_1x8", "c1", c1, m18, tables=["max"])
    c2 = t5_base_onnx_graph()
    subs2 = prune_graph(c2, 2)
    enc = max((i for i, s in enumerate(subs2) if count_candidates(c2, s) < 10000),
              key=lambda i: count_candidates(c2, subs2[i]))
    dec = max(range(len(subs2)), key=lambda i: count_candidates(c2, subs2[i]))
    plan_case("c2_1x8", "c2_t5", c2, m18, tables=[enc], slices=[(dec, 512)])
    c3 = trim_and_group(gen_wide_classifier(100000, 2048, blocks=16, batch=32))
    plan_case("c3_2x4", "c3", c3, m24)
    plan_case("c3_2x4_slow", "c3", c3, m24_slow)
    c4 = trim_and_group(gen_transformer_stack(48, d_model=6144, heads=48))
    plan_case("c4_1x8", "c4", c4, m18)
    plan_case("c4_2x4", "c4", c4, m24)
    plan_case("c4_2x4_slow", "c4", c4, m24_slow)

    # --- fold stress (config 4 scale-up): only hashes are committed; the graph is
    #     regenerated by paper_2302_00247_b200.workloads.transformer_stack ----------------
    stress = []
    for L in (480, 7000):
        t0 = time.perf_counter()
        g = trim_and_group(gen_transformer_stack(L))
        for md in (2, 3):
            subs = prune_graph(g, md)
            stress.append({"layers": L, "min_dup": md, "nodes": len(g),
                           "graph_sha": sha(dump_graph(g)), "prune_sha": sha(prune_doc(subs)),
                           "blocks": len(subs),
                           "multiplicities": sorted(s.multiplicity for s in subs)})
        print(f"  fold stress L={L}: {len(g)} nodes, {time.perf_counter() - t0:.1f}s", flush=True)

    out = {"generator": "tests/golden/make_golden.py", "reference": "shardplan 0.1.0",
           "cases": cases, "fold_stress": stress}
    with open(os.path.join(HERE, "cases.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"wrote {len(cases)} cases in {time.perf_counter() - t_start:.1f}s")


if __name__ == "__main__":
    main()
