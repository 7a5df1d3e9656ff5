"""Per-block scoring results of the c5 throughput tables in walk mode at
SP_FLOW_SPLIT=1 vs the default split, whole and in 2 / 8 shards."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_2302_00247_b200._native import Backend
from paper_2302_00247_b200.api_types import ClusterSpec
from paper_2302_00247_b200.dist import merge_scores
from paper_2302_00247_b200.lowering import lower
from paper_2302_00247_b200.search import Session, fold_blocks
from paper_2302_00247_b200.workloads import motif_dag

be = Backend(0)
low = lower(motif_dag(0, "throughput"))
ses = Session.open(low, be)
ba = fold_blocks(low, 2, session=ses)
off, nodes = ba.templates_csr()
t = be.tables(ses.dgraph, off, nodes, ClusterSpec.from_mesh("1x8"), 1 << 20, 4 << 20)
be.set_mode("walk")
k = lambda rs: [(r.candidates, r.valid, r.has_best, r.best_index, r.best_total, r.best_num_split) for r in rs]
os.environ["SP_FLOW_SPLIT"] = "1"
ref = k(be.score(t))
for split in ("1", "4"):
    os.environ["SP_FLOW_SPLIT"] = split
    for n in (1, 2, 8):
        got = k(merge_scores([be.score(t, s, n) for s in range(n)]) if n > 1 else be.score(t))
        bad = [b for b in range(len(ref)) if got[b] != ref[b]]
        print("split", split, "n", n, "bad blocks", len(bad), [(b, ref[b], got[b]) for b in bad[:3]], flush=True)
t.close()
