"""c5 walk: per-block results merged over N simulated-rank shares (score(t, s, n))
equal the whole search, with the root relief (incl. the largest block's
relieved tail) at several settings."""
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
ref = k(be.score(t))
for relief in ("10", "20", "60"):
    os.environ["SP_ROOT_RELIEF"] = relief
    for n in (4, 8):
        got = k(merge_scores([be.score(t, s, n) for s in range(n)]))
        bad = [b for b in range(len(ref)) if got[b] != ref[b]]
        print("relief", relief, "n", n, "bad", len(bad), bad[:3], flush=True)
t.close()
