"""A/B of the two multi-kernel fold paths on one graph (diagnostic)."""
import json
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
from paper_2302_00247_b200._native import Backend  # noqa: E402
from paper_2302_00247_b200.blocks import to_prune_doc  # noqa: E402
from paper_2302_00247_b200.lowering import lower  # noqa: E402
from paper_2302_00247_b200.search import Session, fold_blocks  # noqa: E402
from paper_2302_00247_b200.workloads import motif_dag  # noqa: E402

be = Backend(0)
g = motif_dag(0, sys.argv[1] if len(sys.argv) > 1 else "parity")
low = lower(g)
ses = Session.open(low, be)
os.environ.pop("SP_FOLD_SORT", None)
a = to_prune_doc(low, fold_blocks(low, 2, session=ses))
os.environ["SP_FOLD_SORT"] = "1"
b = to_prune_doc(low, fold_blocks(low, 2, session=ses))
print("blocks", len(a), len(b), "equal", a == b)
for i, (x, y) in enumerate(zip(a, b)):
    if x != y:
        print("first diff at block", i, "prefix", x[0], y[0], "T", len(x[1]), len(y[1]), "R", len(x[2]), len(y[2]))
        if x[1] != y[1]:
            for t, (p, q) in enumerate(zip(x[1], y[1])):
                if p != q:
                    print("template pos", t, p, q)
                    break
        for j, (p, q) in enumerate(zip(x[2], y[2])):
            if p != q:
                print("instance", j, "prefix", p[0], q[0])
                for t, (u, w) in enumerate(zip(p[1], q[1])):
                    if u != w:
                        print("  member", t, u, w)
                        break
                break
        px, py = [p[0] for p in x[2]], [p[0] for p in y[2]]
        print("only hash:", sorted(set(px) - set(py))[:10], "only sort:", sorted(set(py) - set(px))[:10])
        print("hash order ok:", px == sorted(px), "sort order ok:", py == sorted(py))
        print("hash[20:28]", px[20:28])
        print("sort[20:28]", py[20:28])
        break
