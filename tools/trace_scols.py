"""Diagnostics: run GPU and oracle on a kNN instance with sparsify_cols traced, report the
interfaces whose ranks differ (SPQR_TRACE_SCOLS in both engines)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
dump = sys.argv[2] if len(sys.argv) > 2 else None
out = os.environ.get("OUT", "gpurun_out")
for k in ("gpu", "orc"):
    for ext in ("", ".G", ".R"):
        try:
            os.remove(f"{out}/trace_{k}.txt{ext}")
        except OSError:
            pass
from paper_2102_09878_b200.problems import knn_geometric
p = knn_geometric(N, seed=0, levels=int(np.log2(N)) - 4)
kw = dict(eps=p.eps, levels=p.levels, coords=p.coords)
os.environ["SPQR_TRACE_SCOLS"] = f"{out}/trace_gpu.txt" + (f":{dump}" if dump else "")
import paper_2102_09878_b200 as P
g = P.Pipeline(p.A, **kw)
os.environ["SPQR_TRACE_SCOLS"] = f"{out}/trace_orc.txt" + (f":{dump}" if dump else "")
import oracle as O
o = O.Pipeline(p.A, **kw)
def load(f):
    d, order = {}, []
    for line in open(f):
        t = line.split()
        if t[0] == "S":
            continue
        if t[0] == "m":  # row move: m <cluster> row <row> tgt <front>
            key, val = ("m", int(t[1]), int(t[3])), (int(t[5]),)
        elif t[0] == "e":  # elimination: e <cluster> rows <n> tcols <n> 0
            key, val = ("e", int(t[1])), (int(t[3]), int(t[5]))
        else:  # r / p: <kind> <cluster> a <n> b <n> c <n>
            key, val = (t[0], int(t[1])), (int(t[3]), int(t[5]), int(t[7]))
        d.setdefault(key, []).append(val)
        order.append(key)
    return d, order
(a, oa), (b, ob) = load(f"{out}/trace_gpu.txt"), load(f"{out}/trace_orc.txt")
diff = [k for k in ob if a.get(k) != b.get(k)]
print("records", len(a), len(b), "differing", len(set(diff)))
print("first differences in the oracle's order (e = elimination rows/cols, m = row move target,\n"
      "r = sparsify_rows p2/nw/keep, p = sparsify_cols cs/nG/rank):")
seen = set()
for k in diff:
    if k in seen:
        continue
    seen.add(k)
    print(" ", k, "gpu", a.get(k), "oracle", b.get(k))
    if len(seen) >= 10:
        break
