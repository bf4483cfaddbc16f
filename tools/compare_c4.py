"""BASELINE config 4 at full size: GPU engine vs CPU oracle, per-stage interface widths."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import knn_geometric
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
p = knn_geometric(N, seed=0, levels=int(np.log2(N)) - 4)
kw = dict(eps=p.eps, levels=p.levels, coords=p.coords)
t0 = time.time(); g = P.Pipeline(p.A, **kw); tg = time.time() - t0
t0 = time.time(); o = O.Pipeline(p.A, **kw); to = time.time() - t0
print(f"N={N} gpu {tg:.1f}s oracle {to:.1f}s | nW {g.nW} vs {o.nW} | nnz_w {g.nnz_w} vs {o.nnz_w}", flush=True)
print("perm equal", np.array_equal(g.perm(), o.perm()), "owner equal", np.array_equal(g.owner(), o.owner()))
for a, b in zip(g.stages(), o.stages()):
    fa, fb = np.asarray(a["front_cols"]), np.asarray(b["front_cols"])
    if len(fa) != len(fb):
        print(f"  stage {a['stage']}: {len(fa)} vs {len(fb)} interfaces"); continue
    d = np.nonzero(fa != fb)[0]
    if len(d):
        print(f"  stage {a['stage']}: {len(d)} of {len(fa)} widths differ; gpu-oracle {np.unique(fa[d] - fb[d], return_counts=True)}")
