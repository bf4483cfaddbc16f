"""GPU engine vs CPU oracle on the 3D tall problem at reduced size: per-stage interface widths,
nW / nnz(W), CGLS iterations (parity check for the large-front kernels)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
L = int(sys.argv[2]) if len(sys.argv) > 2 else None
p = tall_grid(n, dim=3, seed=0)
kw = dict(eps=p.eps, levels=L or p.levels, coords=p.coords)
t0 = time.time(); g = P.Pipeline(p.A, **kw); tg = time.time() - t0
t0 = time.time(); o = O.Pipeline(p.A, **kw); to = time.time() - t0
xg, rg = g.solve(p.b); xo, ro = o.solve(p.b)
print(f"n={n} L={kw['levels']} gpu {tg:.2f}s oracle {to:.2f}s | nW {g.nW} vs {o.nW} | nnz_w {g.nnz_w} vs {o.nnz_w} | "
      f"iters {rg['iterations']} vs {ro['iterations']}", flush=True)
for a, b in zip(g.stages(), o.stages()):
    fa, fb = np.asarray(a["front_cols"]), np.asarray(b["front_cols"])
    if len(fa) != len(fb) or not np.array_equal(fa, fb):
        d = np.nonzero(fa != fb)[0] if len(fa) == len(fb) else []
        print(f"  stage {a['stage']}: {len(fa)} vs {len(fb)} fronts; differing widths at {list(d[:10])} "
              f"gpu {list(fa[d[:10]]) if len(d) else ''} oracle {list(fb[d[:10]]) if len(d) else ''}")
