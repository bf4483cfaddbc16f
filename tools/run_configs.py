"""Run BASELINE configs 3 and 4 at full size on the GPU (and the oracle on C3)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid, knn_geometric

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
if which == "c3":
    p = tall_grid(48, dim=3, seed=0)
else:
    p = knn_geometric(1 << 20, seed=0, levels=16)
print(p.name, p.A.shape, p.A.nnz, "levels", p.levels, "eps", p.eps, flush=True)
t0 = time.time()
g = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
t1 = time.time()
x, r = g.solve(p.b)
t = g.times()
print(f"GPU create {t1-t0:.2f}s (partition {t['t_partition']:.2f}s factor {t['t_factorize']:.2f}s) solve {r['t_solve']:.3f}s "
      f"iters {r['iterations']} conv {r['converged']} res {r['residual_history'][-1]:.2e} nW {g.nW} nnz_w {g.nnz_w}", flush=True)
ks = g.kernel_stats()
print("kernels", {k: (round(v["ms"], 1) if isinstance(v, dict) else v) for k, v in ks.items()} if isinstance(ks, dict) else ks)
st = g.stages()
print("top cols per stage", [s['top_cols'] for s in st])
if which == "c3" and os.environ.get("ORACLE"):
    import oracle as O
    t0 = time.time()
    o = O.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    xo, ro = o.solve(p.b)
    tt = o.times()
    print(f"oracle factor {tt['t_factorize']:.2f}s solve {ro['t_solve']:.2f}s iters {ro['iterations']} res {ro['residual_history'][-1]:.2e} nW {o.nW} nnz_w {o.nnz_w}")
