import sys, os, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = tall_grid(n)
L = p.levels or None
for rep in range(int(os.environ.get("REPS", "2"))):
    t0 = time.time()
    g = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    t1 = time.time()
    x, r = g.solve(p.b)
    t2 = time.time()
    print(f"n={n} create {t1-t0:.3f}s solve {t2-t1:.3f}s times {g.times()} iters {r['iterations']} conv {r['converged']} res {r['residual_history'][-1]:.2e}")
    print("nW", g.nW, "nnz_w", g.nnz_w, "batches", g.nbatches, "launches", g.launches, "syncs", g.syncs, "h2d MB", g.h2d_bytes/1e6, "d2h MB", g.d2h_bytes/1e6, "sweep launches", g.sweep_launches)
for s in g.stages():
    print(s['stage'], len(s['front_cols']), "te %.3f ts %.3f tsp %.3f tm %.3f" % (s['t_eliminate'], s['t_scale'], s['t_sparsify'], s['t_merge']))
