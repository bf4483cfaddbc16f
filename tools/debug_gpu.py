import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid, random_full_rank
rng = np.random.default_rng(132)
A = rng.standard_normal((6, 1, 1))
out, tau, sg, info = P.qr_apply_batched(A, 1)
print("qr1x1 in", A.ravel(), "out", out.ravel(), "tau", tau.ravel(), "sign", sg.ravel(), "info", info)
A = rng.standard_normal((2, 3, 2))
out, tau, sg, info = P.qr_apply_batched(A, 2)
print("qr3x2 sign", sg, [O.householder_qr(A[b])[2] for b in range(2)])
cases = []
for eps in (0.0, 1e-2):
    for L in (1, 2, 3):
        cases.append(("rand", random_full_rank(120, 70, 4, seed=3), None, L, eps, 0))
for n, L in ((8, 2), (12, 3), (16, 4), (32, 6)):
    p = tall_grid(n, seed=1)
    for eps in (0.0, 1e-2):
        cases.append((f"grid{n}", p.A, p.coords, L, eps, 1))
for name, A, coords, L, eps, skip in cases:
    try:
        g = P.Pipeline(A, eps=eps, levels=L, skip_levels=skip, coords=coords)
        o = O.Pipeline(A, eps=eps, levels=L, skip_levels=skip, coords=coords)
        so, sgs = o.stages(), g.stages()
        bad = [ (a['stage'], len(a['front_cols']), len(b['front_cols'])) for a, b in zip(so, sgs) if not np.array_equal(a['front_cols'], b['front_cols'])]
        po = o.rows()[0]; pg = g.rows()[0]
        print(name, L, eps, "ok nW", o.nW, g.nW, "nnzw", o.nnz_w, g.nnz_w, "pivots_eq", np.array_equal(po, pg), "stage mismatches", bad[:3])
    except Exception as e:
        print(name, L, eps, "ERROR", type(e).__name__, str(e)[:200])
