"""Build the C2 factorization several times in one process and print nW / nnz_w / iterations
(a data race shows up as run-to-run differences)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = tall_grid(n)
for rep in range(int(os.environ.get("REPS", "3"))):
    g = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    x, r = g.solve(p.b)
    print(f"rep {rep} nW {g.nW} nnz_w {g.nnz_w} iters {r['iterations']}", flush=True)
