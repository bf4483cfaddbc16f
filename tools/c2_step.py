"""One bench step of the headline workload (BASELINE config 2, C2): spaQR factorization +
preconditioned CGLS solve through the public API, for ncu launch lists
(tools/ncu_traffic.py).  WARM=<k> runs k unprofiled-in-spirit warm-up steps first (use
ncu --launch-skip to skip them)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_09878_b200 as P  # noqa: E402
from paper_2102_09878_b200.problems import tall_grid  # noqa: E402

p = tall_grid(int(os.environ.get("N", "512")))
for _ in range(int(os.environ.get("WARM", "0")) + 1):
    g = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    x, rep = g.solve(p.b)
t = g.times()
print(f"launches factorize {g.launches} solve {t['solve_launches']} iters {rep['iterations']} "
      f"factorize_event_ms {t['factorize_event_ms']:.1f} solve_event_ms {t['solve_event_ms']:.2f}")
