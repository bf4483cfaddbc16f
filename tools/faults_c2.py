"""Minor page faults and wall time of C2 factorizations (host allocation behaviour)."""
import os, sys, time, resource
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid
p = tall_grid(512)
for rep in range(int(os.environ.get("REPS", "3"))):
    f0 = resource.getrusage(resource.RUSAGE_SELF).ru_minflt
    t0 = time.time()
    g = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    t1 = time.time()
    f1 = resource.getrusage(resource.RUSAGE_SELF).ru_minflt
    print(f"rep {rep} create {t1 - t0:.3f}s factorize_event {g.times()['factorize_event_ms'] / 1e3:.3f}s minflt {f1 - f0}", flush=True)
    del g
