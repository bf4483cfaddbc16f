"""C2 factorization wall time vs host thread count (median of REPS after one warm-up)."""
import os, subprocess, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, time
sys.path.insert(0, %r)
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid
p = tall_grid(512)
ts = []
for rep in range(int(os.environ.get("REPS", "4")) + 1):
    g = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    if rep: ts.append(g.times()["factorize_event_ms"] / 1e3)
    del g
print(" ".join(f"{t:.3f}" for t in ts))
''' % ROOT
print("cpus", os.cpu_count(), flush=True)
for nt in sys.argv[1:]:
    env = dict(os.environ, OMP_NUM_THREADS=nt)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip()
    ts = [float(x) for x in out.split()] if out else []
    print(f"threads {nt:>3s}: median {statistics.median(ts):.3f} s  all {out}", flush=True)
