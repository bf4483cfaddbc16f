"""C5 CPQR leg only: 256x256 interface, sigma_i = 0.8^i, eps 1e-2, per batch size (device time)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.microbench import run_cpqr
from paper_2102_09878_b200.problems import decaying_interface
B = decaying_interface(256, 0.8, seed=0)
for nb in (64, 1024, 4096):
    rank, ms = run_cpqr(B, nb, 1e-2)
    print(os.environ.get("SPQR_CPQR_PATH", "auto"), "batch", nb, "rank", int(rank), f"{ms:.3f} ms", flush=True)
