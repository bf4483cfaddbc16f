"""One C5 front-QR shape timed in this process (env switches are read once per process):
python tools/c5_one.py <shape index 0..2> [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import microbench as mb  # noqa: E402

SHAPES = [(128, 32, 256, 4096), (512, 128, 256, 1024), (4096, 1024, 256, 64)]
m, n, k, nb = SHAPES[int(sys.argv[1])]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ms = mb.run_ours(m, n, k, nb, reps=reps)
tf = mb.qr_flops(m, n, k) * nb / ms / 1e9
env = {k_: v for k_, v in os.environ.items() if k_.startswith("SPQR_")}
print(f"{m}x{n}+{k} x{nb}  {env}  {ms:.3f} ms  {tf:.2f} TF/s  {100 * tf / mb.FP64_PEAK:.1f} %", flush=True)
