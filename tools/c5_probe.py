"""C5 front-QR probe: device ms / TFLOP/s of spqr_qr_apply_batched_dev for given shapes
(m n k batch ...), best of 5; run under different SPQR_* environment settings to compare paths."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_09878_b200 as P  # noqa: E402


def run(m, n, k, nb, reps=5):
    L = P.lib()
    ntot = n + k
    g = torch.Generator(device="cuda").manual_seed(0)
    A0 = torch.randn(nb, ntot, m, dtype=torch.float64, device="cuda", generator=g)
    tau = torch.empty(nb, n, dtype=torch.float64, device="cuda")
    sg = torch.empty(nb, n, dtype=torch.float64, device="cuda")
    info = torch.empty(nb, dtype=torch.int32, device="cuda")
    best = 1e30
    for r in range(reps + 1):
        A = A0.clone()
        torch.cuda.synchronize()
        ms = C.c_float()
        rc = L.spqr_qr_apply_batched_dev(nb, m, n, ntot, C.c_void_p(A.data_ptr()), C.c_void_p(tau.data_ptr()),
                                         C.c_void_p(sg.data_ptr()), C.c_void_p(info.data_ptr()), C.byref(ms))
        assert rc == 0
        if r > 0:
            best = min(best, ms.value)
    fl = (2 * m * n * n - 2 / 3 * n ** 3 + 4 * m * n * k - 2 * n * n * k) * nb
    return best, fl / best / 1e9


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    tag = os.environ.get("TAG", "")
    for i in range(0, len(a), 4):
        m, n, k, nb = a[i:i + 4]
        ms, tf = run(m, n, k, nb)
        print(f"{tag:24s} {m}x{n}+{k} x{nb}: {ms:8.3f} ms {tf:7.2f} TF/s {tf / 37.1 * 100:5.1f}%", flush=True)
