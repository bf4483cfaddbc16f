"""k_qr_wy phase profile (SPQR_WY_PROF=1): 128x32+256 fronts at several batch sizes
(148 = one CTA per SM: uncontended latencies)."""
import sys, os, ctypes as C, torch
sys.path.insert(0, os.getcwd())
import paper_2102_09878_b200 as P
L = P.lib()
for nb in [int(a) for a in sys.argv[1:]] or [148, 4096]:
    m, n, k = 128, 32, 256
    ntot = n + k
    A0 = torch.randn(nb, ntot, m, dtype=torch.float64, device="cuda")
    tau = torch.empty(nb, n, dtype=torch.float64, device="cuda"); sg = torch.empty_like(tau)
    info = torch.empty(nb, dtype=torch.int32, device="cuda")
    best = 1e9
    for r in range(3):
        A = A0.clone(); torch.cuda.synchronize(); ms = C.c_float()
        L.spqr_qr_apply_batched_dev(nb, m, n, ntot, C.c_void_p(A.data_ptr()), C.c_void_p(tau.data_ptr()), C.c_void_p(sg.data_ptr()), C.c_void_p(info.data_ptr()), C.byref(ms))
        if r: best = min(best, ms.value)
    print(m, n, k, nb, f"{best:.3f} ms", flush=True)
