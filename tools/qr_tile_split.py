import sys, os, ctypes as C, torch
sys.path.insert(0, os.getcwd())
import paper_2102_09878_b200 as P
L = P.lib()
for (m, n, k, nb) in [(128, 32, 0, 4096), (128, 32, 64, 4096), (128, 32, 128, 4096), (128, 32, 256, 4096)]:
    ntot = n + k
    A0 = torch.randn(nb, ntot, m, dtype=torch.float64, device="cuda")
    tau = torch.empty(nb, n, dtype=torch.float64, device="cuda"); sg = torch.empty_like(tau)
    info = torch.empty(nb, dtype=torch.int32, device="cuda")
    best = 1e9
    for r in range(4):
        A = A0.clone(); torch.cuda.synchronize(); ms = C.c_float()
        L.spqr_qr_apply_batched_dev(nb, m, n, ntot, C.c_void_p(A.data_ptr()), C.c_void_p(tau.data_ptr()), C.c_void_p(sg.data_ptr()), C.c_void_p(info.data_ptr()), C.byref(ms))
        if r: best = min(best, ms.value)
    print(m, n, k, nb, f"{best:.3f} ms")
