"""BASELINE config 5: front-QR microbenchmark on B200.

Batches of i.i.d. N(0,1) fronts: 4096 x (128x32), 1024 x (512x128), 64 x (4096x1024); per
block Householder QR + Q^T applied to a 256-column neighbour block (one fused call), plus a
truncated CPQR (eps 1e-2) of a 256x256 interface with sigma_i = 0.8^i.  Reports device time
(CUDA events), FP64 TFLOP/s against the measured DMMA peak, and GB/s against measured HBM.
Comparator: torch.geqrf + torch.ormqr (cuSOLVER) on the same batch.
"""
import json
import os
import sys
import time

import numpy as np
import torch
import ctypes as C

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_09878_b200 as P  # noqa: E402

FP64_PEAK = 37.1   # TF/s, tools/fp64_peak (DMMA m8n8k4, B200, this pool)
HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6538.9


def qr_flops(m, n, k):
    return 2 * m * n * n - 2 / 3 * n ** 3 + 4 * m * n * k - 2 * n * n * k


def run_ours(m, n, k, nb, reps=3):
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
    return best


def run_cpqr(B, nb, eps, reps=3):
    """truncated CPQR of nb copies of B on the device (spqr_cpqr_batched_dev), best of reps"""
    L = P.lib()
    m, n = B.shape
    A0 = torch.from_numpy(np.asfortranarray(B).T.copy()).to("cuda").reshape(1, n, m).repeat(nb, 1, 1).contiguous()
    rank = torch.empty(nb, dtype=torch.int32, device="cuda")
    best = 1e30
    for r in range(reps + 1):
        A = A0.clone()
        torch.cuda.synchronize()
        ms = C.c_float()
        rc = L.spqr_cpqr_batched_dev(nb, m, n, C.c_void_p(A.data_ptr()), eps, C.c_void_p(rank.data_ptr()), C.byref(ms))
        assert rc == 0
        if r > 0:
            best = min(best, ms.value)
    rk = rank.cpu().numpy()
    assert (rk == rk[0]).all()
    return rk[0], best


def run_torch(m, n, k, nb, reps=2):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(nb, m, n, dtype=torch.float64, device="cuda", generator=g)
    X = torch.randn(nb, m, k, dtype=torch.float64, device="cuda", generator=g)
    best = 1e30
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a, t = torch.geqrf(A)
        torch.ormqr(a, t, X, left=True, transpose=True)
        e1.record()
        torch.cuda.synchronize()
        if r > 0:
            best = min(best, e0.elapsed_time(e1))
    return best


def main():
    out = {"fp64_peak_tflops": FP64_PEAK, "hbm_gbs": HBM, "shapes": []}
    shapes = [(128, 32, 4096), (512, 128, 1024), (4096, 1024, 64)]
    only = os.environ.get("MB_ONLY")
    if only is not None:
        shapes = [shapes[int(only)]]
    for (m, n, nb) in shapes:
        k = 256
        ms = run_ours(m, n, k, nb)
        fl = qr_flops(m, n, k) * nb
        by = 16.0 * m * (n + k) * nb
        row = {"shape": f"{m}x{n}+{k}", "batch": nb, "ms": round(ms, 3), "TFLOP/s": round(fl / ms / 1e9, 2),
               "frac_fp64": round(fl / ms / 1e9 / FP64_PEAK, 3), "GB/s": round(by / ms / 1e6, 1),
               "frac_hbm": round(by / ms / 1e6 / HBM, 3)}
        try:
            if os.environ.get("MB_NO_TORCH"):
                raise RuntimeError("skipped")
            tm = run_torch(m, n, k, nb)
            row["torch_geqrf_ormqr_ms"] = round(tm, 3)
        except Exception as e:  # comparator only
            row["torch_geqrf_ormqr_ms"] = f"failed: {e}"[:80]
        out["shapes"].append(row)
        print(row, flush=True)
    if os.environ.get("MB_ONLY") is not None:
        return
    # CPQR 256x256, sigma_i = 0.8^i, eps 1e-2: one interface per block of each batch size, device time
    from paper_2102_09878_b200.problems import decaying_interface
    B = decaying_interface(256, 0.8, seed=0)
    m = n = 256
    for nb in (64, 1024, 4096):
        rank, ms = run_cpqr(B, nb, 1e-2)
        r = int(rank)
        fl = sum(4.0 * (m - j) * (n - j - 1) for j in range(r)) + 2.0 * m * n
        by = 8.0 * m * n + 8.0 * r * n  # single-pass ideal: read the block, write R
        row = {"shape": "cpqr 256x256 eps 1e-2", "batch": nb, "rank": r, "ms": round(ms, 3),
               "GFLOP/s": round(fl * nb / ms / 1e6, 1), "GB/s": round(by * nb / ms / 1e6, 1),
               "frac_hbm": round(by * nb / ms / 1e6 / HBM, 4)}
        out.setdefault("cpqr", []).append(row)
        print(row, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
