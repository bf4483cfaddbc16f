"""Structure fingerprint of a full-size BASELINE config, for parity at sizes where the CPU
checker runs for minutes to an hour: run the oracle (or the reference, oracle/_ref) HERE on
the CPU and save the fingerprint; tools/parity_check.py recomputes it with the GPU pipeline on
the box and compares.  Fingerprint: nW, nnz(W), CGLS iterations / final residual, sha256 of
perm, row owner, pivot rows, sorted dropped and trailing rows, and every stage's interface
widths (saved in full).

usage: python tools/parity_dump.py c3|c4|c2 [oracle|ref] out.npz
"""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_09878_b200.problems import knn_geometric, tall_grid  # noqa: E402


def problem(which):
    if which == "c2":
        return tall_grid(512)
    if which == "c3":
        return tall_grid(48, dim=3, seed=0)
    if which == "c4":
        return knn_geometric(1 << 20, seed=0, levels=16)
    if which.startswith("knn"):
        n = int(which[3:])
        return knn_geometric(n, seed=0, levels=int(np.log2(n)) - 4)
    raise ValueError(which)


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def fingerprint(P, p):
    t0 = time.time()
    pipe = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    t1 = time.time()
    x, rep = pipe.solve(p.b)
    A = p.A
    rel = float(np.linalg.norm(A.T @ (p.b - A @ x)) / np.linalg.norm(A.T @ p.b))
    pr, dr, tr = pipe.rows()
    st = pipe.stages()
    fp = dict(nW=pipe.nW, nnz_w=pipe.nnz_w, iterations=rep["iterations"], rel_residual=rel,
              perm=h(pipe.perm()), owner=h(pipe.owner()), pivot_row=h(pr), dropped=h(np.sort(dr)),
              trailing=h(np.sort(tr)), t_factorize=t1 - t0)
    widths = {f"stage_{s['stage']}": np.asarray(s["front_cols"], np.int32) for s in st}
    return fp, widths


if __name__ == "__main__":
    which, impl, out = sys.argv[1], sys.argv[2], sys.argv[3]
    if impl == "ref":
        from oracle import ref as M
    else:
        import oracle as M
    p = problem(which)
    fp, widths = fingerprint(M, p)
    print(which, impl, fp, flush=True)
    np.savez_compressed(out, **{k: np.array(v) for k, v in fp.items()}, **widths)
