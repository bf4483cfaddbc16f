"""GPU side of tools/parity_dump.py: run the GPU pipeline on the same config and compare with a
saved CPU fingerprint.  Prints one line per item and 'PARITY OK' / 'PARITY DIFF'.

usage: python tools/parity_check.py c3|c4|c2 cpu_fingerprint.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.parity_dump import fingerprint, problem  # noqa: E402

if __name__ == "__main__":
    import paper_2102_09878_b200 as P
    which, path = sys.argv[1], sys.argv[2]
    ref = np.load(path)
    p = problem(which)
    fp, widths = fingerprint(P, p)
    ok = True
    for k in ("nW", "nnz_w", "perm", "owner", "pivot_row", "dropped", "trailing"):
        same = str(fp[k]) == str(ref[k])
        ok &= same
        print(f"{k:10s} {'same' if same else 'DIFF'}  gpu {fp[k]}  cpu {ref[k]}")
    it_ok = abs(int(fp["iterations"]) - int(ref["iterations"])) <= 1
    res_ok = abs(float(fp["rel_residual"]) - float(ref["rel_residual"])) <= 1e-10
    ok &= it_ok and res_ok
    print(f"iterations {fp['iterations']} vs {int(ref['iterations'])}; rel residual {fp['rel_residual']:.3e} vs "
          f"{float(ref['rel_residual']):.3e}")
    nd = 0
    for k, w in widths.items():
        r = ref[k] if k in ref else None
        if r is None or len(r) != len(w) or not np.array_equal(r, w):
            nd += 1
            if r is not None and len(r) == len(w):
                d = np.nonzero(r != w)[0]
                print(f"  {k}: {len(d)} of {len(w)} widths differ (gpu-cpu {np.unique(w[d] - r[d], return_counts=True)})")
            else:
                print(f"  {k}: {len(w)} vs {None if r is None else len(r)} interfaces")
    ok &= nd == 0
    print(f"stages with identical interface widths: {len(widths) - nd} of {len(widths)}; GPU factor {fp['t_factorize']:.2f} s")
    print("PARITY OK" if ok else "PARITY DIFF")
