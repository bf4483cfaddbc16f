"""Subtree-split analysis of a full-size config on the GPU engine: for G = 2, 4,
8 ranks, the share of the factorization's flops each rank would own (load balance of the
subtree partition), the bytes crossing ranks per phase, and per stage.

usage: python tools/subtree_split.py c2|c4 [G ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.parity_dump import problem  # noqa: E402

import paper_2102_09878_b200 as P  # noqa: E402

which = sys.argv[1]
Gs = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
p = problem(which)
base = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
stages = [s["stage"] for s in base.stages()]
front_bytes = None
print(f"{which}: N={p.A.shape[1]} M={p.A.shape[0]} nW={base.nW} nnz(W)={base.nnz_w}")
PH = ["stack rows", "R to holders", "scols holders", "merges"]
for G in Gs:
    g = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords, ranks=G)
    assert (g.nW, g.nnz_w) == (base.nW, base.nnz_w)
    rs = g.rank_stats()
    fl, cr = rs["flops"], rs["cross"]
    tot = fl.sum(axis=0)
    lg = G.bit_length() - 1
    sub = fl[[i for i, s in enumerate(stages[: len(fl)]) if s > lg]].sum(axis=0)
    print(f"\nG={G}: owned flops per rank (whole factorization) {np.array2string(tot / 1e9, precision=2)} GFLOP; "
          f"max/mean {tot.max() / tot.mean():.2f}")
    print(f"  subtree stages (k > {lg}): max/mean {sub.max() / max(sub.mean(), 1):.2f}; "
          f"rank-0 top levels {fl[[i for i, s in enumerate(stages[:len(fl)]) if s <= lg]].sum() / 1e9:.2f} GFLOP")
    print("  cross-rank bytes: " + ", ".join(f"{PH[q]} {cr[:, q].sum() / 1e6:.1f} MB" for q in range(4)) +
          f"; total {cr.sum() / 1e6:.1f} MB (NVLink 5 at 900 GB/s: {cr.sum() / 900e9 * 1e3:.2f} ms)")
    print("  per stage (stage: cross MB | owned GFLOP max/mean):")
    for i in range(len(fl)):
        s = stages[i] if i < len(stages) else "-"
        m = fl[i].mean()
        print(f"    {s}: {cr[i].sum() / 1e6:8.2f} MB | {fl[i].max() / 1e9:7.3f} / {m / 1e9:7.3f}")
