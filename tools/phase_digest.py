"""Find the first phase where the GPU engine's state differs from the oracle's (parity
diagnostics).  Both engines write one record per stage-level phase (end of the stage's
eliminations, scale, sparsify_rows, sparsify_cols, merge) with, per live front: cluster, #rows,
#keys and hashes of its row-id list, its (key, width) list and (with *_DIGEST_VALUES=1) its
significance pattern (row-key blocks with squared norm > 1e-20 x the front's largest).

  CPU:  ORC_DIGEST=cpu.bin [ORC_DIGEST_VALUES=1] python tools/phase_digest.py run c4 oracle
  GPU:  SPQR_DIGEST=gpu.bin [SPQR_DIGEST_VALUES=1] python tools/phase_digest.py run c4 gpu
  diff: python tools/phase_digest.py diff cpu.bin gpu.bin
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PHASES = ["eliminated", "scale", "sparsify_rows", "sparsify_cols", "merge"]


def read(path):
    raw = open(path, "rb").read()
    out, o = [], 0
    while o < len(raw):
        ph, st, nf = np.frombuffer(raw, np.int32, 3, o)
        o += 12
        rec = np.frombuffer(raw, np.int32, 3 * nf, o).reshape(nf, 3)
        o += 12 * nf
        hs = np.frombuffer(raw, np.uint64, 3 * nf, o).reshape(nf, 3)
        o += 24 * nf
        out.append((int(ph), int(st), rec, hs))
    return out


def table(rec, hs):
    # fronts with neither rows nor keys carry no state; the engines keep them differently
    keep = (rec[:, 1] > 0) | (rec[:, 2] > 0)
    return {int(c): (int(r), int(k), int(a), int(b), int(v)) for (c, r, k), (a, b, v) in zip(rec[keep], hs[keep])}


def diff(a_path, b_path, limit=12):
    A, B = read(a_path), read(b_path)
    ia = {(p, s): (r, h) for p, s, r, h in A}
    for p, s, rec, hs in B:
        if (p, s) not in ia:
            continue
        ta, tb = table(*ia[(p, s)]), table(rec, hs)
        bad = []
        for c in sorted(set(ta) | set(tb)):
            x, y = ta.get(c), tb.get(c)
            if x is None or y is None:
                bad.append((c, "only cpu" if y is None else "only gpu", x, y))
                continue
            what = [n for n, i in (("nrows", 0), ("nkeys", 1), ("rows", 2), ("keys", 3), ("values", 4)) if x[i] != y[i]]
            if what:
                bad.append((c, ",".join(what), x[:2], y[:2]))
        tag = f"stage {s:2d} {PHASES[p]:14s}"
        if bad:
            print(f"{tag} {len(bad)} of {len(tb)} fronts differ")
            for c, w, x, y in bad[:limit]:
                print(f"    cluster {c}: {w}  cpu {x}  gpu {y}")
            return s, p, [c for c, *_ in bad]
        print(f"{tag} {len(tb)} fronts identical")
    print("no differing phase")
    return None


def run(which, side):
    from tools.parity_dump import problem
    p = problem(which)
    if side == "oracle":
        import oracle as O
        pipe = O.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    else:
        import paper_2102_09878_b200 as P
        pipe = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    print(side, "nW", pipe.nW, "nnz_w", pipe.nnz_w)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3])
    else:
        diff(sys.argv[2], sys.argv[3])
