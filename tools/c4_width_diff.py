"""Locate the interfaces whose sparsify_cols rank differs between the GPU engine and a CPU
fingerprint (tools/parity_dump.py), dump their G (SPQR_DUMP_G) from the GPU engine, and
report the truncated-CPQR stop margins on it: for each differing interface, the GPU and oracle
ranks on the same G, the pivot norm at the cut relative to eps*|R11| and the singular values
of G around eps*sigma_1.

usage: python tools/c4_width_diff.py c4 tests/golden/c4_oracle_fingerprint.npz
"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.parity_dump import problem  # noqa: E402

which, path = sys.argv[1], sys.argv[2]
ref = np.load(path)
import paper_2102_09878_b200 as P  # noqa: E402

p = problem(which)
views = {}


os.environ["SPQR_OBSERVE_STRUCTURE_ONLY"] = "1"  # structure only: no block downloads per phase


def obs(ph, st, de, v):
    if ph == "sparsify_cols":
        views[st] = [c for c in sorted(v["fronts"]) if len(v["cols"][c]) > 0]


g = P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords, observer=obs)
targets = []
for s in g.stages():
    k = f"stage_{s['stage']}"
    w = np.asarray(s["front_cols"])
    if k in ref and len(ref[k]) == len(w):
        d = np.nonzero(ref[k] != w)[0]
        if len(d):
            print(k, "differs at", d[:5], "gpu", w[d[:5]], "cpu", ref[k][d[:5]])
            targets.append((s["stage"], int(d[0])))
del g
for st, idx in targets[:1]:
    # the interface with that position among the stage's nonzero-width fronts at snapshot
    # time (after sparsify_cols, as StageStats.front_cols)
    cand = views[st]
    print("stage", st, "candidate clusters near index", cand[max(0, idx - 2): idx + 3])
    c = cand[idx]
    out = f"gpurun_out/G_{st}_{c}.bin"
    env = dict(os.environ, SPQR_DUMP_G=f"{st}:{c}:{out}")
    env.pop("SPQR_OBSERVE_STRUCTURE_ONLY", None)
    subprocess.run([sys.executable, "-c", f"""
import sys; sys.path.insert(0, '.')
from tools.parity_dump import problem
import paper_2102_09878_b200 as P
p = problem('{which}')
P.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
"""], env=env, check=True)
    raw = open(out, "rb").read()
    cs, nG = np.frombuffer(raw[:8], np.int32)
    G = np.frombuffer(raw[8:], np.float64).reshape(nG, cs).T.copy()
    import oracle as O
    og = O.cpqr(G, p.eps)
    gg = P.cpqr_batched(G[None], p.eps)[0]
    sv = np.linalg.svd(G, compute_uv=False)
    r11 = abs(og["r11"])
    print(f"cluster {c}: G {cs}x{nG}; rank oracle {og['rank']} gpu {gg['rank']}; r11 {r11:.6e}")
    Rd = np.abs(np.diag(og["R"][:, og["perm"]])) if og["rank"] else np.zeros(0)
    print("  |R_kk| / (eps r11) for the kept pivots (last 3):", (Rd[-3:] / (p.eps * r11)))
    rel = sv / sv[0]
    near = np.argsort(np.abs(rel - p.eps))[:3]
    print("  singular values / sigma_1 nearest eps:", [(int(i), float(rel[i])) for i in sorted(near)],
          " relative distance to eps:", [float(abs(rel[i] - p.eps) / p.eps) for i in sorted(near)])
