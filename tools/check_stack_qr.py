"""Diagnostics: the dumped elimination stack through the GPU batched QR vs the oracle."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2102_09878_b200 as P
def load(f):
    b = open(f, 'rb').read(); m, n, cs = np.frombuffer(b[:12], np.int32)
    return np.frombuffer(b[12:], np.float64).reshape(n, m).T.copy(), int(cs)
S, cs = load(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/stack_gpu.bin')
V, t, s, R = O.householder_qr(S[:, :cs])
X = O.apply_reflectors(V, t, s, S[:, cs:], "left_t")
for path in ("auto", "smem", "blocked", "tile_dmma"):
    os.environ.pop("SPQR_QR_PATH", None); os.environ.pop("SPQR_TILE_DMMA", None)
    if path == "tile_dmma": os.environ["SPQR_TILE_DMMA"] = "1"
    elif path != "auto": os.environ["SPQR_QR_PATH"] = path
    out, tau, sg, info = P.qr_apply_batched(S[None].copy(), cs)
    G = out[0]
    print(path, "R err", np.abs(np.triu(G[:cs, :cs]) - R).max(), "trailing err", np.abs(G[:, cs:] - X).max(),
          "rows>=cs err", np.abs(G[cs:, cs:] - X[cs:]).max())
os.environ.pop("SPQR_QR_PATH", None); os.environ.pop("SPQR_TILE_DMMA", None)
out, tau, sg, info = P.qr_apply_batched(S[None].copy(), cs)
G = out[0]
np.set_printoptions(precision=4, suppress=True, linewidth=150)
d = np.abs(G[:, cs:] - X).max(axis=1)
print("per-row max diff:", d)
print("gpu tau", tau[0]); print("orc tau", t)
print("gpu row 21", G[21, cs:]); print("orc row 21", X[21])
print("col tails:", [float((S[k+1:, k]**2).sum()) for k in range(cs)])
