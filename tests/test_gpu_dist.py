"""The distributed factorization (spqr_pipeline_create_dist): 2 and 4 processes,
each with its own CUDA context (here all on GPU 0 — no kernel of one rank waits on another;
the ranks exchange over a gloo group on the host), each holding and eliminating its own
subtree through the stages before the first scale_all, the top-separator fronts re-merged on
every rank after each stage; rank 0 receives the other subtrees and finishes.  Rank 0's factorization must be
the single-process one: same ordering, W factor count, nnz(W), pivot / dropped / trailing rows,
every stage's widths, the same W sweeps and the same CGLS solve."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys, json
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid, knn_geometric
dist.init_process_group("gloo", init_method="env://")
rank, ws = dist.get_rank(), dist.get_world_size()
cases = {"grid64": lambda: tall_grid(64), "knn": lambda: knn_geometric(8192, seed=2, levels=8),
         "grid3d": lambda: tall_grid(20, dim=3, seed=1), "c2": lambda: tall_grid(512),
         "c3": lambda: tall_grid(48, dim=3, seed=0), "c4": lambda: knn_geometric(1 << 20, seed=0, levels=16)}
if os.environ["CASE"].startswith("sing"):  # singular leaf fronts (test_gpu_pipeline's matrices)
    import scipy.sparse as sp
    case = os.environ["CASE"]
    if case in ("singA", "singB"):  # one row couples the two columns of one leaf: "rows couple"
        D = np.zeros((9, 6))
        D[0, 0], D[0, 1] = 1.0, 2.0
        for j in range(2, 6):
            D[2 * j - 3, j] = 3.0
            D[2 * j - 2, j] = 0.5
        parts = [0, 0, 1, 1, 1, 1] if case == "singA" else [1, 1, 0, 0, 0, 0]
    else:  # a leaf whose stack QR meets an exactly zero pivot
        D = np.zeros((11, 7))
        D[0, 0], D[0, 1], D[1, 2], D[2, 2] = 1.5, -2.25, 2.0, 0.5
        for j in range(3, 7):
            D[2 * j - 3, j] = 3.0
            D[2 * j - 2, j] = -0.75
        parts = [0, 0, 0, 1, 1, 1, 1]
    A = sp.csc_matrix(D)
    kw = dict(eps=0.0, levels=1, parts=parts)
    try:
        P.Pipeline(A, dist_group=dist.group.WORLD, **kw)
        got = None
    except P.SingularFrontError as e:
        got = (e.cluster, str(e))
    if rank == 0:
        try:
            P.Pipeline(A, **kw)
            want = None
        except P.SingularFrontError as e:
            want = (e.cluster, str(e))
        assert want is not None and got == want, (got, want)
    dist.barrier()
    print(json.dumps({"rank": rank, "error": got}))
    dist.destroy_process_group()
    sys.exit(0)
p = cases[os.environ["CASE"]]()
kw = dict(eps=p.eps, levels=p.levels, coords=p.coords)
g = P.Pipeline(p.A, dist_group=dist.group.WORLD, **kw)
out = {"rank": rank, "root": bool(g.is_root), "bytes": g.dist_bytes}
if rank == 0:
    ref = P.Pipeline(p.A, **kw)
    assert (g.nW, g.nnz_w, g.ndropped, g.ntrailing) == (ref.nW, ref.nnz_w, ref.ndropped, ref.ntrailing), \
        ((g.nW, g.nnz_w, g.ndropped, g.ntrailing), (ref.nW, ref.nnz_w, ref.ndropped, ref.ntrailing))
    assert np.array_equal(g.perm(), ref.perm())
    a, b = g.rows(), ref.rows()
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(np.sort(a[1]), np.sort(b[1])) and np.array_equal(np.sort(a[2]), np.sort(b[2]))
    for s1, s2 in zip(g.stages(), ref.stages()):
        assert np.array_equal(s1["front_cols"], s2["front_cols"]), s1["stage"]
    z = np.random.default_rng(0).standard_normal(g.N)
    for f in ("w_solve", "wt_solve"):
        d = np.linalg.norm(getattr(g, f)(z) - getattr(ref, f)(z)) / np.linalg.norm(getattr(ref, f)(z))
        assert d <= 1e-12, (f, d)
        out[f] = d
    x1, r1 = g.solve(p.b)
    x2, r2 = ref.solve(p.b)
    assert r1["iterations"] == r2["iterations"]
    assert abs(r1["residual_history"][-1] - r2["residual_history"][-1]) <= 1e-10
    out["iters"] = r1["iterations"]
else:
    assert not g.is_root
    try:
        g.solve(p.b)
        raise AssertionError("a non-root rank solved")
    except RuntimeError:
        pass
dist.barrier()
print(json.dumps(out))
dist.destroy_process_group()
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(ws, case, timeout):
    port = _free_port()
    procs = []
    for r in range(ws):
        env = dict(os.environ, ROOT=ROOT, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(ws), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CASE=case)
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=timeout) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, (o[-2000:], e[-4000:])
    return [o.strip().splitlines()[-1] for o, _ in outs]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("ws", [2, 4])
@pytest.mark.parametrize("case", ["grid64", "knn", "grid3d"])
def test_distributed_factorization_matches_single_process(ws, case):
    print(_run(ws, case, 550))


@pytest.mark.timeout(900)
def test_distributed_c2_full_size():
    """BASELINE config 2 at full size across 2 ranks: identical to the single-process run."""
    print(_run(2, "c2", 850))


@pytest.mark.timeout(1500)
@pytest.mark.parametrize("case,ws", [("c3", 4), ("c4", 2)])
def test_distributed_full_size_3d_and_knn(case, ws):
    """BASELINE configs 3 (4 ranks) and 4 (2 ranks) at full size: identical to the single-process run."""
    print(_run(ws, case, 1400))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case", ["singA", "singB", "singP"])
def test_distributed_singular_front_error(case):
    """A singular leaf on rank 0's side (singA, singP) or on rank 1's (singB): rank 0 raises the
    SingularFrontError — cluster and reason — the single-process factorization raises."""
    print(_run(2, case, 280))
