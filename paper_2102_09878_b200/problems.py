"""Seeded synthetic least-squares problems for the BASELINE.json configs.

The reference's own generator (proj/src/problems.cpp:281-319, inverse Poisson)
is not what BASELINE.json asks for, so these are new.  All problems are FP64,
returned as canonical CSC (scipy.sparse.csc_matrix, sorted indices, no explicit
zeros) together with per-column coordinates (the geometric nested-dissection
input, partition.cpp:26-49) and a right-hand side b ~ N(0,1).

RNG: numpy PCG64 seeded with the documented seed (default 0).  Ambiguities
resolved as SURVEY.md Appendix B proposes: random-row neighbours are distinct
and in-grid; kNN row i < N uses point i (it carries the +2 diagonal boost).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class Problem:
    name: str
    A: sp.csc_matrix        # M x N, canonical CSC
    coords: np.ndarray      # N x dim, float64
    b: np.ndarray           # M
    levels: int
    eps: float

    @property
    def shape(self):
        return self.A.shape


def _canon(rows, cols, vals, m, n) -> sp.csc_matrix:
    A = sp.csc_matrix((vals, (rows, cols)), shape=(m, n))
    A.sum_duplicates()
    A.eliminate_zeros()
    A.sort_indices()
    A.indptr = A.indptr.astype(np.int32)
    A.indices = A.indices.astype(np.int32)
    return A


def _pick_neighbours(rng, cells, dims, k):
    """k distinct in-grid face neighbours of each cell (random order)."""
    d = len(dims)
    coord = np.stack(np.unravel_index(cells, dims), axis=1)
    offs = []
    for a in range(d):
        for s in (-1, 1):
            o = np.zeros(d, dtype=np.int64)
            o[a] = s
            offs.append(o)
    offs = np.array(offs)                                     # 2d x d
    nb = coord[:, None, :] + offs[None, :, :]                 # c x 2d x d
    ok = np.all((nb >= 0) & (nb < np.array(dims)), axis=2)    # c x 2d
    key = rng.random(ok.shape)
    key[~ok] = np.inf
    order = np.argsort(key, axis=1)[:, :k]
    sel = np.take_along_axis(nb, order[:, :, None], axis=1)   # c x k x d
    flat = np.ravel_multi_index(tuple(sel[:, :, a] for a in range(d)), dims)
    return flat


def tall_grid(n: int, dim: int = 2, seed: int = 0, levels: int | None = None,
              eps: float | None = None) -> Problem:
    """2D (dim=2, 5-point, M=2N) or 3D (dim=3, 7-point, M=3N) tall problem."""
    rng = np.random.default_rng(seed)
    dims = (n,) * dim
    N = n ** dim
    cells = np.arange(N, dtype=np.int64)
    coord = np.stack(np.unravel_index(cells, dims), axis=1)
    rows, cols, vals = [cells], [cells], [2.0 * dim + rng.random(N)]
    for a in range(dim):
        for s in (-1, 1):
            nb = coord.copy()
            nb[:, a] += s
            ok = (nb[:, a] >= 0) & (nb[:, a] < n)
            j = np.ravel_multi_index(tuple(nb[ok].T), dims)
            rows.append(cells[ok])
            cols.append(j)
            vals.append(-1.0 + 0.1 * rng.standard_normal(int(ok.sum())))
    extra = (dim - 1) * N       # 2D: N extra rows of 3 nnz; 3D: 2N rows of 4 nnz
    k = dim                     # neighbours per extra row
    rc = rng.integers(0, N, size=extra)
    nbs = _pick_neighbours(rng, rc, dims, k)
    rid = N + np.arange(extra, dtype=np.int64)
    rows.append(rid)
    cols.append(rc)
    vals.append(rng.standard_normal(extra))
    for t in range(k):
        rows.append(rid)
        cols.append(nbs[:, t])
        vals.append(rng.standard_normal(extra))
    M = N + extra
    A = _canon(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), M, N)
    b = rng.standard_normal(M)
    if levels is None:
        levels = {64: 8, 512: 14}.get(n, 0) if dim == 2 else {48: 12}.get(n, 0)
    if eps is None:
        eps = 1e-3 if (dim == 2 and n == 64) else 1e-2
    return Problem(f"tall{dim}d_n{n}", A, coord.astype(np.float64), b, levels, eps)


def knn_geometric(N: int, seed: int = 0, levels: int = 16, eps: float = 1e-2) -> Problem:
    """Config 4: N points U[0,1)^2, M = 4N rows of a point and its 4 exact NNs."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    pts = rng.random((N, 2))
    M = 4 * N
    centre = np.concatenate([np.arange(N), rng.integers(0, N, size=M - N)])
    _, nn = cKDTree(pts).query(pts, k=5)
    # nn[:,0] is the point itself (distinct points with probability 1)
    sel = nn[centre]                                    # M x 5
    vals = rng.standard_normal((M, 5))
    vals[:N, 0] += 2.0
    rows = np.repeat(np.arange(M), 5)
    A = _canon(rows, sel.ravel(), vals.ravel(), M, N)
    b = rng.standard_normal(M)
    return Problem(f"knn_N{N}", A, pts, b, levels, eps)


def random_full_rank(m: int, n: int, extra_per_col: int, seed: int) -> sp.csc_matrix:
    """Test helper shaped like test_factorize.cpp:43-50 (structural diagonal 3+U(-1,1))."""
    rng = np.random.default_rng(seed)
    r = [np.arange(n)]
    c = [np.arange(n)]
    v = [3.0 + rng.uniform(-1, 1, n)]
    r.append(rng.integers(0, m, size=n * extra_per_col))
    c.append(np.repeat(np.arange(n), extra_per_col))
    v.append(rng.uniform(-1, 1, n * extra_per_col))
    return _canon(np.concatenate(r), np.concatenate(c), np.concatenate(v), m, n)


def microbench_blocks(m: int, n: int, batch: int, seed: int = 0):
    """Config 5: i.i.d. N(0,1) fronts (batch x m x n, column-major per block)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((batch, n, m)).transpose(0, 2, 1).copy(order="C")


def decaying_interface(n: int = 256, ratio: float = 0.8, seed: int = 0) -> np.ndarray:
    """Config 5 CPQR block: U diag(ratio^i) V^T with Haar U, V (QR of Gaussians)."""
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = ratio ** np.arange(n)
    return np.asfortranarray((U * s) @ V.T)
