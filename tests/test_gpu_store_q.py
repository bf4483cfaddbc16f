"""GPU parity of the orthogonal row factors Q (FactorizeOptions::store_q, factorize.h:16):
RowReflects recorded at eliminate (factorize.cpp:324-330), scale_all (:483), sparsify_rows
(:514-519) and sparsify_cols (:583-588), applied by Factorization::q_apply_t / q_apply
(transforms.cpp:113-127), and written / read with the SPQRFW01 file (transforms.cpp:230-237,
277-286).  Tests follow test_factorize.cpp:52-90,124-224 and test_serialization.cpp:62-110."""
import numpy as np
import pytest

import oracle as O
from paper_2102_09878_b200.problems import knn_geometric, random_full_rank, tall_grid

pytestmark = pytest.mark.gpu


def _P():
    import paper_2102_09878_b200 as P
    return P


def probe_identity(A, F, nprobe, rng):
    """test_factorize.cpp:52-73: max deviation of Q^T A W^{-1} from the pivot-scattered [I; 0]."""
    piv, _, _ = F.rows()
    worst = 0.0
    for _ in range(nprobe):
        z = rng.uniform(-1, 1, F.N)
        y = F.q_apply_t(A @ F.w_solve(z))
        expect = np.zeros(F.M)
        expect[piv] = z
        worst = max(worst, np.abs(y - expect).max() / np.linalg.norm(z))
    return worst


def q_solve(F, b):
    """test_factorize.cpp:75-84: u = W^{-1} gather(Q^T b) at the pivot rows."""
    piv, _, _ = F.rows()
    return F.w_solve(F.q_apply_t(b)[piv])


@pytest.mark.parametrize("case", ["grid_eps", "knn_eps", "grid_exact"])
def test_q_matches_oracle(case):
    """Q^T y and Q y agree with the oracle's (same factors in the same order)."""
    if case == "grid_eps":
        p = tall_grid(32, seed=5)
        kw = dict(eps=1e-2, levels=6, coords=p.coords)
    elif case == "knn_eps":
        p = knn_geometric(4096, seed=6, levels=6)
        kw = dict(eps=1e-2, levels=6, coords=p.coords)
    else:
        p = tall_grid(16, seed=7)
        kw = dict(eps=0.0, levels=4, coords=p.coords)
    g = _P().Pipeline(p.A, store_q=True, **kw)
    o = O.Pipeline(p.A, store_q=True, **kw)
    assert g.nW == o.nW and g.nQ == o.nQ > 0
    rng = np.random.default_rng(1)
    for _ in range(3):
        y = rng.standard_normal(g.M)
        for f in ("q_apply_t", "q_apply"):
            a, b = getattr(g, f)(y), getattr(o, f)(y)
            assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(y), f
        # orthogonality round trip (test_factorize.cpp:216-222)
        assert np.linalg.norm(g.q_apply(g.q_apply_t(y)) - y) <= 1e-11 * np.linalg.norm(y)


def test_store_q_leaves_w_unchanged():
    """store_q only records: W, the row sets and the solve are those of the plain run."""
    p = tall_grid(32, seed=8)
    kw = dict(eps=1e-2, levels=6, coords=p.coords)
    a = _P().Pipeline(p.A, **kw)
    b = _P().Pipeline(p.A, store_q=True, **kw)
    assert a.nQ == -1 and b.nQ > 0
    assert (a.nW, a.nnz_w, a.ndropped, a.ntrailing) == (b.nW, b.nnz_w, b.ndropped, b.ntrailing)
    for x, y in zip(a.rows(), b.rows()):
        assert np.array_equal(x, y)
    z = np.random.default_rng(2).standard_normal(a.N)
    assert np.array_equal(a.w_solve(z), b.w_solve(z))
    with pytest.raises(RuntimeError):
        a.q_apply_t(np.zeros(a.M))


@pytest.mark.parametrize("trial", range(3))
def test_exact_elimination_is_permuted_identity(trial):
    """test_factorize.cpp:124-147: with eps = 0, Q^T A W^{-1} = [I; 0] scattered to the pivot
    rows (through spaqr_factorize on the pipeline's hierarchy, store_q set)."""
    A0 = random_full_rank(100, 60, 4, seed=10 + trial)
    g = _P().Pipeline(A0, eps=0.0, levels=2, skip_levels=0)
    F = _P().spaqr_factorize(g.scaled(), g.hierarchy(), g.owner(), eps=0.0, skip_levels=0, store_q=True)
    assert F.ndropped == 0 and F.nQ > 0
    assert probe_identity(g.scaled(), F, 20, np.random.default_rng(trial)) <= 1e-10


def test_exact_factorization_q_solve_is_dense_least_squares():
    """test_factorize.cpp:149-171: u = W^{-1} gather(Q^T b) solves min ||A u - b||."""
    A0 = random_full_rank(150, 90, 4, seed=21)
    g = _P().Pipeline(A0, eps=0.0, levels=2, skip_levels=0)
    A = g.scaled()
    F = _P().spaqr_factorize(A, g.hierarchy(), g.owner(), eps=0.0, skip_levels=0, store_q=True)
    b = np.random.default_rng(3).uniform(-1, 1, A.shape[0])
    u = q_solve(F, b)
    ref = np.linalg.lstsq(A.toarray(), b, rcond=None)[0]
    assert np.linalg.norm(u - ref) <= 1e-10 * np.linalg.norm(ref)


def test_q_survives_the_factor_file(tmp_path):
    """test_serialization.cpp:62-110: a store_q factorization written and read back keeps Q; the
    GPU's file matches the oracle's reader (nQ) and q_apply_t is bit-identical after the load."""
    p = tall_grid(24, seed=9)
    g = _P().Pipeline(p.A, eps=1e-2, levels=5, skip_levels=1, coords=p.coords, store_q=True)
    path = tmp_path / "q.spqrfw"
    g.save(path)
    F = _P().Factorization.load(path)
    assert F.nQ == g.nQ > 0 and F.nW == g.nW
    y = np.random.default_rng(4).standard_normal(g.M)
    assert np.array_equal(F.q_apply_t(y), g.q_apply_t(y))
    assert np.array_equal(F.q_apply(y), g.q_apply(y))
    # the oracle's restated reader sees the same Q section
    _, v = O.factor_file_apply(str(path), "q_apply_t", y)
    assert np.linalg.norm(v - g.q_apply_t(y)) <= 1e-12 * np.linalg.norm(y)


@pytest.mark.timeout(900)
def test_q_matches_oracle_3d_blocked_fronts():
    """A 3D problem whose top fronts exceed the tile kernels (> 2 MB: the blocked QR path,
    mbqr.cu) and whose large interfaces run on the cluster CPQR: Q still matches the oracle."""
    p = tall_grid(24, dim=3, seed=3)
    kw = dict(eps=p.eps, levels=p.levels, coords=p.coords)
    g = _P().Pipeline(p.A, store_q=True, **kw)
    o = O.Pipeline(p.A, store_q=True, **kw)
    assert g.nW == o.nW and g.nQ == o.nQ > 0
    y = np.random.default_rng(7).standard_normal(g.M)
    for f in ("q_apply_t", "q_apply"):
        a, b = getattr(g, f)(y), getattr(o, f)(y)
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(y), f
