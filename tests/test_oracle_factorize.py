"""Oracle pinning: engine + sweeps + CGLS against the reference's own known
answers and properties (proj/tests/test_factorize.cpp, test_solve.cpp).  The
reference's structured instances use its inverse-Poisson generator
(out of scope here); the BASELINE tall-grid generator stands in."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from paper_2102_09878_b200.problems import random_full_rank, tall_grid


def check_row_accounting(P):  # test_factorize.cpp:85-96
    pr, dr, tr = P.rows()
    assert np.all(pr >= 0) and np.all(pr < P.M)
    assert len(set(pr.tolist())) == P.N
    allr = np.concatenate([pr, dr, tr])
    assert len(allr) == P.M and len(set(allr.tolist())) == P.M


def test_identity_factors_to_identity():  # :100-122
    n = 40
    A = sp.identity(n, format="csc")
    P = O.Pipeline(A, eps=0.0, levels=1)
    assert P.ndropped == 0 and P.ntrailing == 0
    z = np.random.default_rng(1).uniform(-1, 1, n)
    w = P.w_apply(z)
    assert np.array_equal(w, z)
    assert np.array_equal(P.w_solve(w), z)


def _probe_identity(P, nprobe, rng):  # :52-73
    A = P.scaled()
    pr, _, _ = P.rows()
    worst = 0.0
    for _ in range(nprobe):
        z = rng.uniform(-1, 1, P.N)
        u = P.w_solve(z)
        y = P.q_apply_t(A @ u)
        e = np.zeros(P.M)
        e[pr] = z
        worst = max(worst, np.abs(y - e).max() / np.linalg.norm(z))
    return worst


def test_exact_elimination_is_permuted_identity():  # :124-147
    rng = np.random.default_rng(7)
    for t in range(3):
        P = O.Pipeline(random_full_rank(100, 60, 4, seed=t), eps=0.0, levels=2, store_q=True)
        assert P.ndropped == 0
        assert _probe_identity(P, 20, rng) <= 1e-10
        check_row_accounting(P)
    p = tall_grid(8)
    P = O.Pipeline(p.A, eps=0.0, levels=O.default_num_levels(64), coords=p.coords, store_q=True)
    assert P.ndropped == 0
    assert _probe_identity(P, 20, rng) <= 1e-10


def test_exact_factorization_solves_dense_ls():  # :149-171 (via Q^T b + W^{-1})
    rng = np.random.default_rng(11)
    for A0, coords, L in [(random_full_rank(150, 90, 4, seed=5), None, 2)]:
        P = O.Pipeline(A0, eps=0.0, levels=L, coords=coords, store_q=True)
        A = P.scaled().toarray()
        b = rng.uniform(-1, 1, P.M)
        y = P.q_apply_t(b)
        pr, _, _ = P.rows()
        u = P.w_solve(y[pr])
        ref = np.linalg.lstsq(A, b, rcond=None)[0]
        assert np.linalg.norm(u - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("eps", [0.0, 1e-2])
def test_transforms_round_trip(eps):  # :173-225
    rng = np.random.default_rng(13)
    p = tall_grid(16, seed=7)
    P = O.Pipeline(p.A, eps=eps, levels=O.default_num_levels(256), skip_levels=1, coords=p.coords, store_q=True)
    for _ in range(10):
        z = rng.uniform(-1, 1, P.N)
        nz = np.linalg.norm(z)
        assert np.linalg.norm(P.w_solve(P.w_apply(z)) - z) <= 1e-12 * nz
        assert np.linalg.norm(P.wt_solve(P.wt_apply(z)) - z) <= 1e-12 * nz
        assert np.linalg.norm(P.w_apply(P.w_solve(z)) - z) <= 1e-12 * nz
        a, b = rng.uniform(-1, 1, P.N), rng.uniform(-1, 1, P.N)
        assert abs(P.wt_apply(a) @ b - a @ P.w_apply(b)) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(b) * 10
        y = rng.uniform(-1, 1, P.M)
        assert np.linalg.norm(P.q_apply(P.q_apply_t(y)) - y) <= 1e-11 * np.linalg.norm(y)


def test_row_accounting_across_configurations():  # :227-253
    p = tall_grid(12, seed=9)
    for eps in (0.0, 1e-2, 1e-1):
        for skip in (0, 2):
            P = O.Pipeline(p.A, eps=eps, levels=2, skip_levels=skip, coords=p.coords)
            check_row_accounting(P)
            if eps == 0.0:
                assert P.ndropped == 0
    for t in range(3):
        P = O.Pipeline(random_full_rank(120, 70, 5, seed=17 + t), eps=1e-2, levels=2, skip_levels=0)
        check_row_accounting(P)


def test_sparsification_compresses():  # :255-303
    p = tall_grid(24, seed=21)
    L = O.default_num_levels(24 * 24)
    F0 = O.Pipeline(p.A, eps=0.0, levels=L, coords=p.coords)
    Fm = O.Pipeline(p.A, eps=1e-2, levels=L, skip_levels=1, coords=p.coords)
    F1 = O.Pipeline(p.A, eps=1e-1, levels=L, skip_levels=1, coords=p.coords)
    assert F1.ndropped > 0
    assert F1.nnz_w < F0.nnz_w

    def last_top(P):
        t = 0
        for s in P.stages():
            if s["top_cols"] > 0:
                t = s["top_cols"]
        return t

    assert last_top(F1) <= last_top(Fm) <= last_top(F0)
    assert last_top(F1) < last_top(F0)
    st = F1.stages()
    assert len(st) == L + 1
    prev = 0
    for i, s in enumerate(st):
        assert s["stage"] == L + 1 - i
        assert s["nnz_w"] >= prev
        prev = s["nnz_w"]
        assert np.all(s["front_aspect"] > 0)


@pytest.mark.parametrize("levels,eps,skip", [(2, 1e-2, 0), (2, 0.0, 0), (3, 1e-1, 1)])
def test_engine_invariants(levels, eps, skip):  # :309-444
    p = tall_grid(12, seed=25)
    P = O.Pipeline(p.A, eps=eps, levels=levels, skip_levels=skip, coords=p.coords, check_invariants=True)
    assert P.violations == 0
    ph = P.phases()
    cl = P.clusters()
    L1 = P.L + 1
    i = 0
    for k in range(L1, 0, -1):
        for cid, c in enumerate(cl):
            if c["level"] == k and c["stage"] == k:
                assert ph[i] == ("eliminate", k, cid)
                i += 1
        if eps > 0 and k >= 2 and L1 - k >= skip:  # scale is gated by the skip window (factorize.cpp:763)
            assert [ph[i][0], ph[i + 1][0], ph[i + 2][0]] == ["scale", "sparsify_rows", "sparsify_cols"]
            i += 3
        if k >= 2:
            assert ph[i][0] == "merge"
            i += 1
    assert i == len(ph)
    check_row_accounting(P)


def test_rank_deficiency_raises_singular_front():  # :446-481
    D = np.zeros((9, 6))
    D[0, 0], D[0, 1] = 1.0, 2.0
    for j in range(2, 6):
        D[2 * j - 3, j] = 3.0
        D[2 * j - 2, j] = 0.5
    with pytest.raises(O.SingularFrontError) as e:
        O.Pipeline(sp.csc_matrix(D), eps=0.0, levels=1, parts=[0, 0, 1, 1, 1, 1])
    assert e.value.cluster >= 0 and "rows couple" in str(e.value) and "singular front" in str(e.value)
    D = np.zeros((11, 7))
    D[0, 0], D[0, 1], D[1, 2], D[2, 2] = 1.5, -2.25, 2.0, 0.5
    for j in range(3, 7):
        D[2 * j - 3, j] = 3.0
        D[2 * j - 2, j] = -0.75
    with pytest.raises(O.SingularFrontError) as e:
        O.Pipeline(sp.csc_matrix(D), eps=0.0, levels=1, parts=[0, 0, 0, 1, 1, 1, 1])
    assert e.value.cluster >= 0 and "pivot" in str(e.value)


def test_shape_validation():  # :483-495
    wide = sp.csc_matrix(np.eye(3, 5))
    with pytest.raises(ValueError):
        O.Pipeline(wide, eps=1e-2, levels=1)


# ----------------------------------------------------------------- solve
def test_cgls_identity_one_iteration_bitwise():  # test_solve.cpp:66-84
    n = 30
    b = np.random.default_rng(2).standard_normal(n)
    u, rep = O.cgls_plain(sp.identity(n, format="csc"), b)
    assert rep["converged"] and rep["iterations"] == 1
    assert list(rep["residual_history"]) == [1.0, 0.0]
    assert np.array_equal(u, b)


def test_exact_factorization_preconditions_to_immediate_convergence():  # :86-104
    p = tall_grid(8, seed=5)
    P = O.Pipeline(p.A, eps=0.0, levels=O.default_num_levels(64), coords=p.coords)
    b = np.random.default_rng(7).standard_normal(P.M)
    x, rep = P.solve(b, tol=1e-10)
    assert rep["converged"] and rep["iterations"] <= 3 and rep["dropped_rows"] == 0


def test_csne_matches_dense_ls():  # :106-139
    rng = np.random.default_rng(23)
    A0 = random_full_rank(200, 120, 4, seed=23)
    P = O.Pipeline(A0, eps=0.0, levels=2, solver="direct")
    for _ in range(3):
        b = rng.standard_normal(200)
        x, rep = P.solve(b, direct=True)
        ref = np.linalg.lstsq(A0.toarray(), b, rcond=None)[0]
        assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)
        assert rep["iterations"] == 1 and len(rep["residual_history"]) == 2
        assert rep["residual_history"][1] <= 1e-12 and rep["converged"]


def test_preconditioning_cuts_iterations():  # :172-217
    p = tall_grid(24, seed=3)
    P = O.Pipeline(p.A, eps=1e-2, levels=O.default_num_levels(576), skip_levels=1, coords=p.coords)
    b = np.random.default_rng(5).standard_normal(P.M)
    x, pre = P.solve(b, tol=1e-10, maxit=2000)
    u, plain = O.cgls_plain(P.scaled(), b, tol=1e-10, maxit=2000)
    assert pre["converged"] and plain["converged"]
    assert pre["iterations"] <= 50 and plain["iterations"] >= 4 * pre["iterations"]
    h = pre["residual_history"]
    assert len(h) == pre["iterations"] + 1 and h[0] == 1.0 and np.all(np.isfinite(h))


def test_weighted_reporting():  # :219-239
    p = tall_grid(8, seed=5)
    A = p.A.copy()
    d = np.sqrt(np.asarray(A.multiply(A).sum(axis=0))).ravel()
    As = A @ sp.diags(1.0 / d)
    b = np.random.default_rng(11).standard_normal(A.shape[0])
    u, rep = O.cgls_plain(As, b, tol=0.0, maxit=5, weights=d)
    r = b - As @ u
    expected = np.linalg.norm(A.T @ r) / np.linalg.norm(A.T @ b)
    assert rep["residual_history"][-1] == pytest.approx(expected, rel=1e-10)


def test_direct_kind_forces_exact():  # :320-341
    p = tall_grid(8, seed=19)
    b = np.random.default_rng(19).standard_normal(p.A.shape[0])
    Pe = O.Pipeline(p.A, eps=0.0, coords=p.coords)
    Pd = O.Pipeline(p.A, eps=0.5, solver="direct", coords=p.coords)
    xe, re = Pe.solve(b)
    xd, rd = Pd.solve(b)
    assert re["iterations"] == rd["iterations"]
    assert np.abs(xe - xd).max() == 0.0
