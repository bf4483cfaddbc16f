"""Oracle pinning: dense kernels against the reference's own property and
known-answer tests (proj/tests/test_dense_kernels.cpp).  numpy's LAPACK SVD
stands in for Eigen::JacobiSVD as the rank oracle."""
import numpy as np
import pytest

import oracle as O


def rmat(rng, m, n):
    return rng.uniform(-1.0, 1.0, size=(m, n))


def rrank(rng, m, n, r):
    return rmat(rng, m, r) @ rmat(rng, r, n)


def svd_rank(B, rel):  # test_dense_kernels.cpp:25-33
    if B.size == 0:
        return 0
    s = np.linalg.svd(B, compute_uv=False)
    if s.size == 0 or s[0] == 0.0:
        return 0
    return int(np.sum(s > rel * s[0]))


def test_householder_qr_reconstructs_with_sign_convention():  # :37-65
    rng = np.random.default_rng(7)
    for _ in range(40):
        n = 1 + int(rng.integers(12))
        m = n + int(rng.integers(20))
        B = rmat(rng, m, n)
        V, tau, sg, R = O.householder_qr(B)
        assert R.shape == (n, n)
        assert np.all(np.diag(R) >= 0)
        assert np.all(np.tril(R, -1) == 0.0)
        RZ = np.zeros((m, n))
        RZ[:n] = R
        RZ = O.apply_reflectors(V, tau, sg, RZ, "left")
        nb = 1.0 + np.linalg.norm(B)
        assert np.linalg.norm(RZ - B) <= 1e-12 * nb
        Cm = O.apply_reflectors(V, tau, sg, B, "left_t")
        assert np.linalg.norm(Cm[:n] - R) <= 1e-12 * nb
        if m > n:
            assert np.linalg.norm(Cm[n:]) <= 1e-12 * nb


def test_known_answers():  # SPEC dense-kernels examples: [3;4] -> R = [5]; I4 -> I4
    V, tau, sg, R = O.householder_qr(np.array([[3.0], [4.0]]))
    assert abs(R[0, 0] - 5.0) <= 1e-15
    V, tau, sg, R = O.householder_qr(np.eye(4))
    assert np.allclose(R, np.eye(4), atol=0, rtol=0)


def test_reflector_applies_agree_with_dense_q():  # :67-96
    rng = np.random.default_rng(11)
    for _ in range(20):
        n = 1 + int(rng.integers(8))
        m = n + int(rng.integers(10))
        V, tau, sg, R = O.householder_qr(rmat(rng, m, n))
        Q = O.apply_reflectors(V, tau, sg, np.eye(m), "left")
        assert np.linalg.norm(Q.T @ Q - np.eye(m)) <= 1e-12 * m
        X = rmat(rng, m, 5)
        assert np.linalg.norm(O.apply_reflectors(V, tau, sg, X, "left") - Q @ X) <= 1e-12 * (1 + np.linalg.norm(X))
        assert np.linalg.norm(O.apply_reflectors(V, tau, sg, X, "left_t") - Q.T @ X) <= 1e-12 * (1 + np.linalg.norm(X))
        Z = rmat(rng, 4, m)
        assert np.linalg.norm(O.apply_reflectors(V, tau, sg, Z, "right") - Z @ Q) <= 1e-12 * (1 + np.linalg.norm(Z))
        assert np.linalg.norm(O.apply_reflectors(V, tau, sg, Z, "right_t") - Z @ Q.T) <= 1e-12 * (1 + np.linalg.norm(Z))


def test_blocked_and_rank1_paths_agree():  # apply_raw's two branches (dense_kernels.cpp:61-85)
    rng = np.random.default_rng(3)
    V, tau, sg, R = O.householder_qr(rmat(rng, 30, 9))
    X = rmat(rng, 30, 7)
    blocked = O.apply_reflectors(V, tau, sg, X, "left_t")
    cols = np.column_stack([O.apply_reflectors(V, tau, sg, X[:, [j]], "left_t") for j in range(7)])
    assert np.abs(blocked - cols).max() <= 1e-13


def test_truncated_cpqr_obeys_truncation_rule():  # :98-135
    rng = np.random.default_rng(23)
    for trial in range(40):
        m = 2 + int(rng.integers(20))
        n = 2 + int(rng.integers(20))
        r0 = 1 + int(rng.integers(min(m, n)))
        B = rrank(rng, m, n, r0)
        eps = 1e-8 if trial % 2 else 1e-4
        T = O.cpqr(B, eps)
        r = T["rank"]
        assert r <= min(m, n) and T["R"].shape == (r, n) and len(T["perm"]) >= r
        prev = np.inf
        for i in range(r):
            d = T["R"][i, T["perm"][i]]
            assert d >= 0 and d >= eps * T["r11"] * (1 - 1e-10) and d <= prev * (1 + 1e-10)
            prev = d
        Q = O.apply_reflectors(T["V"], T["tau"], T["sign"], np.eye(m), "left")
        E = B - Q[:, :r] @ T["R"]
        for j in range(n):
            assert np.linalg.norm(E[:, j]) <= 10 * eps * T["r11"] + 1e-13 * (1 + np.linalg.norm(B))
        assert np.linalg.norm(E) <= 10 * eps * T["r11"] * np.sqrt(min(m, n) - r) + 1e-12 * (1 + np.linalg.norm(B))


def test_truncated_cpqr_rank_matches_svd():  # :137-149
    rng = np.random.default_rng(31)
    for _ in range(30):
        m = 3 + int(rng.integers(25))
        n = 3 + int(rng.integers(25))
        r0 = 1 + int(rng.integers(min(m, n)))
        B = rrank(rng, m, n, r0)
        assert O.cpqr(B, 1e-10)["rank"] == svd_rank(B, 1e-10)


def test_truncated_cpqr_edge_cases():  # :151-201
    rng = np.random.default_rng(41)
    T = O.cpqr(np.zeros((6, 4)), 1e-8)
    assert T["rank"] == 0 and T["r11"] == 0.0
    assert O.cpqr(np.zeros((6, 4)), 0.0)["rank"] == 0
    B = rmat(rng, 9, 5)
    T = O.cpqr(B, 0.0)
    assert T["rank"] == 5
    Q = O.apply_reflectors(T["V"], T["tau"], T["sign"], np.eye(9), "left")
    assert np.linalg.norm(B - Q[:, :5] @ T["R"]) <= 1e-12 * (1 + np.linalg.norm(B))
    B = np.zeros((4, 3))
    B[:, 0] = 1.0
    T = O.cpqr(B, 0.0)
    assert T["rank"] == 3
    Q = O.apply_reflectors(T["V"], T["tau"], T["sign"], np.eye(4), "left")
    assert np.linalg.norm(B - Q[:, :3] @ T["R"]) <= 1e-13
    for _ in range(20):
        B = rrank(rng, 12, 10, 6)
        prev = 99
        for eps in (1e-12, 1e-8, 1e-4, 1e-2, 1e-1):
            r = O.cpqr(B, eps)["rank"]
            assert r <= prev
            prev = r
    assert O.cpqr(rmat(rng, 3, 14), 1e-10)["rank"] == 3
    assert O.cpqr(rmat(rng, 14, 3), 1e-10)["rank"] == 3
    # SPEC examples: diag(1, 1e-8), eps 1e-2 -> rank 1
    assert O.cpqr(np.diag([1.0, 1e-8]), 1e-2)["rank"] == 1


def test_cpqr_decaying_spectrum_rank():  # BASELINE config 5: sigma_i = 0.8^i, eps 1e-2 -> 21
    from paper_2102_09878_b200.problems import decaying_interface
    B = decaying_interface(256, 0.8, seed=0)
    T = O.cpqr(B, 1e-2)
    # pivoted-QR diagonals track but do not equal singular values: the rule is
    # |R_ii| >= eps |R_11| (dense_kernels.cpp:156-158), so rank >= svd rank.
    assert svd_rank(B, 1e-2) == 21
    assert 21 <= T["rank"] <= 25


def test_triangular_solves_all_modes():  # :203-228
    rng = np.random.default_rng(57)
    for _ in range(25):
        n = 1 + int(rng.integers(10))
        R = np.triu(rmat(rng, n, n))
        R[np.diag_indices(n)] = 1.0 + np.abs(np.diag(R))
        B = rmat(rng, n, 4)
        nb = 1 + np.linalg.norm(B)
        assert np.linalg.norm(R @ O.tri_solve_upper(R, B, "left", False) - B) <= 1e-11 * nb
        assert np.linalg.norm(R.T @ O.tri_solve_upper(R, B, "left", True) - B) <= 1e-11 * nb
        Cm = rmat(rng, 4, n)
        nc = 1 + np.linalg.norm(Cm)
        assert np.linalg.norm(O.tri_solve_upper(R, Cm, "right", False) @ R - Cm) <= 1e-11 * nc
        assert np.linalg.norm(O.tri_solve_upper(R, Cm, "right", True) @ R.T - Cm) <= 1e-11 * nc
    # SPEC: R=[[2,1],[0,1]], B=(3,1)^T -> X=(1,1)^T
    X = O.tri_solve_upper(np.array([[2.0, 1.0], [0.0, 1.0]]), np.array([[3.0], [1.0]]))
    assert np.array_equal(X, np.ones((2, 1)))


def test_singular_diagonals_rejected():  # :230-240
    R = np.eye(3)
    R[1, 1] = 0.0
    with pytest.raises(O.SingularFrontError):
        O.check_diag_invertible(R)
    with pytest.raises(O.SingularFrontError):
        O.tri_solve_upper(R, np.ones((3, 2)))
    R[1, 1] = 1e-320
    with pytest.raises(O.SingularFrontError):
        O.check_diag_invertible(R)
    R[1, 1] = 1e-300
    O.check_diag_invertible(R)
