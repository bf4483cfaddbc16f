"""GPU parity of the engine- and solver-level boundary (include/spaqr_b200.h):
spaqr_factorize on a caller-supplied hierarchy and row ownership (factorize.h:51-53),
cgls(A, W, b, u, opt, weights) (solve.h:30-31), and SPQRFW01 factor files loaded onto the
GPU (load_factorization, transforms.cpp:242-289) — against the oracle and the reference."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from oracle import ref as R
from paper_2102_09878_b200.problems import knn_geometric, tall_grid

pytestmark = pytest.mark.gpu


def _P():
    import paper_2102_09878_b200 as P
    return P


def _close(a, b, tol):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) <= tol * max(np.linalg.norm(b), 1.0)


@pytest.mark.parametrize("case", ["grid", "knn", "exact"])
def test_factorize_on_given_hierarchy_matches_pipeline_and_oracle(case):
    if case == "grid":
        p = tall_grid(32, seed=2)
        kw = dict(eps=1e-2, levels=6, coords=p.coords)
    elif case == "knn":
        p = knn_geometric(4096, seed=3, levels=6)
        kw = dict(eps=1e-2, levels=6, coords=p.coords)
    else:
        p = tall_grid(16, seed=4)
        kw = dict(eps=0.0, levels=4, coords=p.coords)
    g = _P().Pipeline(p.A, **kw)
    o = O.Pipeline(p.A, **kw)
    F = _P().spaqr_factorize(g.scaled(), g.hierarchy(), g.owner(), eps=kw["eps"])
    assert (F.nW, F.nnz_w, F.ndropped, F.ntrailing) == (g.nW, g.nnz_w, g.ndropped, g.ntrailing) == \
           (o.nW, o.nnz_w, o.ndropped, o.ntrailing)
    for a, b in zip(F.rows(), o.rows()):
        assert np.array_equal(np.sort(a), np.sort(b))
    assert np.array_equal(F.rows()[0], o.rows()[0])
    for a, b in zip(F.stages(), o.stages()):
        assert a["stage"] == b["stage"] and np.array_equal(a["front_cols"], b["front_cols"])
    z = np.random.default_rng(0).uniform(-1, 1, F.N)
    for name in ("w_apply", "w_solve", "wt_apply", "wt_solve"):
        assert _close(getattr(F, name)(z), getattr(o, name)(z), 1e-10)
    # the scaled, permuted matrix and ownership are the oracle's, bit for bit
    As, Ao = g.scaled(), o.scaled()
    assert np.array_equal(As.indptr, Ao.indptr) and np.array_equal(As.indices, Ao.indices)
    assert np.array_equal(As.data, Ao.data)


def test_cgls_with_given_factor_matches_reference_cgls():
    p = tall_grid(32, seed=6)
    kw = dict(eps=1e-2, levels=6, coords=p.coords)
    g = _P().Pipeline(p.A, **kw)
    F = _P().spaqr_factorize(g.scaled(), g.hierarchy(), g.owner(), eps=1e-2)
    As = g.scaled()
    u, rep = _P().cgls(As, F, p.b, tol=1e-12, maxit=500, weights=g.weights())
    x, rp = g.solve(p.b)  # Pipeline::solve = cgls on the same W, then unscale
    assert rep["iterations"] == rp["iterations"] and rep["converged"]
    assert np.allclose(rep["residual_history"], rp["residual_history"], rtol=1e-8, atol=1e-13)
    perm, w = g.perm(), g.weights()
    xu = np.zeros_like(x)
    xu[perm] = u / w
    assert _close(xu, x, 1e-9)
    o = O.Pipeline(p.A, **kw)
    xo, ro = o.solve(p.b)
    assert abs(ro["iterations"] - rep["iterations"]) <= 1


def test_plain_cgls_matches_oracle():
    p = tall_grid(24, seed=8)
    A = p.A.tocsc()
    u, rep = _P().cgls(A, None, p.b, tol=1e-10, maxit=400)
    uo, ro = O.cgls_plain(A, p.b, tol=1e-10, maxit=400)
    assert abs(rep["iterations"] - ro["iterations"]) <= 1
    rel = lambda x: np.linalg.norm(A.T @ (p.b - A @ x)) / np.linalg.norm(A.T @ p.b)
    assert abs(rel(u) - rel(uo)) <= 1e-10


@pytest.mark.parametrize("writer", ["gpu", "oracle", "reference"])
def test_factor_file_loads_onto_gpu_and_solves(writer, tmp_path):
    """factor once, solve many: a saved W (written by the GPU, the oracle or the reference's
    own save_factorization) loads onto the GPU; its sweeps and a CGLS with it match."""
    if writer == "reference" and not R.available():
        pytest.skip("oracle/_ref unavailable")
    p = tall_grid(32, seed=9)
    kw = dict(eps=1e-2, levels=6, coords=p.coords)
    o = O.Pipeline(p.A, **kw)
    path = tmp_path / "w.spqr"
    if writer == "gpu":
        _P().Pipeline(p.A, **kw).save(path)
    elif writer == "oracle":
        o.save(path)
    else:
        R.Pipeline(p.A, **kw).save(path)
    F = _P().Factorization.load(path)
    assert (F.M, F.N, F.nW, F.nnz_w) == (o.M, o.N, o.nW, o.nnz_w)
    for a, b in zip(F.rows(), o.rows()):
        assert np.array_equal(a, b)
    z = np.random.default_rng(1).uniform(-1, 1, F.N)
    for name in ("w_apply", "w_solve", "wt_apply", "wt_solve"):
        assert _close(getattr(F, name)(z), getattr(o, name)(z), 1e-10)
    u, rep = _P().cgls(o.scaled(), F, p.b, weights=o.weights())
    xo, ro = o.solve(p.b)
    assert abs(rep["iterations"] - ro["iterations"]) <= 1 and rep["converged"]
    F2 = _P().Factorization.load(path)  # a second handle from the same file: independent state
    assert _close(F2.w_solve(z), F.w_solve(z), 0.0)


def test_boundary_errors_follow_the_reference():
    p = tall_grid(12, seed=1)
    g = _P().Pipeline(p.A, eps=1e-2, levels=3, coords=p.coords)
    with pytest.raises(ValueError, match="row_owner size mismatch"):
        _P().spaqr_factorize(g.scaled(), g.hierarchy(), g.owner()[:-1])
    bad = dict(g.hierarchy())
    bad["finest_of_col"] = np.full(g.N, 10 ** 6, np.int32)
    with pytest.raises(ValueError):
        _P().spaqr_factorize(g.scaled(), bad, g.owner())
    with pytest.raises(ValueError, match="at least as many rows"):
        _P().Pipeline(sp.random(4, 9, density=0.5, format="csc", random_state=1) + sp.eye(4, 9), eps=0.0, levels=1)
    with pytest.raises(ValueError, match="right-hand side length mismatch"):
        g.solve(np.ones(g.M - 1))
    with pytest.raises(ValueError):
        g.w_solve(np.ones(g.N + 1))
    with pytest.raises(ValueError, match="coordinate row count"):
        _P().Pipeline(p.A, eps=1e-2, levels=3, coords=p.coords[:-1])


def test_factor_file_errors(tmp_path):
    path = tmp_path / "junk.spqr"
    path.write_bytes(b"NOTAFILE" + b"\0" * 64)
    with pytest.raises(RuntimeError, match="bad magic"):
        _P().Factorization.load(path)
    p = tall_grid(12, seed=1)
    good = tmp_path / "w.spqr"
    _P().Pipeline(p.A, eps=1e-2, levels=3, coords=p.coords).save(good)
    data = good.read_bytes()
    trunc = tmp_path / "t.spqr"
    trunc.write_bytes(data[: len(data) // 2])
    with pytest.raises(RuntimeError, match="truncated"):
        _P().Factorization.load(trunc)
    with pytest.raises(RuntimeError, match="cannot open"):
        _P().Factorization.load(tmp_path / "missing.spqr")
