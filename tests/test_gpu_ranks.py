"""Subtree-split accounting on the GPU engine (FactorizeOptions::ranks): a
pipeline created with ranks = G reports, per stage, the flops each rank of a G-GPU subtree
split would own and the bytes that would cross ranks, and factors exactly as with ranks = 1."""
import numpy as np
import pytest

from paper_2102_09878_b200.problems import knn_geometric, tall_grid

pytestmark = pytest.mark.gpu


def _P():
    import paper_2102_09878_b200 as P
    return P


@pytest.mark.parametrize("G", [2, 4, 8])
def test_rank_accounting_leaves_the_factorization_unchanged(G):
    p = tall_grid(64)
    kw = dict(eps=p.eps, levels=p.levels, coords=p.coords)
    a = _P().Pipeline(p.A, **kw)
    b = _P().Pipeline(p.A, ranks=G, **kw)
    assert a.rank_stats() is None
    assert (a.nW, a.nnz_w, a.ndropped, a.ntrailing) == (b.nW, b.nnz_w, b.ndropped, b.ntrailing)
    for x, y in zip(a.rows(), b.rows()):
        assert np.array_equal(x, y)
    rs = b.rank_stats()
    assert rs["ranks"] == G
    # the owner map is the host plan's
    plan = _P().rank_plan(p.A, G, levels=p.levels, coords=p.coords)
    assert np.array_equal(rs["owner"], plan["owner"])
    # every rank owns work; the accounted flops cover the engine's QR and CPQR work
    fl = rs["flops"]
    assert np.all(fl.sum(axis=0) > 0)
    t = b.times()
    assert fl.sum() >= 0.999 * t["qr_flops"]
    # subtrees meet only along the top separators: some traffic, far below the front data
    assert rs["cross"].sum() > 0


def test_rank_accounting_knn():
    p = knn_geometric(4096, seed=5, levels=8)
    g = _P().Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords, ranks=4)
    rs = g.rank_stats()
    assert rs["flops"].shape[1] == 4 and np.all(rs["flops"].sum(axis=0) > 0)
