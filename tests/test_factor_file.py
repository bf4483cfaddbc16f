"""SPQRFW01 factor files (save_factorization / load_factorization, transforms.cpp:129-289;
the reference's tests: test_serialization.cpp:62-200).

CPU: the oracle's writer and reader round-trip bit for bit, reject a bad magic, and the
file layout is the documented one (parsed here independently).
GPU: the B200 pipeline's file parses to the same structure as the oracle's (indices exact,
values within FP64 tolerance) and, loaded by the oracle's reader, reproduces the GPU's own
W sweeps."""
import os
import struct

import numpy as np
import pytest

import oracle as O
from paper_2102_09878_b200.problems import tall_grid


def parse(path):
    """Independent reader of the SPQRFW01 layout."""
    b = open(path, "rb").read()
    pos = 0

    def i64():
        nonlocal pos
        v = struct.unpack_from("<q", b, pos)[0]
        pos += 8
        return v

    def f64s(n):
        nonlocal pos
        v = np.frombuffer(b, "<f8", n, pos).copy()
        pos += 8 * n
        return v

    def ivec():
        n = i64()
        return np.array([i64() for _ in range(n)], np.int64)

    def mat():
        r, c = i64(), i64()
        return f64s(r * c).reshape(r, c, order="F")

    def vec():
        return f64s(i64())

    assert b[:8] == b"SPQRFW01"
    pos = 8
    out = dict(M=i64(), N=i64(), eps=f64s(1)[0], pivot_row=ivec(), dropped=ivec(), trailing=ivec(), W=[])
    for _ in range(i64()):
        tag = i64()
        if tag == 0:
            out["W"].append(("tri", ivec(), mat(), ivec(), mat()))
        else:
            assert tag == 1
            out["W"].append(("rot", ivec(), mat(), vec(), vec()))
    out["has_q"] = i64()
    if out["has_q"]:
        for _ in range(i64()):
            ivec(), mat(), vec(), vec()
    assert pos == len(b), "trailing bytes"
    return out


def _problem():
    p = tall_grid(24, seed=5)
    return p, dict(eps=1e-2, levels=5, coords=p.coords)


def test_oracle_file_round_trip_and_layout(tmp_path):
    p, kw = _problem()
    o = O.Pipeline(p.A, **kw)
    f = tmp_path / "w.spqr"
    o.save(f)
    d = parse(f)
    assert (d["M"], d["N"]) == p.A.shape and d["eps"] == kw["eps"] and len(d["W"]) == o.nW and d["has_q"] == 0
    pr, dr, tr = o.rows()
    assert np.array_equal(d["pivot_row"], pr) and np.array_equal(np.sort(d["dropped"]), np.sort(dr))
    z = np.random.default_rng(1).standard_normal(p.A.shape[1])
    for mode in ("w_apply", "w_solve", "wt_apply", "wt_solve"):
        dims, v = O.factor_file_apply(f, mode, z)
        assert dims == (p.A.shape[0], p.A.shape[1], o.nW)
        assert np.array_equal(v, getattr(o, mode)(z))  # bit-exact through the file
    bad = tmp_path / "bad.spqr"
    bad.write_bytes(b"NOTSPQR!" + f.read_bytes()[8:])
    with pytest.raises(RuntimeError, match="bad magic"):
        O.factor_file_apply(bad, "w_solve")
    short = tmp_path / "short.spqr"
    short.write_bytes(f.read_bytes()[:200])
    with pytest.raises(RuntimeError):
        O.factor_file_apply(short, "w_solve")


@pytest.mark.gpu
def test_gpu_file_matches_oracle_and_loads(tmp_path):
    import paper_2102_09878_b200 as P
    p, kw = _problem()
    o, g = O.Pipeline(p.A, **kw), P.Pipeline(p.A, **kw)
    fo, fg = tmp_path / "o.spqr", tmp_path / "g.spqr"
    o.save(fo)
    g.save(fg)
    a, b = parse(fg), parse(fo)
    assert (a["M"], a["N"], a["eps"], a["has_q"]) == (b["M"], b["N"], b["eps"], b["has_q"])
    for key in ("pivot_row", "dropped", "trailing"):
        assert np.array_equal(np.sort(a[key]), np.sort(b[key])), key
    assert np.array_equal(a["pivot_row"], b["pivot_row"])
    assert len(a["W"]) == len(b["W"])
    for x, y in zip(a["W"], b["W"]):
        assert x[0] == y[0] and np.array_equal(x[1], y[1])
        if x[0] == "tri":
            assert np.array_equal(x[3], y[3])
            s = 1 + np.abs(y[2]).max()
            assert np.allclose(x[2], y[2], atol=1e-10 * s) and np.allclose(x[4], y[4], atol=1e-10 * s)
        else:
            assert np.allclose(x[2], y[2], atol=1e-10) and np.allclose(x[3], y[3], atol=1e-12)
            assert np.array_equal(x[4], y[4])
    # the reference-layout file written by the GPU, read back by the (restated) reference loader
    z = np.random.default_rng(2).standard_normal(p.A.shape[1])
    for mode in ("w_apply", "w_solve", "wt_apply", "wt_solve"):
        _, v = O.factor_file_apply(fg, mode, z)
        gz = getattr(g, mode)(z)
        assert np.allclose(v, gz, atol=1e-10 * (1 + np.abs(gz).max())), mode
