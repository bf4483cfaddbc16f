"""Run profile JSON (make_profile / validate_profile, proj/src/profile.cpp:42-188; the
reference's checks: tests/test_profile.cpp).  CPU: the document built from the oracle
validates, quartiles follow the reference's interpolation, the validator reports the
reference's messages.  GPU: the B200 profile validates and its per-stage structure equals
the oracle's (times aside)."""
import json

import numpy as np
import pytest

import oracle as O
from paper_2102_09878_b200.problems import tall_grid
from paper_2102_09878_b200.profile import _quartiles, make_profile, validate_profile


def test_quartiles_interpolate_like_the_reference():
    q = _quartiles([4, 1, 3, 2])
    assert q == {"min": 1.0, "q1": 1.75, "median": 2.5, "q3": 3.25, "max": 4.0}
    assert _quartiles([]) == {"min": 0.0, "q1": 0.0, "median": 0.0, "q3": 0.0, "max": 0.0}
    assert _quartiles([7])["median"] == 7.0


def test_oracle_profile_validates_and_validator_messages():
    p = tall_grid(16, seed=2)
    o = O.Pipeline(p.A, eps=1e-2, levels=4, coords=p.coords)
    x, rep = o.solve(p.b)
    text = make_profile(o, rep, eps=1e-2)
    assert validate_profile(text) == ""
    j = json.loads(text)
    assert len(j["levels"]) == o.nstages and j["totals"]["nnz_w"] == o.nnz_w
    assert j["solve"]["iterations"] == rep["iterations"] and len(j["solve"]["residuals"]) == len(rep["residual_history"])
    assert validate_profile("{") == "profile: not valid JSON"
    bad = dict(j)
    del bad["totals"]
    assert validate_profile(json.dumps(bad)) == "profile: missing 'totals'"
    bad = json.loads(text)
    bad["version"] = 2
    assert validate_profile(json.dumps(bad)) == "profile: unsupported version"
    bad = json.loads(text)
    bad["levels"][0]["merge"] = -1.0
    assert validate_profile(json.dumps(bad)) == "levels[]: negative phase time 'merge'"
    bad = json.loads(text)
    bad["matrix"]["rows"] = 1.5
    assert validate_profile(json.dumps(bad)) == "matrix: 'rows' has the wrong type"
    bad = json.loads(text)
    bad["solve"]["converged"] = 1
    assert validate_profile(json.dumps(bad)) == "solve: missing boolean 'converged'"


@pytest.mark.gpu
def test_gpu_profile_matches_oracle_structure():
    import paper_2102_09878_b200 as P
    p = tall_grid(64, seed=0)
    kw = dict(eps=1e-3, levels=8, coords=p.coords)
    o, g = O.Pipeline(p.A, **kw), P.Pipeline(p.A, **kw)
    _, ro = o.solve(p.b)
    _, rg = g.solve(p.b)
    jo = json.loads(make_profile(o, ro, eps=1e-3))
    tg = make_profile(g, rg, eps=1e-3)
    assert validate_profile(tg) == ""
    jg = json.loads(tg)
    assert jg["matrix"] == jo["matrix"] and jg["options"] == jo["options"]
    assert len(jg["levels"]) == len(jo["levels"])
    for a, b in zip(jg["levels"], jo["levels"]):
        for k in ("stage", "interface_cols", "aspect", "top_rows", "top_cols", "nnz_w"):
            assert a[k] == b[k], (k, a[k], b[k])
    for k in ("nnz_w", "dropped_rows", "trailing_rows"):
        assert jg["totals"][k] == jo["totals"][k]
    assert abs(jg["solve"]["iterations"] - jo["solve"]["iterations"]) <= 1
    assert jg["device"]["front_qr"]["launches"] > 0
