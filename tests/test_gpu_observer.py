"""The reference's per-phase engine invariants (proj/tests/test_factorize.cpp:309-415), checked
on the GPU engine through its observer hook (FactorizeObserver / EngineView,
factorize.h:31-43; spqr_engine_view in include/spaqr_b200.h):

* row conservation at every phase: live rows + pivots + dropped + trailing == M;
* couplings stay on one root-to-leaf path of the hierarchy (ClusterHierarchy::related);
* an elimination leaves non-participant fronts untouched (their old rows and blocks), and
  keys a front gains carry only appended rows — per dependency wave on the GPU, whose
  participants are the fronts holding a block of any cluster of the wave;
* the phase sequence: per stage the eliminations in ascending cluster order (the waves, in
  order, concatenate to exactly the oracle's elimination sequence), then scale /
  sparsify_rows / sparsify_cols inside the sparsification window, then merge.
"""
import numpy as np
import pytest

import oracle as O
from paper_2102_09878_b200.problems import random_full_rank, tall_grid

pytestmark = pytest.mark.gpu


def _P():
    import paper_2102_09878_b200 as P
    return P


def _related_fn(h):
    par = np.asarray(h["tree_parent"])
    node = [c["tree_node"] for c in h["clusters"]]
    anc = {}

    def ancestors(t):
        if t not in anc:
            s, u = set(), t
            while u >= 0:
                s.add(u)
                u = par[u]
            anc[t] = s
        return anc[t]

    def related(a, b):  # partition.cpp:223-229
        ta, tb = node[a], node[b]
        return ta in ancestors(tb) or tb in ancestors(ta)
    return related


def _run(A, **kw):
    snaps = []
    g = _P().Pipeline(A, observer=lambda ph, st, de, v: snaps.append((ph, st, de, v)), **kw)
    return g, snaps


def _invariant_violations(g, snaps):
    related = _related_fn(g.hierarchy())
    bad = []
    prev = None
    for ph, st, de, v in snaps:
        live = sum(len(f["rows"]) for f in v["fronts"].values())
        if live + v["pivots"] + v["dropped"] + v["trailing"] != g.M:
            bad.append(("rows", ph, st))
        for c, f in v["fronts"].items():
            for key, blk in f["blocks"].items():
                if key != c and blk.size and not related(c, key) and np.any(blk != 0.0):
                    bad.append(("coupling", ph, st, c, key))
        if ph == "eliminate" and prev is not None:
            wave = set(v["wave"])
            for c, nf in v["fronts"].items():
                of = prev["fronts"].get(c)
                if of is None or wave & set(of["blocks"]):
                    continue  # new front, or a participant of the wave
                onr = len(of["rows"])
                if len(nf["rows"]) < onr or not np.array_equal(nf["rows"][:onr], of["rows"]):
                    bad.append(("nonpart_rows", st, c))
                    continue
                for key, blk in of["blocks"].items():
                    if blk.shape[1] == 0:
                        continue
                    nb = nf["blocks"].get(key)
                    if nb is None or nb.shape[1] != blk.shape[1] or not np.array_equal(nb[:onr], blk):
                        bad.append(("nonpart_block", st, c, key))
                for key, blk in nf["blocks"].items():
                    if key not in of["blocks"] and blk.shape[1] > 0 and onr > 0 and np.any(blk[:onr] != 0.0):
                        bad.append(("fresh_key", st, c, key))
        prev = v
    return bad


@pytest.mark.parametrize("levels,eps,skip", [(2, 1e-2, 0), (2, 0.0, 0), (3, 1e-1, 1)])
def test_engine_invariants_at_every_phase(levels, eps, skip):
    """The reference test's configurations (test_factorize.cpp:404-407; its inverse-Poisson
    instance replaced by the tall grid, as in tests/test_ref_pins_oracle.py)."""
    p = tall_grid(12, seed=25)
    kw = dict(eps=eps, levels=levels, skip_levels=skip, coords=p.coords)
    g, snaps = _run(p.A, **kw)
    assert snaps, "observer never called"
    assert _invariant_violations(g, snaps) == []
    # phase pattern and elimination order against the oracle's observer
    o = O.Pipeline(p.A, check_invariants=True, **kw)
    assert o.violations == 0
    oph = o.phases()
    flat = []
    for ph, st, de, v in snaps:
        if ph == "eliminate":
            assert v["wave"] == sorted(v["wave"]) and de == v["wave"][0]
            flat += [("eliminate", st, c) for c in v["wave"]]
        else:
            flat.append((ph, st, -1))
    assert flat == [(a, b, c) for a, b, c in oph]
    # the final state accounts for every row
    last = snaps[-1][3]
    pr, dr, tr = g.rows()
    assert last["pivots"] + last["dropped"] + sum(len(f["rows"]) for f in last["fronts"].values()) + \
        last["trailing"] == g.M == len(pr) - (pr < 0).sum() + len(dr) + len(tr)


def test_engine_invariants_random_matrix():  # test_factorize.cpp:408 (random_full_rank, graph bisection)
    A = random_full_rank(140, 80, 4, seed=23)
    g, snaps = _run(A, eps=1e-2, levels=2, skip_levels=0)
    assert _invariant_violations(g, snaps) == []


def test_observer_via_spaqr_factorize_and_widths():
    """spaqr_factorize's observer: the active widths after sparsify_cols are the stage's
    interface widths (StageStats.front_cols), and the observer sees the same phases as the
    pipeline's."""
    p = tall_grid(24, seed=3)
    g, snaps_p = _run(p.A, eps=1e-2, levels=5, skip_levels=1, coords=p.coords)
    snaps = []
    F = _P().spaqr_factorize(g.scaled(), g.hierarchy(), g.owner(), eps=1e-2, skip_levels=1,
                             observer=lambda ph, st, de, v: snaps.append((ph, st, de, v)))
    assert [(a, b, c) for a, b, c, _ in snaps] == [(a, b, c) for a, b, c, _ in snaps_p]
    stages = {s["stage"]: s for s in F.stages()}
    for ph, st, de, v in snaps:
        if ph == "sparsify_cols":
            widths = [len(v["cols"][c]) for c in sorted(v["fronts"]) if len(v["cols"][c]) > 0]
            assert widths == list(stages[st]["front_cols"])
