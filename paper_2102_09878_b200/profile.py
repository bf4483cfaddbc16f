"""Run profile document (the reference's make_profile / validate_profile,
proj/src/profile.cpp:42-188, schema proj/docs/profile.schema.json).

make_profile(pipeline, report) builds the version-1 JSON document from a
pipeline's per-stage statistics (StageStats: phase times, interface widths and
aspect ratios, top separator size, nnz(W)) and a solve report.  The B200
pipeline adds one extra top-level object, "device", with the CUDA-event time,
algorithmic bytes and launch count of every kernel family; the reference's
validator ignores unknown keys, so the document stays valid for both.

validate_profile(text) restates the reference's checker and returns "" for a
valid document or the reference's error message for the first problem found.
"""
from __future__ import annotations

import json
import math

SOLVER_NAMES = ("spaqr", "direct", "diag")


def _quartiles(values):
    """Linear-interpolation quantiles of an unsorted sample, 0 for an empty one (profile.cpp:15-26)."""
    v = sorted(float(x) for x in values)

    def q(p):
        if not v:
            return 0.0
        pos = p * (len(v) - 1)
        lo = int(math.floor(pos))
        hi = min(lo + 1, len(v) - 1)
        frac = pos - lo
        return (1.0 - frac) * v[lo] + frac * v[hi]

    return {"min": q(0.0), "q1": q(0.25), "median": q(0.5), "q3": q(0.75), "max": q(1.0)}


def make_profile(p, report=None, eps=None, skip=3, solver="spaqr", tol=1e-12, maxit=500):
    """JSON text of the run profile for pipeline `p` (the B200 Pipeline or the oracle's),
    `report` = the dict returned by p.solve(...) or None."""
    stages = p.stages() if solver != "diag" else []
    levels = []
    for st in stages:
        levels.append({"stage": int(st["stage"]), "factorize": float(st["t_eliminate"]),
                       "reassign": float(st["t_reassign"]), "scale": float(st["t_scale"]),
                       "sparsify": float(st["t_sparsify"]), "merge": float(st["t_merge"]),
                       "interface_cols": _quartiles(st["front_cols"]), "aspect": _quartiles(st["front_aspect"]),
                       "top_rows": int(st["top_rows"]), "top_cols": int(st["top_cols"]), "nnz_w": int(st["nnz_w"])})
    t = p.times()
    doc = {
        "version": 1,
        "matrix": {"rows": int(p.M), "cols": int(p.N), "nnz": int(getattr(p, "nnz_A", 0) or getattr(p, "nnz", 0))},
        "options": {"eps": float(eps if eps is not None else getattr(p, "eps", 0.0)),
                    "levels": int(p.L) if stages else 0, "skip": int(skip), "solver": solver, "tol": float(tol),
                    "maxit": int(maxit)},
        "levels": levels,
        "totals": {"t_partition": float(t["t_partition"]), "t_factorize": float(t["t_factorize"]),
                   "t_solve": float(report["t_solve"]) if report else 0.0, "nnz_w": int(p.nnz_w),
                   "dropped_rows": int(p.ndropped), "trailing_rows": int(p.ntrailing)},
        "solve": {"iterations": int(report["iterations"]) if report else 0,
                  "converged": bool(report["converged"]) if report else False,
                  "residuals": [float(r) for r in report["residual_history"]] if report else []},
    }
    if hasattr(p, "kernel_stats"):
        doc["device"] = {k: {"ms": v["ms"], "bytes": v["bytes"], "launches": v["launches"]}
                         for k, v in p.kernel_stats().items()}
        doc["device"]["factorize_event_ms"] = float(t.get("factorize_event_ms", 0.0))
        doc["device"]["solve_event_ms"] = float(t.get("solve_event_ms", 0.0))
    return json.dumps(doc, indent=2) + "\n"


def _need(j, key, kind, where):
    if not isinstance(j, dict) or key not in j:
        return f"{where}: missing '{key}'"
    v = j[key]
    if kind == "num":
        ok = isinstance(v, (int, float)) and not isinstance(v, bool)
    elif kind == "int":
        ok = isinstance(v, int) and not isinstance(v, bool)
    else:
        ok = isinstance(v, str)
    return "" if ok else f"{where}: '{key}' has the wrong type"


def validate_profile(text):
    """"" when `text` is a valid version-1 profile, else the first error (profile.cpp:116-188)."""
    try:
        j = json.loads(text)
    except ValueError:
        return "profile: not valid JSON"
    for k in ("version", "matrix", "options", "levels", "totals", "solve"):
        if not isinstance(j, dict) or k not in j:
            return f"profile: missing '{k}'"
    if j["version"] != 1:
        return "profile: unsupported version"
    for k in ("rows", "cols", "nnz"):
        e = _need(j["matrix"], k, "int", "matrix")
        if e:
            return e
    o = j["options"]
    for k in ("eps", "tol"):
        e = _need(o, k, "num", "options")
        if e:
            return e
    for k in ("levels", "skip", "maxit"):
        e = _need(o, k, "int", "options")
        if e:
            return e
    e = _need(o, "solver", "str", "options")
    if e:
        return e
    if not isinstance(j["levels"], list):
        return "profile: 'levels' is not an array"
    for lv in j["levels"]:
        for k in ("factorize", "reassign", "scale", "sparsify", "merge"):
            e = _need(lv, k, "num", "levels[]")
            if e:
                return e
            if lv[k] < 0.0:
                return f"levels[]: negative phase time '{k}'"
        for k in ("stage", "top_rows", "top_cols", "nnz_w"):
            e = _need(lv, k, "int", "levels[]")
            if e:
                return e
        for k in ("interface_cols", "aspect"):
            if k not in lv or not isinstance(lv[k], dict):
                return f"levels[]: missing object '{k}'"
            for qk in ("min", "q1", "median", "q3", "max"):
                e = _need(lv[k], qk, "num", k)
                if e:
                    return e
    t = j["totals"]
    for k in ("t_partition", "t_factorize", "t_solve"):
        e = _need(t, k, "num", "totals")
        if e:
            return e
        if t[k] < 0.0:
            return f"totals: negative time '{k}'"
    for k in ("nnz_w", "dropped_rows", "trailing_rows"):
        e = _need(t, k, "int", "totals")
        if e:
            return e
    s = j["solve"]
    e = _need(s, "iterations", "int", "solve")
    if e:
        return e
    if "converged" not in s or not isinstance(s["converged"], bool):
        return "solve: missing boolean 'converged'"
    if "residuals" not in s or not isinstance(s["residuals"], list):
        return "solve: missing array 'residuals'"
    return ""
