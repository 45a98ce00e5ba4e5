"""Hybrid cost model evaluation, Eq. 9 (TEST INFRASTRUCTURE).

  T(X) = RF(X)  if s <= max(s_profile)      (interpolation)
         PR(X)  if s >  max(s_profile)      (extrapolation)

* RF: mean of the exported regression trees ("mean aggregation";
  50 trees, depth 10, seed 42 per PAPER.md:287, 331).  Each tree is walked as
  written: go left iff x[feature] <= threshold, leaf value at the end.
* PR: least squares polynomial of degree 1..3 chosen by AIC,
  fitted in x = s / scale (R-26), AIC = n ln(max(RSS/n, 1e-12 var(y))) + 2k,
  k = degree + 1, ties -> lowest degree.
* The bundle is read from the text format documented in include/paradyse.h
  (pds_load_costs).  This reader is the oracle's own.

Pins (tests/test_oracle_costmodel.py): forest evaluation == sklearn
RandomForestRegressor.predict (an independent library routine) on random
probes; AIC picks degree 1 on exactly linear and 2 on exactly quadratic data
(hand-computed AIC); Eq. 9 boundary at s_profile_max and +1
(SPEC.md:328-329).  "parity unpinned": the paper's own RF predictions (no data).
"""
from __future__ import annotations

import numpy as np


def features(pi, enabled, h, n, L, s, norm):
    """One-hot over the enabled set (R-25) + normalised (h, n, L) + s."""
    oh = [1.0 if e == pi else 0.0 for e in sorted(enabled)]
    (h0, h1), (n0, n1), (l0, l1), (s0, s1) = norm
    def nz(v, a, b):
        return 0.0 if b == a else (v - a) / (b - a)
    return np.array(oh + [nz(h, h0, h1), nz(n, n0, n1), nz(L, l0, l1), nz(s, s0, s1)])


def tree_predict(tree, x):
    node = 0
    while tree["left"][node] >= 0:
        if x[tree["feature"][node]] <= tree["threshold"][node]:
            node = tree["left"][node]
        else:
            node = tree["right"][node]
    return tree["value"][node]


def forest_predict(trees, x):
    acc = 0.0
    for tr in trees:
        acc += tree_predict(tr, x)
    return acc / len(trees)


def poly_eval(coef, scale, s):
    """numpy polyfit order: highest degree first (Horner)."""
    x = s / scale
    acc = 0.0
    for c in coef:
        acc = acc * x + c
    return acc


def aic(y, yhat, k):
    n = len(y)
    rss = float(np.sum((np.asarray(y) - np.asarray(yhat)) ** 2))
    floor = 1e-12 * float(np.var(y)) if np.var(y) > 0 else 1e-300
    return n * np.log(max(rss / n, floor)) + 2 * k


def nondecreasing(coef, x0, x1, grid=4097):
    """Reading R-26b's admissibility, checked the plain way: the derivative is >= 0 at
    every point of a fine grid on [x0, x1] (plus both ends)."""
    d = np.polyder(np.asarray(coef, dtype=np.float64))
    xs = np.linspace(x0, x1, grid)
    return bool(np.all(np.polyval(d, xs) >= -1e-15 * max(1.0, float(np.max(np.abs(d))))))


def fit_poly(s, y, scale=None, degrees=(1, 2, 3), s_extrap_max=None):
    """Degree 1..3 by AIC.  s_extrap_max (reading R-26b): only
    degrees whose fit is non-decreasing on [min s, s_extrap_max] are candidates."""
    s = np.asarray(s, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    scale = float(s.max()) if scale is None else scale
    x = s / scale
    best = None
    for d in degrees:
        if len(np.unique(x)) < d + 1:
            continue
        coef = np.polyfit(x, y, d)
        if s_extrap_max is not None and not nondecreasing(coef, float(x.min()), s_extrap_max / scale):
            continue
        a = aic(y, np.polyval(coef, x), d + 1)
        if best is None or a < best[0] - 1e-12:
            best = (a, d, coef)
    if best is None:
        raise ValueError("fit_poly: insufficient points (SPEC.md:317)")
    return best[1], best[2], scale


def predict_time(entry, x_feat, s):
    """Eq. 9 dispatch; returns (value, branch)."""
    if s <= entry["s_profile_max"]:
        return forest_predict(entry["trees"], x_feat), "rf"
    return poly_eval(entry["poly_coef"], entry["poly_scale"], s), "pr"


def read_bundle(path):
    """Parse the `pds_bundle 1` text format (include/paradyse.h)."""
    tok = open(path).read().split()
    it = iter(tok)
    def nxt():
        return next(it)
    assert nxt() == "pds_bundle" and nxt() == "1"
    hdr = {}
    for _ in range(7):
        k = nxt()
        hdr[k] = int(nxt()) if k not in ("capacity", "reserve") else float(nxt())
    k = nxt()
    if k == "kv":                     # optional Llama-variant fields (R-GQA / R-SWIGLU)
        hdr["kv"] = int(nxt())
        assert nxt() == "act"
        hdr["act"] = int(nxt())
        k = nxt()
    norm = []
    assert k == "norm"
    for _ in range(4):
        norm.append((float(nxt()), float(nxt())))
    assert nxt() == "n_strat"
    ns = int(nxt())
    strat = {}
    for _ in range(ns):
        assert nxt() == "strategy"
        sid = int(nxt())
        e = {}
        assert nxt() == "s_profile_max"
        e["s_profile_max"] = float(nxt())
        assert nxt() == "poly"
        deg = int(nxt())
        e["poly_scale"] = float(nxt())
        e["poly_coef"] = [float(nxt()) for _ in range(deg + 1)]
        assert nxt() == "trees"
        nt = int(nxt())
        trees = []
        for _ in range(nt):
            assert nxt() == "tree"
            nn = int(nxt())
            tr = dict(feature=[], threshold=[], left=[], right=[], value=[])
            for _ in range(nn):
                tr["feature"].append(int(nxt()))
                tr["threshold"].append(float(nxt()))
                tr["left"].append(int(nxt()))
                tr["right"].append(int(nxt()))
                tr["value"].append(float(nxt()))
            trees.append(tr)
        e["trees"] = trees
        strat[sid] = e
    assert nxt() == "end"
    return dict(hdr=hdr, norm=norm, strat=strat)
