"""Pins for oracle/costmodel.py, flops.py, layouts.py and the synth generators."""
import math
import os

import numpy as np
import pytest

from oracle import costmodel as CM
from oracle import flops, layer, layouts
from synth import HIST, normal, round_bf16, sample_lengths

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- flops
def test_spec_flops_c1_is_2_pow_30():
    assert flops.spec_fwd_flops_noncausal(256, 512) == 2 ** 30
    # s-doubling: attention term x4, linear terms x2
    f1 = flops.spec_fwd_flops_noncausal(256, 512)
    f2 = flops.spec_fwd_flops_noncausal(256, 1024)
    assert f2 - 2 * f1 == 2 * (4 * 1024 ** 2 * 256 - 2 * 4 * 512 ** 2 * 256) // 2


def test_flops_match_executed_matmul_shapes():
    # count 2 m n k over the matmuls oracle.layer actually executes (non-causal)
    h, n, F, s = 16, 2, 64, 12
    from synth import layer_inputs
    d = layer_inputs(h, n, F, s)
    y, c = layer.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"],
                           d["g2"], n=n, causal=False)
    mm = 0
    mm += 2 * s * c["qkv"].shape[-1] * h          # U W_qkv
    dh = h // n
    mm += n * (2 * s * s * dh) * 2                # QK^T and PV per head
    mm += 2 * s * h * h                           # A W_proj
    mm += 2 * s * c["h"].shape[-1] * h           # V2 W_in
    mm += 2 * s * h * c["g"].shape[-1]            # G W_out
    assert mm == flops.spec_fwd_flops_noncausal(h, s)
    assert flops.layer_flops(h, s, F, causal=False) == 3 * mm
    # causal model FLOPs per token: 72 h^2 + 6 s h at F = 4h (SURVEY O-7)
    assert flops.layer_flops_per_token(4096, 4096) == 72 * 4096 ** 2 + 6 * 4096 * 4096


# ---------------------------------------------------------------- layouts
def test_table2_fixture():
    rows = [l.strip().split("|") for l in open(os.path.join(GOLD, "table2.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 8
    for r in rows:
        assert tuple(r[1:]) == layouts.TABLE2[r[0]], r[0]


def test_spec_layout_examples_and_closure():
    assert layouts.spec_layout("act", 1024, 4, s=8)[0] == (1, 2, 1024)
    assert layouts.spec_layout("w_qkv", 1024, 4)[0] == (768, 1024)
    assert layouts.spec_layout("w_out", 1024, 1)[0] == (4096, 1024)
    spec = layouts.TABLE2["Specification"]
    for a in layouts.STRATEGY_LAYOUT.values():
        for b in layouts.STRATEGY_LAYOUT.values():
            assert layouts.compatible(layouts.TABLE2[a], layouts.TABLE2[b])
    assert not layouts.compatible(layouts.TABLE2["Megatron-LM TP"][0], spec[0])
    with pytest.raises(ValueError):
        layouts.spec_layout("act", 64, 3, s=8)


# ---------------------------------------------------------------- cost model
def test_aic_degree_selection():
    s = np.array([1024, 2048, 4096, 8192, 16384, 32768], dtype=float)
    d, coef, sc = CM.fit_poly(s, 3.0 + 2e-4 * s)
    assert d == 1
    d, coef, sc = CM.fit_poly(s, 1.0 + 1e-4 * s + 3e-9 * s * s)
    assert d == 2
    # hand-computed AIC on exactly quadratic data: degree-1 residual is large
    x = s / sc
    c1 = np.polyfit(x, 1.0 + 1e-4 * s + 3e-9 * s * s, 1)
    y = 1.0 + 1e-4 * s + 3e-9 * s * s
    rss1 = float(np.sum((np.polyval(c1, x) - y) ** 2))
    assert CM.aic(y, np.polyval(c1, x), 2) == pytest.approx(6 * math.log(rss1 / 6) + 4)
    with pytest.raises(ValueError):
        CM.fit_poly([5.0], [1.0])


def _write_bundle(path, forests, polys, smax, norm):
    with open(path, "w") as f:
        f.write("pds_bundle 1\nP 1 h 64 n 4 ffn 256 L 4 capacity 1e9 reserve 0\n")
        f.write("norm " + " ".join(f"{a!r} {b!r}" for a, b in norm) + "\n")
        f.write(f"n_strat {len(forests)}\n")
        for sid, rf in forests.items():
            deg, coef, sc = polys[sid]
            f.write(f"strategy {sid} s_profile_max {smax!r} poly {deg} {sc!r} "
                    + " ".join(repr(float(c)) for c in coef) + "\n")
            f.write(f"trees {len(rf.estimators_)}\n")
            for est in rf.estimators_:
                tr = est.tree_
                f.write(f"tree {tr.node_count}\n")
                for i in range(tr.node_count):
                    f.write(f"{int(tr.feature[i])} {float(tr.threshold[i])!r} "
                            f"{int(tr.children_left[i])} {int(tr.children_right[i])} "
                            f"{float(tr.value[i].ravel()[0])!r}\n")
        f.write("end\n")


def test_forest_eval_matches_sklearn_and_eq9(tmp_path):
    from sklearn.ensemble import RandomForestRegressor
    rng = np.random.default_rng(0)
    s = np.sort(rng.integers(512, 32768, size=40)).astype(float)
    norm = [(64, 64), (4, 4), (4, 4), (float(s.min()), float(s.max()))]
    feats = np.stack([CM.features(0, [0, 1], 64, 4, 4, v, norm) for v in s])
    y = 1e-3 * s + 1e-8 * s * s + rng.normal(0, 0.01, size=s.size)
    rf = RandomForestRegressor(n_estimators=50, max_depth=10, random_state=42).fit(feats, y)
    rf2 = RandomForestRegressor(n_estimators=50, max_depth=10, random_state=42).fit(feats, y)
    probes = np.stack([CM.features(0, [0, 1], 64, 4, 4, v, norm)
                       for v in rng.uniform(512, 32768, size=50)])
    assert np.array_equal(rf.predict(probes), rf2.predict(probes))
    path = tmp_path / "b.txt"
    _write_bundle(path, {0: rf, 1: rf2}, {0: CM.fit_poly(s, y), 1: CM.fit_poly(s, y)},
                  float(s.max()), norm)
    b = CM.read_bundle(str(path))
    ours = np.array([CM.forest_predict(b["strat"][0]["trees"], p) for p in probes])
    ref = rf.predict(probes)
    assert np.max(np.abs(ours - ref) / np.abs(ref)) < 1e-12
    e = b["strat"][0]
    f_at = CM.features(0, [0, 1], 64, 4, 4, s.max(), norm)
    assert CM.predict_time(e, f_at, s.max())[1] == "rf"
    assert CM.predict_time(e, f_at, s.max() + 1)[1] == "pr"


# ---------------------------------------------------------------- synth
def test_generator_counter_property_and_bf16():
    a = normal(42, 1, (1000,))
    b = normal(42, 1, (2000,))
    assert np.array_equal(a, b[:1000])               # counter-based: prefix-stable
    assert np.array_equal(round_bf16(a), a)
    assert abs(a.mean()) < 0.1 and abs(a.std() - 1) < 0.1


def test_dataset_histograms():
    # Table 3: empirical frequencies within 2% at 1e4 samples
    for name in ("githubcode", "grch38"):
        pct, smax = HIST[name]
        lens = sample_lengths(name, 10000, seed=42)
        assert lens.max() <= smax
        edges = [0, 4096, 8192, 16384, 32768, 65536, 131072, 10 ** 9]
        cnt = np.histogram(lens, bins=edges)[0] / len(lens)
        p = np.asarray(pct) / np.sum(pct)
        assert np.all(np.abs(cnt - p) < 0.02), (name, cnt, p)
    assert np.isclose(sum(HIST["grch38"][0]), 99.1)   # renormalised (R-29)


def test_table5_saving_and_case_study():
    # context pins: Saving = (Time - Time_full) / Time for every Table 5 row
    rows = [(3173.80, 2799.45, 11.80), (2795.91, 2799.45, -0.13), (2813.13, 2799.45, 0.49),
            (1741.99, 1724.13, 1.03), (2657.04, 2622.89, 1.29), (2800.49, 2799.45, 0.04)]
    for t, tf, sv in rows:
        assert round(100 * (t - tf) / t, 2) == sv
    assert math.isclose(329728 / 117248 - 1, 1.8122, rel_tol=1e-4)
    total = 2.5 + 5 + 22 + 1
    assert 30.5 <= total <= 31.5 and abs(22 / 31.3 - 0.702) < 1e-3


def test_nondecreasing_pins():
    # reading R-26b's admissibility on closed forms (numpy coefficient order)
    assert CM.nondecreasing([1.0, 0.0], 0.0, 10.0)              # x
    assert not CM.nondecreasing([-1.0, 0.0], 0.0, 10.0)         # -x
    assert not CM.nondecreasing([1.0, -1.0, 0.0], 0.0, 1.0)     # x^2 - x falls on [0, 1/2)
    assert CM.nondecreasing([1.0, -1.0, 0.0], 0.5, 3.0)         # ... and rises after
    assert CM.nondecreasing([1.0, 0.0, 0.0, 0.0], -1.0, 1.0)    # x^3: derivative 3x^2 >= 0
    assert not CM.nondecreasing([-1.0, 3.0, 0.0, 0.0], 0.0, 4.0)  # -x^3 + 3x^2: falls past x = 2
    assert CM.nondecreasing([-1.0, 3.0, 0.0, 0.0], 0.0, 2.0)


def test_fit_poly_monotone_reading():
    # a noisy-looking cubic whose leading coefficient is negative extrapolates to a
    # falling (eventually negative) time: not admissible under R-26b, degree 2 is chosen
    s = np.array([1024, 2048, 4096, 8192, 16384, 32768, 65536], dtype=float)
    x = s / s.max()
    y = 0.001 + 0.05 * x + 0.12 * x * x - 0.03 * x ** 3
    d, coef, sc = CM.fit_poly(s, y)
    assert d == 3 and coef[0] < 0                          # plain AIC (exact cubic)
    d, coef, sc = CM.fit_poly(s, y, s_extrap_max=float(1 << 20))
    assert d in (1, 2) and CM.nondecreasing(coef, x.min(), (1 << 20) / sc)
    d2, _, _ = CM.fit_poly(s, y, degrees=(1, 2), s_extrap_max=float(1 << 20))
    assert d2 == d
