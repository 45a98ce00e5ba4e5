"""Host logic of the trace / ablation harness (paper_2511_13198_b200/trace.py): Table 5
columns, switching statistics, and the "w/o RF" bundle (Eq. 9
with every length on the polynomial branch)."""
import os

import pytest

from oracle import costmodel as OC
from paper_2511_13198_b200 import trace as T

BUNDLE = os.path.join(os.path.dirname(T.__file__), "bundles", "h4096_n32_f16384_P1.txt")


def test_pr_only_bundle_takes_polynomial_everywhere():
    full = OC.read_bundle(BUNDLE)
    pr = OC.read_bundle(T.pr_only_bundle(BUNDLE))
    for sid, e in pr["strat"].items():
        assert e["s_profile_max"] == 0.0
        f = full["strat"][sid]
        assert e["poly_coef"] == f["poly_coef"] and e["poly_scale"] == f["poly_scale"]
        nf = len(full["strat"]) + 4                 # one-hot over the bundle's strategies + (h, n, L, s)
        _, branch = OC.predict_time(e, [0.0] * nf, 1024)
        assert branch == "pr"
        _, branch = OC.predict_time(f, [0.0] * nf, 1024)
        assert branch == "rf"


def test_switching_counts():
    recs = [{"s": 1, "plan": "TTTT"}, {"s": 2, "plan": "TTTT"}, {"s": 3, "plan": "TMMM"},
            {"s": 4, "plan": "UMUM"}, {"s": 5, "oom": True}]
    sw = T.switches(recs)
    assert sw == {"plan_changes_between_sequences": 2, "strategy_boundaries_inside_plans": 1 + 3}


def test_time_full_at_and_saving():
    # Table 5 semantics: Time_full = full's cumulative time up to the variant's Seq_len
    full = {"records": [{"s": 10, "cum": 1.0}, {"s": 20, "cum": 3.0}, {"s": 30, "cum": 6.0},
                        {"s": 40, "oom": True}]}
    assert T.time_full_at(full, 20) == 3.0
    assert T.time_full_at(full, 25) == 3.0
    assert T.time_full_at(full, 99) == 6.0
    # the paper's own rows reproduce with Saving = (Time - Time_full) / Time
    for time, tf, saving in ((3173.80, 2799.45, 0.1180), (2795.91, 2799.45, -0.0013), (1741.99, 1724.13, 0.0103)):
        assert abs((time - tf) / time - saving) < 5e-4


def test_bucket_edges():
    assert T.bucket_of(4095) == 0 and T.bucket_of(4096) == 1 and T.bucket_of(131072) == 6


def test_committed_bundles_extrapolate_monotonically():
    """Reading R-26b on the shipped bundles: every strategy's PR branch is positive and
    non-decreasing from s_profile_max to 2^20 (beyond 624K), and the product's fit
    (calibrate.aic_poly) equals the oracle's (degrees 1..2, non-decreasing filter) on the
    stored profile records."""
    import json
    import numpy as np
    from paper_2511_13198_b200 import calibrate as CAL
    for P in (1, 2, 4, 8):
        path = os.path.join(os.path.dirname(T.__file__), "bundles", f"h4096_n32_f16384_P{P}.txt")
        b = OC.read_bundle(path)
        recs = json.load(open(path + ".json"))["records"]
        for sid, e in b["strat"].items():
            ss = np.linspace(e["s_profile_max"], float(1 << 20), 257)
            t = [OC.poly_eval(e["poly_coef"], e["poly_scale"], s) for s in ss]
            assert min(t) > 0 and all(b2 >= a2 for a2, b2 in zip(t, t[1:])), (P, sid)
            s_rec = [r[0] for r in recs[str(sid)]]
            y_rec = [r[1] for r in recs[str(sid)]]
            d, coef, sc = OC.fit_poly(s_rec, y_rec, degrees=(1, 2), s_extrap_max=float(1 << 20))
            d2, coef2, sc2 = CAL.aic_poly(s_rec, y_rec)
            assert d == d2 and sc == sc2 and np.allclose(coef, coef2, rtol=1e-12, atol=0), (P, sid)
            assert np.allclose(coef, e["poly_coef"], rtol=1e-12, atol=0), (P, sid)


def test_predicted_trace_adaptive_never_slower_than_a_static_strategy():
    """--predict (host-only contexts, no GPU): with gamma = 0 the adaptive plan is the
    least-time feasible plan of Algorithm 1's candidate space, which contains every
    feasible uniform plan, so per sequence its predicted time is <= every static
    strategy that can run that sequence, and it trains at least as long."""
    from paper_2511_13198_b200 import binding as B
    model = B.Model(h=4096, n_heads=32, ffn=16384, n_layers=32)
    for P in (1, 8):
        path = os.path.join(os.path.dirname(T.__file__), "bundles", f"h4096_n32_f16384_P{P}.txt")
        lens = [8192 * k for k in (1, 2, 3, 5, 8, 13, 21, 34, 55, 78)]
        ad = T.predict_trace(B, model, path, lens, 32, 0.0)
        t_ad = {r["s"]: r["seconds"] for r in ad["records"] if "seconds" in r}
        for name, pi in T.STATIC:
            st = T.predict_trace(B, model, path, lens, 32, 0.0, fixed=pi)
            assert ad["max_s_trained"] >= st["max_s_trained"], (P, name)
            for r in st["records"]:
                if "seconds" in r:
                    assert t_ad[r["s"]] <= r["seconds"] * (1 + 1e-12), (P, name, r["s"])


def test_planner_crossovers_at_p8():
    """The selector's value at P = 8 (host-only context, committed P = 8 bundle, the
    bundle's per-GPU capacity): short sequences run uniformly on the fastest strategy,
    the 624K sequence (north_star) gets a feasible plan that must mix in a
    memory-saving strategy (no static time-optimal plan fits), and the L = 32 frontier
    of the adaptive plan exceeds every static strategy's."""
    from paper_2511_13198_b200 import binding as B
    model = B.Model(h=4096, n_heads=32, ffn=16384, n_layers=32)
    path = os.path.join(os.path.dirname(T.__file__), "bundles", "h4096_n32_f16384_P8.txt")
    ctx = B.Context(model, P=8, device=-1)
    ctx.load_costs(path)
    t_short = ctx.cost_eval(8192)[0]
    plan, flags = ctx.plan(8192, 32)
    assert not flags & B.PLAN_INFEASIBLE
    assert len(set(plan)) == 1 and t_short[plan[0]] == min(t for i, t in enumerate(t_short) if i in set(plan) | {0})
    plan, flags = ctx.plan(638976, 32)
    assert not flags & B.PLAN_INFEASIBLE
    assert set(plan) & {B.METP, B.METP_FULL}
    ctx.close()
    unit = 128 * 64
    fr = {pi: T.predict_frontier(B, model, path, 32, unit, fixed=pi)["s"] for pi in range(B.N_STRATEGIES)}
    ad = T.predict_frontier(B, model, path, 32, unit)["s"]
    assert ad >= 638976 and all(ad >= v for v in fr.values())


@pytest.mark.parametrize("n_kv,act", [(None, 0), (8, 0), (8, 1), (32, 1)])
def test_calibrate_comm_model_equals_oracle_formula(n_kv, act):
    """The modelled bundles' collective bytes (calibrate.comm_bytes_per_rank) equal the
    oracle's formula (oracle/flops.comm_bytes, itself pinned to the simulated comm logs),
    MHA and the Llama variant, every strategy, P = 2 / 4 / 8."""
    from oracle import flops as OF
    from paper_2511_13198_b200 import calibrate as CAL
    h, n, F = 4096, 32, 11264
    for P in (2, 4, 8):
        for s in (8192, 65536):
            for pi in range(6):
                got = CAL.comm_bytes_per_rank(pi, h, F, s, P, n, n_kv, act)
                ref = OF.comm_bytes(pi, h, s, P, F, n=n, n_kv=n_kv, act="swiglu" if act else "gelu")
                assert got == pytest.approx(ref, rel=1e-12, abs=1.0), (pi, P, s)
