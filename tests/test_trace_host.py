"""Host logic of the trace / ablation harness (paper_2511_13198_b200/trace.py): Table 5
columns, switching statistics, and the "w/o RF" bundle (Eq. 9
with every length on the polynomial branch)."""
import os

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
        _, branch = OC.predict_time(e, [0.0] * 9, 1024)
        assert branch == "pr"
        _, branch = OC.predict_time(f, [0.0] * 9, 1024)
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
