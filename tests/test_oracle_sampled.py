"""Pin of oracle/sampled.py (SURVEY O-9): the row-sampled oracle equals the full
unsharded oracle (oracle.layer, itself pinned by autograd / finite differences /
closed forms) with the same sparse cotangent, to 1e-12, at sizes the full oracle
finishes in a second.  A dropped term anywhere (a K/V row range, a missing dX1 on
rows R, the RoPE^T of dQ, the causal key limit) fails one of these."""
import numpy as np
import pytest

from oracle import layer as OL
from oracle import sampled as OS
from synth import layer_inputs


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("h,n,F,s,causal,R", [
    (64, 2, 256, 96, True, [0, 5, 40, 95]),
    (128, 4, 512, 256, True, [3, 100, 101, 200]),          # max R < s - 1: rows beyond get dX = 0
    (128, 2, 256, 128, False, [1, 64, 127]),
    (256, 4, 1024, 512, True, [0, 127, 128, 300, 511]),
])
def test_sampled_equals_full_oracle(h, n, F, s, causal, R):
    d = layer_inputs(h, n, F, s, 1, seed=5)
    R = np.array(R)
    dy = np.zeros((s, 1, h))
    dy[R, 0] = d["dy"][R, 0]
    y, c = OL.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], n=n,
                        causal=causal)
    g = OL.layer_bwd(dy, c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], n=n,
                     causal=causal)
    r = OS.sampled_layer(d["x"][:, 0], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], n,
                         R, dy[R, 0], causal=causal)
    assert _rel(r["y"], y[R, 0]) < 1e-12
    assert _rel(r["o"], c["o"][R, 0]) < 1e-12
    assert _rel(r["z"], c["z"][R, 0]) < 1e-12
    assert _rel(r["lse"], c["lse"][0][:, R]) < 1e-12
    assert _rel(r["dx"], g["dx"][:, 0]) < 1e-12
    for k in ("dw_qkv", "dw_proj", "dw_in", "dw_out", "dg1", "dg2"):
        assert _rel(r[k], g[k]) < 1e-12, k
    if causal and R.max() < s - 1:
        assert np.all(r["dx"][R.max() + 1:] == 0.0)


def test_sampled_rejects_unsorted_rows():
    d = layer_inputs(64, 2, 256, 64, 1, seed=1)
    with pytest.raises(AssertionError):
        OS.sampled_layer(d["x"][:, 0], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], 2,
                         [5, 3], np.zeros((2, 64)))


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("il", [False, True])
def test_sampled_llama_variant_equals_full_oracle(causal, il):
    """GQA + SwiGLU (R-GQA / R-SWIGLU) in the row-sampled oracle, plain and interleaved
    (the device's spec layout) W_in, against oracle.layer's full Llama layer."""
    from oracle.shard import il_perm
    h, n, n_kv, F, s = 128, 4, 2, 256, 256
    d = layer_inputs(h, n, F, s, 1, seed=8, n_kv=n_kv, act="swiglu")
    R = np.array([2, 77, 130, 250])
    dy = np.zeros((s, 1, h))
    dy[R, 0] = d["dy"][R, 0]
    kw = dict(n=n, causal=causal, n_kv=n_kv, act="swiglu")
    y, c = OL.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    g = OL.layer_bwd(dy, c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    pm = il_perm(F)
    w_in = d["w_in"][:, pm] if il else d["w_in"]
    r = OS.sampled_layer(d["x"][:, 0], d["w_qkv"], d["w_proj"], w_in, d["w_out"], d["g1"], d["g2"], n,
                         R, dy[R, 0], causal=causal, n_kv=n_kv, act="swiglu", il=il)
    assert _rel(r["y"], y[R, 0]) < 1e-12
    assert _rel(r["z"], c["z"][R, 0]) < 1e-12
    assert _rel(r["dx"], g["dx"][:, 0]) < 1e-12
    assert _rel(r["dw_in"], g["dw_in"][:, pm] if il else g["dw_in"]) < 1e-12
    for k in ("dw_qkv", "dw_proj", "dw_out", "dg1", "dg2"):
        assert _rel(r[k], g[k]) < 1e-12, k
