"""Pins for oracle/layer.py against what the paper and mathematics fix."""
import math

import numpy as np
import pytest
import torch

from oracle import layer as L
from synth import layer_inputs


def _inputs(h=16, n=2, ffn=64, s=8, b=1, seed=3):
    d = layer_inputs(h, n, ffn, s, b, seed=seed)
    return d


def test_attention_single_token_is_v():
    # s = 1 => softmax over one key is 1, attention output = V
    rng = np.random.default_rng(0)
    q, k, v = rng.normal(size=(3, 1, 8))
    a, lse = L.attention_fwd(q, k, v)
    assert np.array_equal(a, v)
    assert np.isclose(lse[0], float(q[0] @ k[0]) / math.sqrt(8))


def test_attention_identical_keys_is_causal_prefix_mean():
    # identical keys => constant scores => uniform weights over the causal prefix,
    # A_t = mean(V[0..t]) and LSE_t = log(t+1) + q_t.k / sqrt(d) (closed form)
    rng = np.random.default_rng(1)
    s, d = 13, 8
    q = rng.normal(size=(s, d))
    k = np.tile(rng.normal(size=(1, d)), (s, 1))
    v = rng.normal(size=(s, d))
    a, lse = L.attention_fwd(q, k, v, causal=True, block=4)
    for t in range(s):
        assert np.allclose(a[t], v[: t + 1].mean(axis=0), atol=1e-13)
        assert np.isclose(lse[t], math.log(t + 1) + q[t] @ k[0] / math.sqrt(d), atol=1e-13)
    a2, _ = L.attention_fwd(q, k, v, causal=False)
    assert np.allclose(a2, np.tile(v.mean(axis=0), (s, 1)), atol=1e-13)


def test_attention_naive_loops():
    # a hand-rolled loop oracle on s <= 4 agrees to 1e-12
    rng = np.random.default_rng(2)
    s, d = 4, 6
    q, k, v = rng.normal(size=(3, s, d))
    a, _ = L.attention_fwd(q, k, v, causal=True, block=2)
    for t in range(s):
        w = [math.exp(sum(q[t, j] * k[u, j] for j in range(d)) / math.sqrt(d)) for u in range(t + 1)]
        z = sum(w)
        for j in range(d):
            ref = sum(w[u] * v[u, j] for u in range(t + 1)) / z
            assert abs(a[t, j] - ref) < 1e-12


def test_rope_identity_at_zero_and_relative():
    d = 16
    rng = np.random.default_rng(4)
    x = rng.normal(size=(1, d))
    c, s = L.rope_cos_sin([0], d)
    assert np.array_equal(L.rope_apply(x, c, s), x)
    # q.k after RoPE depends only on the position difference (rotation property)
    q, k = rng.normal(size=(2, 1, d))
    def dot(tq, tk):
        cq, sq = L.rope_cos_sin([tq], d)
        ck, sk = L.rope_cos_sin([tk], d)
        return float(L.rope_apply(q, cq, sq)[0] @ L.rope_apply(k, ck, sk)[0])
    assert np.isclose(dot(7, 3), dot(1007, 1003), atol=1e-9)
    assert np.isclose(dot(5, 5), float(q[0] @ k[0]), atol=1e-12)
    # complex view: pair (x_k, x_{k+d/2}) is multiplied by exp(i t theta^(-2k/d))
    t = 11
    c1, s1 = L.rope_cos_sin([t], d)
    r = L.rope_apply(x, c1, s1)[0]
    for kk in range(d // 2):
        z = complex(x[0, kk], x[0, kk + d // 2]) * np.exp(1j * t * 10000.0 ** (-2 * kk / d))
        assert np.isclose(r[kk], z.real) and np.isclose(r[kk + d // 2], z.imag)
    # backward is the transpose rotation: <R x, y> == <x, R^T y>
    y = rng.normal(size=(1, d))
    assert np.isclose(float(L.rope_apply(x, c1, s1)[0] @ y[0]),
                      float(x[0] @ L.rope_apply_t(y, c1, s1)[0]))


def test_rmsnorm_and_gelu_closed_forms():
    from scipy.stats import norm
    rng = np.random.default_rng(5)
    x = rng.normal(size=(5, 1, 32)) * 3
    u, xhat, r = L.rmsnorm(x, np.ones(32), eps=0.0)
    assert np.allclose(np.mean(u * u, axis=-1), 1.0)
    u2, _, _ = L.rmsnorm(7.0 * x, np.ones(32), eps=0.0)   # scale invariance
    assert np.allclose(u, u2)
    z = np.linspace(-6, 6, 101)
    assert np.allclose(L.gelu(z), z * norm.cdf(z), atol=1e-15)
    assert np.allclose(L.gelu_grad(z), norm.cdf(z) + z * norm.pdf(z), atol=1e-14)


def test_zero_w_in_gives_zero_z():
    # W_in = 0 => Z = GELU(0) W_out = 0 and Y = X1
    d = _inputs()
    y, c = L.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], np.zeros_like(d["w_in"]), d["w_out"],
                       d["g1"], d["g2"], n=2)
    assert np.array_equal(c["z"], np.zeros_like(c["z"]))
    assert np.array_equal(y, c["x1"])


def _torch_layer(x, w_qkv, w_proj, w_in, w_out, g1, g2, n, causal=True, eps=1e-5):
    """Independent torch fp64 implementation from library routines
    (F.rms_norm, F.scaled_dot_product_attention, F.gelu)."""
    import torch.nn.functional as F
    s, b, h = x.shape
    d = h // n
    def norm(t, g):
        return F.rms_norm(t, (h,), g, eps=eps)
    u = norm(x, g1)
    qkv = u @ w_qkv
    q, k, v = qkv.split(h, dim=-1)
    def heads(t):
        return t.reshape(s, b, n, d).permute(1, 2, 0, 3)
    q, k, v = heads(q), heads(k), heads(v)
    pos = torch.arange(s, dtype=torch.float64)
    inv = 10000.0 ** (-2 * torch.arange(d // 2, dtype=torch.float64) / d)
    ang = pos[:, None] * inv[None, :]
    cos = torch.cat([ang.cos(), ang.cos()], -1)
    sin = torch.cat([ang.sin(), ang.sin()], -1)
    def rot(t):
        t1, t2 = t[..., : d // 2], t[..., d // 2:]
        return t * cos + torch.cat([-t2, t1], -1) * sin
    a = F.scaled_dot_product_attention(rot(q), rot(k), v, is_causal=causal)
    a = a.permute(2, 0, 1, 3).reshape(s, b, h)
    x1 = x + a @ w_proj
    y = x1 + F.gelu(norm(x1, g2) @ w_in) @ w_out
    return y


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("b", [1, 2])
def test_layer_fwd_bwd_vs_torch_autograd(causal, b):
    d = _inputs(h=16, n=4, ffn=48, s=9, b=b, seed=7)
    y, c = L.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"],
                       n=4, causal=causal)
    g = L.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"],
                    n=4, causal=causal)
    names = ["x", "w_qkv", "w_proj", "w_in", "w_out", "g1", "g2"]
    tt = {k: torch.tensor(d[k], dtype=torch.float64, requires_grad=True) for k in names}
    yt = _torch_layer(*(tt[k] for k in names), n=4, causal=causal)
    assert np.allclose(yt.detach().numpy(), y, rtol=1e-12, atol=1e-12)
    yt.backward(torch.tensor(d["dy"]))
    for k, gk in [("x", "dx"), ("w_qkv", "dw_qkv"), ("w_proj", "dw_proj"), ("w_in", "dw_in"),
                  ("w_out", "dw_out"), ("g1", "dg1"), ("g2", "dg2")]:
        ref = tt[k].grad.numpy()
        err = np.linalg.norm(ref - g[gk]) / np.linalg.norm(ref)
        assert err < 1e-12, (k, err)


def test_layer_bwd_finite_differences():
    d = _inputs(h=8, n=2, ffn=16, s=5, b=1, seed=11)
    args = dict(n=2)
    def loss(dd):
        y, _ = L.layer_fwd(dd["x"], dd["w_qkv"], dd["w_proj"], dd["w_in"], dd["w_out"], dd["g1"],
                           dd["g2"], **args)
        return float(np.sum(y * d["dy"]))
    y, c = L.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **args)
    g = L.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **args)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for key, gkey in [("x", "dx"), ("w_qkv", "dw_qkv"), ("w_proj", "dw_proj"), ("w_in", "dw_in"),
                      ("w_out", "dw_out"), ("g1", "dg1"), ("g2", "dg2")]:
        for _ in range(3):
            idx = tuple(rng.integers(0, n) for n in d[key].shape)
            dp = {k: v.copy() for k, v in d.items()}
            dm = {k: v.copy() for k, v in d.items()}
            dp[key][idx] += eps
            dm[key][idx] -= eps
            fd = (loss(dp) - loss(dm)) / (2 * eps)
            an = g[gkey][idx]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (key, idx, fd, an)


# ---------------------------------------------------------------- Llama variant (NEXT-3)
def _llama_inputs(h=16, n=4, n_kv=2, ffn=128, s=9, b=1, seed=5):
    return layer_inputs(h, n, ffn, s, b, seed=seed, n_kv=n_kv, act="swiglu")


def _torch_llama(x, w_qkv, w_proj, w_in, w_out, g1, g2, n, n_kv, causal=True, eps=1e-5):
    """Independent torch fp64 Llama block from library routines: F.rms_norm,
    F.scaled_dot_product_attention(enable_gqa=True), F.silu (SwiGLU with
    w_in = [W_gate | W_up])."""
    import torch.nn.functional as F
    s, b, h = x.shape
    d = h // n
    u = F.rms_norm(x, (h,), g1, eps=eps)
    q, k, v = (u @ w_qkv).split([n * d, n_kv * d, n_kv * d], dim=-1)
    def heads(t, m):
        return t.reshape(s, b, m, d).permute(1, 2, 0, 3)
    q, k, v = heads(q, n), heads(k, n_kv), heads(v, n_kv)
    pos = torch.arange(s, dtype=torch.float64)
    inv = 10000.0 ** (-2 * torch.arange(d // 2, dtype=torch.float64) / d)
    ang = pos[:, None] * inv[None, :]
    cos = torch.cat([ang.cos(), ang.cos()], -1)
    sin = torch.cat([ang.sin(), ang.sin()], -1)
    def rot(t):
        t1, t2 = t[..., : d // 2], t[..., d // 2:]
        return t * cos + torch.cat([-t2, t1], -1) * sin
    a = F.scaled_dot_product_attention(rot(q), rot(k), v, is_causal=causal, enable_gqa=True)
    x1 = x + a.permute(2, 0, 1, 3).reshape(s, b, h) @ w_proj
    gate, up = (F.rms_norm(x1, (h,), g2, eps=eps) @ w_in).chunk(2, dim=-1)
    return x1 + (F.silu(gate) * up) @ w_out


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("n_kv", [1, 2, 4])
def test_llama_layer_vs_torch_autograd(causal, n_kv):
    d = _llama_inputs(n_kv=n_kv, b=2)
    kw = dict(n=4, causal=causal, n_kv=n_kv, act="swiglu")
    y, c = L.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    g = L.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    names = ["x", "w_qkv", "w_proj", "w_in", "w_out", "g1", "g2"]
    tt = {k: torch.tensor(d[k], dtype=torch.float64, requires_grad=True) for k in names}
    yt = _torch_llama(*(tt[k] for k in names), n=4, n_kv=n_kv, causal=causal)
    assert np.allclose(yt.detach().numpy(), y, rtol=1e-12, atol=1e-12)
    yt.backward(torch.tensor(d["dy"]))
    for k, gk in [("x", "dx"), ("w_qkv", "dw_qkv"), ("w_proj", "dw_proj"), ("w_in", "dw_in"),
                  ("w_out", "dw_out"), ("g1", "dg1"), ("g2", "dg2")]:
        ref = tt[k].grad.numpy()
        err = np.linalg.norm(ref - g[gk]) / np.linalg.norm(ref)
        assert err < 1e-12, (k, err)


def test_gqa_equals_mha_with_repeated_kv_heads():
    """GQA is MHA whose key / value heads are copies within each query group: the
    forward and dx agree, dW_q agrees, and dW_k / dW_v are the group sums of the
    MHA gradients of the copies (a wrong head mapping breaks all three)."""
    h, n, n_kv = 32, 8, 2
    d = layer_inputs(h, n, 64, 11, 1, seed=9, n_kv=n_kv)
    dh = h // n
    grp = n // n_kv
    wq, wk, wv = np.split(d["w_qkv"], [n * dh, (n + n_kv) * dh], axis=1)
    rep = lambda w: np.concatenate([w[:, (i // grp) * dh:(i // grp + 1) * dh] for i in range(n)], axis=1)
    w_mha = np.concatenate([wq, rep(wk), rep(wv)], axis=1)
    args = (d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"])
    y1, c1 = L.layer_fwd(d["x"], d["w_qkv"], *args, n=n, n_kv=n_kv)
    y2, c2 = L.layer_fwd(d["x"], w_mha, *args, n=n)
    assert np.allclose(y1, y2, rtol=1e-13, atol=1e-13)
    g1 = L.layer_bwd(d["dy"], c1, d["w_qkv"], *args, n=n, n_kv=n_kv)
    g2 = L.layer_bwd(d["dy"], c2, w_mha, *args, n=n)
    assert np.allclose(g1["dx"], g2["dx"], rtol=1e-12, atol=1e-12)
    gq, gk, gv = np.split(g1["dw_qkv"], [n * dh, (n + n_kv) * dh], axis=1)
    mq, mk, mv = np.split(g2["dw_qkv"], [n * dh, 2 * n * dh], axis=1)
    assert np.allclose(gq, mq, rtol=1e-12, atol=1e-12)
    for gg, mm in ((gk, mk), (gv, mv)):
        for j in range(n_kv):
            ref = sum(mm[:, i * dh:(i + 1) * dh] for i in range(j * grp, (j + 1) * grp))
            assert np.allclose(gg[:, j * dh:(j + 1) * dh], ref, rtol=1e-12, atol=1e-12)


def test_swiglu_closed_forms():
    x = np.linspace(-6, 6, 97)
    # SiLU = x sigma(x): sigma(0) = 1/2, odd part; SiLU' by central differences
    assert L.silu(np.array([0.0]))[0] == 0.0
    assert np.allclose(L.silu(x) - L.silu(-x), x, rtol=0, atol=1e-15)
    e = 1e-6
    assert np.allclose(L.silu_grad(x), (L.silu(x + e) - L.silu(x - e)) / (2 * e), rtol=0, atol=1e-8)
    # W_up = 0 => Z = 0 (the gate cannot leak through)
    d = _llama_inputs()
    F = d["w_out"].shape[0]
    d["w_in"][:, F:] = 0.0
    y, c = L.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"],
                       n=4, n_kv=2, act="swiglu")
    assert np.array_equal(c["z"], np.zeros_like(c["z"]))
    # the interleaved spec layout and the plain halves give the same G and dH
    from oracle.shard import il_perm
    hp = np.random.default_rng(1).standard_normal((5, 2 * 128))
    pm = il_perm(128)
    assert np.array_equal(L.ffn_act(hp[:, pm], "swiglu", il=True), L.ffn_act(hp, "swiglu"))
    dg = np.random.default_rng(2).standard_normal((5, 128))
    assert np.array_equal(L.ffn_act_bwd(dg, hp[:, pm], "swiglu", il=True), L.ffn_act_bwd(dg, hp, "swiglu")[:, pm])


def test_llama_finite_differences():
    d = _llama_inputs(h=8, n=2, n_kv=1, ffn=64, s=5, seed=13)
    args = dict(n=2, n_kv=1, act="swiglu")
    def loss(dd):
        y, _ = L.layer_fwd(dd["x"], dd["w_qkv"], dd["w_proj"], dd["w_in"], dd["w_out"], dd["g1"],
                           dd["g2"], **args)
        return float(np.sum(y * d["dy"]))
    y, c = L.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **args)
    g = L.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **args)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for key, gkey in [("x", "dx"), ("w_qkv", "dw_qkv"), ("w_in", "dw_in"), ("w_out", "dw_out")]:
        for _ in range(3):
            idx = tuple(rng.integers(0, n) for n in d[key].shape)
            dp = {k: v.copy() for k, v in d.items()}
            dm = {k: v.copy() for k, v in d.items()}
            dp[key][idx] += eps
            dm[key][idx] -= eps
            fd = (loss(dp) - loss(dm)) / (2 * eps)
            an = g[gkey][idx]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (key, idx, fd, an)


# ---------------------------------------------------------------- varlen packing (NEXT-3)
def _torch_packed(x, w_qkv, w_proj, w_in, w_out, g1, g2, n, lens, causal=True, eps=1e-5):
    """Independent torch fp64 route for a PACKED stream: one SDPA call over all T tokens
    with a block-diagonal (causal) boolean mask and RoPE positions that restart at every
    sequence start (the packing semantics, written the other way round)."""
    import torch.nn.functional as F
    T, b, h = x.shape
    d = h // n
    u = F.rms_norm(x, (h,), g1, eps=eps)
    q, k, v = (u @ w_qkv).split(h, dim=-1)
    heads = lambda t: t.reshape(T, b, n, d).permute(1, 2, 0, 3)  # noqa: E731
    q, k, v = heads(q), heads(k), heads(v)
    seq = torch.repeat_interleave(torch.arange(len(lens)), torch.tensor(lens))
    starts = torch.tensor(np.concatenate([[0], np.cumsum(lens)[:-1]]))
    pos = (torch.arange(T) - starts[seq]).to(torch.float64)
    inv = 10000.0 ** (-2 * torch.arange(d // 2, dtype=torch.float64) / d)
    ang = pos[:, None] * inv[None, :]
    cos = torch.cat([ang.cos(), ang.cos()], -1)
    sin = torch.cat([ang.sin(), ang.sin()], -1)
    def rot(t):
        t1, t2 = t[..., : d // 2], t[..., d // 2:]
        return t * cos + torch.cat([-t2, t1], -1) * sin
    allowed = seq[:, None] == seq[None, :]
    if causal:
        allowed &= torch.arange(T)[None, :] <= torch.arange(T)[:, None]
    a = F.scaled_dot_product_attention(rot(q), rot(k), v, attn_mask=allowed)
    x1 = x + a.permute(2, 0, 1, 3).reshape(T, b, h) @ w_proj
    return x1 + F.gelu(F.rms_norm(x1, (h,), g2, eps=eps) @ w_in) @ w_out


@pytest.mark.parametrize("causal", [True, False])
def test_varlen_layer_vs_torch_packed(causal):
    lens = [5, 1, 7, 3]
    d = _inputs(h=16, n=4, ffn=48, s=sum(lens), b=1, seed=29)
    kw = dict(n=4, causal=causal)
    y, cs = L.layer_fwd_varlen(d["x"], lens, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    g = L.layer_bwd_varlen(d["dy"], cs, lens, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    names = ["x", "w_qkv", "w_proj", "w_in", "w_out", "g1", "g2"]
    tt = {k: torch.tensor(d[k], dtype=torch.float64, requires_grad=True) for k in names}
    yt = _torch_packed(*(tt[k] for k in names), n=4, lens=lens, causal=causal)
    assert np.allclose(yt.detach().numpy(), y, rtol=1e-12, atol=1e-12)
    yt.backward(torch.tensor(d["dy"]))
    for k, gk in [("x", "dx"), ("w_qkv", "dw_qkv"), ("w_in", "dw_in"), ("w_out", "dw_out"), ("g1", "dg1")]:
        ref = tt[k].grad.numpy()
        assert np.linalg.norm(ref - g[gk]) / np.linalg.norm(ref) < 1e-12, k
    # one sequence is the plain layer
    y1, _ = L.layer_fwd_varlen(d["x"], [sum(lens)], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"],
                               d["g2"], **kw)
    y2, _ = L.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    assert np.array_equal(y1, y2)
