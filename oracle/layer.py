"""Unsharded ParaDySe layer, forward and backward, in fp64 (TEST INFRASTRUCTURE).

Follows PAPER.md Eqs. 1-4 (section "Problem Formulation")
with the north_star additions read as DESIGN.md R-1..R-7:

  pre-norm Llama block   X1 = X + MHA(RMSNorm_1(X)),  Y = X1 + FFN(RMSNorm_2(X1))
  Eq. 1  [Q|K|V] = U W_qkv
  RoPE   rotate-half pairs (k, k+d/2), global positions, theta = 10000 (R-3)
  Eq. 2  A = softmax(Q K^T / sqrt(d) + causal mask) V, per head (R-1)
  Eq. 3  O = A W_proj
  Eq. 4  Z = GELU(V2 W_in) W_out, exact erf GELU   (R-4)

Llama variant (the paper's LLaMA of Table 4, PAPER.md:317;
readings R-GQA / R-SWIGLU of DESIGN.md):
  GQA     n_kv key/value heads (n_kv | n); query head i attends with key/value
          head i // (n / n_kv); w_qkv [h, (n + 2 n_kv) d] columns [Q | K | V]
  SwiGLU  FFN(v) = (SiLU(v W_gate) * (v W_up)) W_down, SiLU(x) = x sigma(x);
          w_in [h, 2F] columns [W_gate | W_up], w_out [F, h]

Shapes (b = batch, the boundary layout [s, b, h] of Table 2 / R-10):
  x [s, b, h]; w_qkv [h, 3h] columns [Q | K | V], head i at columns i*d;
  w_proj [h, h]; w_in [h, F]; w_out [F, h]; g1, g2 [h].

Pins (tests/test_oracle_layer.py): s = 1 => attention = V;
GQA = MHA with every key/value head repeated over its query group (forward, dx,
and dW_k / dW_v = the group sums of the repeated copies); SwiGLU with W_up = 0
=> Z = 0, torch fp64 autograd (F.silu, SDPA with enable_gqa);
W_in = 0 => Z = 0; RoPE at t = 0 is the identity; naive
triple-loop attention on s <= 4; torch.float64 autograd (an independent
library routine) for every gradient; central finite differences.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

EPS = 1e-5
ROPE_THETA = 10000.0


def rmsnorm(x, g, eps=EPS):
    """r = (mean_j x_j^2 + eps)^(-1/2); xhat = x r; u = xhat * g  (R-2)."""
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    xhat = x * r
    return xhat * g, xhat, r[..., 0]


def rmsnorm_bwd(du, xhat, r, g):
    """dx = r (a - xhat mean(a xhat)), a = du * g;  dg = sum_tokens du * xhat."""
    a = du * g
    dx = r[..., None] * (a - xhat * np.mean(a * xhat, axis=-1, keepdims=True))
    dg = np.sum(du * xhat, axis=tuple(range(du.ndim - 1)))
    return dx, dg


def rope_cos_sin(positions, d, theta=ROPE_THETA):
    """cos/sin of angle t * theta^(-2k/d), k < d/2, angles in fp64 (R-3)."""
    k = np.arange(d // 2, dtype=np.float64)
    inv = theta ** (-2.0 * k / d)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def rope_apply(x, cos, sin):
    """Rotate-half: x'_k = x_k c - x_{k+d/2} s ; x'_{k+d/2} = x_k s + x_{k+d/2} c.
    x [..., s, d] with cos/sin [s, d/2]."""
    d2 = x.shape[-1] // 2
    a, b = x[..., :d2], x[..., d2:]
    return np.concatenate([a * cos - b * sin, a * sin + b * cos], axis=-1)


def rope_apply_t(dx, cos, sin):
    """Transpose rotation (by -angle), the RoPE backward (O-2 step 5)."""
    d2 = dx.shape[-1] // 2
    a, b = dx[..., :d2], dx[..., d2:]
    return np.concatenate([a * cos + b * sin, -a * sin + b * cos], axis=-1)


def gelu(x):
    """GELU(x) = x Phi(x), exact erf form (R-4)."""
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def gelu_grad(x):
    """d GELU / dx = Phi(x) + x phi(x)."""
    phi = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    return 0.5 * (1.0 + erf(x / math.sqrt(2.0))) + x * phi


def silu(x):
    """SiLU(x) = x sigma(x) (R-SWIGLU)."""
    return x / (1.0 + np.exp(-x))


def silu_grad(x):
    """d SiLU / dx = sigma(x) (1 + x (1 - sigma(x)))."""
    sg = 1.0 / (1.0 + np.exp(-x))
    return sg * (1.0 + x * (1.0 - sg))


IL = 64   # SwiGLU interleave of the spec layout (R-SWIGLU): gate block j, then up block j


def _gate_up(hpre, il):
    """Views of the gate and up pre-activations.  il=False: plain [gate | up] halves
    (the unsharded w_in); il=True: the spec layout's blocks of IL columns
    [gate_0 | up_0 | gate_1 | up_1 | ...] (every rank shard and every gather of them)."""
    F2 = hpre.shape[-1]
    if not il:
        return hpre[..., :F2 // 2], hpre[..., F2 // 2:]
    blk = hpre.reshape(hpre.shape[:-1] + (F2 // (2 * IL), 2, IL))
    return blk[..., 0, :], blk[..., 1, :]


def ffn_act(hpre, act="gelu", il=False):
    """G = GELU(H) (Eq. 4), or SwiGLU's G = SiLU(H_gate) * H_up."""
    if act == "gelu":
        return gelu(hpre)
    if act != "swiglu":
        raise ValueError(act)
    gate, up = _gate_up(hpre, il)
    g = silu(gate) * up
    return g.reshape(hpre.shape[:-1] + (hpre.shape[-1] // 2,))


def ffn_act_bwd(dg, hpre, act="gelu", il=False):
    """dH from dG: GELU'(H) dG, or SwiGLU's dH_gate = dG H_up SiLU'(H_gate),
    dH_up = dG SiLU(H_gate), in the layout of hpre."""
    if act == "gelu":
        return dg * gelu_grad(hpre)
    if act != "swiglu":
        raise ValueError(act)
    gate, up = _gate_up(hpre, il)
    dgv = dg.reshape(gate.shape)
    dh = np.empty_like(hpre)
    dgate, dup = _gate_up(dh, il)
    dgate[...] = dgv * up * silu_grad(gate)
    dup[...] = dgv * silu(gate)
    return dh


def attention_fwd(q, k, v, causal=True, block=256):
    """Eq. 2 for one (batch, head): q, k, v [s, d].  Returns (A [s,d], LSE [s]).
    Computed in row blocks so no s x s buffer exists; each block is the plain
    definition (softmax over the allowed keys)."""
    s, d = q.shape
    scale = 1.0 / math.sqrt(d)
    out = np.empty_like(q)
    lse = np.empty(s)
    for r0 in range(0, s, block):
        r1 = min(s, r0 + block)
        kmax = r1 if causal else s
        sc = (q[r0:r1] @ k[:kmax].T) * scale
        if causal:
            t = np.arange(r0, r1)[:, None]
            u = np.arange(kmax)[None, :]
            sc = np.where(u <= t, sc, -np.inf)
        m = sc.max(axis=1, keepdims=True)
        e = np.exp(sc - m)
        z = e.sum(axis=1, keepdims=True)
        out[r0:r1] = (e / z) @ v[:kmax]
        lse[r0:r1] = (m + np.log(z))[:, 0]
    return out, lse


def attention_bwd(q, k, v, o, lse, do, causal=True, block=256):
    """Backward of Eq. 2 for one (batch, head) (O-2 step 4):
    D = rowsum(dO o O); P = exp(S - LSE); dV = P^T dO; dP = dO V^T;
    dS = P o (dP - D); dQ = dS K / sqrt(d); dK = dS^T Q / sqrt(d)."""
    s, d = q.shape
    scale = 1.0 / math.sqrt(d)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    D = np.sum(do * o, axis=1)
    for r0 in range(0, s, block):
        r1 = min(s, r0 + block)
        kmax = r1 if causal else s
        sc = (q[r0:r1] @ k[:kmax].T) * scale
        p = np.exp(sc - lse[r0:r1, None])
        if causal:
            t = np.arange(r0, r1)[:, None]
            u = np.arange(kmax)[None, :]
            p = np.where(u <= t, p, 0.0)
        dv[:kmax] += p.T @ do[r0:r1]
        dp = do[r0:r1] @ v[:kmax].T
        ds = p * (dp - D[r0:r1, None])
        dq[r0:r1] += (ds @ k[:kmax]) * scale
        dk[:kmax] += (ds.T @ q[r0:r1]) * scale
    return dq, dk, dv


def _split_heads(m, n):
    """[s, b, n*d] -> [b, n, s, d]"""
    s, b, hd = m.shape
    return m.reshape(s, b, n, hd // n).transpose(1, 2, 0, 3)


def _merge_heads(m):
    """[b, n, s, d] -> [s, b, n*d]"""
    b, n, s, d = m.shape
    return m.transpose(2, 0, 1, 3).reshape(s, b, n * d)


def _qkv_split(qkv, n, n_kv):
    """[s, b, (n + 2 n_kv) d] laid out [Q | K | V] -> heads [b, n|n_kv, s, d]."""
    nk = n if n_kv is None else n_kv
    d = qkv.shape[-1] // (n + 2 * nk)
    hq, hk = n * d, nk * d
    return (_split_heads(qkv[..., :hq], n), _split_heads(qkv[..., hq:hq + hk], nk),
            _split_heads(qkv[..., hq + hk:], nk), nk, d)


def mha_core_fwd(qkv, n, positions, causal=True, theta=ROPE_THETA, n_kv=None):
    """RoPE + Eq. 2 on a [s, b, (n + 2 n_kv) d] tensor laid out [Q | K | V] (head i
    at columns i*d of each block; n_kv = None: n, MHA).  Query head i uses key /
    value head i // (n / n_kv) (GQA).  Returns (A [s, b, n d], LSE [b, n, s])."""
    q, k, v, nk, d = _qkv_split(qkv, n, n_kv)
    grp = n // nk
    cos, sin = rope_cos_sin(positions, d, theta)
    qr = rope_apply(q, cos, sin)
    kr = rope_apply(k, cos, sin)
    a = np.empty_like(q)
    lse = np.empty(q.shape[:3])
    for bi in range(q.shape[0]):
        for hi in range(n):
            a[bi, hi], lse[bi, hi] = attention_fwd(qr[bi, hi], kr[bi, hi // grp], v[bi, hi // grp], causal)
    return _merge_heads(a), lse


def mha_core_bwd(da_m, qkv, a_m, lse, n, positions, causal=True, theta=ROPE_THETA, n_kv=None):
    """Backward of mha_core_fwd from its saved inputs only (pre-RoPE qkv, the
    attention output A and LSE): returns d[Q|K|V] (pre-RoPE), the layout of qkv;
    a key / value head's gradient sums over its query group."""
    q, k, v, nk, d = _qkv_split(qkv, n, n_kv)
    grp = n // nk
    cos, sin = rope_cos_sin(positions, d, theta)
    qr = rope_apply(q, cos, sin)
    kr = rope_apply(k, cos, sin)
    a = _split_heads(a_m, n)
    da = _split_heads(da_m, n)
    dq = np.empty_like(qr)
    dk = np.zeros_like(kr)
    dv = np.zeros_like(v)
    for bi in range(qr.shape[0]):
        for hi in range(n):
            j = hi // grp
            gq, gk, gv = attention_bwd(qr[bi, hi], kr[bi, j], v[bi, j], a[bi, hi], lse[bi, hi], da[bi, hi], causal)
            dq[bi, hi] = gq
            dk[bi, j] += gk
            dv[bi, j] += gv
    dq = rope_apply_t(dq, cos, sin)
    dk = rope_apply_t(dk, cos, sin)
    return np.concatenate([_merge_heads(dq), _merge_heads(dk), _merge_heads(dv)], axis=-1)


def layer_fwd(x, w_qkv, w_proj, w_in, w_out, g1, g2, n, causal=True, eps=EPS,
              theta=ROPE_THETA, n_kv=None, act="gelu"):
    """O-1: one unsharded layer forward.  Returns (y, cache) where cache holds
    every intermediate named in O-1 (O and Z are the sublayer deltas, R-34).
    n_kv / act: the Llama variant (GQA, SwiGLU with w_in = [W_gate | W_up])."""
    s = x.shape[0]
    pos = np.arange(s)
    u, xhat1, r1 = rmsnorm(x, g1, eps)
    qkv = u @ w_qkv                                       # Eq. 1
    a, lse = mha_core_fwd(qkv, n, pos, causal, theta, n_kv)  # RoPE + Eq. 2
    o = a @ w_proj                                        # Eq. 3
    x1 = x + o
    v2, xhat2, r2 = rmsnorm(x1, g2, eps)
    hpre = v2 @ w_in                                      # Eq. 4
    g = ffn_act(hpre, act)
    z = g @ w_out
    y = x1 + z
    cache = dict(u=u, xhat1=xhat1, r1=r1, qkv=qkv, a=a, lse=lse, o=o, x1=x1,
                 v2=v2, xhat2=xhat2, r2=r2, h=hpre, g=g, z=z, y=y, pos=pos)
    return y, cache


def layer_bwd(dy, cache, w_qkv, w_proj, w_in, w_out, g1, g2, n, causal=True,
              theta=ROPE_THETA, n_kv=None, act="gelu"):
    """O-2: analytic VJP of layer_fwd.  Returns dict of dx and all weight grads."""
    c = cache
    # FFN (O-2 step 1)
    dz = dy
    dw_out = np.tensordot(c["g"], dz, axes=([0, 1], [0, 1]))
    dg = dz @ w_out.T
    dh = ffn_act_bwd(dg, c["h"], act)
    dw_in = np.tensordot(c["v2"], dh, axes=([0, 1], [0, 1]))
    dv2 = dh @ w_in.T
    # RMSNorm2 (step 2)
    dx1n, dg2 = rmsnorm_bwd(dv2, c["xhat2"], c["r2"], g2)
    dx1 = dy + dx1n
    # projection (step 3)
    dw_proj = np.tensordot(c["a"], dx1, axes=([0, 1], [0, 1]))
    da = dx1 @ w_proj.T
    # attention + RoPE (steps 4-5)
    dqkv = mha_core_bwd(da, c["qkv"], c["a"], c["lse"], n, c["pos"], causal, theta, n_kv)
    # QKV (step 6)
    dw_qkv = np.tensordot(c["u"], dqkv, axes=([0, 1], [0, 1]))
    du = dqkv @ w_qkv.T
    # RMSNorm1 (step 7)
    dxn, dg1 = rmsnorm_bwd(du, c["xhat1"], c["r1"], g1)
    dx = dx1 + dxn
    return dict(dx=dx, dw_qkv=dw_qkv, dw_proj=dw_proj, dw_in=dw_in, dw_out=dw_out,
                dg1=dg1, dg2=dg2, dx1=dx1, dqkv=dqkv)


def layer_fwd_varlen(x, lens, w_qkv, w_proj, w_in, w_out, g1, g2, n, **kw):
    """Varlen packing (reading R-VARLEN): the token axis of
    x [T, 1, h] holds len(lens) independent sequences back to back.  By definition the
    packed layer is the unsharded layer (O-1) applied to each sequence — attention
    stays inside a sequence and its RoPE positions start at 0 — so this is that loop.
    Returns (y [T, 1, h], per-sequence caches); o / z taps concatenated in the caches."""
    ys, caches = [], []
    o = 0
    for L in lens:
        y, c = layer_fwd(x[o:o + L], w_qkv, w_proj, w_in, w_out, g1, g2, n, **kw)
        ys.append(y)
        caches.append(c)
        o += L
    if o != x.shape[0]:
        raise ValueError(f"sum(lens)={o} != tokens {x.shape[0]}")
    return np.concatenate(ys, axis=0), caches


def layer_bwd_varlen(dy, caches, lens, w_qkv, w_proj, w_in, w_out, g1, g2, n, **kw):
    """Backward of layer_fwd_varlen: dx concatenated, weight and gain gradients summed
    over the sequences (they share the weights)."""
    out = None
    dxs = []
    o = 0
    for L, c in zip(lens, caches):
        g = layer_bwd(dy[o:o + L], c, w_qkv, w_proj, w_in, w_out, g1, g2, n, **kw)
        dxs.append(g["dx"])
        if out is None:
            out = {k: v.copy() for k, v in g.items() if k.startswith("dw") or k.startswith("dg")}
        else:
            for k in out:
                out[k] += g[k]
        o += L
    out["dx"] = np.concatenate(dxs, axis=0)
    return out
