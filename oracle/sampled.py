"""Row-sampled exact oracle for full-size parity (TEST INFRASTRUCTURE).

SURVEY §8(c) O-9, "sparse-cotangent row-sampled" parity: pick a set R of query rows
and set dY = 0 outside R.  Then, exactly (no approximation, fp64):

* forward rows R of Y, of the sublayer deltas O and Z (reading R-34) and LSE need
  U, K, V for every row (O(s h^2)) but attention only for the rows in R
  (O(|R| s h)) — Eq. 1-4 of PAPER.md:101-106 restricted to rows R;
* backward with dY = 0 outside R: dZ, dH, dX1 and dA vanish outside R, so every
  weight gradient and dgamma needs only the FFN / projection rows R, dQ rows R and
  the dK / dV rows <= max R (causal: the keys the sampled queries saw); dX is exact
  on every row (rows > max R of a causal layer get exactly 0).

The arithmetic follows oracle.layer step by step (O-1 / O-2): the same rmsnorm,
rope, gelu building blocks; only the row restriction differs.  Cost
O(s h^2 + |R| s h), so 7B-sized layers at s = 32K-128K stay within seconds to
minutes on the host cores.

Pin (tests/test_oracle_sampled.py): at s <= 512 every output equals oracle.layer's
full fwd / bwd with the same sparse dY (Y, O, Z, LSE on rows R; dX on every row;
every dW and dgamma) to 1e-12, causal and non-causal, several h / n.
"""
from __future__ import annotations

import math

import numpy as np

from .layer import (EPS, ROPE_THETA, ffn_act, ffn_act_bwd, rmsnorm, rmsnorm_bwd, rope_apply,
                    rope_apply_t, rope_cos_sin)


def sampled_layer(x, w_qkv, w_proj, w_in, w_out, g1, g2, n, R, dy_r, causal=True, eps=EPS,
                  theta=ROPE_THETA, n_kv=None, act="gelu", il=False):
    """x [s, h] (b = 1), weights as oracle.layer (w_qkv [h, (n + 2 n_kv) d] = [Q | K | V]
    column blocks, head i at columns i*d; n_kv = None: n), R sorted distinct row
    indices, dy_r [|R|, h] the non-zero rows of dY (weights may be float32 arrays of
    bf16-exact values: every product is formed in fp64).  act / il: the FFN activation
    (oracle.layer.ffn_act; il = SwiGLU's interleaved spec layout of w_in).  Returns dict:
    y, o, z [|R|, h], lse [n, |R|] (rows R), and dx [s, h], dw_qkv, dw_proj, dw_in,
    dw_out, dg1, dg2 (exact for the sparse dY)."""
    R = np.asarray(R)
    assert np.all(np.diff(R) > 0), "R must be sorted and distinct"
    x = np.asarray(x, dtype=np.float64)        # weights may be float32 holding bf16-exact values
    s, h = x.shape
    d = h // n
    nk = n if n_kv is None else n_kv
    grp = n // nk
    hk = nk * d
    kmax = int(R.max()) + 1 if causal else s          # keys any sampled query sees
    # ---------------- forward (O-1 restricted to rows R)
    u, xhat1, r1 = rmsnorm(x, g1, eps)
    wq, wk, wv = w_qkv[:, :h], w_qkv[:, h:h + hk], w_qkv[:, h + hk:]
    kf = u[:kmax] @ wk                                 # Eq. 1, K / V rows < kmax
    vf = u[:kmax] @ wv
    qr = u[R] @ wq
    cos, sin = rope_cos_sin(np.arange(kmax), d, theta)
    scale = 1.0 / math.sqrt(d)
    krot = np.empty_like(kf)
    qrot = np.empty_like(qr)
    a = np.zeros((len(R), h))
    lse = np.zeros((n, len(R)))
    for j in range(nk):
        cj = slice(j * d, (j + 1) * d)
        krot[:, cj] = rope_apply(kf[:, cj], cos, sin)
    for hh in range(n):
        c = slice(hh * d, (hh + 1) * d)
        cj = slice((hh // grp) * d, (hh // grp + 1) * d)  # the head's key / value head (GQA)
        qrot[:, c] = rope_apply(qr[:, c], cos[R], sin[R])
        for i, t in enumerate(R):
            nt = t + 1 if causal else s                # causal mask (R-1)
            sc = krot[:nt, cj] @ qrot[i, c] * scale    # Eq. 2
            mx = sc.max()
            e = np.exp(sc - mx)
            a[i, c] = (e / e.sum()) @ vf[:nt, cj]
            lse[hh, i] = mx + math.log(e.sum())
    o = a @ w_proj                                      # Eq. 3
    x1 = x[R] + o
    v2, xhat2, r2 = rmsnorm(x1, g2, eps)
    hp = v2 @ w_in                                      # Eq. 4
    gg = ffn_act(hp, act, il)
    z = gg @ w_out
    y = x1 + z
    # ---------------- backward (O-2 with dY = 0 outside R)
    dgg = dy_r @ w_out.T
    dh = ffn_act_bwd(dgg, hp, act, il)
    dw_out = gg.T @ dy_r
    dw_in = v2.T @ dh
    dv2 = dh @ w_in.T
    dx1n, dg2 = rmsnorm_bwd(dv2, xhat2, r2, g2)
    dx1 = dy_r + dx1n
    dw_proj = a.T @ dx1
    da = dx1 @ w_proj.T
    dq_r = np.zeros((len(R), h))
    dk = np.zeros((kmax, hk))
    dv = np.zeros((kmax, hk))
    for hh in range(n):
        c = slice(hh * d, (hh + 1) * d)
        cj = slice((hh // grp) * d, (hh // grp + 1) * d)
        for i, t in enumerate(R):
            nt = t + 1 if causal else s
            p = np.exp(krot[:nt, cj] @ qrot[i, c] * scale - lse[hh, i])
            dd = da[i, c] @ a[i, c]                    # D_t = sum_j dA_tj A_tj
            dv[:nt, cj] += np.outer(p, da[i, c])       # a key / value head sums its group
            ds = p * (vf[:nt, cj] @ da[i, c] - dd)
            dq_r[i, c] = (ds @ krot[:nt, cj]) * scale
            dk[:nt, cj] += np.outer(ds, qrot[i, c]) * scale
    for hh in range(n):                                 # RoPE^T (O-2 step 5)
        c = slice(hh * d, (hh + 1) * d)
        dq_r[:, c] = rope_apply_t(dq_r[:, c], cos[R], sin[R])
    for j in range(nk):
        cj = slice(j * d, (j + 1) * d)
        dk[:, cj] = rope_apply_t(dk[:, cj], cos, sin)
    # O-2 step 6, dW_qkv = U^T dQKV and dU = dQKV W_qkv^T, over the non-zero rows of
    # dQKV only: dQ lives on rows R, dK / dV on rows < kmax
    dkv = np.concatenate([dk, dv], axis=1)
    dw_qkv = np.empty((h, h + 2 * hk))
    dw_qkv[:, :h] = u[R].T @ dq_r
    dw_qkv[:, h:] = u[:kmax].T @ dkv
    du = np.zeros((s, h))
    du[:kmax] = dkv @ w_qkv[:, h:].T
    du[R] += dq_r @ wq.T
    dxn, dg1 = rmsnorm_bwd(du, xhat1, r1, g1)
    dx = dxn
    dx[R] += dx1
    return dict(y=y, o=o, z=z, lse=lse, dx=dx, dw_qkv=dw_qkv, dw_proj=dw_proj, dw_in=dw_in,
                dw_out=dw_out, dg1=dg1, dg2=dg2)
