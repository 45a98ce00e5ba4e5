"""Parity at BASELINE's full size (7B layer: h=4096, n=32, d=128, F=16384) in the
bench's launch configuration (P = 1 context, planned strategy), on sampled outputs
the oracle computes one by one ("sparse-cotangent row-sampled"):

* forward: rows R of Y, of the sublayer deltas O and Z (R-34) and LSE — each needs
  U, K, V for all rows (O(s h^2)) plus attention for the rows in R;
* backward with dY = 0 outside R: every weight gradient and dgamma exactly (they
  only see rows R of the FFN / projection and the K/V rows <= max R of attention),
  dX on sampled rows, and dX == 0 exactly on rows > max R.

The oracle side is assembled from oracle.layer building blocks in fp64 on the
same bf16 inputs.  Tolerance: relative L2 1e-2 (north_star bf16 path).
"""
import math

import numpy as np
import pytest
import torch

from oracle import layer as OL
from synth import round_bf16

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2511_13198_b200 import binding as B
    from tests.gpu_util import dev_bf16, host, rel

H, NH, F = 4096, 32, 16384
D = H // NH


def _inputs(s, seed):
    rng = np.random.default_rng(seed)
    g = lambda *sh, std=1.0, mean=0.0: round_bf16(mean + std * rng.standard_normal(sh))
    return dict(x=g(s, H), w_qkv=g(H, 3 * H, std=H ** -0.5), w_proj=g(H, H, std=H ** -0.5),
                w_in=g(H, F, std=H ** -0.5), w_out=g(F, H, std=F ** -0.5),
                g1=g(H, std=0.1, mean=1.0), g2=g(H, std=0.1, mean=1.0), dyR=None)


@pytest.mark.parametrize("s,pi", [(4096, 0), (4096, 1), (4096, 2), (4096, 3),
                                  (32768, 0)])      # the bench's longest length, its planned strategy
def test_fullsize_sampled(s, pi):
    d = _inputs(s, 11 + pi)
    R = np.array([5, 700, 1500, s // 2 + 3, s - 700, s - 2, s - 1]) if pi == 0 else np.array([3, 1024, s // 2 + 11, s - 129])
    rng = np.random.default_rng(99)
    dy = np.zeros((s, H))
    dy[R] = round_bf16(rng.standard_normal((len(R), H)))
    # ---------------- GPU (bench configuration: P = 1 context)
    model = B.Model(h=H, n_heads=NH, ffn=F)
    ctx = B.Context(model)
    w = dict(w_qkv_t=dev_bf16(d["w_qkv"].T), w_proj=dev_bf16(d["w_proj"]), w_in_t=dev_bf16(d["w_in"].T),
             w_out=dev_bf16(d["w_out"]), g1=dev_bf16(d["g1"]), g2=dev_bf16(d["g2"]))
    gr = {k: torch.zeros(v.shape, dtype=torch.float32, device="cuda") for k, v in w.items()}
    W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
    G = B.Grads(*(gr[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
    x = dev_bf16(d["x"])
    y = torch.empty_like(x)
    o = torch.empty_like(x)
    z = torch.empty_like(x)
    dx = torch.empty_like(x)
    tdy = dev_bf16(dy)
    st = torch.cuda.current_stream().cuda_stream
    ctx.debug_taps(o.data_ptr(), z.data_ptr())
    sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
    ctx.layer_bwd(pi, tdy.data_ptr(), sv, W, G, dx.data_ptr(), st)
    torch.cuda.synchronize()
    ctx.close()
    # ---------------- oracle, rows R (fp64)
    X = d["x"]
    u, xhat1, r1 = OL.rmsnorm(X, d["g1"])
    Wq, Wk, Wv = d["w_qkv"][:, :H], d["w_qkv"][:, H:2 * H], d["w_qkv"][:, 2 * H:]
    Kf = u @ Wk
    Vf = u @ Wv
    Qr = u[R] @ Wq
    cosf, sinf = OL.rope_cos_sin(np.arange(s), D)
    scale = 1.0 / math.sqrt(D)
    A = np.zeros((len(R), H))
    lse = np.zeros((NH, len(R)))
    Krot = np.empty_like(Kf)
    Qrot = np.empty_like(Qr)
    for hh in range(NH):
        sl = slice(hh * D, (hh + 1) * D)
        Krot[:, sl] = OL.rope_apply(Kf[:, sl], cosf, sinf)
        Qrot[:, sl] = OL.rope_apply(Qr[:, sl], cosf[R], sinf[R])
        for i, t in enumerate(R):
            sc = Krot[: t + 1, sl] @ Qrot[i, sl] * scale
            m = sc.max()
            e = np.exp(sc - m)
            A[i, sl] = (e / e.sum()) @ Vf[: t + 1, sl]
            lse[hh, i] = m + math.log(e.sum())
    O = A @ d["w_proj"]
    X1 = X[R] + O
    v2, xhat2, r2 = OL.rmsnorm(X1, d["g2"])
    Hp = v2 @ d["w_in"]
    Gg = OL.gelu(Hp)
    Z = Gg @ d["w_out"]
    Y = X1 + Z
    assert rel(host(o)[R], O) < 1e-2
    assert rel(host(z)[R], Z) < 1e-2
    assert rel(host(y)[R], Y) < 1e-2
    # ---------------- backward with dY = 0 outside R
    dYR = dy[R]
    dGg = dYR @ d["w_out"].T
    dH = dGg * OL.gelu_grad(Hp)
    dW_out = Gg.T @ dYR
    dW_in = v2.T @ dH
    dV2 = dH @ d["w_in"].T
    dx1n, dg2 = OL.rmsnorm_bwd(dV2, xhat2, r2, d["g2"])
    dX1 = dYR + dx1n
    dW_proj = A.T @ dX1
    dA = dX1 @ d["w_proj"].T
    dQr = np.zeros((len(R), H))
    dK = np.zeros((s, H))
    dV = np.zeros((s, H))
    for hh in range(NH):
        sl = slice(hh * D, (hh + 1) * D)
        for i, t in enumerate(R):
            p = np.exp(Krot[: t + 1, sl] @ Qrot[i, sl] * scale - lse[hh, i])
            Dt = dA[i, sl] @ A[i, sl]
            dV[: t + 1, sl] += np.outer(p, dA[i, sl])
            dS = p * (Vf[: t + 1, sl] @ dA[i, sl] - Dt)
            dQr[i, sl] = (dS @ Krot[: t + 1, sl]) * scale
            dK[: t + 1, sl] += np.outer(dS, Qrot[i, sl]) * scale
    for hh in range(NH):   # RoPE^T
        sl = slice(hh * D, (hh + 1) * D)
        dK[:, sl] = OL.rope_apply_t(dK[:, sl], cosf, sinf)
        dQr[:, sl] = OL.rope_apply_t(dQr[:, sl], cosf[R], sinf[R])
    dQKV = np.concatenate([np.zeros((s, H)), dK, dV], axis=1)
    dQKV[R, :H] = dQr
    dW_qkv = u.T @ dQKV
    dU = dQKV @ d["w_qkv"].T
    dxn, dg1 = OL.rmsnorm_bwd(dU, xhat1, r1, d["g1"])
    dXf = dxn
    dXf[R] += dX1
    assert rel(host(gr["w_out"]), dW_out) < 1e-2
    assert rel(host(gr["w_in_t"]), dW_in.T) < 1e-2
    assert rel(host(gr["w_proj"]), dW_proj) < 1e-2
    assert rel(host(gr["w_qkv_t"]), dW_qkv.T) < 1e-2
    assert rel(host(gr["g1"]), dg1) < 1e-2
    assert rel(host(gr["g2"]), dg2) < 1e-2
    sample = np.concatenate([R, np.arange(0, s, 97)])
    gx = host(dx)
    assert rel(gx[sample], dXf[sample]) < 1e-2
    assert np.all(gx[R.max() + 1:] == 0.0)            # no gradient beyond the last cotangent row
