"""Per-strategy sharded simulations of one layer, fwd + bwd, fp64 (TEST INFRASTRUCTURE).

Each function f_{pi} maps spec-layout input shards + spec-layout weight shards
to spec-layout output shards on a simulated Grid (Eqs. 7-8, PAPER.md:228-232;
"identical parameter lists ... and return types").  The
dataflows are those of SURVEY §8(c) O-5 / DESIGN.md:

  MegatronTS: AllGather on s before MHA / FFN, column-
      parallel QKV / FC1, row-parallel proj / FC2, ReduceScatter after.
  UlyssesZ   (R-12): ZeRO3-style AllGather of the weight
      shards, All-to-All sequence->heads around attention and back.
  METP       (R-11 "R-METP"): the TS dataflow split into
      c waves (wave k = local rows [k s/(Pc), (k+1) s/(Pc)) of every shard),
      per-wave AG / RS, attention over the full position-ordered Q/K/V (a
      query-chunk x KV-chunk loop), FFN intermediates recomputed in backward.

Every saved activation is registered in the grid's memory ledger with its
device byte size (bf16 = 2 B, fp32 statistics = 4 B) and the backward reads
ONLY registered tensors, so the ledger is an honest recount of what must be
kept between forward and backward (pin for oracle/memory.py).

Pins: every strategy at every P in {1, 2, 4, 8} reproduces layer.layer_fwd /
layer_bwd to <= 1e-12 (north_star); switched chains equal the
L-layer unsharded stack; comm-log multisets match the
documented signature.  METP's true external schedule is
"parity unpinned" beyond that invariant.
"""
from __future__ import annotations

import copy

import numpy as np

from .layer import (EPS, ROPE_THETA, ffn_act, ffn_act_bwd, gelu, gelu_grad, mha_core_bwd, mha_core_fwd,
                    rmsnorm, rmsnorm_bwd, rope_apply, rope_apply_t, rope_cos_sin)

TS, UZ, METP, CZ, METP_FULL, COL = 0, 1, 2, 3, 4, 5
NAMES = {TS: "MegatronTS", UZ: "UlyssesZ", METP: "METP", CZ: "MegatronCZ", METP_FULL: "METP-full",
         COL: "ColossalZ"}


class Cfg:
    def __init__(self, h, n, ffn, causal=True, eps=EPS, theta=ROPE_THETA, metp_chunks=None,
                 metp_recompute="ffn", n_kv=None, act="gelu"):
        self.h, self.n, self.ffn = h, n, ffn
        # Llama variant (NEXT-3, R-GQA / R-SWIGLU), every strategy
        self.n_kv = n if n_kv is None else n_kv
        self.act = act
        self.causal, self.eps, self.theta = causal, eps, theta
        self.metp_chunks = metp_chunks
        if metp_recompute not in ("ffn", "full"):
            raise ValueError(f"metp_recompute must be 'ffn' or 'full', not {metp_recompute!r}")
        self.metp_recompute = metp_recompute      # R-11 / SURVEY O-6: 'full' also recomputes QKV


def _save(grid, r, saved, name, arr, bpe):
    saved[name] = arr
    saved.setdefault("_ids", []).append(grid.track(r, arr.size * bpe, "saved"))


def _release(grid, saved):
    for hid in saved.pop("_ids", []):
        grid.release(hid)


def _apply_norm(x, r, g):
    """Recompute u = x r g from the saved input and rstd (no new statistics)."""
    return x * r[..., None] * g


def _nkv_local(cfg, P):
    return cfg.n_kv // P


def _act(h, cfg):
    """G of a spec-layout (interleaved for SwiGLU) FC1 output."""
    return ffn_act(h, cfg.act, il=True)


def _act_bwd(dg, h, cfg):
    return ffn_act_bwd(dg, h, cfg.act, il=True)


def _zero_grads(W):
    p = len(W["w_qkv_t"])
    return {k: [np.zeros_like(a) for a in W[src]] for k, src in
            [("dw_qkv_t", "w_qkv_t"), ("dw_proj", "w_proj"), ("dw_in_t", "w_in_t"),
             ("dw_out", "w_out"), ("dg1", "g1"), ("dg2", "g2")]} | {"_p": p}


# ------------------------------------------------------------------ MegatronTS
def ts_fwd(grid, xs, W, cfg):
    P = grid.p
    s = xs[0].shape[0] * P
    nl = cfg.n // P
    pos = np.arange(s)
    saved = [dict() for _ in range(P)]
    u, r1 = [], []
    for r in range(P):
        ur, _, rr = rmsnorm(xs[r], W["g1"][r], cfg.eps)
        u.append(ur)
        r1.append(rr)
    U = grid.all_gather(u)                                         # AG(u)
    qkv = [U[r] @ W["w_qkv_t"][r].T for r in range(P)]             # column-parallel Eq. 1
    att = [mha_core_fwd(qkv[r], nl, pos, cfg.causal, cfg.theta, _nkv_local(cfg, P)) for r in range(P)]
    opart = [att[r][0] @ W["w_proj"][r] for r in range(P)]        # row-parallel Eq. 3
    o = grid.reduce_scatter(opart)                                 # RS(o)
    x1 = [xs[r] + o[r] for r in range(P)]
    v, r2 = [], []
    for r in range(P):
        vr, _, rr = rmsnorm(x1[r], W["g2"][r], cfg.eps)
        v.append(vr)
        r2.append(rr)
    V = grid.all_gather(v)                                         # AG(v)
    hpre = [V[r] @ W["w_in_t"][r].T for r in range(P)]
    zpart = [_act(hpre[r], cfg) @ W["w_out"][r] for r in range(P)]
    z = grid.reduce_scatter(zpart)                                 # RS(z)
    y = [x1[r] + z[r] for r in range(P)]
    for r in range(P):
        sv = saved[r]
        _save(grid, r, sv, "x", xs[r], 2)
        _save(grid, r, sv, "r1", r1[r], 4)
        _save(grid, r, sv, "qkv", qkv[r], 2)
        _save(grid, r, sv, "a", att[r][0], 2)
        _save(grid, r, sv, "lse", att[r][1], 4)
        _save(grid, r, sv, "x1", x1[r], 2)
        _save(grid, r, sv, "r2", r2[r], 4)
        _save(grid, r, sv, "h", hpre[r], 2)
    return y, saved, dict(o=o, z=z)


def ts_bwd(grid, dys, saved, W, cfg, grads):
    P = grid.p
    s = dys[0].shape[0] * P
    nl = cfg.n // P
    pos = np.arange(s)
    sv = saved
    dZ = grid.all_gather(dys)                                      # AG(dz)
    v = [_apply_norm(sv[r]["x1"], sv[r]["r2"], W["g2"][r]) for r in range(P)]
    V = grid.all_gather(v)                                         # AG(v) re-gather
    dvpart = []
    for r in range(P):
        hp = sv[r]["h"]
        dg = dZ[r] @ W["w_out"][r].T
        dh = _act_bwd(dg, hp, cfg)
        grads["dw_out"][r] += np.tensordot(_act(hp, cfg), dZ[r], axes=([0, 1], [0, 1]))
        grads["dw_in_t"][r] += np.tensordot(dh, V[r], axes=([0, 1], [0, 1]))
        dvpart.append(dh @ W["w_in_t"][r])
    dv = grid.reduce_scatter(dvpart)                               # RS(dv)
    dx1, dg2 = [], []
    for r in range(P):
        xhat2 = sv[r]["x1"] * sv[r]["r2"][..., None]
        d, dgr = rmsnorm_bwd(dv[r], xhat2, sv[r]["r2"], W["g2"][r])
        dx1.append(dys[r] + d)
        dg2.append(dgr)
    dX1 = grid.all_gather(dx1)                                     # AG(dx1)
    u = [_apply_norm(sv[r]["x"], sv[r]["r1"], W["g1"][r]) for r in range(P)]
    dqkv = []
    for r in range(P):
        da = dX1[r] @ W["w_proj"][r].T
        grads["dw_proj"][r] += np.tensordot(sv[r]["a"], dX1[r], axes=([0, 1], [0, 1]))
        dqkv.append(mha_core_bwd(da, sv[r]["qkv"], sv[r]["a"], sv[r]["lse"], nl, pos,
                                 cfg.causal, cfg.theta, _nkv_local(cfg, P)))
    U = grid.all_gather(u)                                         # AG(u) re-gather
    dupart = []
    for r in range(P):
        grads["dw_qkv_t"][r] += np.tensordot(dqkv[r], U[r], axes=([0, 1], [0, 1]))
        dupart.append(dqkv[r] @ W["w_qkv_t"][r])
    du = grid.reduce_scatter(dupart)                               # RS(du)
    dx, dg1 = [], []
    for r in range(P):
        xhat1 = sv[r]["x"] * sv[r]["r1"][..., None]
        d, dgr = rmsnorm_bwd(du[r], xhat1, sv[r]["r1"], W["g1"][r])
        dx.append(dx1[r] + d)
        dg1.append(dgr)
    _finish_dgamma(grid, grads, dg1, dg2)
    for r in range(P):
        _release(grid, sv[r])
    return dx


def _finish_dgamma(grid, grads, dg1, dg2):
    P = grid.p
    cat = grid.all_reduce([np.concatenate([dg1[r], dg2[r]]) for r in range(P)])  # AR(dg1||dg2)
    hh = dg1[0].shape[0]
    for r in range(P):
        grads["dg1"][r] += cat[r][:hh]
        grads["dg2"][r] += cat[r][hh:]


# ------------------------------------------------------------------ UlyssesZ
def _gather_weights(grid, W):
    return dict(
        w_qkv_t=grid.all_gather(W["w_qkv_t"]),   # rows: head-group-major [g0 Q,K,V | g1 ...]
        w_proj=grid.all_gather(W["w_proj"]),
        w_in_t=grid.all_gather(W["w_in_t"]),
        w_out=grid.all_gather(W["w_out"]),
    )


def uz_fwd(grid, xs, W, cfg):
    P = grid.p
    sl = xs[0].shape[0]
    s = sl * P
    nl = cfg.n // P
    Wf = _gather_weights(grid, W)                                  # 4 x AG(W)
    saved = [dict() for _ in range(P)]
    u, r1, qkv_loc = [], [], []
    for r in range(P):
        ur, _, rr = rmsnorm(xs[r], W["g1"][r], cfg.eps)
        u.append(ur)
        r1.append(rr)
        qkv_loc.append(ur @ Wf["w_qkv_t"][r].T)     # [s/P, b, 3h], head-group-major columns
    # A2A seq -> heads: send column block j (3h/P wide) to rank j, concat along s
    qkv = grid.all_to_all(qkv_loc, split_axis=2, concat_axis=0)
    att = [mha_core_fwd(qkv[r], nl, np.arange(s), cfg.causal, cfg.theta, _nkv_local(cfg, P))
           for r in range(P)]
    # A2A heads -> seq: send row block j (s/P rows) to rank j, concat along columns
    afull = grid.all_to_all([att[r][0] for r in range(P)], split_axis=0, concat_axis=2)
    o = [afull[r] @ Wf["w_proj"][r] for r in range(P)]
    x1 = [xs[r] + o[r] for r in range(P)]
    y, z = [], []
    for r in range(P):
        vr, _, rr = rmsnorm(x1[r], W["g2"][r], cfg.eps)
        hp = vr @ Wf["w_in_t"][r].T
        zr = _act(hp, cfg) @ Wf["w_out"][r]
        z.append(zr)
        y.append(x1[r] + zr)
        sv = saved[r]
        _save(grid, r, sv, "x", xs[r], 2)
        _save(grid, r, sv, "r1", r1[r], 4)
        _save(grid, r, sv, "qkv", qkv[r], 2)
        _save(grid, r, sv, "a", att[r][0], 2)
        _save(grid, r, sv, "lse", att[r][1], 4)
        _save(grid, r, sv, "afull", afull[r], 2)
        _save(grid, r, sv, "x1", x1[r], 2)
        _save(grid, r, sv, "r2", rr, 4)
        _save(grid, r, sv, "h", hp, 2)
    return y, saved, dict(o=o, z=z)


def uz_bwd(grid, dys, saved, W, cfg, grads):
    P = grid.p
    sl = dys[0].shape[0]
    s = sl * P
    nl = cfg.n // P
    sv = saved
    Wf = _gather_weights(grid, W)                                  # 4 x AG(W) again
    dwo, dwi, dwp, dwq = [], [], [], []
    dx1, dg2, dafull = [], [], []
    for r in range(P):
        hp = sv[r]["h"]
        v = _apply_norm(sv[r]["x1"], sv[r]["r2"], W["g2"][r])
        dg = dys[r] @ Wf["w_out"][r].T
        dh = _act_bwd(dg, hp, cfg)
        dwo.append(np.tensordot(_act(hp, cfg), dys[r], axes=([0, 1], [0, 1])))
        dwi.append(np.tensordot(dh, v, axes=([0, 1], [0, 1])))
        dv = dh @ Wf["w_in_t"][r]
        xhat2 = sv[r]["x1"] * sv[r]["r2"][..., None]
        d, dgr = rmsnorm_bwd(dv, xhat2, sv[r]["r2"], W["g2"][r])
        dx1.append(dys[r] + d)
        dg2.append(dgr)
        dafull.append(dx1[r] @ Wf["w_proj"][r].T)
        dwp.append(np.tensordot(sv[r]["afull"], dx1[r], axes=([0, 1], [0, 1])))
    # A2A(dO): seq -> heads (column block j to rank j)
    da = grid.all_to_all(dafull, split_axis=2, concat_axis=0)
    dqkv = [mha_core_bwd(da[r], sv[r]["qkv"], sv[r]["a"], sv[r]["lse"], nl, np.arange(s),
                         cfg.causal, cfg.theta, _nkv_local(cfg, P)) for r in range(P)]
    # A2A(dQKV): heads -> seq (row block j to rank j, concat along columns)
    dqkv_loc = grid.all_to_all(dqkv, split_axis=0, concat_axis=2)
    dx, dg1 = [], []
    for r in range(P):
        u = _apply_norm(sv[r]["x"], sv[r]["r1"], W["g1"][r])
        dwq.append(np.tensordot(dqkv_loc[r], u, axes=([0, 1], [0, 1])))
        du = dqkv_loc[r] @ Wf["w_qkv_t"][r]
        xhat1 = sv[r]["x"] * sv[r]["r1"][..., None]
        d, dgr = rmsnorm_bwd(du, xhat1, sv[r]["r1"], W["g1"][r])
        dx.append(dx1[r] + d)
        dg1.append(dgr)
    # ZeRO3: reduce-scatter full local dW (fp32) into spec shards
    for key, full in (("dw_qkv_t", dwq), ("dw_proj", dwp), ("dw_in_t", dwi), ("dw_out", dwo)):
        part = grid.reduce_scatter(full, axis=0, bpe=4)
        for r in range(P):
            grads[key][r] += part[r]
    _finish_dgamma(grid, grads, dg1, dg2)
    for r in range(P):
        _release(grid, sv[r])
    return dx


# ------------------------------------------------------------------ METP (R-METP)
def _wave_rows(sl, c, k):
    w = sl // c
    return slice(k * w, (k + 1) * w)


def _wave_positions(P, sl, c, k):
    """Global positions of the AG'd wave-k rows, rank-major: r' s/P + k s/(Pc) + j."""
    w = sl // c
    return np.concatenate([r * sl + k * w + np.arange(w) for r in range(P)])


def metp_chunks(cfg, P):
    return cfg.metp_chunks if cfg.metp_chunks else P


def metp_fwd(grid, xs, W, cfg):
    P = grid.p
    sl = xs[0].shape[0]
    s = sl * P
    nl = cfg.n // P
    c = metp_chunks(cfg, P)
    if sl % c:
        raise ValueError(f"s/P={sl} not divisible by metp_chunks={c} (SPEC.md:184)")
    hq = (cfg.n + 2 * cfg.n_kv) * (cfg.h // cfg.n) // P     # local Q | K | V columns
    b = xs[0].shape[1]
    saved = [dict() for _ in range(P)]
    u, r1 = [], []
    for r in range(P):
        ur, _, rr = rmsnorm(xs[r], W["g1"][r], cfg.eps)
        u.append(ur)
        r1.append(rr)
    qkv = [np.zeros((s, b, hq)) for _ in range(P)]     # full-s, position-ordered
    for k in range(c):
        rows = _wave_rows(sl, c, k)
        Uw = grid.all_gather([u[r][rows] for r in range(P)])       # AG(u) wave k
        posw = _wave_positions(P, sl, c, k)
        for r in range(P):
            qkv[r][posw] = Uw[r] @ W["w_qkv_t"][r].T
    # attention over the full sequence (query-chunk x KV-chunk two-level loop)
    att = [mha_core_fwd(qkv[r], nl, np.arange(s), cfg.causal, cfg.theta, _nkv_local(cfg, P))
           for r in range(P)]
    o = [np.zeros_like(xs[r]) for r in range(P)]
    for k in range(c):
        rows = _wave_rows(sl, c, k)
        posw = _wave_positions(P, sl, c, k)
        ow = grid.reduce_scatter([att[r][0][posw] @ W["w_proj"][r] for r in range(P)])  # RS(o)
        for r in range(P):
            o[r][rows] = ow[r]
    x1 = [xs[r] + o[r] for r in range(P)]
    v, r2 = [], []
    for r in range(P):
        vr, _, rr = rmsnorm(x1[r], W["g2"][r], cfg.eps)
        v.append(vr)
        r2.append(rr)
    z = [np.zeros_like(xs[r]) for r in range(P)]
    for k in range(c):
        rows = _wave_rows(sl, c, k)
        Vw = grid.all_gather([v[r][rows] for r in range(P)])       # AG(v) wave k
        zw = grid.reduce_scatter([_act(Vw[r] @ W["w_in_t"][r].T, cfg) @ W["w_out"][r]
                                  for r in range(P)])             # RS(z) wave k
        for r in range(P):
            z[r][rows] = zw[r]
    y = [x1[r] + z[r] for r in range(P)]
    for r in range(P):
        sv = saved[r]
        _save(grid, r, sv, "x", xs[r], 2)
        _save(grid, r, sv, "r1", r1[r], 4)
        if cfg.metp_recompute == "ffn":           # 'full': QKV recomputed in backward
            _save(grid, r, sv, "qkv", qkv[r], 2)
        _save(grid, r, sv, "a", att[r][0], 2)
        _save(grid, r, sv, "lse", att[r][1], 4)
        _save(grid, r, sv, "x1", x1[r], 2)
        _save(grid, r, sv, "r2", r2[r], 4)
    return y, saved, dict(o=o, z=z)


def metp_bwd(grid, dys, saved, W, cfg, grads):
    P = grid.p
    sl = dys[0].shape[0]
    s = sl * P
    nl = cfg.n // P
    c = metp_chunks(cfg, P)
    sv = saved
    dx1 = [np.zeros_like(d) for d in dys]
    dg2 = [np.zeros(cfg.h) for _ in range(P)]
    for k in range(c):   # FFN backward, recomputing v, H, G per wave
        rows = _wave_rows(sl, c, k)
        dZw = grid.all_gather([dys[r][rows] for r in range(P)])    # AG(dz) wave k
        vloc = [_apply_norm(sv[r]["x1"][rows], sv[r]["r2"][rows], W["g2"][r]) for r in range(P)]
        Vw = grid.all_gather(vloc)                                 # AG(v) wave k
        dvpart = []
        for r in range(P):
            hp = Vw[r] @ W["w_in_t"][r].T
            dg = dZw[r] @ W["w_out"][r].T
            dh = _act_bwd(dg, hp, cfg)
            grads["dw_out"][r] += np.tensordot(_act(hp, cfg), dZw[r], axes=([0, 1], [0, 1]))
            grads["dw_in_t"][r] += np.tensordot(dh, Vw[r], axes=([0, 1], [0, 1]))
            dvpart.append(dh @ W["w_in_t"][r])
        dvw = grid.reduce_scatter(dvpart)                          # RS(dv) wave k
        for r in range(P):
            xhat2 = sv[r]["x1"][rows] * sv[r]["r2"][rows][..., None]
            d, dgr = rmsnorm_bwd(dvw[r], xhat2, sv[r]["r2"][rows], W["g2"][r])
            dx1[r][rows] = dys[r][rows] + d
            dg2[r] += dgr
    hl = cfg.h // P
    b = dys[0].shape[1]
    da = [np.zeros((s, b, hl)) for _ in range(P)]
    for k in range(c):   # projection backward per wave
        rows = _wave_rows(sl, c, k)
        posw = _wave_positions(P, sl, c, k)
        dX1w = grid.all_gather([dx1[r][rows] for r in range(P)])   # AG(dx1) wave k
        for r in range(P):
            da[r][posw] = dX1w[r] @ W["w_proj"][r].T
            grads["dw_proj"][r] += np.tensordot(sv[r]["a"][posw], dX1w[r], axes=([0, 1], [0, 1]))
    if cfg.metp_recompute == "full":   # QKV recompute: per wave AG(u) and the QKV GEMM again
        qkv = [np.zeros((s, b, (cfg.n + 2 * cfg.n_kv) * (cfg.h // cfg.n) // P)) for _ in range(P)]
        for k in range(c):
            rows = _wave_rows(sl, c, k)
            posw = _wave_positions(P, sl, c, k)
            uloc = [_apply_norm(sv[r]["x"][rows], sv[r]["r1"][rows], W["g1"][r]) for r in range(P)]
            Uw = grid.all_gather(uloc)                             # AG(u) wave k (recompute)
            for r in range(P):
                qkv[r][posw] = Uw[r] @ W["w_qkv_t"][r].T
    else:
        qkv = [sv[r]["qkv"] for r in range(P)]
    dqkv = [mha_core_bwd(da[r], qkv[r], sv[r]["a"], sv[r]["lse"], nl, np.arange(s),
                         cfg.causal, cfg.theta, _nkv_local(cfg, P)) for r in range(P)]
    dx = [np.zeros_like(d) for d in dys]
    dg1 = [np.zeros(cfg.h) for _ in range(P)]
    for k in range(c):   # QKV backward per wave
        rows = _wave_rows(sl, c, k)
        posw = _wave_positions(P, sl, c, k)
        uloc = [_apply_norm(sv[r]["x"][rows], sv[r]["r1"][rows], W["g1"][r]) for r in range(P)]
        Uw = grid.all_gather(uloc)                                 # AG(u) wave k
        dupart = []
        for r in range(P):
            grads["dw_qkv_t"][r] += np.tensordot(dqkv[r][posw], Uw[r], axes=([0, 1], [0, 1]))
            dupart.append(dqkv[r][posw] @ W["w_qkv_t"][r])
        duw = grid.reduce_scatter(dupart)                          # RS(du) wave k
        for r in range(P):
            xhat1 = sv[r]["x"][rows] * sv[r]["r1"][rows][..., None]
            d, dgr = rmsnorm_bwd(duw[r], xhat1, sv[r]["r1"][rows], W["g1"][r])
            dx[r][rows] = dx1[r][rows] + d
            dg1[r] += dgr
    _finish_dgamma(grid, grads, dg1, dg2)
    for r in range(P):
        _release(grid, sv[r])
    return dx


# ------------------------------------------------------------------ MegatronCZ
# Megatron-LM CP + ZeRO3 (reading R-CZ): weights gathered
# ZeRO3-style as in UlyssesZ, every GEMM local on the rank's s/P rows; the context-
# parallel attention all-gathers the sequence's Q/K/V and computes the rank's own
# query rows against every key (causal: keys <= the query position).  In backward the
# key / value gradients of every rank's queries are reduce-scattered back to the rows'
# owners.  The W_qkv spec shard [Q_r; K_r; V_r] is gathered part by part so the full
# weight is [Q all; K all; V all] (one attention call over all heads), and its
# gradient is reduce-scattered part by part back into the spec layout.

def _gather_qkv_parts(grid, W, h, n=None, n_kv=None):
    """3 x AG of the spec shards' Q, K, V rows -> [Q all; K all; V all] ([(n + 2 n_kv) d, h];
    GQA: the K and V parts are n_kv d / P rows per shard)."""
    P = grid.p
    hl = h // P
    hkl = hl if n is None or n_kv is None else n_kv * (h // n) // P
    bounds = [(0, hl), (hl, hl + hkl), (hl + hkl, hl + 2 * hkl)]
    parts = [grid.all_gather([W["w_qkv_t"][r][a:b] for r in range(P)])[0] for a, b in bounds]
    return np.concatenate(parts, axis=0)


def _rep_kv(x, grp):
    """GQA: key / value heads [b, n_kv, rows, d] -> one copy per query head [b, n, rows, d]."""
    return np.repeat(x, grp, axis=1) if grp > 1 else x


def _fold_kv(g, grp):
    """GQA: per-query-head gradients [b, n, rows, d] -> summed per key / value head."""
    if grp == 1:
        return g
    b, n, rows, d = g.shape
    return g.reshape(b, n // grp, grp, rows, d).sum(axis=2)


# causally balanced ("zigzag") placement: the s positions are cut into 2P half-chunks
# of c = s/(2P); rank r computes the queries of half-chunks r and 2P-1-r, which it
# receives (with their K, V) by point-to-point sends from their boundary owners, and
# the keys / values travel around the ring in P steps (K/V of rank (r - k) mod P at
# step k), so every rank holds O(u) of them at a time.  Each (query half-chunk, key
# half-chunk) pair is a full block, a causal diagonal block, or empty; at every ring
# step every rank has two full-block equivalents of work.  Partial results merge by
# the log-sum-exp identity; the backward runs the same ring with each K/V block's fp32
# dK / dV accumulator travelling with it (P passes: it comes home), using the merged
# LSE.  Results return to the boundary layout by the reverse point-to-point exchange.

def _zz(j, P):
    """Zigzag owner of half-chunk j (of 2P)."""
    return j if j < P else 2 * P - 1 - j


def _zig(r, P):
    """The half-chunks rank r computes, in position order."""
    return (r, 2 * P - 1 - r)


def _zig_positions(r, P, c):
    a, b = _zig(r, P)
    return np.concatenate([np.arange(a * c, (a + 1) * c), np.arange(b * c, (b + 1) * c)])


def _to_zigzag(grid, X, bpe=2):
    """Boundary rows [s/P, ...] per rank -> zigzag rows [half-chunk r ; half-chunk 2P-1-r]."""
    P = grid.p
    c = X[0].shape[0] // 2
    recv = grid.permute([[X[r][:c], X[r][c:]] for r in range(P)],
                        [[_zz(2 * r, P), _zz(2 * r + 1, P)] for r in range(P)], bpe)
    out = []
    for r in range(P):
        ids = [hc for src in range(P) for hc in (2 * src, 2 * src + 1) if _zz(hc, P) == r]
        byid = dict(zip(ids, recv[r]))
        out.append(np.concatenate([byid[j] for j in _zig(r, P)], axis=0))
    return out


def _from_zigzag(grid, Z, bpe=2):
    """Zigzag rows per rank -> boundary rows (the reverse exchange)."""
    P = grid.p
    c = Z[0].shape[0] // 2
    recv = grid.permute([[Z[r][:c], Z[r][c:]] for r in range(P)],
                        [[j // 2 for j in _zig(r, P)] for r in range(P)], bpe)
    out = []
    for q in range(P):
        ids = [hc for src in range(P) for hc in _zig(src, P) if hc // 2 == q]
        byid = dict(zip(ids, recv[q]))
        out.append(np.concatenate([byid[2 * q], byid[2 * q + 1]], axis=0))
    return out


def _heads(x, n):
    """[rows, b, n*d] -> [b, n, rows, d]"""
    rows, b, hd = x.shape
    return x.reshape(rows, b, n, hd // n).transpose(1, 2, 0, 3)


def _unheads(x):
    b, n, rows, d = x.shape
    return x.transpose(2, 0, 1, 3).reshape(rows, b, n * d)


def _pair_fwd(q, k, v, pq, pk, causal):
    """Softmax attention of queries q [b, n, rq, d] over keys k / values v [b, n, rk, d]
    alone (Eq. 2 restricted to these keys), causal by global position: (O, LSE); rows
    with no visible key have O = 0, LSE = -inf."""
    sc = np.einsum("bnqd,bnkd->bnqk", q, k) / np.sqrt(q.shape[-1])
    if causal:
        sc = np.where(pk[None, None, None, :] > pq[None, None, :, None], -np.inf, sc)
    m = np.max(sc, axis=-1, keepdims=True)
    m_safe = np.where(np.isfinite(m), m, 0.0)
    e = np.exp(sc - m_safe)
    l = np.sum(e, axis=-1, keepdims=True)
    o = np.einsum("bnqk,bnkd->bnqd", e, v) / np.where(l > 0, l, 1.0)
    lse = np.where(l[..., 0] > 0, m_safe[..., 0] + np.log(np.where(l[..., 0] > 0, l[..., 0], 1.0)), -np.inf)
    return o, lse


def _merge(o1, l1, o2, l2):
    """log-sum-exp merge of two partial softmax results over disjoint key sets."""
    lse = np.logaddexp(l1, l2)
    fin = np.isfinite(lse)
    w1 = np.where(fin, np.exp(np.where(fin, l1 - np.where(fin, lse, 0.0), -np.inf)), 0.0)
    w2 = np.where(fin, np.exp(np.where(fin, l2 - np.where(fin, lse, 0.0), -np.inf)), 0.0)
    return w1[..., None] * o1 + w2[..., None] * o2, lse


def _pair_bwd(q, k, v, do, lse, D, pq, pk, causal):
    """The pair's share of the attention backward given the MERGED row LSE and
    D = rowsum(dO o O): P = exp(S - LSE) on the visible keys; dV = P^T dO;
    dS = P o (dO V^T - D); dQ = dS K / sqrt(d); dK = dS^T Q / sqrt(d)."""
    scale = 1.0 / np.sqrt(q.shape[-1])
    sc = np.einsum("bnqd,bnkd->bnqk", q, k) * scale
    p = np.exp(sc - lse[..., None])
    if causal:
        p = np.where(pk[None, None, None, :] > pq[None, None, :, None], 0.0, p)
    dv = np.einsum("bnqk,bnqd->bnkd", p, do)
    ds = p * (np.einsum("bnqd,bnkd->bnqk", do, v) - D[..., None])
    return np.einsum("bnqk,bnkd->bnqd", ds, k) * scale, np.einsum("bnqk,bnqd->bnkd", ds, q) * scale, dv


def cz_fwd(grid, xs, W, cfg):
    P = grid.p
    sl = xs[0].shape[0]
    s = sl * P
    h, n, nk = cfg.h, cfg.n, cfg.n_kv
    grp = n // nk
    c = sl // 2
    if sl % 2:
        raise ValueError("MegatronCZ: s must be divisible by 2P (zigzag half-chunks)")
    wq = _gather_qkv_parts(grid, W, h, n, nk)
    wp = grid.all_gather(W["w_proj"])[0]
    wi = grid.all_gather(W["w_in_t"])[0]
    wo = grid.all_gather(W["w_out"])[0]
    d = h // n
    saved = [dict() for _ in range(P)]
    r1, qkv_b = [], []
    for r in range(P):
        ur, _, rr = rmsnorm(xs[r], W["g1"][r], cfg.eps)
        r1.append(rr)
        qkv = ur @ wq.T                                            # [s/P, b, h + 2 hk], [Q | K | V] all heads
        hk = nk * d
        cos, sin = rope_cos_sin(np.arange(r * sl, (r + 1) * sl), d, cfg.theta)
        qr = _unheads(rope_apply(_heads(qkv[..., :h], n), cos, sin))
        kr = _unheads(rope_apply(_heads(qkv[..., h:h + hk], nk), cos, sin))
        qkv_b.append(np.concatenate([qr, kr, qkv[..., h + hk:]], axis=-1))   # RoPE at global positions
    qkvz = _to_zigzag(grid, qkv_b)                                 # SendRecv(QKV): boundary -> zigzag
    pos = [_zig_positions(r, P, c) for r in range(P)]
    q = [_heads(qkvz[r][..., :h], n) for r in range(P)]
    kv = [qkvz[r][..., h:] for r in range(P)]                      # travels around the ring
    kv_pos = list(pos)
    o_acc = [np.zeros_like(q[r]) for r in range(P)]
    l_acc = [np.full(q[r].shape[:-1], -np.inf) for r in range(P)]
    for k in range(P):
        for r in range(P):
            kk = _rep_kv(_heads(kv[r][..., :nk * d], nk), grp)
            vv = _rep_kv(_heads(kv[r][..., nk * d:], nk), grp)
            for ai in range(2):
                qa = slice(ai * c, (ai + 1) * c)
                for bi in range(2):
                    kb = slice(bi * c, (bi + 1) * c)
                    if cfg.causal and kv_pos[r][kb][0] > pos[r][qa][-1]:
                        continue                                   # key half-chunk after every query
                    o_p, l_p = _pair_fwd(q[r][:, :, qa], kk[:, :, kb], vv[:, :, kb], pos[r][qa],
                                         kv_pos[r][kb], cfg.causal)
                    o_acc[r][:, :, qa], l_acc[r][:, :, qa] = _merge(o_acc[r][:, :, qa], l_acc[r][:, :, qa],
                                                                   o_p, l_p)
        if k < P - 1:
            kv = grid.ring_pass(kv, bpe=2)                         # K/V of rank r - k - 1 next
            kv_pos = [kv_pos[(r - 1) % P] for r in range(P)]
    a_all = _from_zigzag(grid, [_unheads(o_acc[r]) for r in range(P)])   # SendRecv(O): back to boundary
    y, o, z = [], [], []
    for r in range(P):
        a_r = a_all[r]
        o_r = a_r @ wp
        x1 = xs[r] + o_r
        vr, _, rr2 = rmsnorm(x1, W["g2"][r], cfg.eps)
        hp = vr @ wi.T
        z_r = _act(hp, cfg) @ wo
        o.append(o_r)
        z.append(z_r)
        y.append(x1 + z_r)
        sv = saved[r]
        _save(grid, r, sv, "x", xs[r], 2)
        _save(grid, r, sv, "r1", r1[r], 4)
        _save(grid, r, sv, "qkv", qkvz[r], 2)                      # zigzag rows, post-RoPE
        _save(grid, r, sv, "a", a_r, 2)                            # boundary rows
        _save(grid, r, sv, "lse", l_acc[r], 4)                     # zigzag rows
        _save(grid, r, sv, "x1", x1, 2)
        _save(grid, r, sv, "r2", rr2, 4)
        _save(grid, r, sv, "h", hp, 2)
    return y, saved, dict(o=o, z=z)


def cz_bwd(grid, dys, saved, W, cfg, grads):
    P = grid.p
    sl = dys[0].shape[0]
    h, n, nk = cfg.h, cfg.n, cfg.n_kv
    grp = n // nk
    d = h // n
    hk = nk * d
    c = sl // 2
    sv = saved
    wq = _gather_qkv_parts(grid, W, h, n, nk)
    wp = grid.all_gather(W["w_proj"])[0]
    wi = grid.all_gather(W["w_in_t"])[0]
    wo = grid.all_gather(W["w_out"])[0]
    dwo, dwi, dwp, dwq = [], [], [], []
    dx1, dg2, da = [], [], []
    for r in range(P):
        hp = sv[r]["h"]
        v = _apply_norm(sv[r]["x1"], sv[r]["r2"], W["g2"][r])
        dg = dys[r] @ wo.T
        dh = _act_bwd(dg, hp, cfg)
        dwo.append(np.tensordot(_act(hp, cfg), dys[r], axes=([0, 1], [0, 1])))
        dwi.append(np.tensordot(dh, v, axes=([0, 1], [0, 1])))
        xhat2 = sv[r]["x1"] * sv[r]["r2"][..., None]
        dd, dgr = rmsnorm_bwd(dh @ wi, xhat2, sv[r]["r2"], W["g2"][r])
        dx1.append(dys[r] + dd)
        dg2.append(dgr)
        da.append(dx1[r] @ wp.T)                                   # dA, boundary rows
        dwp.append(np.tensordot(sv[r]["a"], dx1[r], axes=([0, 1], [0, 1])))
    oz = _to_zigzag(grid, [sv[r]["a"] for r in range(P)])          # SendRecv(O) -> zigzag
    doz = _to_zigzag(grid, da)                                     # SendRecv(dO) -> zigzag
    pos = [_zig_positions(r, P, c) for r in range(P)]
    q = [_heads(sv[r]["qkv"][..., :h], n) for r in range(P)]
    do_h = [_heads(doz[r], n) for r in range(P)]
    D = [np.sum(do_h[r] * _heads(oz[r], n), axis=-1) for r in range(P)]
    lse = [sv[r]["lse"] for r in range(P)]
    kv = [sv[r]["qkv"][..., h:] for r in range(P)]
    kv_pos = list(pos)
    dkv = [np.zeros_like(kv[r]) for r in range(P)]                 # travels with its K/V block (fp32)
    dq = [np.zeros_like(q[r]) for r in range(P)]
    for k in range(P):
        for r in range(P):
            kk = _rep_kv(_heads(kv[r][..., :hk], nk), grp)
            vv = _rep_kv(_heads(kv[r][..., hk:], nk), grp)
            dk_h = np.zeros_like(kk)
            dv_h = np.zeros_like(vv)
            for ai in range(2):
                qa = slice(ai * c, (ai + 1) * c)
                for bi in range(2):
                    kb = slice(bi * c, (bi + 1) * c)
                    if cfg.causal and kv_pos[r][kb][0] > pos[r][qa][-1]:
                        continue
                    gq, gk, gv = _pair_bwd(q[r][:, :, qa], kk[:, :, kb], vv[:, :, kb], do_h[r][:, :, qa],
                                           lse[r][:, :, qa], D[r][:, :, qa], pos[r][qa], kv_pos[r][kb],
                                           cfg.causal)
                    dq[r][:, :, qa] += gq
                    dk_h[:, :, kb] += gk
                    dv_h[:, :, kb] += gv
            dkv[r] = dkv[r] + np.concatenate([_unheads(_fold_kv(dk_h, grp)), _unheads(_fold_kv(dv_h, grp))],
                                             axis=-1)
        if k < P - 1:
            kv = grid.ring_pass(kv, bpe=2)
            kv_pos = [kv_pos[(r - 1) % P] for r in range(P)]
        dkv = grid.ring_pass(dkv, bpe=4)                           # P passes: home after the last
    dqkvz = []
    for r in range(P):
        cos, sin = rope_cos_sin(pos[r], d, cfg.theta)              # RoPE^T at the zigzag positions
        dqr = _unheads(rope_apply_t(dq[r], cos, sin))
        dkr = _unheads(rope_apply_t(_heads(dkv[r][..., :hk], nk), cos, sin))
        dqkvz.append(np.concatenate([dqr, dkr, dkv[r][..., hk:]], axis=-1))
    dqkv = _from_zigzag(grid, dqkvz)                               # SendRecv(dQKV) -> boundary
    dx, dg1 = [], []
    for r in range(P):
        u = _apply_norm(sv[r]["x"], sv[r]["r1"], W["g1"][r])
        dwq.append(np.tensordot(dqkv[r], u, axes=([0, 1], [0, 1])))   # [3h, h], [Q; K; V] all
        du = dqkv[r] @ wq
        xhat1 = sv[r]["x"] * sv[r]["r1"][..., None]
        dd, dgr = rmsnorm_bwd(du, xhat1, sv[r]["r1"], W["g1"][r])
        dx.append(dx1[r] + dd)
        dg1.append(dgr)
    # ZeRO3 reduce-scatters (fp32): W_qkv^T part by part back into [Q_r; K_r; V_r]
    qparts = [grid.reduce_scatter([dwq[r][a:b] for r in range(P)], axis=0, bpe=4)
              for a, b in ((0, h), (h, h + hk), (h + hk, h + 2 * hk))]
    for r in range(P):
        grads["dw_qkv_t"][r] += np.concatenate([qparts[i][r] for i in range(3)], axis=0)
    for key, full in (("dw_proj", dwp), ("dw_in_t", dwi), ("dw_out", dwo)):
        part = grid.reduce_scatter(full, axis=0, bpe=4)
        for r in range(P):
            grads[key][r] += part[r]
    _finish_dgamma(grid, grads, dg1, dg2)
    for r in range(P):
        _release(grid, sv[r])
    return dx


# ------------------------------------------------------------------ ColossalZ (RSA)
# Reading R-COL: Colossal-AI sequence parallelism + ZeRO3 weights
# (PAPER.md:220).  Weights and every GEMM as MegatronCZ (local boundary rows); the
# attention is Ring Self-Attention on the contiguous boundary chunks: the keys pass
# around the ring and every rank materialises its rows' full score matrix
# [n, s/P, s] (quadratic memory, the paper's reason to exclude it),
# a plain row softmax gives the probabilities (saved for the backward), then the
# values pass around the ring for O = P V.  Backward: values again (dP = dO V^T,
# dV partials travelling with their block), dS = P o (dP - D), keys again (dQ = dS K,
# dK partials travelling with their block).

def _ring_blocks(grid, blocks, bpe):
    """P steps of the ring: yields (step, blocks held now) and passes after each step but
    the last (P - 1 RingPass)."""
    P = grid.p
    for k in range(P):
        yield k, blocks
        if k < P - 1:
            blocks = grid.ring_pass(blocks, bpe=bpe)


def colossal_fwd(grid, xs, W, cfg):
    P = grid.p
    sl = xs[0].shape[0]
    s = sl * P
    h, n, nk = cfg.h, cfg.n, cfg.n_kv
    grp = n // nk
    d = h // n
    hk = nk * d
    wq = _gather_qkv_parts(grid, W, h, n, nk)
    wp = grid.all_gather(W["w_proj"])[0]
    wi = grid.all_gather(W["w_in_t"])[0]
    wo = grid.all_gather(W["w_out"])[0]
    saved = [dict() for _ in range(P)]
    r1, qkv_b = [], []
    for r in range(P):
        ur, _, rr = rmsnorm(xs[r], W["g1"][r], cfg.eps)
        r1.append(rr)
        qkv = ur @ wq.T
        cos, sin = rope_cos_sin(np.arange(r * sl, (r + 1) * sl), d, cfg.theta)
        qr = _unheads(rope_apply(_heads(qkv[..., :h], n), cos, sin))
        kr = _unheads(rope_apply(_heads(qkv[..., h:h + hk], nk), cos, sin))
        qkv_b.append(np.concatenate([qr, kr, qkv[..., h + hk:]], axis=-1))
    q = [_heads(qkv_b[r][..., :h], n) for r in range(P)]
    b = xs[0].shape[1]
    scores = [np.zeros((b, n, sl, s)) for _ in range(P)]
    for k, kb in _ring_blocks(grid, [qkv_b[r][..., h:h + hk] for r in range(P)], 2):    # ring of K
        for r in range(P):
            j = (r - k) % P
            scores[r][..., j * sl:(j + 1) * sl] = np.einsum("bnqd,bnkd->bnqk", q[r],
                                                            _rep_kv(_heads(kb[r], nk), grp)) / np.sqrt(d)
    probs = []
    for r in range(P):
        sc = scores[r]
        if cfg.causal:
            pos_q = np.arange(r * sl, (r + 1) * sl)
            sc = np.where(np.arange(s)[None, None, None, :] > pos_q[None, None, :, None], -np.inf, sc)
        m = np.max(sc, axis=-1, keepdims=True)
        e = np.exp(sc - m)
        probs.append(e / np.sum(e, axis=-1, keepdims=True))
    o = [np.zeros_like(q[r]) for r in range(P)]
    for k, vb in _ring_blocks(grid, [qkv_b[r][..., h + hk:] for r in range(P)], 2):     # ring of V
        for r in range(P):
            j = (r - k) % P
            o[r] += np.einsum("bnqk,bnkd->bnqd", probs[r][..., j * sl:(j + 1) * sl], _rep_kv(_heads(vb[r], nk), grp))
    y, oo, z = [], [], []
    for r in range(P):
        a_r = _unheads(o[r])
        o_r = a_r @ wp
        x1 = xs[r] + o_r
        vr, _, rr2 = rmsnorm(x1, W["g2"][r], cfg.eps)
        hp = vr @ wi.T
        z_r = _act(hp, cfg) @ wo
        oo.append(o_r)
        z.append(z_r)
        y.append(x1 + z_r)
        sv = saved[r]
        _save(grid, r, sv, "x", xs[r], 2)
        _save(grid, r, sv, "r1", r1[r], 4)
        _save(grid, r, sv, "qkv", qkv_b[r], 2)                     # boundary rows, post-RoPE
        _save(grid, r, sv, "a", a_r, 2)
        _save(grid, r, sv, "probs", probs[r], 2)                   # [b, n, s/P, s]: quadratic
        _save(grid, r, sv, "x1", x1, 2)
        _save(grid, r, sv, "r2", rr2, 4)
        _save(grid, r, sv, "h", hp, 2)
    return y, saved, dict(o=oo, z=z)


def colossal_bwd(grid, dys, saved, W, cfg, grads):
    P = grid.p
    sl = dys[0].shape[0]
    h, n, nk = cfg.h, cfg.n, cfg.n_kv
    grp = n // nk
    d = h // n
    hk = nk * d
    sv = saved
    wq = _gather_qkv_parts(grid, W, h, n, nk)
    wp = grid.all_gather(W["w_proj"])[0]
    wi = grid.all_gather(W["w_in_t"])[0]
    wo = grid.all_gather(W["w_out"])[0]
    dwo, dwi, dwp, dwq = [], [], [], []
    dx1, dg2, da = [], [], []
    for r in range(P):
        hp = sv[r]["h"]
        v = _apply_norm(sv[r]["x1"], sv[r]["r2"], W["g2"][r])
        dg = dys[r] @ wo.T
        dh = _act_bwd(dg, hp, cfg)
        dwo.append(np.tensordot(_act(hp, cfg), dys[r], axes=([0, 1], [0, 1])))
        dwi.append(np.tensordot(dh, v, axes=([0, 1], [0, 1])))
        xhat2 = sv[r]["x1"] * sv[r]["r2"][..., None]
        dd, dgr = rmsnorm_bwd(dh @ wi, xhat2, sv[r]["r2"], W["g2"][r])
        dx1.append(dys[r] + dd)
        dg2.append(dgr)
        da.append(dx1[r] @ wp.T)
        dwp.append(np.tensordot(sv[r]["a"], dx1[r], axes=([0, 1], [0, 1])))
    do_h = [_heads(da[r], n) for r in range(P)]
    D = [np.sum(do_h[r] * _heads(sv[r]["a"], n), axis=-1) for r in range(P)]
    probs = [sv[r]["probs"] for r in range(P)]
    dp = [np.zeros_like(probs[r]) for r in range(P)]
    dvacc = [np.zeros_like(sv[r]["qkv"][..., h + hk:]) for r in range(P)]
    for k, vb in _ring_blocks(grid, [sv[r]["qkv"][..., h + hk:] for r in range(P)], 2):  # ring of V
        for r in range(P):
            j = (r - k) % P
            blk = slice(j * sl, (j + 1) * sl)
            dp[r][..., blk] = np.einsum("bnqd,bnkd->bnqk", do_h[r], _rep_kv(_heads(vb[r], nk), grp))
            dvacc[r] = dvacc[r] + _unheads(_fold_kv(np.einsum("bnqk,bnqd->bnkd", probs[r][..., blk], do_h[r]), grp))
        dvacc = grid.ring_pass(dvacc, bpe=4)                        # dV partials travel home (P passes)
    ds = [probs[r] * (dp[r] - D[r][..., None]) / np.sqrt(d) for r in range(P)]
    q = [_heads(sv[r]["qkv"][..., :h], n) for r in range(P)]
    dq = [np.zeros_like(q[r]) for r in range(P)]
    dkacc = [np.zeros_like(sv[r]["qkv"][..., h:h + hk]) for r in range(P)]
    for k, kb in _ring_blocks(grid, [sv[r]["qkv"][..., h:h + hk] for r in range(P)], 2):  # ring of K
        for r in range(P):
            j = (r - k) % P
            blk = slice(j * sl, (j + 1) * sl)
            dq[r] += np.einsum("bnqk,bnkd->bnqd", ds[r][..., blk], _rep_kv(_heads(kb[r], nk), grp))
            dkacc[r] = dkacc[r] + _unheads(_fold_kv(np.einsum("bnqk,bnqd->bnkd", ds[r][..., blk], q[r]), grp))
        dkacc = grid.ring_pass(dkacc, bpe=4)
    dx, dg1 = [], []
    for r in range(P):
        cos, sin = rope_cos_sin(np.arange(r * sl, (r + 1) * sl), d, cfg.theta)
        dqkv = np.concatenate([_unheads(rope_apply_t(dq[r], cos, sin)),
                               _unheads(rope_apply_t(_heads(dkacc[r], nk), cos, sin)), dvacc[r]], axis=-1)
        u = _apply_norm(sv[r]["x"], sv[r]["r1"], W["g1"][r])
        dwq.append(np.tensordot(dqkv, u, axes=([0, 1], [0, 1])))
        du = dqkv @ wq
        xhat1 = sv[r]["x"] * sv[r]["r1"][..., None]
        dd, dgr = rmsnorm_bwd(du, xhat1, sv[r]["r1"], W["g1"][r])
        dx.append(dx1[r] + dd)
        dg1.append(dgr)
    qparts = [grid.reduce_scatter([dwq[r][a:b] for r in range(P)], axis=0, bpe=4)
              for a, b in ((0, h), (h, h + hk), (h + hk, h + 2 * hk))]
    for r in range(P):
        grads["dw_qkv_t"][r] += np.concatenate([qparts[i][r] for i in range(3)], axis=0)
    for key, full in (("dw_proj", dwp), ("dw_in_t", dwi), ("dw_out", dwo)):
        part = grid.reduce_scatter(full, axis=0, bpe=4)
        for r in range(P):
            grads[key][r] += part[r]
    _finish_dgamma(grid, grads, dg1, dg2)
    for r in range(P):
        _release(grid, sv[r])
    return dx


def _full(cfg):
    """METP-full (strategy 4) = R-METP with metp_recompute = 'full' (SURVEY O-5 / O-6),
    a strategy of its own so the planner can choose it per layer."""
    c = copy.copy(cfg)
    c.metp_recompute = "full"
    return c


def metp_full_fwd(grid, xs, W, cfg):
    return metp_fwd(grid, xs, W, _full(cfg))


def metp_full_bwd(grid, dys, saved, W, cfg, grads):
    return metp_bwd(grid, dys, saved, W, _full(cfg), grads)


REGISTRY = {TS: (ts_fwd, ts_bwd), UZ: (uz_fwd, uz_bwd), METP: (metp_fwd, metp_bwd), CZ: (cz_fwd, cz_bwd),
            METP_FULL: (metp_full_fwd, metp_full_bwd), COL: (colossal_fwd, colossal_bwd)}


def layer_fwd(pi, grid, xs, W, cfg):
    """Registry lookup f_pi — the uniform signature."""
    if pi not in REGISTRY:
        raise KeyError(f"unknown strategy {pi} (SPEC.md:244)")
    return REGISTRY[pi][0](grid, xs, W, cfg)


def layer_bwd(pi, grid, dys, saved, W, cfg, grads):
    if pi not in REGISTRY:
        raise KeyError(f"unknown strategy {pi} (SPEC.md:244)")
    return REGISTRY[pi][1](grid, dys, saved, W, cfg, grads)


def new_grads(W):
    g = _zero_grads(W)
    g.pop("_p")
    return g
