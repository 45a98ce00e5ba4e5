"""Spec-layout shards — Table 2 "Specification" row (TEST INFRASTRUCTURE).

  activations X_MHA, O, X_FFN, Z : b x s/p x h, rank r owns positions
                                   [r s/P, (r+1) s/P) (R-10; stored [s/P, b, h])
  W_qkv   stored (3h/p x h)^T    : rank r holds the 3h/P x h block made of the
                                   Q rows of head group r, then its K rows, then
                                   its V rows; group r = heads [r n/P, (r+1) n/P) (R-9)
  W_proj  h/p x h                : rows [r h/P, (r+1) h/P)
  W_in    stored (4h/p x h)^T    : rows [r F/P, (r+1) F/P) of W_in^T
  W_out   4h/p x h               : rows [r F/P, (r+1) F/P)
  g1, g2                         : replicated

Llama variant (NEXT-3; readings R-GQA / R-SWIGLU): with n_kv key/value heads the
W_qkv shard holds the Q rows of head group r (n/P heads), then the K rows of KV
group r (n_kv/P heads), then its V rows ((n + 2 n_kv) d / P x h); with SwiGLU,
W_in [h, 2F] = [W_gate | W_up] is stored with its columns interleaved in blocks of
64 (gate block j, then up block j: `il_perm`), transposed, and row-sharded, so
every shard and every row-wise gather of shards keeps whole (gate, up) pairs.

The transposed storage of W_qkv / W_in is the paper's so a
ZeRO3 row-wise AllGather is memory-contiguous.  Pins: shard/unshard round
trip is exact; Table 2 fixture (tests/test_oracle_layouts.py).
"""
from __future__ import annotations

import numpy as np


def check_div(name, val, p):
    if val % p:
        raise ValueError(f"{name}={val} not divisible by P={p} (SPEC.md:184)")


def shard_act(x, p):
    check_div("s", x.shape[0], p)
    return [c.copy() for c in np.split(x, p, axis=0)]


def unshard_act(shards):
    return np.concatenate(shards, axis=0)


def shard_wqkv_t(w_qkv, n, p, n_kv=None):
    """w_qkv [h, (n + 2 n_kv) d] ([Q | K | V] columns) -> list of transposed
    ((n + 2 n_kv) d / P x h) blocks: Q of head group r, K and V of KV group r."""
    h = w_qkv.shape[0]
    nk = n if n_kv is None else n_kv
    check_div("n", n, p)
    check_div("n_kv", nk, p)
    d = w_qkv.shape[1] // (n + 2 * nk)
    gq, gk = (n // p) * d, (nk // p) * d
    base = (0, n * d, (n + nk) * d)
    width = (gq, gk, gk)
    out = []
    for r in range(p):
        cols = [w_qkv[:, base[i] + r * width[i]: base[i] + (r + 1) * width[i]] for i in range(3)]
        out.append(np.concatenate(cols, axis=1).T.copy())
    return out


def unshard_wqkv_t(shards, n, n_kv=None):
    p = len(shards)
    h = shards[0].shape[1]
    nk = n if n_kv is None else n_kv
    d = shards[0].shape[0] * p // (n + 2 * nk)
    gq, gk = (n // p) * d, (nk // p) * d
    base = (0, n * d, (n + nk) * d)
    width = (gq, gk, gk)
    w = np.empty((h, (n + 2 * nk) * d))
    for r, blk_t in enumerate(shards):
        blk = blk_t.T
        o = 0
        for i in range(3):
            w[:, base[i] + r * width[i]: base[i] + (r + 1) * width[i]] = blk[:, o:o + width[i]]
            o += width[i]
    return w


def il_perm(F, il=64):
    """Column order of the spec-layout SwiGLU W_in: for each block j of `il` FFN
    columns, the gate columns [j il, (j+1) il) then the up columns F + [j il, (j+1) il)."""
    if F % il:
        raise ValueError(f"ffn={F} not divisible by the interleave {il}")
    idx = []
    for j in range(F // il):
        idx.extend(range(j * il, (j + 1) * il))
        idx.extend(range(F + j * il, F + (j + 1) * il))
    return np.array(idx)


def shard_rows(w, p):
    check_div("rows", w.shape[0], p)
    return [c.copy() for c in np.split(w, p, axis=0)]


def shard_weights(dense, n, p, n_kv=None, act="gelu"):
    """Dense oracle weights -> per-rank spec-layout shards (dict of lists)."""
    w_in = dense["w_in"]
    if act == "swiglu":
        w_in = w_in[:, il_perm(w_in.shape[1] // 2)]
    return dict(
        w_qkv_t=shard_wqkv_t(dense["w_qkv"], n, p, n_kv),
        w_proj=shard_rows(dense["w_proj"], p),
        w_in_t=shard_rows(w_in.T, p),
        w_out=shard_rows(dense["w_out"], p),
        g1=[dense["g1"].copy() for _ in range(p)],
        g2=[dense["g2"].copy() for _ in range(p)],
    )


def unshard_grads(gsh, n, n_kv=None, act="gelu"):
    """Per-rank spec-layout gradient shards -> dense oracle-orientation grads."""
    dw_in = np.concatenate(gsh["dw_in_t"], axis=0).T
    if act == "swiglu":
        plain = np.empty_like(dw_in)
        plain[:, il_perm(dw_in.shape[1] // 2)] = dw_in
        dw_in = plain
    return dict(
        dw_qkv=unshard_wqkv_t(gsh["dw_qkv_t"], n, n_kv),
        dw_proj=np.concatenate(gsh["dw_proj"], axis=0),
        dw_in=dw_in,
        dw_out=np.concatenate(gsh["dw_out"], axis=0),
        dg1=gsh["dg1"][0],
        dg2=gsh["dg2"][0],
    )
