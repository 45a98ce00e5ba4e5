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


def shard_wqkv_t(w_qkv, n, p):
    """w_qkv [h, 3h] ([Q | K | V] columns) -> list of (3h/P x h) transposed blocks."""
    h = w_qkv.shape[0]
    check_div("n", n, p)
    d = h // n
    g = (n // p) * d
    out = []
    for r in range(p):
        cols = []
        for blk in range(3):
            c0 = blk * h + r * g
            cols.append(w_qkv[:, c0:c0 + g])
        out.append(np.concatenate(cols, axis=1).T.copy())
    return out


def unshard_wqkv_t(shards, n):
    p = len(shards)
    h = shards[0].shape[1]
    d = h // n
    g = (n // p) * d
    w = np.empty((h, 3 * h))
    for r, blk_t in enumerate(shards):
        blk = blk_t.T
        for b in range(3):
            w[:, b * h + r * g: b * h + (r + 1) * g] = blk[:, b * g:(b + 1) * g]
    return w


def shard_rows(w, p):
    check_div("rows", w.shape[0], p)
    return [c.copy() for c in np.split(w, p, axis=0)]


def shard_weights(dense, n, p):
    """Dense oracle weights -> per-rank spec-layout shards (dict of lists)."""
    return dict(
        w_qkv_t=shard_wqkv_t(dense["w_qkv"], n, p),
        w_proj=shard_rows(dense["w_proj"], p),
        w_in_t=shard_rows(dense["w_in"].T, p),
        w_out=shard_rows(dense["w_out"], p),
        g1=[dense["g1"].copy() for _ in range(p)],
        g2=[dense["g2"].copy() for _ in range(p)],
    )


def unshard_grads(gsh, n):
    """Per-rank spec-layout gradient shards -> dense oracle-orientation grads."""
    return dict(
        dw_qkv=unshard_wqkv_t(gsh["dw_qkv_t"], n),
        dw_proj=np.concatenate(gsh["dw_proj"], axis=0),
        dw_in=np.concatenate(gsh["dw_in_t"], axis=0).T,
        dw_out=np.concatenate(gsh["dw_out"], axis=0),
        dg1=gsh["dg1"][0],
        dg2=gsh["dg2"][0],
    )
