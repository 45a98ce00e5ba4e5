"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no norm, no attention, no GEMM,
no cost model).  It only draws numbers:

* ``normal(seed, tensor_id, shape, std, mean)`` — a counter-based generator
  (splitmix64 of ``(seed, tensor_id, flat index)`` -> Box-Muller), so any
  element can be regenerated independently of the others.  Values are rounded
  to the nearest bf16 (round-to-nearest-even) and returned as float64 arrays
  that hold bf16-exact values, so the fp64 oracle and the bf16 device path see
  the *same* numbers.
* ``bf16_bits(a)`` — the raw uint16 bf16 encoding of a bf16-exact float64
  array (for uploading to the device without another rounding step).
* ``layer_inputs(...)`` — the recipe of DESIGN.md §"Input recipe": x ~ N(0,1),
  W ~ N(0, 1/h), gamma ~ 1 + N(0, 0.1^2), dY ~ N(0,1).
* ``sample_lengths(...)`` — Table 3 length histograms,
  log-uniform within buckets (reading R-30).
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
    z = x
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
    return z ^ (z >> np.uint64(31))


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 (RNE), returned as float64."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = (u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """uint16 encoding of a bf16-exact float64 array."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(bits: np.ndarray) -> np.ndarray:
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)


def normal(seed: int, tensor_id: int, shape, std: float = 1.0, mean: float = 0.0,
           bf16: bool = True) -> np.ndarray:
    n = int(np.prod(shape)) if len(shape) else 1
    idx = np.arange(n, dtype=np.uint64)
    key = np.uint64((seed & 0xFFFFFF) << 40 | (tensor_id & 0xFFFF) << 24)
    a = _splitmix64(_splitmix64(idx * np.uint64(2) + key))
    b = _splitmix64(_splitmix64(idx * np.uint64(2) + np.uint64(1) + key))
    u1 = ((a >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    u2 = (b >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    v = (mean + std * z).reshape(shape)
    return round_bf16(v) if bf16 else v


# tensor ids of the recipe (stable: tests and bench rely on them)
TID = dict(x=1, w_qkv=2, w_proj=3, w_in=4, w_out=5, g1=6, g2=7, dy=8)


def layer_inputs(h: int, n_heads: int, ffn: int, s: int, b: int = 1, seed: int = 42,
                 layer: int = 0, n_kv: int | None = None, act: str = "gelu"):
    """Dense (unsharded) inputs of one layer in the oracle's orientation.

    Returns a dict of bf16-exact float64 arrays:
      x [s, b, h]; w_qkv [h, (n + 2 n_kv) d] (columns [Q | K | V], head i at i*d;
      n_kv = n_heads unless given: GQA); w_proj [h, h]; w_in [h, ffn] (SwiGLU:
      [h, 2 ffn] = [W_gate | W_up]); w_out [ffn, h]; g1, g2 [h]; dy [s, b, h].
    """
    off = 16 * layer
    std_w = 1.0 / np.sqrt(h)
    nk = n_heads if n_kv is None else n_kv
    wq = (n_heads + 2 * nk) * (h // n_heads)
    fin = 2 * ffn if act == "swiglu" else ffn
    return dict(
        x=normal(seed, TID["x"] + off, (s, b, h)),
        w_qkv=normal(seed, TID["w_qkv"] + off, (h, wq), std=std_w),
        w_proj=normal(seed, TID["w_proj"] + off, (h, h), std=std_w),
        w_in=normal(seed, TID["w_in"] + off, (h, fin), std=std_w),
        w_out=normal(seed, TID["w_out"] + off, (ffn, h), std=1.0 / np.sqrt(ffn)),
        g1=normal(seed, TID["g1"] + off, (h,), std=0.1, mean=1.0),
        g2=normal(seed, TID["g2"] + off, (h,), std=0.1, mean=1.0),
        dy=normal(seed, TID["dy"] + off, (s, b, h)),
    )


# Table 3: bucket edges in tokens (K = 1024, reading R-30)
K = 1024
BUCKETS = [(256, 4 * K), (4 * K, 8 * K), (8 * K, 16 * K), (16 * K, 32 * K),
           (32 * K, 64 * K), (64 * K, 128 * K), (128 * K, None)]
HIST = {
    "githubcode": ([65.7, 14.5, 9.8, 5.1, 2.7, 1.1, 1.1], 309 * K),
    "grch38": ([3.5, 26.4, 28.7, 21.2, 11.9, 5.5, 1.9], 624 * K),
}


def sample_lengths(dataset: str, n: int, seed: int = 42) -> np.ndarray:
    """n lengths from the Table 3 histogram of ``dataset`` (renormalised, R-29),
    log-uniform within each bucket; the open last bucket is capped at the
    dataset maximum (R-30).  Deterministic in ``seed``."""
    pct, smax = HIST[dataset]
    p = np.asarray(pct, dtype=np.float64)
    p = p / p.sum()
    rng = np.random.default_rng(seed)
    bucket = rng.choice(len(p), size=n, p=p)
    u = rng.random(n)
    out = np.empty(n, dtype=np.int64)
    for i, (bk, uu) in enumerate(zip(bucket, u)):
        lo, hi = BUCKETS[bk]
        hi = smax + 1 if hi is None else hi
        v = int(np.exp(np.log(lo) + uu * (np.log(hi) - np.log(lo))))
        out[i] = min(max(v, lo), hi - 1)
    return out


def pad_to(s: int, multiple: int) -> int:
    return ((s + multiple - 1) // multiple) * multiple
