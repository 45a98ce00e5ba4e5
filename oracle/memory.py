"""Per-layer, per-rank memory model in bytes (TEST INFRASTRUCTURE).

Eq. 6 constrains sum_l M_{pi_l}(X) < OOM.  The paper's memory
model was learned from profiles and is admitted to be coarse;
this build reads M analytically (R-22, SURVEY O-6):

  units   u = (s/P) b h 2 B      l = (s/P) b 4 B      lam = (n/P) s b 4 B
  persistent W = (3h^2 + h^2 + 2hF)/P (2 + 4) + 2h (2 + 4)   (bf16 weights + fp32 grads)
  saved   TS   = 6u + (F/h)u + 2l + lam   x, r1, QKV(3u), A(1u), LSE, x1, r2, H(F/h u)
          UZ   = 7u + (F/h)u + 2l + lam   as TS + post-A2A attention output (1u)
          METP = 6u + 2l + lam            (metp_recompute = ffn: H recomputed)
          METP = 3u + 2l + lam            (metp_recompute = full: QKV recomputed too)
  plan    sum_l (W + saved_{pi_l}) + max_{pi enabled} transient_pi + reserve < capacity

Pin: the saved formula equals the simulated grid's ledger recount of the
tensors the sharded simulations keep for backward (tests/test_oracle_memory.py,
SPEC.md:99); the C1 worked example of SURVEY O-6.  The transient term is the
workspace plan of the CUDA path written out independently;
"parity unpinned" against a measured device peak until the T5 measurement.
"""
from __future__ import annotations

TS, UZ, METP = 0, 1, 2


def units(h, n, s, P, b=1):
    sl = s // P
    return sl * b * h * 2, sl * b * 4, (n // P) * s * b * 4


def persistent(h, ffn, P):
    return (4 * h * h + 2 * h * ffn) // P * 6 + 2 * h * 6


def saved(pi, h, n, ffn, s, P, b=1, metp_recompute="ffn"):
    u, l, lam = units(h, n, s, P, b)
    f = ffn // h
    if pi == TS:
        return (6 + f) * u + 2 * l + lam
    if pi == UZ:
        return (7 + f) * u + 2 * l + lam
    if pi == METP:
        return (6 if metp_recompute == "ffn" else 3) * u + 2 * l + lam
    raise KeyError(pi)


def transient(pi, h, n, ffn, s, P, b=1, metp_chunks=None):
    """Workspace bytes of the CUDA path's buffer plan, per rank.

    Buffers (bf16 unless noted), with u = one [s/P, b, h] activation:
      TS   fwd: gather P u, partial P u, G (F/h) P?  -> see formulas below
    The plan is written as max(fwd, bwd) of the live-buffer maxima.
    """
    u, l, lam = units(h, n, s, P, b)
    f = ffn // h
    sl_rows = s // P
    if pi == TS:
        fwd = 2 * P * u + f * u + 2 * u
        bwd = P * u + 2 * f * u + 5 * u + 2 * P * u
        return max(fwd, bwd)
    if pi == UZ:
        wfull = (4 * h * h + 2 * h * ffn) * 2
        dwfull = max(3 * h * h, h * h, h * ffn) * 4
        fwd = wfull + 3 * u + 2 * u + f * u * 2
        bwd = wfull + dwfull + 2 * f * u + 6 * u + 3 * u
        return max(fwd, bwd)
    if pi == METP:
        c = metp_chunks or P
        w = P * u // c
        fwd = 3 * w + f * w + 2 * u
        bwd = 3 * w + 3 * f * w + 5 * u + 2 * u
        return max(fwd, bwd)
    raise KeyError(pi)


def layer_bytes(pi, h, n, ffn, s, P, b=1, metp_recompute="ffn"):
    """M_pi(s) of Eq. 6 for one layer: persistent + saved."""
    return persistent(h, ffn, P) + saved(pi, h, n, ffn, s, P, b, metp_recompute)
