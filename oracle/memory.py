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

TS, UZ, METP, CZ = 0, 1, 2, 3


def units(h, n, s, P, b=1):
    sl = s // P
    return sl * b * h * 2, sl * b * 4, (n // P) * s * b * 4


def persistent(h, ffn, P):
    return (4 * h * h + 2 * h * ffn) // P * 6 + 2 * h * 6


def saved(pi, h, n, ffn, s, P, b=1, metp_recompute="ffn"):
    u, l, lam = units(h, n, s, P, b)
    f = ffn // h
    if pi == TS or pi == CZ:           # CZ saves its local rows of the same tensors
        return (6 + f) * u + 2 * l + lam
    if pi == UZ:
        return (7 + f) * u + 2 * l + lam
    if pi == METP:
        return (6 if metp_recompute == "ffn" else 3) * u + 2 * l + lam
    raise KeyError(pi)


def _al(x):
    return (x + 255) // 256 * 256


def _norm_bwd_grid(rows):
    return min((rows + 3) // 4, 444)   # 148 SMs x 3 resident 256-thread blocks


def transient(pi, h, n, ffn, s, P, b=1, metp_chunks=None, metp_recompute="ffn"):
    """Workspace bytes per rank of the CUDA path's buffer plan,
    each buffer rounded up to 256 B.  Written out from the plan table, not shared
    with the library (tests compare it with pds_mem_bytes).  Token buffers hold
    rows = positions x b (layout [s, b, h])."""
    sl = s // P
    u = sl * b * h * 2
    lam = (n // P) * s * b * 4
    hl, Fl = h // P, ffn // P
    small = _al(2 * h * 4)
    S, SL = s * b, sl * b                  # token rows (all / this rank)
    if pi == TS:
        bufs = [S * h * 2, S * h * 2, S * Fl * 2, S * Fl * 2, lam, _norm_bwd_grid(SL) * h * 4,
                max(Fl, 3 * hl) * S * 2, h * S * 2, h * max(Fl, 3 * hl) * 2]
        if P > 1:
            bufs.append(S * h * 2)      # second gather buffer: bwd re-gathers prefetched

    elif pi == UZ:
        bufs = [3 * h * h * 2, h * h * 2, ffn * h * 2, ffn * h * 2, max(3 * h, ffn) * h * 4,
                u, 3 * u, 3 * u, SL * ffn * 2, SL * ffn * 2, 3 * u, 3 * u, u, lam,
                _norm_bwd_grid(SL) * h * 4, max(ffn, 3 * h) * SL * 2, h * SL * 2, h * max(ffn, 3 * h) * 2]
    elif pi == CZ:
        # full weights + fp32 dW (ZeRO3), gathered Q/K/V of the whole context and the
        # all-rows dQ/dK/dV partials (RS in place), local FFN / attention scratch
        bufs = [3 * h * h * 2, h * h * 2, ffn * h * 2, ffn * h * 2, max(3 * h, ffn) * h * 4,
                u, S * 3 * h * 2, S * 3 * h * 2, SL * ffn * 2, SL * ffn * 2, u, u, lam,
                _norm_bwd_grid(SL) * h * 4, max(ffn, 3 * h) * SL * 2, h * SL * 2, h * max(ffn, 3 * h) * 2]
    elif pi == METP:
        c = metp_chunks or P
        w = sl // c * b                    # rows of one wave per rank
        uw = w * h * 2
        bufs = [u, u, P * uw, P * uw, P * uw, P * w * Fl * 2, P * w * Fl * 2, P * w * Fl * 2,
                S * hl * 2, S * 3 * hl * 2, lam, _norm_bwd_grid(w) * h * 4,
                max(Fl, 3 * hl) * P * w * 2, h * P * w * 2, h * max(Fl, 3 * hl) * 2]
        if metp_recompute == "full":
            bufs.append(S * 3 * hl * 2)     # QKV (fwd, then recomputed in bwd), not saved
    else:
        raise KeyError(pi)
    return sum(_al(x) for x in bufs) + small


def layer_bytes(pi, h, n, ffn, s, P, b=1, metp_recompute="ffn"):
    """M_pi(s) of Eq. 6 for one layer: persistent + saved."""
    return persistent(h, ffn, P) + saved(pi, h, n, ffn, s, P, b, metp_recompute)
