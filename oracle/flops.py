"""FLOP and communication-byte model of one layer (TEST INFRASTRUCTURE).

* SPEC.md:298 forward FLOPs (non-causal, MHA + FFN): (8 b s h^2 + 4 b s^2 h) + 16 b s h^2
  -> exactly 2^30 at C1 (h = 256, s = 512, b = 1).
* Model FLOPs per token, causal (SURVEY O-7, the roofline numerator of bench.py):
    fwd  2 (3h^2 + h^2 + 2hF) + 2 s h       (= 24 h^2 + 2 s h at F = 4h)
    bwd  2 x fwd                            (dX and dW GEMMs; dQ, dK, dV)
    total 72 h^2 + 6 s h at F = 4h
* Comm bytes per rank per layer fwd+bwd (O-7), payload (P-1)/P x full.

Pins: C1 value 2^30; the 4x / 2x scaling under s-doubling; the
matmul shapes actually executed by oracle.layer (tests/test_oracle_flops.py);
the comm bytes equal the simulated grid's comm log (tests/test_oracle_strategies.py).
"""
from __future__ import annotations


def spec_fwd_flops_noncausal(h, s, b=1):
    return (8 * b * s * h * h + 4 * b * s * s * h) + 16 * b * s * h * h


def layer_flops_per_token(h, s, ffn=None, causal=True):
    """Model FLOPs per token for fwd+bwd of one layer."""
    f = 4 * h if ffn is None else ffn
    lin = 2 * (3 * h * h + h * h + 2 * h * f)
    att = (2 if causal else 4) * s * h
    return 3 * (lin + att)


def layer_flops(h, s, ffn=None, causal=True, b=1):
    return layer_flops_per_token(h, s, ffn, causal) * s * b


def comm_bytes(pi, h, s, P, ffn=None, b=1, metp_recompute="ffn", n=None, n_kv=None, act="gelu"):
    """Bytes each rank sends per layer (fwd + bwd), payload convention SPEC.md:109.
    METP with metp_recompute='full' re-gathers u once more (SURVEY O-5 table).
    Llama variant (R-GQA / R-SWIGLU): n / n_kv heads give the Q|K|V width (n + 2 n_kv) d
    (3h for MHA) and the K (V) width n_kv d; SwiGLU weighs 3 h F instead of 2 h F."""
    f = 4 * h if ffn is None else ffn
    if P == 1:
        return 0
    fr = (P - 1) / P
    act_b = s * b * h * 2
    ar = 2 * fr * 2 * h * 4
    hk = h if n is None or n_kv is None else n_kv * (h // n)       # K (V) width, all heads
    qw = h + 2 * hk                                                # Q | K | V width
    wb = qw * h + h * h + (3 if act == "swiglu" else 2) * h * f   # weight elements per layer
    if pi in (0, 2, 4):      # TS / METP / METP-full (same bytes, c x more messages)
        extra = 1 if (pi == 4 or (pi == 2 and metp_recompute == "full")) else 0
        return int(round((10 + extra) * fr * act_b + ar))
    if pi == 1:
        a2a = 2 * fr * (s // P) * b * (qw + h) * 2
        return int(round(a2a + fr * wb * (2 + 2 + 4) + ar))
    if pi == 3:              # CZ (ring, zigzag), ZeRO3 weights as UZ
        c = s // (2 * P)                                       # half-chunk (positions)
        # half-chunks whose zigzag owner (j < P ? j : 2P-1-j) is not their boundary
        # owner j // 2 move in each boundary <-> zigzag exchange; per-rank mean
        moved = sum(1 for j in range(2 * P) if (j if j < P else 2 * P - 1 - j) != j // 2)
        zig = moved * c * b * (qw + h + h + h + qw) * 2 / P    # QKV, O | O, dO, dQKV
        kv = (s // P) * b * 2 * hk                             # one rank's K/V block (elements)
        ring = 2 * (P - 1) * kv * 2 + P * kv * 4               # K/V fwd + bwd (bf16), dK/dV (fp32)
        return int(round(zig + ring + fr * wb * (2 + 2 + 4) + ar))
    if pi == 5:              # ColossalZ (RSA), ZeRO3 weights as UZ
        kb = (s // P) * b * hk                                 # one rank's K (or V) block (elements)
        ring = 4 * (P - 1) * kb * 2 + 2 * P * kb * 4           # K, V fwd + V, K bwd (bf16); dV, dK (fp32)
        return int(round(ring + fr * wb * (2 + 2 + 4) + ar))
    raise KeyError(pi)
