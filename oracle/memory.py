"""Per-layer, per-rank memory model in bytes (TEST INFRASTRUCTURE).

Eq. 6 constrains sum_l M_{pi_l}(X) < OOM.  The paper's memory
model was learned from profiles and is admitted to be coarse;
this build reads M analytically (R-22, SURVEY O-6):

  units   u = (s/P) b h 2 B      l = (s/P) b 4 B      lam = (n/P) s b 4 B
  persistent W = (3h^2 + h^2 + 2hF)/P (2 + 4) + 2h (2 + 4)   (bf16 weights + fp32 grads)
  saved   TS   = 6u + (F/h)u + 2l + lam   x, r1, QKV(3u), A(1u), LSE, x1, r2, H(F/h u)
          UZ   = 7u + (F/h)u + 2l + lam   as TS + post-A2A attention output (1u)
          METP = 6u + 2l + lam            (metp_recompute = ffn: H recomputed)
          METP = 3u + 2l + lam            (metp_recompute = full, and METP-full: QKV recomputed too)
          COL  = 6u + (F/h)u + 2l + n (s/P) s b 2   ColossalZ (RSA): the probabilities instead of LSE
  plan    sum_l (W + saved_{pi_l}) + max_{pi in plan} workspace_pi + reserve < capacity (R-22)

Llama variant (NEXT-3, R-GQA / R-SWIGLU; every strategy): the saved Q/K/V
is (n + 2 n_kv)/n x 3u/3 = q u with q = (n + 2 n_kv)/n instead of 3u, the saved FFN
pre-activation H is (2F/h) u ([gate | up]) instead of (F/h) u, and the weights are
W = (q h^2 + h^2 + 3hF)/P (2 + 4) + 2h (2 + 4).

Pins: the saved formula equals the simulated grid's ledger recount of the
tensors the sharded simulations keep for backward (tests/test_oracle_strategies.py,
SPEC.md:99); the C1 worked example of SURVEY O-6.  The transient (workspace) term
of the plan is NOT modelled here exactly — it is a property of an implementation's
buffer plan.  `transient_floor` is the dataflow lower bound (O-5 / O-6); the
library's exact workspace is pinned by measuring its device allocation
(tests/test_gpu_memory.py).  "parity unpinned" for an exact oracle transient.
"""
from __future__ import annotations

TS, UZ, METP, CZ, METP_FULL, COL = 0, 1, 2, 3, 4, 5


def units(h, n, s, P, b=1):
    sl = s // P
    return sl * b * h * 2, sl * b * 4, (n // P) * s * b * 4


def persistent(h, ffn, P, n=None, n_kv=None, act="gelu"):
    qkv = 3 * h * h if n is None or n_kv is None else (n + 2 * n_kv) * (h // n) * h
    fc = (3 if act == "swiglu" else 2) * h * ffn
    return (qkv + h * h + fc) // P * 6 + 2 * h * 6


def saved(pi, h, n, ffn, s, P, b=1, metp_recompute="ffn", n_kv=None, act="gelu"):
    u, l, lam = units(h, n, s, P, b)
    nk = n if n_kv is None else n_kv
    qkv = (s // P) * b * (n + 2 * nk) * (h // n) * 2       # local Q | K | V rows (3u for MHA)
    hb = (s // P) * b * (2 if act == "swiglu" else 1) * ffn * 2   # FFN pre-activation H
    if pi == TS or pi == CZ:           # CZ saves its local rows of the same tensors
        return 3 * u + qkv + hb + 2 * l + lam
    if pi == UZ:
        return 4 * u + qkv + hb + 2 * l + lam
    if pi == METP:
        return (3 * u + qkv if metp_recompute == "ffn" else 3 * u) + 2 * l + lam
    if pi == METP_FULL:
        return 3 * u + 2 * l + lam
    if pi == COL:                      # ColossalZ (R-COL): TS's tensors minus LSE, plus the
        return 3 * u + qkv + hb + 2 * l + n * (s // P) * s * b * 2     # softmax probabilities [n, s/P, s] bf16
    raise KeyError(pi)


def valid(pi, h, n, ffn, s, P, metp_chunks=None, n_kv=None, act="gelu"):
    """Reading R-15: the library runs a strategy at (s, P) only when
    P | s, P | n, 128 | s/P (tile rows), 64 | F/P, for METP / METP-full also
    c | s/P and 128 | s/(P c) (c = metp_chunks, default P), and for MegatronCZ
    128 | s/(2P) (its zigzag half-chunks, R-CZ); the Llama variant (GQA n_kv, SwiGLU)
    needs P | n_kv, n_kv | n.  Never padded."""
    if s <= 0 or s % P or n % P or (s // P) % 128 or ffn % P or (ffn // P) % 64:
        return False
    nk = n if n_kv is None else n_kv
    if nk % P or n % nk:               # Llama variant (GQA): P | n_kv, n_kv | n
        return False
    if pi in (METP, METP_FULL):
        c = metp_chunks or P
        sl = s // P
        if sl % c or (sl // c) % 128:
            return False
    if pi == CZ and (s // P) % 256:      # R-CZ: zigzag half-chunks of s/(2P) positions, 128 | s/(2P)
        return False
    return True


def transient_floor(pi, h, n, ffn, s, P, b=1, metp_chunks=None):
    """A LOWER BOUND on any implementation's per-rank workspace (bytes) for one layer,
    from the dataflow of SURVEY O-5 / O-6 (not from this build's buffer table): the
    non-saved tensors that must be live together at one step of the strategy.

      TS    the row-parallel FC2 step: its input G = GELU(H) [s, F/P] (not saved,
            (F/h) u) and its output partial [s, h] before the RS (P u)   -> (P + F/h) u
      UZ    FC2 with the gathered W_out [F, h] (bf16), local G [s/P, F] and output
            [s/P, h]; backward: the full local fp32 dW_out [F, h] beside G   -> max of both
      CZ    a ring step of the backward: the incoming K/V block (2u), the block's
            travelling dK/dV partial and its successor (2 x 2u, bf16-equivalent), the
            zigzag dO and O (2u) and the dQ partial (u); UZ's FC2 step in its own
            phase                                                            -> max of both
      METP  one wave of TS's FC2 step: G [P w, F/P] and partial [P w, h], w = s/(P c)
            rows of each rank, plus the gathered wave input [P w, h]      -> (2P/c + F/(h c)) u
      METP-full  as METP plus the recomputed Q/K/V of the own heads [s, 3h/P] (3u)

    O-6's TS ~ 2P u fwd / (2P + 8) u bwd and METP ~ (2P/c + 8/c + 2) u are estimates of
    an implementation; this floor keeps only what the dataflow cannot avoid.  Pin: the
    library's workspace is never below it (tests/test_planner_host.py), and the
    library's reported workspace equals its measured device allocation
    (tests/test_gpu_memory.py) — "parity unpinned" for any exact transient value."""
    u, _, _ = units(h, n, s, P, b)
    f = ffn // h
    if pi == TS:
        return (P + f) * u
    uz = max((f + 1) * u + ffn * h * 2, ffn * h * 4 + f * u)
    if pi == UZ:
        return uz
    if pi == CZ:
        return max(9 * u, uz)
    if pi == COL:                      # RSA: the fp32 score matrix of the own rows [n, s/P, s]
        return max(n * (s // P) * s * b * 4, uz)
    c = metp_chunks or P
    base = (2 * P * u + f * u) // c
    if pi == METP:
        return base
    if pi == METP_FULL:
        return base + 3 * u
    raise KeyError(pi)


def layer_bytes(pi, h, n, ffn, s, P, b=1, metp_recompute="ffn", n_kv=None, act="gelu"):
    """M_pi(s) of Eq. 6 for one layer: persistent + saved."""
    return (persistent(h, ffn, P, n, n if n_kv is None else n_kv, act)
            + saved(pi, h, n, ffn, s, P, b, metp_recompute, n_kv, act))
