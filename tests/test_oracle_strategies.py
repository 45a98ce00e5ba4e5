"""Pins for oracle/strategies.py: every strategy at every P reproduces the
unsharded layer (north_star), switched chains,
comm signatures, and the ledger = memory model."""
from collections import Counter

import numpy as np
import pytest

from oracle import flops, layer, memory, shard
from oracle import strategies as S
from oracle.grid import Grid
from synth import layer_inputs

H, N, F = 32, 8, 128


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _run(pi, P, d, s, causal=True, chunks=None):
    g = Grid(P)
    cfg = S.Cfg(H, N, F, causal=causal, metp_chunks=chunks)
    W = shard.shard_weights(d, N, P)
    xs = shard.shard_act(d["x"], P)
    ys, saved, taps = S.layer_fwd(pi, g, xs, W, cfg)
    fwd_log = list(g.comm_log)
    grads = S.new_grads(W)
    dxs = S.layer_bwd(pi, g, shard.shard_act(d["dy"], P), saved, W, cfg, grads)
    return g, ys, taps, dxs, grads, fwd_log


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("pi", [S.TS, S.UZ, S.METP, S.CZ, S.COL])
def test_strategy_equals_unsharded(pi, P):
    s = 32
    d = layer_inputs(H, N, F, s, 1, seed=21)
    y_ref, c = layer.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"],
                               d["g2"], n=N)
    g_ref = layer.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"],
                            d["g2"], n=N)
    g, ys, taps, dxs, grads, _ = _run(pi, P, d, s, chunks=2 if pi == S.METP else None)
    assert _rel(shard.unshard_act(ys), y_ref) < 1e-12
    assert _rel(shard.unshard_act(taps["o"]), c["o"]) < 1e-12       # sublayer deltas (R-34)
    assert _rel(shard.unshard_act(taps["z"]), c["z"]) < 1e-12
    assert _rel(shard.unshard_act(dxs), g_ref["dx"]) < 1e-12
    dense = shard.unshard_grads(grads, N)
    for k in ("dw_qkv", "dw_proj", "dw_in", "dw_out", "dg1", "dg2"):
        assert _rel(dense[k], g_ref[k]) < 1e-12, k
    # shard indexing: rank r's gradient shard is the oracle's rank-r slice (O-4)
    ref_sh = shard.shard_weights(dict(w_qkv=g_ref["dw_qkv"], w_proj=g_ref["dw_proj"],
                                      w_in=g_ref["dw_in"], w_out=g_ref["dw_out"],
                                      g1=g_ref["dg1"], g2=g_ref["dg2"]), N, P)
    for r in range(P):
        assert _rel(grads["dw_qkv_t"][r], ref_sh["w_qkv_t"][r]) < 1e-12
        assert _rel(grads["dw_in_t"][r], ref_sh["w_in_t"][r]) < 1e-12
    # every saved tensor released after backward
    assert all(g.live_bytes(r) == 0 for r in range(P))


@pytest.mark.parametrize("P", [1, 2, 4])
def test_noncausal_and_batch(P):
    s = 16
    d = layer_inputs(H, N, F, s, 2, seed=5)
    y_ref, c = layer.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"],
                               d["g2"], n=N, causal=False)
    for pi in (S.TS, S.UZ, S.METP, S.CZ, S.COL):
        _, ys, _, _, _, _ = _run(pi, P, d, s, causal=False)
        assert _rel(shard.unshard_act(ys), y_ref) < 1e-12


def _signature(log):
    return Counter(e["primitive"] for e in log)


def test_comm_signatures_and_bytes_c1():
    # C1: h=256, n=4, F=1024, s=512, P=2 (SURVEY O-5 table) — run at reduced s with
    # the same structure, then check the byte formula at the C1 shape
    s, P = 16, 2
    d = layer_inputs(H, N, F, s, 1, seed=2)
    for pi, fwd_sig, all_sig in [
        (S.TS, {"AllGather": 2, "ReduceScatter": 2},
         {"AllGather": 6, "ReduceScatter": 4, "AllReduce": 1}),
        (S.UZ, {"AllGather": 4, "AllToAll": 2},
         {"AllGather": 8, "AllToAll": 4, "ReduceScatter": 4, "AllReduce": 1}),
        (S.METP, {"AllGather": 4, "ReduceScatter": 4},     # c = P = 2 waves
         {"AllGather": 12, "ReduceScatter": 8, "AllReduce": 1}),
        # CZ (ring, zigzag): 6 weight AGs (W_qkv^T in its Q, K, V parts) per pass; fwd
        # SendRecv(QKV -> zigzag), P - 1 K/V ring passes, SendRecv(O -> boundary); bwd
        # SendRecv(O, dO -> zigzag), P - 1 K/V passes + P fp32 dK/dV passes,
        # SendRecv(dQKV -> boundary), the 6 fp32 dW reduce-scatters, AR(dgamma)
        (S.CZ, {"AllGather": 6, "SendRecv": 2, "RingPass": 1},
         {"AllGather": 12, "SendRecv": 5, "RingPass": 4, "ReduceScatter": 6, "AllReduce": 1}),
        # ColossalZ (RSA): weights as CZ; fwd K ring and V ring (P - 1 each); bwd V ring and
        # K ring (P - 1 each) plus the fp32 dV and dK accumulators (P passes each)
        (S.COL, {"AllGather": 6, "RingPass": 2},
         {"AllGather": 12, "RingPass": 8, "ReduceScatter": 6, "AllReduce": 1}),
    ]:
        g, _, _, _, _, flog = _run(pi, P, d, s)
        assert _signature(flog) == Counter(fwd_sig), pi
        assert _signature(g.comm_log) == Counter(all_sig), pi
        total = sum(e["bytes"] for e in g.comm_log)
        assert total == flops.comm_bytes(pi, H, s, P, F), (pi, total)
    # C1 numbers of SURVEY O-5 from the same formula
    assert flops.comm_bytes(S.TS, 256, 512, 2) == 1310720 + 2048
    assert flops.comm_bytes(S.UZ, 256, 512, 2) == 3670016 + 2048


@pytest.mark.parametrize("P", [2, 4])
def test_switched_chain_equals_stack(P):
    # random strategy sequences, no collective between layers
    s, Ln = 16, 4
    rng = np.random.default_rng(P)
    layers = [layer_inputs(H, N, F, s, 1, seed=9, layer=i) for i in range(Ln)]
    x = layers[0]["x"]
    dy = layers[0]["dy"]
    for trial in range(3):
        plan = list(rng.integers(0, 6, size=Ln))
        # dense stack
        yd = x
        caches = []
        for i in range(Ln):
            w = layers[i]
            yd, c = layer.layer_fwd(yd, w["w_qkv"], w["w_proj"], w["w_in"], w["w_out"], w["g1"],
                                    w["g2"], n=N)
            caches.append(c)
        dd = dy
        for i in reversed(range(Ln)):
            w = layers[i]
            dd = layer.layer_bwd(dd, caches[i], w["w_qkv"], w["w_proj"], w["w_in"], w["w_out"],
                                 w["g1"], w["g2"], n=N)["dx"]
        # sharded, switched
        g = Grid(P)
        cfg = S.Cfg(H, N, F)
        Ws = [shard.shard_weights(layers[i], N, P) for i in range(Ln)]
        xs = shard.shard_act(x, P)
        saves = []
        boundary = []
        for i, pi in enumerate(plan):
            n0 = len(g.comm_log)
            xs, sv, _ = S.layer_fwd(int(pi), g, xs, Ws[i], cfg)
            boundary.append(n0)
            saves.append(sv)
        assert _rel(shard.unshard_act(xs), yd) < 1e-12
        ds = shard.shard_act(dy, P)
        for i in reversed(range(Ln)):
            grads = S.new_grads(Ws[i])
            ds = S.layer_bwd(int(plan[i]), g, ds, saves[i], Ws[i], cfg, grads)
        assert _rel(shard.unshard_act(ds), dd) < 1e-12
        # redistribution-free: the log is exactly the concatenation of per-layer signatures
        sig = Counter()
        for pi in plan:
            g2 = Grid(P)
            _run_sig = _run(int(pi), P, layers[0], s)[0]
            sig += _signature(_run_sig.comm_log)
        assert _signature(g.comm_log) == sig


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("pi", [S.TS, S.UZ, S.METP, S.CZ, S.COL])
def test_ledger_equals_memory_model(pi, P):
    # the ledger recount of saved tensors equals the analytic formula
    s = 32
    d = layer_inputs(H, N, F, s, 1, seed=1)
    g = Grid(P)
    cfg = S.Cfg(H, N, F)
    W = shard.shard_weights(d, N, P)
    _, saved, _ = S.layer_fwd(pi, g, shard.shard_act(d["x"], P), W, cfg)
    for r in range(P):
        assert g.live_bytes(r, "saved") == memory.saved(pi, H, N, F, s, P), (pi, P, r)


def test_memory_c1_worked_example():
    # SURVEY O-6 worked example at C1 (P = 2)
    h, n, F, s, P = 256, 4, 1024, 512, 2
    assert memory.units(h, n, s, P) == (131072, 1024, 4096)
    assert memory.persistent(h, F, P) == 2362368
    assert memory.saved(S.TS, h, n, F, s, P) == 1316864
    assert memory.saved(S.UZ, h, n, F, s, P) == 1447936
    assert memory.saved(S.METP, h, n, F, s, P) == 792576
    assert memory.saved(S.METP, h, n, F, s, P, metp_recompute="full") == 399360


def test_memory_ordering():
    # SPEC.md:254 / SURVEY pins: METP saves less than TS and UZ at every s, P > 1
    for s in (4096, 65536, 638976):
        for P in (2, 4, 8):
            m = [memory.saved(pi, 4096, 32, 16384, s, P) for pi in (S.TS, S.UZ, S.METP)]
            assert m[2] < m[0] and m[2] < m[1]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_metp_full_recompute_equals_unsharded(P):
    # metp_recompute = 'full' (SURVEY O-5 / O-6): QKV is not saved but recomputed in the
    # backward from per-wave re-gathers of u; the layer is still the unsharded layer
    s = 32
    d = layer_inputs(H, N, F, s, 1, seed=23)
    y_ref, c = layer.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"],
                               d["g2"], n=N)
    g_ref = layer.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"],
                            d["g2"], n=N)
    g = Grid(P)
    cfg = S.Cfg(H, N, F, metp_chunks=2, metp_recompute="full")
    W = shard.shard_weights(d, N, P)
    ys, saved, taps = S.layer_fwd(S.METP, g, shard.shard_act(d["x"], P), W, cfg)
    for r in range(P):
        assert "qkv" not in saved[r]
        assert g.live_bytes(r, "saved") == memory.saved(S.METP, H, N, F, s, P, metp_recompute="full")
    n_fwd = len(g.comm_log)
    grads = S.new_grads(W)
    dxs = S.layer_bwd(S.METP, g, shard.shard_act(d["dy"], P), saved, W, cfg, grads)
    assert _rel(shard.unshard_act(ys), y_ref) < 1e-12
    assert _rel(shard.unshard_act(dxs), g_ref["dx"]) < 1e-12
    dense = shard.unshard_grads(grads, N)
    for k in ("dw_qkv", "dw_proj", "dw_in", "dw_out", "dg1", "dg2"):
        assert _rel(dense[k], g_ref[k]) < 1e-12, k
    if P > 1:
        # signature: the 'ffn' backward plus c = 2 extra wave gathers of u
        bwd = _signature(g.comm_log[n_fwd:])
        assert bwd == Counter({"AllGather": 8 + 2, "ReduceScatter": 4, "AllReduce": 1})
        assert sum(e["bytes"] for e in g.comm_log) == flops.comm_bytes(S.METP, H, s, P, F,
                                                                         metp_recompute="full")
    assert all(g.live_bytes(r) == 0 for r in range(P))


def test_metp_full_recompute_halves_saved_bytes():
    # SURVEY O-6: METP saves 6u + 2l + lam ('ffn') or 3u + 2l + lam ('full')
    for s, P in ((4096, 1), (65536, 2), (638976, 8)):
        u, l, lam = memory.units(4096, 32, s, P)
        ffn = memory.saved(S.METP, 4096, 32, 16384, s, P)
        full = memory.saved(S.METP, 4096, 32, 16384, s, P, metp_recompute="full")
        assert ffn - full == 3 * u
    with pytest.raises(ValueError):
        S.Cfg(H, N, F, metp_recompute="qkv")


# ---------------------------------------------------------------- Llama variant (NEXT-3)
@pytest.mark.parametrize("P,n_kv", [(1, 2), (2, 2), (2, 4), (4, 4)])
@pytest.mark.parametrize("pi", [S.TS, S.UZ, S.METP, S.METP_FULL, S.CZ, S.COL])
def test_llama_variant_equals_unsharded(pi, P, n_kv):
    """GQA (n_kv key/value heads) + SwiGLU (interleaved spec layout, R-SWIGLU): every
    strategy that runs the variant reproduces the unsharded Llama layer, per-rank
    gradient shards included, and its ledger equals the memory formula."""
    s, ffn = 32, 256
    d = layer_inputs(H, N, ffn, s, 2, seed=23, n_kv=n_kv, act="swiglu")
    kw = dict(n=N, n_kv=n_kv, act="swiglu")
    y_ref, c = layer.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    g_ref = layer.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], **kw)
    g = Grid(P)
    cfg = S.Cfg(H, N, ffn, metp_chunks=2 if pi in (S.METP, S.METP_FULL) else None, n_kv=n_kv, act="swiglu")
    W = shard.shard_weights(d, N, P, n_kv=n_kv, act="swiglu")
    ys, saved, taps = S.layer_fwd(pi, g, shard.shard_act(d["x"], P), W, cfg)
    for r in range(P):
        assert g.live_bytes(r, "saved") == memory.saved(pi, H, N, ffn, s, P, b=2, n_kv=n_kv, act="swiglu")
    grads = S.new_grads(W)
    dxs = S.layer_bwd(pi, g, shard.shard_act(d["dy"], P), saved, W, cfg, grads)
    assert _rel(shard.unshard_act(ys), y_ref) < 1e-12
    assert _rel(shard.unshard_act(taps["z"]), c["z"]) < 1e-12
    assert _rel(shard.unshard_act(dxs), g_ref["dx"]) < 1e-12
    dense = shard.unshard_grads(grads, N, n_kv=n_kv, act="swiglu")
    for k in ("dw_qkv", "dw_proj", "dw_in", "dw_out", "dg1", "dg2"):
        assert _rel(dense[k], g_ref[k]) < 1e-12, k
    ref_sh = shard.shard_weights(dict(w_qkv=g_ref["dw_qkv"], w_proj=g_ref["dw_proj"], w_in=g_ref["dw_in"],
                                      w_out=g_ref["dw_out"], g1=g_ref["dg1"], g2=g_ref["dg2"]), N, P,
                                 n_kv=n_kv, act="swiglu")
    for r in range(P):
        assert _rel(grads["dw_qkv_t"][r], ref_sh["w_qkv_t"][r]) < 1e-12
        assert _rel(grads["dw_in_t"][r], ref_sh["w_in_t"][r]) < 1e-12
    # the simulated comm log's bytes = the formula with the variant's widths
    full = "full" if pi == S.METP_FULL else "ffn"
    assert sum(e["bytes"] for e in g.comm_log) == flops.comm_bytes(pi, H, s, P, ffn, b=2, metp_recompute=full, n=N,
                                                                 n_kv=n_kv, act="swiglu"), pi


def test_llama_variant_validity():
    """P must divide n_kv (GQA head groups stay whole on a rank)."""
    assert memory.valid(S.TS, H, N, 256, 256, 2, n_kv=2, act="swiglu")
    assert memory.valid(S.CZ, H, N, 256, 512, 2, n_kv=2, act="swiglu")
    assert not memory.valid(S.TS, H, N, 256, 512, 4, n_kv=2, act="swiglu")
