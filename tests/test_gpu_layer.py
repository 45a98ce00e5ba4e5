"""Whole-layer parity on B200: every strategy at P = 1 (real context) and P = 2, 4
(loopback group: P virtual ranks, one host thread each, on one GPU) against the
fp64 oracle (north_star: "every strategy ... matches the CPU oracle").

bf16 path tolerance (north_star): relative L2 <= 1e-2 on Y, the sublayer deltas
O and Z (R-34), dX, dX - dY, every weight gradient and dgamma; shard indexing is
checked per rank against the oracle's rank-r slice.
"""
import threading

import numpy as np
import pytest
import torch

from oracle import layer as OL
from oracle import shard as OS
from synth import layer_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2511_13198_b200 import binding as B
    from tests.gpu_util import dev_bf16, host, rel

TOL = 1e-2


class Rank:
    """Device buffers of one (virtual) rank."""

    def __init__(self, W, r, x, dy):
        self.w = {k: dev_bf16(W[k][r]) for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")}
        self.g = {k: torch.zeros(W[src][r].shape, dtype=torch.float32, device="cuda")
                  for k, src in (("dw_qkv_t", "w_qkv_t"), ("dw_proj", "w_proj"), ("dw_in_t", "w_in_t"),
                                 ("dw_out", "w_out"), ("dg1", "g1"), ("dg2", "g2"))}
        self.x = dev_bf16(x.reshape(x.shape[0], -1))
        self.dy = dev_bf16(dy.reshape(dy.shape[0], -1))
        self.y = torch.empty_like(self.x)
        self.dx = torch.empty_like(self.x)
        self.o = torch.empty_like(self.x)
        self.z = torch.empty_like(self.x)

    def weights(self):
        return B.Weights(*(self.w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))

    def grads(self):
        return B.Grads(*(self.g[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))


def run_ranks(model, P, pi_list, ranks_per_layer, x_shards, dy_shards, taps=True, overlap=None, varlen=None,
              logs=None):
    """Run an L-layer stack (plan pi_list) on P loopback ranks; returns per-rank outputs.
    overlap: None = library default, else pds_set_overlap(ctx, overlap)."""
    grp = B.Group(P)
    errs = []
    outs = [None] * P

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                ctx = B.Context(model, group=grp, rank=r)
                if overlap is not None:
                    ctx.set_overlap(overlap)
                if varlen:
                    ctx.set_varlen(varlen)
                if logs is not None:
                    ctx.comm_log(True)
                xs = dev_bf16(x_shards[r].reshape(x_shards[r].shape[0], -1))
                acts = [xs]
                saves = []
                for li, pi in enumerate(pi_list):
                    R = ranks_per_layer[li][r]
                    if taps:
                        ctx.debug_taps(R.o.data_ptr(), R.z.data_ptr())
                    y = torch.empty_like(xs)
                    sv = ctx.layer_fwd(pi, x_shards[r].shape[0] * P, acts[-1].data_ptr(), R.weights(), y.data_ptr(),
                                       st.cuda_stream)
                    acts.append(y)
                    saves.append(sv)
                d = dev_bf16(dy_shards[r].reshape(dy_shards[r].shape[0], -1))
                for li in reversed(range(len(pi_list))):
                    R = ranks_per_layer[li][r]
                    dx = torch.empty_like(d)
                    ctx.layer_bwd(pi_list[li], d.data_ptr(), saves[li], R.weights(), R.grads(), dx.data_ptr(),
                                  st.cuda_stream)
                    d = dx
                st.synchronize()
                outs[r] = (host(acts[-1]), host(d))
                if logs is not None:
                    logs[r] = ctx.read_comm_log()
                ctx.close()
        except Exception as e:  # surfaced in the main thread
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    grp.close()
    if errs:
        raise errs[0]
    return outs


def _check_layer(pi, P, h, n, F, s, seed=1, chunks=0, causal=True, recompute=0, b=1, n_kv=None, act="gelu",
                 varlen=None):
    d = layer_inputs(h, n, F, s, b, seed=seed, n_kv=n_kv, act=act)
    wargs = (d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"])
    kw = dict(n=n, causal=causal, n_kv=n_kv, act=act)
    if varlen:                       # R-VARLEN: the oracle layer per packed sequence
        y_ref, cs = OL.layer_fwd_varlen(d["x"], varlen, *wargs, **kw)
        g_ref = OL.layer_bwd_varlen(d["dy"], cs, varlen, *wargs, **kw)
        c = dict(o=np.concatenate([q["o"] for q in cs]), z=np.concatenate([q["z"] for q in cs]))
    else:
        y_ref, c = OL.layer_fwd(d["x"], *wargs, **kw)
        g_ref = OL.layer_bwd(d["dy"], c, *wargs, **kw)
    W = OS.shard_weights(d, n, P, n_kv=n_kv, act=act)
    xs = OS.shard_act(d["x"], P)
    dys = OS.shard_act(d["dy"], P)
    ranks = [Rank(W, r, xs[r], dys[r]) for r in range(P)]
    model = B.Model(h=h, n_heads=n, ffn=F, metp_chunks=chunks, causal=1 if causal else 0,
                    metp_recompute=recompute, batch=b, n_kv_heads=n_kv or 0, ffn_act=1 if act == "swiglu" else 0)
    outs = run_ranks(model, P, [pi], [ranks], xs, dys, varlen=varlen)
    y = np.concatenate([o[0] for o in outs]).reshape(s, b, h)
    dx = np.concatenate([o[1] for o in outs]).reshape(s, b, h)
    o = np.concatenate([host(R.o) for R in ranks]).reshape(s, b, h)
    z = np.concatenate([host(R.z) for R in ranks]).reshape(s, b, h)
    res = dict(y=rel(y, y_ref), o=rel(o, c["o"]), z=rel(z, c["z"]), dx=rel(dx, g_ref["dx"]),
               dxmdy=rel(dx - d["dy"], g_ref["dx"] - d["dy"]))
    gsh = {k: [host(R.g[k]) for R in ranks] for k in ranks[0].g}
    dense = OS.unshard_grads(gsh, n, n_kv=n_kv, act=act)
    for k in ("dw_qkv", "dw_proj", "dw_in", "dw_out", "dg1", "dg2"):
        res[k] = rel(dense[k], g_ref[k])
    # shard indexing: rank r's gradient shard vs the oracle's rank-r slice (O-4)
    ref_sh = OS.shard_weights(dict(w_qkv=g_ref["dw_qkv"], w_proj=g_ref["dw_proj"], w_in=g_ref["dw_in"],
                                   w_out=g_ref["dw_out"], g1=g_ref["dg1"], g2=g_ref["dg2"]), n, P,
                              n_kv=n_kv, act=act)
    for r in range(P):
        res[f"qkv_shard{r}"] = rel(gsh["dw_qkv_t"][r], ref_sh["w_qkv_t"][r])
        res[f"y_shard{r}"] = rel(outs[r][0].reshape(s // P, b, h), y_ref[r * (s // P):(r + 1) * (s // P)])
    bad = {k: v for k, v in res.items() if not v < TOL}
    assert not bad, (pi, P, bad, res)
    return res


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
def test_layer_p1_c1(pi):
    # C1 shapes (h=256, n=4, d=64, F=1024, s=512), P = 1: every strategy degenerates
    _check_layer(pi, 1, 256, 4, 1024, 512)


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
def test_layer_p2_c1(pi):
    # C1 at P = 2 (the configs[0] case), METP with c = 2 waves
    _check_layer(pi, 2, 256, 4, 1024, 512)


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
def test_layer_p4_d128(pi):
    # d = 128 heads, P = 4, METP c = 2 waves of 128 rows per rank
    _check_layer(pi, 4, 1024, 8, 4096, 1024, chunks=2)


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("P", [1, 2])
def test_layer_batch2(pi, P):
    # b = 2 independent sequences in the [s/P, b, h] boundary layout (Table 1's b,
    # reading Q-35): token rows t*b + bi, attention per sequence, RoPE at position t
    _check_layer(pi, P, 256, 4, 1024, 512, seed=13, b=2, chunks=2 if P == 1 else 0)


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
def test_layer_p4_batch2_d128(pi):
    # b = 2 with d = 128 heads at P = 4 (METP: 2 waves of 128 positions x 2 sequences),
    # tile-overlapped collectives on
    _check_layer(pi, 4, 1024, 8, 4096, 1024, seed=14, b=2, chunks=2)


@pytest.mark.parametrize("pi", [0, 1, 2, 4])
def test_layer_fused_attn_bwd(pi):
    # the opt-in fused attention backward (pds_set_attn_bwd(1)) inside the layer: its fp32
    # dQ accumulator borrows the TS / UZ transposition buffer or METP's ul + vl; b = 2
    # (the accumulator is reused sequence after sequence)
    B.set_attn_bwd(1)
    try:
        _check_layer(pi, 2, 1024, 8, 4096, 1024, seed=21, b=2, chunks=2)
    finally:
        B.set_attn_bwd(0)


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
def test_layer_p8(pi):
    # eight ranks (the paper's node) on the loopback group: s/P = 128 rows,
    # one head per rank; METP with c = 1 wave; MegatronCZ's zigzag half-chunks need
    # 128 | s/(2P): s = 2048 for it
    _check_layer(pi, 8, 1024, 8, 4096, 2048 if pi == 3 else 1024, seed=8, chunks=1)


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
def test_layer_bert_shape_noncausal(pi):
    # Table 4's BERT layer (h = 1024, 16 heads of d = 64, F = 4h, bidirectional) at P = 2
    _check_layer(pi, 2, 1024, 16, 4096, 512, seed=4, causal=False)


@pytest.mark.parametrize("recompute", [0, 1])
@pytest.mark.parametrize("P,h,n,F,s,chunks", [(1, 256, 4, 1024, 512, 2), (2, 256, 4, 1024, 512, 0),
                                              (4, 1024, 8, 4096, 1024, 2)])
def test_layer_metp_recompute_modes(P, h, n, F, s, chunks, recompute):
    # metp_recompute = full: Q/K/V recomputed in backward from re-gathered u (SURVEY O-6).
    # P = 1 with c = 2 waves: a single-segment row remap with an offset (wave 1 of rank 0)
    _check_layer(2, P, h, n, F, s, chunks=chunks, recompute=recompute)


def test_metp_full_equals_ffn_bitwise():
    # the recomputed Q/K/V are the forward's bit for bit, so every output and gradient is
    P, h, n, F, s = 2, 1024, 8, 4096, 1024
    d = layer_inputs(h, n, F, s, 1, seed=12)
    W = OS.shard_weights(d, n, P)
    xs = OS.shard_act(d["x"], P)
    dys = OS.shard_act(d["dy"], P)
    res = []
    for rc in (0, 1):
        ranks = [Rank(W, r, xs[r], dys[r]) for r in range(P)]
        outs = run_ranks(B.Model(h=h, n_heads=n, ffn=F, metp_recompute=rc), P, [2], [ranks], xs, dys)
        res.append((outs, {k: [host(R.g[k]) for R in ranks] for k in ranks[0].g}))
    for r in range(P):
        assert np.array_equal(res[0][0][r][0], res[1][0][r][0])
        assert np.array_equal(res[0][0][r][1], res[1][0][r][1])
        for k in res[0][1]:
            assert np.array_equal(res[0][1][k][r], res[1][1][k][r]), k


def test_layer_ts_odd_chunks_p2():
    # s/P = 384 rows (an odd number of 128-row blocks), tile-overlapped TS vs the oracle
    _check_layer(0, 2, 256, 4, 1024, 768, seed=6)


@pytest.mark.parametrize("pi,P,h,n,F,s,chunks", [
    (0, 2, 2048, 16, 8192, 4096, 0),    # TS, CTA-pair GEMMs, 8 m-blocks per chunk
    (0, 4, 1024, 8, 4096, 2048, 0),     # TS, 1-CTA GEMMs, rotated tile order
    (0, 2, 2048, 16, 8192, 2816, 0),    # TS, 256-row pair tiles straddle chunks
    (2, 2, 2048, 16, 8192, 4096, 2),    # METP, 2 waves of 1024 rows per rank
    (2, 4, 1024, 8, 4096, 2048, 2),     # METP, 4 ranks x 2 waves of 256 rows
    (1, 2, 2048, 16, 8192, 4096, 0),    # UlyssesZ, A2A blocks of 3h/P columns, pair GEMMs
    (1, 4, 1024, 8, 4096, 2048, 0)])    # UlyssesZ, 4 ranks
def test_overlap_bit_identical(pi, P, h, n, F, s, chunks):
    """MegatronTS / METP with the tile-overlapped AG / RS and UlyssesZ with the
    block-gated All-to-Alls (pds_set_overlap 1) equal the in-order collectives (0) bit
    for bit: the same tiles, the same rank-order sums."""
    d = layer_inputs(h, n, F, s, 1, seed=11)
    W = OS.shard_weights(d, n, P)
    xs = OS.shard_act(d["x"], P)
    dys = OS.shard_act(d["dy"], P)
    model = B.Model(h=h, n_heads=n, ffn=F, metp_chunks=chunks)
    res = []
    for ov in (0, 1):
        ranks = [Rank(W, r, xs[r], dys[r]) for r in range(P)]
        outs = run_ranks(model, P, [pi], [ranks], xs, dys, overlap=ov)
        res.append((outs, {k: [host(R.g[k]) for R in ranks] for k in ranks[0].g},
                    [host(R.o) for R in ranks], [host(R.z) for R in ranks]))
    (o0, g0, a0, z0), (o1, g1, a1, z1) = res
    for r in range(P):
        assert np.array_equal(o0[r][0], o1[r][0]), ("y", r)
        assert np.array_equal(o0[r][1], o1[r][1]), ("dx", r)
        assert np.array_equal(a0[r], a1[r]) and np.array_equal(z0[r], z1[r]), ("o/z", r)
        for k in g0:
            assert np.array_equal(g0[k][r], g1[k][r]), (k, r)


def test_switched_chain_p2():
    # a 4-layer stack with a switched plan; boundary tensors pass unchanged (R-31)
    P, h, n, F, s = 2, 256, 4, 1024, 512
    plan = [2, 0, 5, 3, 1, 4]                  # every strategy once, METP-full last
    layers = [layer_inputs(h, n, F, s, 1, seed=5, layer=i) for i in range(len(plan))]
    yd = layers[0]["x"]
    caches = []
    for L in layers:
        yd, cc = OL.layer_fwd(yd, L["w_qkv"], L["w_proj"], L["w_in"], L["w_out"], L["g1"], L["g2"], n=n)
        caches.append(cc)
    dd = layers[0]["dy"]
    for i in reversed(range(len(plan))):
        L = layers[i]
        dd = OL.layer_bwd(dd, caches[i], L["w_qkv"], L["w_proj"], L["w_in"], L["w_out"], L["g1"], L["g2"],
                          n=n)["dx"]
    xs = OS.shard_act(layers[0]["x"], P)
    dys = OS.shard_act(layers[0]["dy"], P)
    rpl = []
    for i in range(len(plan)):
        W = OS.shard_weights(layers[i], n, P)
        rpl.append([Rank(W, r, xs[r], dys[r]) for r in range(P)])
    outs = run_ranks(B.Model(h=h, n_heads=n, ffn=F), P, plan, rpl, xs, dys, taps=False)
    y = np.concatenate([o[0] for o in outs])[:, None, :]
    dx = np.concatenate([o[1] for o in outs])[:, None, :]
    assert rel(y, yd) < TOL
    assert rel(dx, dd) < TOL
    assert rel(dx - layers[0]["dy"], dd - layers[0]["dy"]) < TOL


def test_layer_errors():
    m = B.Model(h=256, n_heads=4, ffn=1024)
    ctx = B.Context(m)
    x = torch.zeros(384, 256, dtype=torch.bfloat16, device="cuda")
    w = B.Weights(*([x.data_ptr()] * 6))
    with pytest.raises(B.PdsError) as e:
        ctx.layer_fwd(7, 384, x.data_ptr(), w, x.data_ptr())
    assert e.value.code == -3
    with pytest.raises(B.PdsError) as e:
        ctx.layer_fwd(0, 200, x.data_ptr(), w, x.data_ptr())      # s/P not a multiple of 128
    assert e.value.code == -2
    ctx.close()


def test_plan_strategy_masks():
    # pds_set_enabled covers every strategy of the bundle: each alone yields its uniform plan
    import os
    from oracle import costmodel as CM
    path = os.path.join(os.path.dirname(B.__file__), "bundles", "h4096_n32_f16384_P1.txt")
    m = B.Model(h=4096, n_heads=32, ffn=16384, n_layers=8)
    ctx = B.Context(m)
    ctx.load_costs(path)
    ctx.set_capacity(1e15, 0.0)
    for pi in sorted(CM.read_bundle(path)["strat"]):
        ctx.set_enabled(1 << pi)
        plan, _ = ctx.plan(8192, 8)
        assert plan == [pi] * 8, (pi, plan)
    with pytest.raises(B.PdsError) as e:
        ctx.set_enabled(1 << B.N_STRATEGIES)
    assert e.value.code == -1
    ctx.close()


@pytest.mark.parametrize("pi,b", [(0, 1), (2, 1), (0, 2), (4, 2)])
def test_step_host(pi, b):
    """pds_layer_step_host (host x, dy in; host y, dx out; copies overlapped on a copy
    stream) equals the device-pointer fwd + bwd bit for bit and the oracle within TOL,
    b = 1 and b = 2 sequences (staging holds s/P x b x h)."""
    h, n, F, s = 256, 4, 1024, 512
    d = layer_inputs(h, n, F, s, b, seed=3)
    y_ref, c = OL.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], n=n)
    g_ref = OL.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], n=n)
    W = OS.shard_weights(d, n, 1)
    R1 = Rank(W, 0, d["x"], d["dy"])
    R2 = Rank(W, 0, d["x"], d["dy"])
    ctx = B.Context(B.Model(h=h, n_heads=n, ffn=F, batch=b))
    st = torch.cuda.current_stream()
    sv = ctx.layer_fwd(pi, s, R1.x.data_ptr(), R1.weights(), R1.y.data_ptr(), st.cuda_stream)
    ctx.layer_bwd(pi, R1.dy.data_ptr(), sv, R1.weights(), R1.grads(), R1.dx.data_ptr(), st.cuda_stream)
    xh, dyh = R2.x.cpu().pin_memory(), R2.dy.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    dxh = torch.empty_like(xh).pin_memory()
    ctx.layer_step_host(pi, s, xh.data_ptr(), dyh.data_ptr(), R2.weights(), R2.grads(), yh.data_ptr(),
                        dxh.data_ptr(), st.cuda_stream)
    # a second, pipelined call on the other staging set with its own host buffers
    R3 = Rank(W, 0, d["x"], d["dy"])
    yh3 = torch.empty_like(xh).pin_memory()
    dxh3 = torch.empty_like(xh).pin_memory()
    ctx.layer_step_host(pi, s, xh.data_ptr(), dyh.data_ptr(), R3.weights(), R3.grads(), yh3.data_ptr(),
                        dxh3.data_ptr(), st.cuda_stream)
    ctx.host_drain(st.cuda_stream)
    st.synchronize()
    assert torch.equal(yh3, yh) and torch.equal(dxh3, dxh)
    assert torch.equal(yh, R1.y.cpu()) and torch.equal(dxh, R1.dx.cpu())
    for k in R1.g:
        assert torch.equal(R1.g[k], R2.g[k]), k
    assert rel(host(yh).reshape(s, b, h), y_ref) < TOL
    assert rel(host(dxh).reshape(s, b, h), g_ref["dx"]) < TOL
    ctx.close()


@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
def test_nccl_one_rank_equals_self(pi):
    """The NCCL backend (a one-rank communicator: pds_create with P = 1 and a unique
    id) runs every collective of the strategy, METP's side-stream wave gathers on a
    split communicator included (c = 2 waves), and must reproduce the no-communicator
    context bit for bit."""
    h, n, F, s = 256, 4, 1024, 512
    d = layer_inputs(h, n, F, s, 1, seed=9)
    W = OS.shard_weights(d, n, 1)
    model = B.Model(h=h, n_heads=n, ffn=F, metp_chunks=2)
    res = []
    for uid in (None, B.nccl_unique_id()):
        R = Rank(W, 0, d["x"], d["dy"])
        ctx = B.Context(model, P=1, rank=0, device=0, uid=uid)
        st = torch.cuda.current_stream()
        sv = ctx.layer_fwd(pi, s, R.x.data_ptr(), R.weights(), R.y.data_ptr(), st.cuda_stream)
        ctx.layer_bwd(pi, R.dy.data_ptr(), sv, R.weights(), R.grads(), R.dx.data_ptr(), st.cuda_stream)
        st.synchronize()
        res.append(R)
        ctx.close()
    a, b = res
    assert torch.equal(a.y, b.y) and torch.equal(a.dx, b.dx)
    for k in a.g:
        assert torch.equal(a.g[k], b.g[k]), k


# ---------------------------------------------------------------- Llama variant (NEXT-3)
@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("P,h,n,n_kv,F,s", [
    (1, 512, 8, 2, 768, 768),        # d = 64, grp 4, an odd count of 256-query CTAs
    (2, 1024, 8, 2, 1536, 1024),     # d = 128, grp 4, one KV head per rank
    (4, 1024, 8, 4, 1024, 2048),     # d = 128, grp 2
])
def test_llama_variant_layer(pi, P, h, n, n_kv, F, s):
    """GQA + SwiGLU layer (R-GQA / R-SWIGLU) on every strategy that runs it, per-rank
    shards included, against the fp64 oracle's Llama layer."""
    chunks = 2 if pi in (2, 4) and P > 1 else 0
    _check_layer(pi, P, h, n, F, s, seed=17, chunks=chunks, n_kv=n_kv, act="swiglu", b=2 if P == 2 else 1)


@pytest.mark.parametrize("n_kv,act", [(2, "gelu"), (8, "swiglu")])
def test_llama_variant_parts_separately(n_kv, act):
    """GQA alone (GELU FFN) and SwiGLU alone (MHA) through MegatronTS at P = 2."""
    _check_layer(0, 2, 1024, 8, 2048, 1024, seed=19, n_kv=n_kv, act=act)



# ---------------------------------------------------------------- varlen packing (NEXT-3)
@pytest.mark.parametrize("pi", [0, 1, 2, 4])
@pytest.mark.parametrize("P,lens,causal", [
    (1, [256, 768, 512], True),
    (2, [256, 768, 512, 512], True),      # sequences straddle the rank boundary
    (2, [512, 1024, 512], False),
    (4, [1280, 256, 512], True),
])
def test_varlen_layer(pi, P, lens, causal):
    """Packed sequences (R-VARLEN): attention block-diagonal per sequence, RoPE
    positions restarting per sequence, against the oracle layer per sequence."""
    chunks = 2 if pi in (2, 4) else 0
    _check_layer(pi, P, 512, 4, 2048, sum(lens), seed=23, chunks=chunks, causal=causal, varlen=lens)


def test_varlen_llama_variant():
    """Packing together with GQA + SwiGLU (the Llama variant) through UlyssesZ at P = 2."""
    _check_layer(1, 2, 1024, 8, 1536, 2048, seed=29, n_kv=2, act="swiglu", varlen=[768, 256, 1024])


def test_varlen_argument_errors():
    ctx = B.Context(B.Model(h=256, n_heads=4, ffn=1024))
    with pytest.raises(B.PdsError) as e:
        ctx.set_varlen([256, 300])
    assert e.value.code == -2                             # every sequence a multiple of 256
    ctx.set_varlen([256, 512])
    d = layer_inputs(256, 4, 1024, 768, 1, seed=3)
    W = OS.shard_weights(d, 4, 1)
    R = Rank(W, 0, d["x"], d["dy"])
    y = torch.empty_like(R.x)
    with pytest.raises(B.PdsError) as e:                  # seq_len must be the packed total
        ctx.layer_fwd(0, 1024, R.x.data_ptr(), R.weights(), y.data_ptr(), 0)
    assert e.value.code == -1
    for pi in (3, 5):
        with pytest.raises(B.PdsError) as e:
            ctx.layer_fwd(pi, 768, R.x.data_ptr(), R.weights(), y.data_ptr(), 0)
        assert e.value.code == -9
    ctx.set_varlen([])                                    # back to one sequence
    sv = ctx.layer_fwd(0, 768, R.x.data_ptr(), R.weights(), y.data_ptr(), 0)
    ctx.saved_release(sv)
    ctx.close()
    with pytest.raises(B.PdsError) as e:
        B.Context(B.Model(h=256, n_heads=4, ffn=1024, batch=2)).set_varlen([256])
    assert e.value.code == -1


# ---------------------------------------------------------------- comm log
@pytest.mark.parametrize("pi", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("overlap", [0, 1])
def test_comm_log_equals_oracle_dataflow(pi, overlap):
    """The device path's collectives (pds_comm_log) at P = 2: the same primitive multiset
    as the oracle simulation of that strategy, and the bytes every rank sends sum to the
    oracle's formula (oracle/flops.comm_bytes, itself equal to the simulated comm log)."""
    from collections import Counter
    from oracle import flops as OF
    from oracle import strategies as S
    from oracle.grid import Grid
    h, n, F, s, P = 256, 4, 1024, 1024, 2
    d = layer_inputs(h, n, F, s, 1, seed=5)
    W = OS.shard_weights(d, n, P)
    xs, dys = OS.shard_act(d["x"], P), OS.shard_act(d["dy"], P)
    ranks = [Rank(W, r, xs[r], dys[r]) for r in range(P)]
    logs = [None] * P
    run_ranks(B.Model(h=h, n_heads=n, ffn=F, metp_chunks=2), P, [pi], [ranks], xs, dys, taps=False,
              overlap=overlap, logs=logs)
    g = Grid(P)
    cfg = S.Cfg(h, n, F, metp_chunks=2)
    ys, saved, _ = S.layer_fwd(pi, g, xs, W, cfg)
    S.layer_bwd(pi, g, dys, saved, W, cfg, S.new_grads(W))
    for r in range(P):
        assert Counter(e["primitive"] for e in logs[r]) == Counter(g.primitives()), (pi, r)
        assert all(e["participants"] == P for e in logs[r])
    total = sum(e["bytes"] for lg in logs for e in lg)
    full = "full" if pi == 4 else "ffn"
    assert total == P * OF.comm_bytes(pi, h, s, P, F, metp_recompute=full), (pi, total)
