"""Per-kernel parity on B200 against the oracle (fp32-accumulate path, reading R-14).

Each kernel is fed bf16 inputs; the oracle computes the same stage in fp64 from
those exact inputs.  Tolerances (relative L2, written per check): fp32 outputs
2e-3 (north_star "fp32-accumulate path"), bf16 outputs 1e-2.
"""
import math

import numpy as np
import pytest
import torch

from oracle import layer as OL
from synth import normal, round_bf16

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2511_13198_b200 import binding as B
    from tests.gpu_util import dev_bf16, dev_f32, host, rel, stream


def _mat(seed, tid, shape, std=1.0):
    return normal(seed, tid, shape, std=std)


GEMM_SHAPES = [(256, 384, 256), (200, 392, 200), (128, 128, 64), (1024, 768, 512), (4096, 4096, 512),
               (344, 1536, 4096), (2368, 2048, 320), (4096, 1536, 4096)]


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("shape", GEMM_SHAPES)
def test_gemm_f32(a_mn, b_mn, shape):
    M, N, K = shape
    A = _mat(1, 1, (M, K), std=1 / math.sqrt(K))
    Bm = _mat(1, 2, (N, K))
    ref = A @ Bm.T
    a_st = A.T.copy() if a_mn else A
    b_st = Bm.T.copy() if b_mn else Bm
    ta, tb = dev_bf16(a_st), dev_bf16(b_st)
    out = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    B.k_gemm(ta.data_ptr(), a_st.shape[1], a_mn, tb.data_ptr(), b_st.shape[1], b_mn, M, N, K,
             out.data_ptr(), N, 2, stream=stream())
    torch.cuda.synchronize()
    assert rel(host(out), ref) < 2e-3
    # fp32 accumulate epilogue: C += A B^T
    B.k_gemm(ta.data_ptr(), a_st.shape[1], a_mn, tb.data_ptr(), b_st.shape[1], b_mn, M, N, K,
             out.data_ptr(), N, 1, stream=stream())
    torch.cuda.synchronize()
    assert rel(host(out), 2 * ref) < 2e-3


def test_gemm_bf16_and_gelu_epilogues():
    M, N, K = 384, 512, 256
    A = _mat(2, 1, (M, K), std=1 / math.sqrt(K))
    W = _mat(2, 2, (N, K))
    ref = A @ W.T
    ta, tw = dev_bf16(A), dev_bf16(W)
    c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    g = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    B.k_gemm(ta.data_ptr(), K, 0, tw.data_ptr(), K, 0, M, N, K, c.data_ptr(), N, 0, stream=stream())
    torch.cuda.synchronize()
    assert rel(host(c), ref) < 1e-2
    B.k_gemm(ta.data_ptr(), K, 0, tw.data_ptr(), K, 0, M, N, K, c.data_ptr(), N, 3, None, g.data_ptr(), N,
             stream=stream())
    torch.cuda.synchronize()
    hb = host(c)
    assert rel(hb, ref) < 1e-2
    assert rel(host(g), OL.gelu(hb)) < 1e-2           # G = GELU(bf16(H))
    # dGELU: C = acc * GELU'(H), aux_out = GELU(H)
    dg = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    g2 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    B.k_gemm(ta.data_ptr(), K, 0, tw.data_ptr(), K, 0, M, N, K, dg.data_ptr(), N, 4, c.data_ptr(),
             g2.data_ptr(), N, stream=stream())
    torch.cuda.synchronize()
    assert rel(host(dg), ref * OL.gelu_grad(hb)) < 1e-2
    assert rel(host(g2), OL.gelu(hb)) < 1e-2


@pytest.mark.parametrize("d", [64, 128])
def test_rope_table_and_gemm_rope(d):
    n_pos = 2048
    t = torch.empty(n_pos, d // 2, 2, dtype=torch.float32, device="cuda")
    B.k_rope_table(t.data_ptr(), n_pos, d, 10000.0, stream())
    torch.cuda.synchronize()
    cos, sin = OL.rope_cos_sin(np.arange(n_pos), d)
    tt = t.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(tt[..., 0] - cos)) < 1e-7 and np.max(np.abs(tt[..., 1] - sin)) < 1e-7
    # large positions: fp64 angle formation keeps the table exact (R-3)
    big = 638976
    tb = torch.empty(big, d // 2, 2, dtype=torch.float32, device="cuda")
    B.k_rope_table(tb.data_ptr(), big, d, 10000.0, stream())
    torch.cuda.synchronize()
    c2, s2 = OL.rope_cos_sin(np.arange(big - 4, big), d)
    last = tb[-4:].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(last[..., 0] - c2)) < 1e-7 and np.max(np.abs(last[..., 1] - s2)) < 1e-7
    # QKV GEMM with fused RoPE; two head groups (Ulysses packing order), rows offset
    heads = 2
    hq = heads * d
    N = 2 * 3 * hq
    M, K = 256, 256
    base = 1000
    A = _mat(3, 1, (M, K), std=1 / math.sqrt(K))
    W = _mat(3, 2, (N, K))
    ref = A @ W.T
    cs, sn = OL.rope_cos_sin(base + np.arange(M), d)
    exp = ref.copy()
    for grp in range(2):
        for blk in range(2):   # Q and K blocks rotate, V does not
            for hh in range(heads):
                c0 = grp * 3 * hq + blk * hq + hh * d
                exp[:, c0:c0 + d] = OL.rope_apply(ref[:, c0:c0 + d], cs, sn)
    ta, tw = dev_bf16(A), dev_bf16(W)
    c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    B.k_gemm_rope(ta.data_ptr(), K, tw.data_ptr(), K, M, N, K, c.data_ptr(), N, t.data_ptr(), d, hq, 0, 0,
                  base, stream())
    torch.cuda.synchronize()
    assert rel(host(c), exp) < 1e-2


@pytest.mark.parametrize("h", [256, 768, 2304, 4096, 8192, 12288])
def test_rmsnorm_fwd_bwd(h):
    # every block-per-row shape: 1 / 2 vectors per thread at <= 4096 (2304: predicated
    # tail), 512 threads with 2 / 3 vectors above (Table 4's LLaMA h = 8192, GPT 12288)
    rows = 300
    x = _mat(4, 1, (rows, h))
    r = _mat(4, 2, (rows, h))
    g = normal(4, 3, (h,), std=0.1, mean=1.0)
    du = _mat(4, 4, (rows, h))
    tx, tr, tg, tdu = dev_bf16(x), dev_bf16(r), dev_bf16(g), dev_bf16(du)
    x1 = torch.empty(rows, h, dtype=torch.bfloat16, device="cuda")
    u = torch.empty(rows, h, dtype=torch.bfloat16, device="cuda")
    rstd = torch.empty(rows, dtype=torch.float32, device="cuda")
    B.k_rmsnorm_fwd(tx.data_ptr(), tr.data_ptr(), tg.data_ptr(), rows, h, 1e-5, x1.data_ptr(), u.data_ptr(),
                    rstd.data_ptr(), stream())
    torch.cuda.synchronize()
    x1r = round_bf16(x + r)
    assert np.array_equal(host(x1), x1r)
    uref, xhat, rref = OL.rmsnorm(x1r, g)
    assert rel(host(rstd), rref) < 2e-3
    assert rel(host(u), uref) < 1e-2
    dx = torch.empty(rows, h, dtype=torch.bfloat16, device="cuda")
    dg = torch.zeros(h, dtype=torch.float32, device="cuda")
    B.k_rmsnorm_bwd(tdu.data_ptr(), x1.data_ptr(), rstd.data_ptr(), tg.data_ptr(), tr.data_ptr(), rows, h,
                    dx.data_ptr(), dg.data_ptr(), stream())
    torch.cuda.synchronize()
    dxr, dgr = OL.rmsnorm_bwd(du, xhat, rref, g)
    assert rel(host(dx), dxr + r) < 1e-2
    assert rel(host(dg), dgr) < 2e-3


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("causal", [1, 0])
@pytest.mark.parametrize("s", [256, 640])
def test_attention_fwd_bwd(d, causal, s):
    _attention_fwd_bwd(d, causal, s)


@pytest.mark.parametrize("s", [256, 640, 1152])
def test_attention_bwd_fused_vs_oracle(s):
    """The fused backward (pds_set_attn_bwd(1); d = 128, causal) against the oracle."""
    B.set_attn_bwd(1)
    try:
        _attention_fwd_bwd(128, 1, s, heads=3)
    finally:
        B.set_attn_bwd(0)


def _attention_fwd_bwd(d, causal, s, heads=2):
    hq = heads * d
    qkv = _mat(5 + d, 1, (s, 3 * hq))
    dout = _mat(5 + d, 2, (s, hq))
    tq, tdo = dev_bf16(qkv), dev_bf16(dout)
    out = torch.empty(s, hq, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(heads, s, dtype=torch.float32, device="cuda")
    B.k_attn_fwd(tq.data_ptr(), 3 * hq, s, heads, d, causal, out.data_ptr(), hq, lse.data_ptr(), stream())
    torch.cuda.synchronize()
    o_gpu = host(out)
    for hh in range(heads):
        q = qkv[:, hh * d:(hh + 1) * d]
        k = qkv[:, hq + hh * d:hq + (hh + 1) * d]
        v = qkv[:, 2 * hq + hh * d:2 * hq + (hh + 1) * d]
        a, l = OL.attention_fwd(q, k, v, causal=bool(causal))
        assert rel(o_gpu[:, hh * d:(hh + 1) * d], a) < 1e-2
        assert rel(host(lse)[hh], l) < 2e-3
    dqkv = torch.empty(s, 3 * hq, dtype=torch.bfloat16, device="cuda")
    B.k_attn_bwd(tq.data_ptr(), 3 * hq, out.data_ptr(), hq, lse.data_ptr(), tdo.data_ptr(), s, heads, d, causal,
                 dqkv.data_ptr(), stream())
    torch.cuda.synchronize()
    g = host(dqkv)
    for hh in range(heads):
        q = qkv[:, hh * d:(hh + 1) * d]
        k = qkv[:, hq + hh * d:hq + (hh + 1) * d]
        v = qkv[:, 2 * hq + hh * d:2 * hq + (hh + 1) * d]
        _, l = OL.attention_fwd(q, k, v, causal=bool(causal))
        dq, dk, dv = OL.attention_bwd(q, k, v, o_gpu[:, hh * d:(hh + 1) * d], l,
                                      dout[:, hh * d:(hh + 1) * d], causal=bool(causal))
        assert rel(g[:, hh * d:(hh + 1) * d], dq) < 1e-2
        assert rel(g[:, hq + hh * d:hq + (hh + 1) * d], dk) < 1e-2
        assert rel(g[:, 2 * hq + hh * d:2 * hq + (hh + 1) * d], dv) < 1e-2


_NWG_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2511_13198_b200 import binding as B
s, heads, d = int(sys.argv[3]), int(sys.argv[4]), 128
B.set_attn_bwd(int(sys.argv[5]))
hq = heads * d
g = torch.Generator().manual_seed(3)
qkv = (torch.randn(s, 3 * hq, generator=g) * 0.5).to(torch.bfloat16).cuda()
dout = torch.randn(s, hq, generator=g).to(torch.bfloat16).cuda()
out = torch.empty(s, hq, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(heads, s, dtype=torch.float32, device="cuda")
dqkv = torch.empty_like(qkv)
B.k_attn_fwd(qkv.data_ptr(), 3 * hq, s, heads, d, 1, out.data_ptr(), hq, lse.data_ptr(), 0)
B.k_attn_bwd(qkv.data_ptr(), 3 * hq, out.data_ptr(), hq, lse.data_ptr(), dout.data_ptr(), s, heads, d, 1,
             dqkv.data_ptr(), 0)
torch.cuda.synchronize()
np.save(sys.argv[2], dqkv.view(torch.int16).cpu().numpy())
"""


def test_attention_bwd_warpgroup_variants_bitwise(tmp_path):
    """(split kernels, the default) dK/dV and dQ kernels with 2 or 4 elementwise warpgroups (PDS_BWD_NWG) do the same
    per-element arithmetic; the MMA k-steps are issued in warpgroup-half order, which
    depends on the count.  So each kernel is bit-identical to the default where the
    count matches (dK/dV: 4 groups, dQ: 2 groups) and equal within fp32 summation
    order otherwise."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for v in ("", "2", "4"):
        f = tmp_path / f"dqkv{v or 'default'}.npy"
        env = dict(os.environ)
        env.pop("PDS_BWD_NWG", None)
        if v:
            env["PDS_BWD_NWG"] = v
        subprocess.run([sys.executable, "-c", _NWG_SCRIPT, root, str(f), "640", "2", "0"], check=True, env=env,
                       timeout=300)
        outs[v] = np.load(f)
    hq = outs[""].shape[1] // 3
    assert np.array_equal(outs[""][:, hq:], outs["4"][:, hq:])       # default dK/dV = 4 groups
    assert np.array_equal(outs[""][:, :hq], outs["2"][:, :hq])       # default dQ = 2 groups
    f32 = {k: (v.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
           for k, v in outs.items()}
    assert rel(f32["2"][:, hq:], f32[""][:, hq:]) < 1e-3
    assert rel(f32["4"][:, :hq], f32[""][:, :hq]) < 1e-3


@pytest.mark.parametrize("s,heads", [(640, 2), (2048, 3), (4096, 5)])
def test_attention_bwd_fused_vs_split(tmp_path, s, heads):
    """The fused backward (one kernel, dQ partials summed over key blocks in a fixed
    order) against the split kernels at the same elementwise warpgroup count (2):
    dK / dV come from the same MMA and elementwise sequence, so they are bit-identical;
    dQ differs only in fp32 summation order (per-key-block partials vs one TMEM
    accumulator).  The fused result is reproducible bit for bit (run twice), and the
    oracle check of the fused path is test_attention_bwd_fused_vs_oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for name, mode, nwg in (("fused", "1", None), ("fused2", "1", None), ("split2", "0", "2")):
        f = tmp_path / f"{name}.npy"
        env = dict(os.environ)
        env.pop("PDS_BWD_NWG", None)
        if nwg:
            env["PDS_BWD_NWG"] = nwg
        subprocess.run([sys.executable, "-c", _NWG_SCRIPT, root, str(f), str(s), str(heads), mode], check=True,
                       env=env, timeout=300)
        outs[name] = np.load(f)
    hq = outs["fused"].shape[1] // 3
    assert np.array_equal(outs["fused"], outs["fused2"])
    assert np.array_equal(outs["fused"][:, hq:], outs["split2"][:, hq:])
    f32 = {k: (v.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
           for k, v in outs.items()}
    assert rel(f32["fused"][:, :hq], f32["split2"][:, :hq]) < 2e-3


# ---------------------------------------------------------------- collective overlap protocol
# The tile-overlapped MegatronTS collectives (pds_set_overlap) rest on two GEMM hooks:
# per-chunk "landed" flags polled by the TMA producer before it loads A rows, and
# per-chunk store counters the reduce-scatter waits on.  Here the chunks really arrive
# (and leave) WHILE the GEMM runs: pinned-host copies on a second stream (copy engine,
# no SM), behind a large dummy copy so the GEMM starts first and has to spin.

@pytest.mark.parametrize("M,N,K,chunk,rot", [(4096, 2048, 2048, 1024, 1024),   # CTA-pair kernel
                                             (1536, 384, 512, 384, 768)])      # 1-CTA kernel, 3 m-blocks/chunk
def test_gemm_waits_for_chunk_flags(M, N, K, chunk, rot):
    A = round_bf16(_mat(3, 1, (M, K), std=1 / math.sqrt(K)))
    W = _mat(3, 2, (N, K))
    tw = dev_bf16(W)
    ta_ref = dev_bf16(A)
    ref = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    B.k_gemm(ta_ref.data_ptr(), K, 0, tw.data_ptr(), K, 0, M, N, K, ref.data_ptr(), N, 0, stream=stream())
    torch.cuda.synchronize()

    a_host = ta_ref.cpu().pin_memory()
    dummy_h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    dummy_d = torch.empty_like(dummy_h, device="cuda")
    ta = torch.full((M, K), float("nan"), dtype=torch.bfloat16, device="cuda")
    flags = torch.zeros(M // chunk, dtype=torch.int32, device="cuda")
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    epoch = 7
    B.k_gemm_sync(ta.data_ptr(), K, tw.data_ptr(), K, M, N, K, out.data_ptr(), N, wait_flags=flags.data_ptr(),
                  epoch=epoch, chunk_rows=chunk, m_rot_rows=rot, stream=sa.cuda_stream)
    with torch.cuda.stream(sb):
        dummy_d.copy_(dummy_h, non_blocking=True)         # ~5-10 ms: the GEMM is already spinning
        for c in [(rot // chunk + i) % (M // chunk) for i in range(M // chunk)]:
            ta[c * chunk:(c + 1) * chunk].copy_(a_host[c * chunk:(c + 1) * chunk], non_blocking=True)
            B.k_stream_write32(sb.cuda_stream, flags.data_ptr() + 4 * c, epoch)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("M,N,K,chunk,rot", [(4096, 2048, 2048, 1024, 2048), (1536, 384, 512, 384, 0)])
def test_gemm_store_counters_gate_chunk_reads(M, N, K, chunk, rot):
    A = _mat(4, 1, (M, K), std=1 / math.sqrt(K))
    W = _mat(4, 2, (N, K))
    ta, tw = dev_bf16(A), dev_bf16(W)
    nch = M // chunk
    ctr = torch.zeros(nch, dtype=torch.int32, device="cuda")
    out = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    got = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    # the reader is enqueued FIRST: each chunk is copied out as soon as its counter says so
    for c in range(nch):
        B.k_stream_wait32(sb.cuda_stream, ctr.data_ptr() + 4 * c, chunk * N // 8)
        with torch.cuda.stream(sb):
            got[c * chunk:(c + 1) * chunk].copy_(out[c * chunk:(c + 1) * chunk], non_blocking=True)
    B.k_gemm_sync(ta.data_ptr(), K, tw.data_ptr(), K, M, N, K, out.data_ptr(), N, done_ctr=ctr.data_ptr(),
                  chunk_rows=chunk, m_rot_rows=rot, stream=sa.cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int16), out.cpu().view(torch.int16))
    assert ctr.cpu().tolist() == [chunk * N // 8] * nch
    assert rel(host(out), A.astype(np.float64) @ W.T) < 1e-2


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("causal", [1, 0])
@pytest.mark.parametrize("s,qn", [(1024, 256), (768, 384)])   # 384: the 256-row forward tiles straddle ranks
def test_attention_query_rows(d, causal, s, qn):
    """Context-parallel attention (MegatronCZ): every rank's query rows against all keys;
    the forward rows are the full attention's, and the per-rank dQ / dK / dV
    contributions sum to the full backward."""
    heads = 2
    hq = heads * d
    qkv = _mat(7 + d, 1, (s, 3 * hq))
    dout = _mat(7 + d, 2, (s, hq))
    tq, tdo = dev_bf16(qkv), dev_bf16(dout)
    ref_o = torch.empty(s, hq, dtype=torch.bfloat16, device="cuda")
    ref_l = torch.empty(heads, s, dtype=torch.float32, device="cuda")
    B.k_attn_fwd(tq.data_ptr(), 3 * hq, s, heads, d, causal, ref_o.data_ptr(), hq, ref_l.data_ptr(), stream())
    acc = torch.zeros(s, 3 * hq, dtype=torch.float32, device="cuda")
    o_rows = []
    for qlo in range(0, s, qn):
        out = torch.empty(qn, hq, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(heads, qn, dtype=torch.float32, device="cuda")
        B.k_attn_fwd_rows(tq.data_ptr(), 3 * hq, s, heads, d, causal, qlo, qn, out.data_ptr(), hq, lse.data_ptr(),
                          stream())
        torch.cuda.synchronize()
        if qlo % 256 == 0:      # same 256-row tiles as the full launch: the same arithmetic
            assert torch.equal(out.view(torch.int16), ref_o[qlo:qlo + qn].view(torch.int16)), qlo
        else:
            assert rel(host(out), host(ref_o[qlo:qlo + qn])) < 2e-3, qlo
        assert torch.allclose(lse, ref_l[:, qlo:qlo + qn], rtol=0, atol=1e-4), qlo
        o_rows.append(out)
        dq = torch.zeros(s, 3 * hq, dtype=torch.bfloat16, device="cuda")
        B.k_attn_bwd_rows(tq.data_ptr(), 3 * hq, out.data_ptr(), hq, lse.data_ptr(), tdo[qlo:qlo + qn].data_ptr(),
                          s, heads, d, causal, qlo, qn, dq.data_ptr(), stream())
        torch.cuda.synchronize()
        acc += dq.float()
    g = host(acc)
    o_gpu = host(torch.cat(o_rows))
    for hh in range(heads):
        q = qkv[:, hh * d:(hh + 1) * d]
        k = qkv[:, hq + hh * d:hq + (hh + 1) * d]
        v = qkv[:, 2 * hq + hh * d:2 * hq + (hh + 1) * d]
        _, l = OL.attention_fwd(q, k, v, causal=bool(causal))
        dqr, dkr, dvr = OL.attention_bwd(q, k, v, o_gpu[:, hh * d:(hh + 1) * d], l, dout[:, hh * d:(hh + 1) * d],
                                         causal=bool(causal))
        assert rel(g[:, hh * d:(hh + 1) * d], dqr) < 1e-2
        assert rel(g[:, hq + hh * d:hq + (hh + 1) * d], dkr) < 1e-2
        assert rel(g[:, 2 * hq + hh * d:2 * hq + (hh + 1) * d], dvr) < 1e-2


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("causal", [1, 0])
def test_attention_ring_pairs(d, causal):
    """Ring attention's pieces (MegatronCZ, R-CZ): the sequence cut into 4 blocks of c
    rows, every query block's attention assembled from (query block, key block) pairs —
    the diagonal pair causal, earlier key blocks full, later ones skipped when causal —
    merged by log-sum-exp (pds_k_attn_merge), equals full attention (oracle); the pair
    backwards accumulated in fp32 (pds_k_attn_bwd_pair, merged LSE, D from
    pds_k_attn_dot) equal the full backward before RoPE^T."""
    heads, c, nb = 2, 256, 4
    s = c * nb
    hq = heads * d
    qkv = _mat(11 + d, 1, (s, 3 * hq))
    dout = _mat(11 + d, 2, (s, hq))
    tq, tdo = dev_bf16(qkv), dev_bf16(dout)
    kv = tq[:, hq:].contiguous()                      # [K | V] of all rows
    o_acc = torch.zeros(s, hq, dtype=torch.float32, device="cuda")
    l_acc = torch.zeros(heads, s, dtype=torch.float32, device="cuda")
    out = torch.empty(s, hq, dtype=torch.bfloat16, device="cuda")
    op = torch.empty(c, hq, dtype=torch.bfloat16, device="cuda")
    lp = torch.empty(heads, c, dtype=torch.float32, device="cuda")
    st = stream()
    for a in range(nb):
        first = True
        for bb in range(nb):
            if causal and bb > a:
                continue
            B.k_attn_fwd_pair(tq[a * c:].data_ptr(), 3 * hq, kv[bb * c:].data_ptr(), 2 * hq, 0, hq, c, c, heads, d,
                              int(causal and bb == a), op.data_ptr(), hq, lp.data_ptr(), st)
            B.k_attn_merge(o_acc[a * c:].data_ptr(), hq, l_acc[:, a * c:].data_ptr(), s, op.data_ptr(), hq,
                           lp.data_ptr(), c, c, heads, d, int(first), out[a * c:].data_ptr(), hq, st)
            first = False
    torch.cuda.synchronize()
    o_gpu = host(out)
    dd = torch.empty(heads, s, dtype=torch.float32, device="cuda")
    B.k_attn_dot(out.data_ptr(), hq, tdo.data_ptr(), s, heads, d, dd.data_ptr(), st)
    dq_acc = torch.zeros(s, hq, dtype=torch.float32, device="cuda")
    dkv_acc = torch.zeros(s, 2 * hq, dtype=torch.float32, device="cuda")
    lse_blk = torch.empty(heads, c, dtype=torch.float32, device="cuda")
    d_blk = torch.empty(heads, c, dtype=torch.float32, device="cuda")
    for a in range(nb):
        lse_blk.copy_(l_acc[:, a * c:(a + 1) * c])
        d_blk.copy_(dd[:, a * c:(a + 1) * c])
        for bb in range(nb):
            if causal and bb > a:
                continue
            B.k_attn_bwd_pair(tq[a * c:].data_ptr(), 3 * hq, kv[bb * c:].data_ptr(), 2 * hq, 0, hq,
                              tdo[a * c:].data_ptr(), hq, lse_blk.data_ptr(), d_blk.data_ptr(), c, c, heads, d,
                              int(causal and bb == a), dq_acc[a * c:].data_ptr(), hq, dkv_acc[bb * c:].data_ptr(),
                              2 * hq, st)
    torch.cuda.synchronize()
    for hh in range(heads):
        q = qkv[:, hh * d:(hh + 1) * d]
        k = qkv[:, hq + hh * d:hq + (hh + 1) * d]
        v = qkv[:, 2 * hq + hh * d:2 * hq + (hh + 1) * d]
        a_ref, l_ref = OL.attention_fwd(q, k, v, causal=bool(causal))
        assert rel(o_gpu[:, hh * d:(hh + 1) * d], a_ref) < 1e-2
        assert np.allclose(host(l_acc)[hh], l_ref, rtol=0, atol=2e-3)
        dqr, dkr, dvr = OL.attention_bwd(q, k, v, o_gpu[:, hh * d:(hh + 1) * d], l_ref,
                                         dout[:, hh * d:(hh + 1) * d], causal=bool(causal))
        assert rel(host(dq_acc)[:, hh * d:(hh + 1) * d], dqr) < 1e-2
        assert rel(host(dkv_acc)[:, hh * d:(hh + 1) * d], dkr) < 1e-2
        assert rel(host(dkv_acc)[:, hq + hh * d:hq + (hh + 1) * d], dvr) < 1e-2


_FWD_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2511_13198_b200 import binding as B
s, heads, d, causal = int(sys.argv[3]), 3, 128, int(sys.argv[4])
hq = heads * d
g = torch.Generator().manual_seed(5)
qkv = (torch.randn(s, 3 * hq, generator=g) * 0.5).to(torch.bfloat16).cuda()
out = torch.empty(s, hq, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(heads, s, dtype=torch.float32, device="cuda")
B.k_attn_fwd(qkv.data_ptr(), 3 * hq, s, heads, d, causal, out.data_ptr(), hq, lse.data_ptr(), 0)
torch.cuda.synchronize()
np.savez(sys.argv[2], out=out.view(torch.int16).cpu().numpy(), lse=lse.cpu().numpy())
"""


@pytest.mark.parametrize("s,causal", [(640, 1), (1536, 1), (1024, 0)])
def test_attention_fwd_pair_kernel_matches(tmp_path, s, causal):
    """The opt-in CTA-pair forward (PDS_ATTN_FWD=pair, cta_group::2) computes every row with
    the same softmax code and the same MMA shapes per row as the default single-CTA
    forward: outputs and LSE agree (ragged pair of 512 rows included)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("1cta", "pair"):
        f = tmp_path / f"{mode}.npz"
        env = dict(os.environ)
        env["PDS_ATTN_FWD"] = mode
        subprocess.run([sys.executable, "-c", _FWD_SCRIPT, root, str(f), str(s), str(causal)], check=True, env=env,
                       timeout=300)
        res[mode] = np.load(f)
    a = (res["1cta"]["out"].view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    b = (res["pair"]["out"].view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert rel(b, a) < 1e-3
    assert np.allclose(res["pair"]["lse"], res["1cta"]["lse"], rtol=0, atol=1e-4)


@pytest.mark.parametrize("s,causal", [(640, 1), (1024, 0), (2304, 1)])
def test_attention_fwd_register_pass_matches(tmp_path, s, causal):
    """The register-pass forward (default: setmaxnreg reallocation, the S row read from TMEM
    once) runs the same arithmetic in the same order as the two-pass softmax
    (PDS_ATTN_FWD=2pass): outputs and LSE are bit-identical."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("2pass", "regs"):
        f = tmp_path / f"{mode}.npz"
        env = dict(os.environ)
        env["PDS_ATTN_FWD"] = mode
        subprocess.run([sys.executable, "-c", _FWD_SCRIPT, root, str(f), str(s), str(causal)], check=True, env=env,
                       timeout=300)
        res[mode] = np.load(f)
    assert np.array_equal(res["regs"]["out"], res["2pass"]["out"])
    assert np.array_equal(res["regs"]["lse"], res["2pass"]["lse"])


@pytest.mark.parametrize("s,causal", [(640, 1), (1024, 0), (2304, 1)])
def test_attention_fwd_split_softmax_matches(tmp_path, s, causal):
    """The opt-in split-softmax forward (PDS_ATTN_FWD=split: two warpgroups per query tile,
    row max / row sum exchanged through shared memory) agrees with the default forward
    (the row sum is added in two partial sums: rounding-level differences only)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("regs", "split"):
        f = tmp_path / f"{mode}.npz"
        env = dict(os.environ)
        env["PDS_ATTN_FWD"] = mode
        subprocess.run([sys.executable, "-c", _FWD_SCRIPT, root, str(f), str(s), str(causal)], check=True, env=env,
                       timeout=300)
        res[mode] = np.load(f)
    a = (res["regs"]["out"].view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    b = (res["split"]["out"].view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert rel(b, a) < 1e-3
    assert np.allclose(res["split"]["lse"], res["regs"]["lse"], rtol=0, atol=1e-5)


# ---------------------------------------------------------------- Llama variant (NEXT-3)
@pytest.mark.parametrize("d,heads,kv_heads", [(128, 4, 1), (128, 4, 2), (64, 8, 2)])
@pytest.mark.parametrize("causal", [1, 0])
@pytest.mark.parametrize("s", [256, 640])
def test_attention_gqa_vs_oracle(d, heads, kv_heads, causal, s):
    """GQA attention (R-GQA): the kernels read key / value head i // grp for query head
    i; the dK / dV kernel sums the group's query heads.  Oracle: oracle.layer's
    per-head attention on the same bf16 inputs, dK / dV summed over the group."""
    hq, hk, grp = heads * d, kv_heads * d, heads // kv_heads
    W = hq + 2 * hk
    qkv = _mat(31 + d, 1, (s, W))
    dout = _mat(31 + d, 2, (s, hq))
    tq, tdo = dev_bf16(qkv), dev_bf16(dout)
    out = torch.empty(s, hq, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(heads, s, dtype=torch.float32, device="cuda")
    B.k_attn_fwd_gqa(tq.data_ptr(), W, s, heads, kv_heads, d, causal, out.data_ptr(), hq, lse.data_ptr(), stream())
    dqkv = torch.zeros(s, W, dtype=torch.bfloat16, device="cuda")
    B.k_attn_bwd_gqa(tq.data_ptr(), W, out.data_ptr(), hq, lse.data_ptr(), tdo.data_ptr(), s, heads, kv_heads, d,
                     causal, dqkv.data_ptr(), stream())
    torch.cuda.synchronize()
    o_gpu, g = host(out), host(dqkv)
    dk_ref = np.zeros((s, hk))
    dv_ref = np.zeros((s, hk))
    for hh in range(heads):
        j = hh // grp
        q = qkv[:, hh * d:(hh + 1) * d]
        k = qkv[:, hq + j * d:hq + (j + 1) * d]
        v = qkv[:, hq + hk + j * d:hq + hk + (j + 1) * d]
        a, l = OL.attention_fwd(q, k, v, causal=bool(causal))
        assert rel(o_gpu[:, hh * d:(hh + 1) * d], a) < 1e-2
        assert rel(host(lse)[hh], l) < 2e-3
        dq, dk, dv = OL.attention_bwd(q, k, v, o_gpu[:, hh * d:(hh + 1) * d], l, dout[:, hh * d:(hh + 1) * d],
                                      causal=bool(causal))
        assert rel(g[:, hh * d:(hh + 1) * d], dq) < 1e-2
        dk_ref[:, j * d:(j + 1) * d] += dk
        dv_ref[:, j * d:(j + 1) * d] += dv
    assert rel(g[:, hq:hq + hk], dk_ref) < 1e-2
    assert rel(g[:, hq + hk:], dv_ref) < 1e-2


@pytest.mark.parametrize("M,F,K", [(384, 256, 256), (1024, 768, 512), (2048, 2048, 1024)])
def test_gemm_swiglu_epilogues(M, F, K):
    """SwiGLU epilogues (R-SWIGLU) against oracle.layer.ffn_act / ffn_act_bwd on the
    interleaved layout: forward H and G = SiLU(bf16 gate) * bf16 up; backward dH (both
    halves), G, and the transposed dH^T / G^T copies the dW GEMMs read."""
    A = _mat(41, 1, (M, K), std=1 / math.sqrt(K))
    Wt = _mat(41, 2, (2 * F, K))                           # W_in^T rows, interleaved
    ta, tw = dev_bf16(A), dev_bf16(Wt)
    hb = torch.empty(M, 2 * F, dtype=torch.bfloat16, device="cuda")
    g = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    B.k_gemm_swiglu(ta.data_ptr(), K, tw.data_ptr(), K, M, 2 * F, K, 0, hb.data_ptr(), 2 * F, g_out=g.data_ptr(),
                    ld_g=F, stream=stream())
    torch.cuda.synchronize()
    H = host(hb)
    assert rel(H, A @ Wt.T) < 1e-2
    assert rel(host(g), OL.ffn_act(H, "swiglu", il=True)) < 1e-2
    # backward: the accumulator is dG = dZ W_out^T (here any [M, F] product)
    dZ = _mat(41, 3, (M, K))
    Wo = _mat(41, 4, (F, K), std=1 / math.sqrt(K))
    tz, to = dev_bf16(dZ), dev_bf16(Wo)
    dh = torch.empty(M, 2 * F, dtype=torch.bfloat16, device="cuda")
    g2 = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    dht = torch.empty(2 * F, M, dtype=torch.bfloat16, device="cuda")
    gt = torch.empty(F, M, dtype=torch.bfloat16, device="cuda")
    B.k_gemm_swiglu(tz.data_ptr(), K, to.data_ptr(), K, M, F, K, 1, dh.data_ptr(), 2 * F, hb.data_ptr(), 2 * F,
                    g2.data_ptr(), F, dht.data_ptr(), gt.data_ptr(), M, stream=stream())
    torch.cuda.synchronize()
    dg = dZ @ Wo.T
    ref_dh = OL.ffn_act_bwd(dg, H, "swiglu", il=True)
    ref_g = OL.ffn_act(H, "swiglu", il=True)
    assert rel(host(dh), ref_dh) < 1e-2
    assert rel(host(g2), ref_g) < 1e-2
    assert rel(host(dht), ref_dh.T) < 1e-2
    assert rel(host(gt), ref_g.T) < 1e-2


def test_gemm_rope_gqa_groups():
    """RoPE epilogue with GQA column groups [Q (hq) | K (hk) | V (hk)]: Q and K columns
    rotated at their row's position, V untouched (oracle.layer.rope_apply)."""
    d, hq, hk, M, K = 128, 512, 128, 256, 256
    N = 2 * (hq + 2 * hk)                                  # two groups (two ranks' blocks)
    A = _mat(43, 1, (M, K), std=1 / math.sqrt(K))
    Wt = _mat(43, 2, (N, K))
    rope = torch.empty(M, d // 2, 2, dtype=torch.float32, device="cuda")
    B.k_rope_table(rope.data_ptr(), M, d, stream=stream())
    ta, tw = dev_bf16(A), dev_bf16(Wt)
    c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    B.k_gemm_rope_gqa(ta.data_ptr(), K, tw.data_ptr(), K, M, N, K, c.data_ptr(), N, rope.data_ptr(), d, hq, hk,
                      stream=stream())
    torch.cuda.synchronize()
    raw = A @ Wt.T
    cos, sin = OL.rope_cos_sin(np.arange(M), d)
    ref = raw.copy()
    for g0 in (0, hq + 2 * hk):
        for c0 in range(g0, g0 + hq + hk, d):
            ref[:, c0:c0 + d] = OL.rope_apply(raw[:, c0:c0 + d], cos, sin)
    assert rel(host(c), ref) < 1e-2


# ---------------------------------------------------------------- dS through HBM
@pytest.mark.parametrize("s,heads", [(256, 2), (640, 3), (1152, 4)])
def test_attention_bwd_ds_path_vs_oracle(s, heads):
    """Backward with dS through HBM (pds_set_attn_bwd(2)): the dK/dV kernel also stores
    dS^T, one batched causal GEMM forms dQ = scale dS K.  Same oracle check as the split
    kernels (causal, d = 128, ragged block counts)."""
    try:
        B.set_attn_bwd(2)
        _attention_fwd_bwd(128, 1, s, heads=heads)
    finally:
        B.set_attn_bwd(0)
