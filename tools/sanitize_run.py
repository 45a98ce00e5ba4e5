"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) at tiny
shapes: every kernel family of libparadyse.so once — both tcgen05 GEMM kernels (CTA
pair and 1-CTA) with every epilogue, the attention forward / backward (d = 64 and 128,
causal and not, full and query-row-range), the norm / transpose / pack kernels — plus
one whole layer fwd + bwd per strategy (P = 1 and a P = 2 loopback group); the Llama
variant (GQA attention, SwiGLU epilogues, a GQA + SwiGLU layer per strategy) and varlen
packing.

  compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py
"""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_13198_b200 import binding as B  # noqa: E402


def r(*sh, std=1.0):
    return (torch.randn(*sh, device="cuda") * std).to(torch.bfloat16)


def kernels():
    st = torch.cuda.current_stream().cuda_stream
    for (M, N, K) in [(256, 512, 256), (128, 128, 64), (384, 256, 320)]:
        a, b = r(M, K), r(N, K)
        c32 = torch.zeros(M, N, device="cuda")
        c16 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        g = torch.empty_like(c16)
        for am in (0, 1):
            for bm in (0, 1):
                aa = a.t().contiguous() if am else a
                bb = b.t().contiguous() if bm else b
                B.k_gemm(aa.data_ptr(), aa.shape[1], am, bb.data_ptr(), bb.shape[1], bm, M, N, K, c32.data_ptr(), N,
                         2, stream=st)
                B.k_gemm(aa.data_ptr(), aa.shape[1], am, bb.data_ptr(), bb.shape[1], bm, M, N, K, c32.data_ptr(), N,
                         1, stream=st)
        B.k_gemm(a.data_ptr(), K, 0, b.data_ptr(), K, 0, M, N, K, c16.data_ptr(), N, 0, stream=st)
        B.k_gemm(a.data_ptr(), K, 0, b.data_ptr(), K, 0, M, N, K, c16.data_ptr(), N, 3, None, g.data_ptr(), N,
                 stream=st)
        d16 = torch.empty_like(c16)
        B.k_gemm(a.data_ptr(), K, 0, b.data_ptr(), K, 0, M, N, K, d16.data_ptr(), N, 4, c16.data_ptr(), g.data_ptr(),
                 N, stream=st)
    for d in (64, 128):
        s, heads = 384, 2
        qkv = r(s, 3 * heads * d, std=0.5)
        out = torch.empty(s, heads * d, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(heads, s, device="cuda")
        dout = r(s, heads * d)
        dqkv = torch.zeros_like(qkv)
        for causal in (1, 0):
            B.k_attn_fwd(qkv.data_ptr(), 3 * heads * d, s, heads, d, causal, out.data_ptr(), heads * d,
                         lse.data_ptr(), st)
            B.k_attn_bwd(qkv.data_ptr(), 3 * heads * d, out.data_ptr(), heads * d, lse.data_ptr(), dout.data_ptr(), s,
                         heads, d, causal, dqkv.data_ptr(), st)
        qn = 128
        out_r = torch.empty(qn, heads * d, dtype=torch.bfloat16, device="cuda")
        lse_r = torch.empty(heads, qn, device="cuda")
        B.k_attn_fwd_rows(qkv.data_ptr(), 3 * heads * d, s, heads, d, 1, 128, qn, out_r.data_ptr(), heads * d,
                          lse_r.data_ptr(), st)
        B.k_attn_bwd_rows(qkv.data_ptr(), 3 * heads * d, out_r.data_ptr(), heads * d, lse_r.data_ptr(),
                          dout[:qn].data_ptr(), s, heads, d, 1, 128, qn, dqkv.data_ptr(), st)
    # GQA attention (4 query heads on 2 / 1 key-value heads) and the SwiGLU epilogues
    for d, heads, kvh in ((128, 4, 2), (64, 4, 1)):
        s = 384
        W = (heads + 2 * kvh) * d
        qkv = r(s, W, std=0.5)
        out = torch.empty(s, heads * d, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(heads, s, device="cuda")
        dout = r(s, heads * d)
        dqkv = torch.zeros_like(qkv)
        for causal in (1, 0):
            B.k_attn_fwd_gqa(qkv.data_ptr(), W, s, heads, kvh, d, causal, out.data_ptr(), heads * d, lse.data_ptr(), st)
            B.k_attn_bwd_gqa(qkv.data_ptr(), W, out.data_ptr(), heads * d, lse.data_ptr(), dout.data_ptr(), s, heads,
                             kvh, d, causal, dqkv.data_ptr(), st)
    M, F, K = 384, 256, 256
    a, wt = r(M, K), r(2 * F, K)
    hb = torch.empty(M, 2 * F, dtype=torch.bfloat16, device="cuda")
    g1 = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    B.k_gemm_swiglu(a.data_ptr(), K, wt.data_ptr(), K, M, 2 * F, K, 0, hb.data_ptr(), 2 * F, g_out=g1.data_ptr(),
                    ld_g=F, stream=st)
    wo = r(F, K)
    dh, dht, gt = (torch.empty(M, 2 * F, dtype=torch.bfloat16, device="cuda"),
                   torch.empty(2 * F, M, dtype=torch.bfloat16, device="cuda"),
                   torch.empty(F, M, dtype=torch.bfloat16, device="cuda"))
    B.k_gemm_swiglu(a.data_ptr(), K, wo.data_ptr(), K, M, F, K, 1, dh.data_ptr(), 2 * F, hb.data_ptr(), 2 * F,
                    g1.data_ptr(), F, dht.data_ptr(), gt.data_ptr(), M, stream=st)
    h, rows = 512, 300
    x, res, gg = r(rows, h), r(rows, h), r(h)
    x1, u = torch.empty_like(x), torch.empty_like(x)
    rstd = torch.empty(rows, device="cuda")
    B.k_rmsnorm_fwd(x.data_ptr(), res.data_ptr(), gg.data_ptr(), rows, h, 1e-5, x1.data_ptr(), u.data_ptr(),
                    rstd.data_ptr(), st)
    dx = torch.empty_like(x)
    dg = torch.zeros(h, device="cuda")
    B.k_rmsnorm_bwd(u.data_ptr(), x1.data_ptr(), rstd.data_ptr(), gg.data_ptr(), res.data_ptr(), rows, h,
                    dx.data_ptr(), dg.data_ptr(), st)
    torch.cuda.synchronize()


def layers():
    from paper_2511_13198_b200.calibrate import make_layer_buffers
    h, n, F, s = 256, 4, 1024, 512
    st = torch.cuda.current_stream().cuda_stream
    model = B.Model(h=h, n_heads=n, ffn=F, metp_chunks=2)
    ctx = B.Context(model)
    w, gr, x, dy = make_layer_buffers(torch, model, 1, s)
    W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
    G = B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for pi in range(B.N_STRATEGIES):
        sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
        ctx.layer_bwd(pi, dy.data_ptr(), sv, W, G, dx.data_ptr(), st)
    ctx.set_varlen([256, 256])                       # varlen packing (TS / UZ / METP / METP-full)
    for pi in (0, 1, 2, 4):
        sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
        ctx.layer_bwd(pi, dy.data_ptr(), sv, W, G, dx.data_ptr(), st)
    torch.cuda.synchronize()
    ctx.close()
    # the Llama variant (GQA 4 -> 2, SwiGLU), every strategy
    lm = B.Model(h=h, n_heads=n, ffn=512, metp_chunks=2, n_kv_heads=2, ffn_act=1)
    ctx = B.Context(lm)
    w, gr, x, dy = make_layer_buffers(torch, lm, 1, s)
    W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
    G = B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for pi in range(B.N_STRATEGIES):
        sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st)
        ctx.layer_bwd(pi, dy.data_ptr(), sv, W, G, dx.data_ptr(), st)
    torch.cuda.synchronize()
    ctx.close()
    # P = 2 loopback group, tile-overlapped collectives on (GEMMs polling flags)
    P = 2
    grp = B.Group(P)
    errs = []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            sm = torch.cuda.Stream()
            with torch.cuda.stream(sm):
                c = B.Context(model, P=P, rank=rank, group=grp)
                w, gr, x, dy = make_layer_buffers(torch, model, P, s, seed=rank)
                W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
                G = B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))
                y, dx = torch.empty_like(x), torch.empty_like(x)
                for pi in range(B.N_STRATEGIES):
                    sv = c.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), sm.cuda_stream)
                    c.layer_bwd(pi, dy.data_ptr(), sv, W, G, dx.data_ptr(), sm.cuda_stream)
                sm.synchronize()
                c.close()
        except Exception as e:      # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(P)]
    [t.start() for t in th]
    [t.join() for t in th]
    grp.close()
    if errs:
        raise errs[0]


if __name__ == "__main__":
    torch.cuda.set_device(0)
    kernels()
    print("kernels ok", flush=True)
    if "--kernels-only" not in sys.argv:
        layers()
        print("layers ok", flush=True)
