"""Attention kernels alone through the kernel-level C ABI (pds_k_attn_fwd / _bwd):
7B head shapes (32 heads, d = 128, causal), TFLOP/s per direction (algorithmic
flops: fwd 2 matmuls, bwd 5, over the causal half).  For A/B of kernel variants run
it under `ncu --clock-control base` (fixed clocks) and compare durations; its own
event timings are subject to the power-capped clock.

  python tools/attn_bench.py --s 16384 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2511_13198_b200 import binding as B
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=16384)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fused", action="store_true", help="fused backward kernel instead of the split dK/dV + dQ")
    ap.add_argument("--ds", action="store_true", help="dS through HBM: dK/dV kernel + batched causal dQ GEMM")
    a = ap.parse_args()
    B.set_attn_bwd(1 if a.fused else 2 if a.ds else 0)
    s, H, d = a.s, a.heads, a.d
    hq = H * d
    qkv = (torch.randn(s, 3 * hq, device="cuda") * 0.5).to(torch.bfloat16)
    out = torch.empty(s, hq, device="cuda", dtype=torch.bfloat16)
    dout = torch.randn(s, hq, device="cuda").to(torch.bfloat16)
    lse = torch.empty(H, s, device="cuda", dtype=torch.float32)
    dqkv = torch.empty_like(qkv)
    st = torch.cuda.current_stream().cuda_stream
    fl = 2.0 * s * s * d * H          # one causal matmul (half of 2 s^2 d) x heads
    for name, fn, mult in (("fwd", lambda: B.k_attn_fwd(qkv.data_ptr(), 3 * hq, s, H, d, 1, out.data_ptr(), hq,
                                                       lse.data_ptr(), st), 2),
                           ("bwd", lambda: B.k_attn_bwd(qkv.data_ptr(), 3 * hq, out.data_ptr(), hq, lse.data_ptr(),
                                                       dout.data_ptr(), s, H, d, 1, dqkv.data_ptr(), st), 5)):
        ts = []
        for r in range(a.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        ms = min(ts)
        tag = (" fused" if a.fused else " ds" if a.ds else "") if name == "bwd" else ""
        print(f"{name}{tag} s={s} {ms:.3f} ms {mult * fl / 2 / ms / 1e9:.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
