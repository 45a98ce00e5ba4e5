"""Per-shape timing of the layer's GEMMs (7B layer, P = 1) through pds_k_gemm.

Shapes of one layer fwd + bwd at sequence length s (h = 4096, F = 16384):
  fwd  QKV (s, 3h, h) TN, proj (s, h, h) NN, FC1 (s, F, h) TN+GELU, FC2 (s, h, F) NN
  bwd  dG (s, F, h) TN+dGELU, dW_out (F, h, s) MM f32+=, dW_in (F, h, s) MM f32+=,
       dV2 (s, h, F) NN, dA (s, h, h) TN, dW_proj (h, h, s) MM f32+=,
       dW_qkv (3h, h, s) MM f32+=, dU (s, h, 3h) NN
(TN: A K-major, B K-major; NN: B MN-major; MM: both MN-major.)
Reports TFLOP/s per shape (CUDA events, median of reps, L2 flushed between reps).
"""
from __future__ import annotations

import argparse
import json


def main():
    import torch
    from . import binding as B
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--probe", action="store_true")
    a = ap.parse_args()
    s, h, F = a.s, 4096, 16384
    shapes = [("QKV", s, 3 * h, h, 0, 0, 0), ("proj", s, h, h, 0, 1, 0), ("FC1", s, F, h, 0, 0, 3),
              ("FC2", s, h, F, 0, 1, 0), ("dG", s, F, h, 0, 0, 4), ("dW_out", F, h, s, 1, 1, 1),
              ("dW_in", F, h, s, 1, 1, 1), ("dV2", s, h, F, 0, 1, 0), ("dA", s, h, h, 0, 0, 0),
              ("dW_proj", h, h, s, 1, 1, 1), ("dW_qkv", 3 * h, h, s, 1, 1, 1), ("dU", s, h, 3 * h, 0, 1, 0)]
    if a.probe:   # isolate operand majors from the epilogue
        shapes = [("TN_bf16", F, h, s, 0, 0, 0), ("TN_f32acc", F, h, s, 0, 0, 1), ("MM_bf16", F, h, s, 1, 1, 0),
                  ("MM_f32acc", F, h, s, 1, 1, 1), ("NT_bf16", F, h, s, 0, 1, 0), ("MT_bf16", F, h, s, 1, 0, 0)]
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    res = {}
    tot_fl = tot_ms = 0.0
    for name, M, N, K, a_mn, b_mn, epi in shapes:
        A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if a_mn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
        Bm = torch.randn(K, N, device="cuda").to(torch.bfloat16) if b_mn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
        C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi in (1, 2) else torch.bfloat16)
        aux_in = torch.randn(M, N, device="cuda").to(torch.bfloat16) if epi == 4 else None
        aux_out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi in (3, 4) else None
        lda = A.shape[1]
        ldb = Bm.shape[1]
        ts = []
        for r in range(a.reps + 2):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            B.k_gemm(A.data_ptr(), lda, a_mn, Bm.data_ptr(), ldb, b_mn, M, N, K, C.data_ptr(), N, epi,
                     aux_in.data_ptr() if aux_in is not None else None,
                     aux_out.data_ptr() if aux_out is not None else None, N, st.cuda_stream)
            e1.record(st)
            e1.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        fl = 2.0 * M * N * K
        res[name] = {"M": M, "N": N, "K": K, "ms": ms, "tflops": fl / ms / 1e9}
        tot_fl += fl
        tot_ms += ms
        print(f"{name:8s} M={M:6d} N={N:6d} K={K:6d} {ms:8.3f} ms {fl / ms / 1e9:7.1f} TF/s", flush=True)
        del A, Bm, C, aux_in, aux_out
    res["total"] = {"ms": tot_ms, "tflops": tot_fl / tot_ms / 1e9}
    print("total", res["total"])
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
