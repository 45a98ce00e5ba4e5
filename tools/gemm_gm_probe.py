"""Long-K TN GEMMs of the 7B layer at s = 16K (FC2 / dV: K = F; dW: K = s) through
pds_k_gemm, for the CTA-pair raster band (PDS_GEMM_GM) under study: run under
`ncu --clock-control base --metrics gpu__time_duration.sum,dram__bytes_read.sum` per band.

  PDS_GEMM_GM=16 ncu ... python tools/gemm_gm_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2511_13198_b200 import binding as B
    st = torch.cuda.current_stream().cuda_stream
    for (M, N, K) in ((16384, 4096, 16384), (16384, 16384, 4096), (32768, 4096, 16384)):
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        Bm = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        B.k_gemm(A.data_ptr(), K, 0, Bm.data_ptr(), K, 0, M, N, K, C.data_ptr(), N, 0, stream=st)
        torch.cuda.synchronize()
        del A, Bm, C


if __name__ == "__main__":
    main()
