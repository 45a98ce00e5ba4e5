"""Timeline of one dQ-kernel CTA (the one with the most key blocks) from a library built
with -DPDS_TRACE: per key block j, clock64 stamps of the MMA warp and of elementwise
warp 4 (see attn_bwd_dq4_kernel); prints per-phase durations in cycles.

  PDS_LIB=paper_2511_13198_b200/libparadyse_trace.so python tools/attn_trace.py --s 16384
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2511_13198_b200 import binding as B
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=16384)
    ap.add_argument("--kernel", default="dq", choices=["dq", "dkdv"])
    a = ap.parse_args()
    s, H, d = a.s, 32, 128
    hq = H * d
    qkv = (torch.randn(s, 3 * hq, device="cuda") * 0.5).to(torch.bfloat16)
    out = torch.empty(s, hq, device="cuda", dtype=torch.bfloat16)
    dout = torch.randn(s, hq, device="cuda").to(torch.bfloat16)
    lse = torch.empty(H, s, device="cuda", dtype=torch.float32)
    dqkv = torch.empty_like(qkv)
    B.k_attn_fwd(qkv.data_ptr(), 3 * hq, s, H, d, 1, out.data_ptr(), hq, lse.data_ptr(), 0)
    for _ in range(2):
        B.k_attn_bwd(qkv.data_ptr(), 3 * hq, out.data_ptr(), hq, lse.data_ptr(), dout.data_ptr(), s, H, d, 1,
                     dqkv.data_ptr(), 0)
    torch.cuda.synchronize()
    nkv = s // 128
    buf = np.zeros((nkv, 8), dtype=np.int64)
    B.call("pds_debug_trace", buf.ctypes.data_as(ctypes.c_void_p), nkv)
    t0 = buf[0, 7]
    names = ["mma: s_free ok", "mma: ds_full ok", "ew: s_full ok", "ew: S loaded", "ew: exps done",
             "ew: dp_full ok", "ew: ds stored", "mma: loop top"]
    if a.kernel == "dkdv":
        names[0] = "mma: p_full ok"
        names[4] = "ew: P stored"
    print("j  " + " | ".join(f"{n:>15s}" for n in names))
    for j in list(range(4)) + list(range(nkv // 2, nkv // 2 + 4)) + [nkv - 2]:
        print(f"{j:3d} " + " | ".join(f"{v - t0:15d}" for v in buf[j]))
    steady = buf[8:nkv - 2]
    per = np.diff(steady[:, 6])
    print("period (ds stored -> next ds stored): median", int(np.median(per)), "cycles")
    ph = {"S ready -> loaded (ew)": steady[:, 3] - steady[:, 2], "loaded -> exps done": steady[:, 4] - steady[:, 3],
          "exps done -> dP ready": steady[:, 5] - steady[:, 4], "dP ready -> dS stored": steady[:, 6] - steady[:, 5],
          "dS stored -> S(j+1) ready": steady[1:, 2] - steady[:-1, 6],
          "mma: ds_full -> next s_free": steady[1:, 0] - steady[:-1, 1]}
    for k, v in ph.items():
        print(f"{k:30s} median {int(np.median(v)):7d}")


if __name__ == "__main__":
    main()
