"""Long-sequence single-layer comparison ("UZ vs METP: tokens/s, peak
memory") and a check of the exact memory model at scale.

For each strategy and each s: one layer fwd + bwd through the C ABI, device-timed
(CUDA events, L2 flushed before), and the library's device memory measured with
cudaMemGetInfo after the forward (saved arena + workspace, the layer's peak: the
backward allocates nothing new) against pds_mem_bytes' saved + transient (reading
R-22: the memory model is the buffer plan itself).  The model's saved set includes
the layer input x, which the caller allocated before the measurement, and the
measurement includes the RoPE table, which the model leaves to the reserve.  On one GPU P = 1, so every
strategy's collectives are identities; the numbers show the compute / memory side
of the trade-off (UZ's full weights and fp32 dW workspace, METP's 6u saved set and
recompute).

  python -m paper_2511_13198_b200.longseq --seqs 65536 131072 --out profiles/x.json
"""
from __future__ import annotations

import argparse
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    import torch
    from . import binding as B
    from .calibrate import make_layer_buffers
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, nargs="+", default=[65536, 131072])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--strategies", default="0,1,2,3", help="subset of 0 (TS), 1 (UZ), 2 (METP), 3 (CZ)")
    ap.add_argument("--metp-recompute", type=int, default=0)
    ap.add_argument("--metp-chunks", type=int, default=0)
    a = ap.parse_args()
    H, N, F, P = 4096, 32, 16384, 1
    model = B.Model(h=H, n_heads=N, ffn=F, n_layers=1, metp_recompute=a.metp_recompute,
                    metp_chunks=a.metp_chunks)
    want = {int(x) for x in a.strategies.split(",")}
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    res = {"model": {"h": H, "n": N, "ffn": F, "metp_recompute": a.metp_recompute, "metp_chunks": a.metp_chunks},
           "P": P, "runs": []}
    for s in a.seqs:
        w, gr, x, dy = make_layer_buffers(torch, model, P, s, seed=7)
        W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
        G = B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))
        y, dx = torch.empty_like(x), torch.empty_like(x)
        for pi, name in ((0, "MegatronTS"), (1, "UlyssesZ"), (2, "METP"), (3, "MegatronCZ")):
            if pi not in want:
                continue
            ctx = B.Context(model)
            saved_b, trans_b, _ = B.mem_bytes(model, P, pi, s)
            torch.cuda.synchronize()
            free0 = torch.cuda.mem_get_info()[0]
            times = []
            measured = None
            for r in range(a.reps + 1):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st.cuda_stream)
                if r == 0:
                    torch.cuda.synchronize()
                    measured = free0 - torch.cuda.mem_get_info()[0]
                ctx.layer_bwd(pi, dy.data_ptr(), sv, W, G, dx.data_ptr(), st.cuda_stream)
                e1.record(st)
                e1.synchronize()
                if r > 0:
                    times.append(e0.elapsed_time(e1) / 1e3)
            t = min(times)
            rec = {"s": s, "strategy": name, "seconds": t, "tokens_per_s": s / t,
                   # model FLOPs of one causal layer fwd + bwd: s (72 h^2 + 6 s h) (SURVEY O-7)
                   "model_tflops": s * (72.0 * H * H + 6.0 * s * H) / t / 1e12,
                   "predicted_saved_bytes": saved_b, "predicted_transient_bytes": trans_b,
                   "predicted_total_bytes": saved_b + trans_b, "measured_library_bytes": measured,
                   "rope_table_bytes": s * (H // N // 2) * 8,
                   # the saved set of the model includes the layer input x (u bytes), which the
                   # caller holds (allocated before the measurement); the rope table is outside it
                   "caller_held_input_bytes": s * H * 2,
                   "measured_plus_input_minus_rope_over_predicted":
                       (measured + s * H * 2 - s * (H // N // 2) * 8) / (saved_b + trans_b)}
            res["runs"].append(rec)
            print(json.dumps(rec), flush=True)
            ctx.close()
            torch.cuda.empty_cache()
        del w, gr, x, dy, y, dx
        torch.cuda.empty_cache()
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
