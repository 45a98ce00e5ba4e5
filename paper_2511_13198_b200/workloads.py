"""The paper's own models (Table 4) on one B200 — SURVEY §8(f) NEXT-3.

  BERT   h = 1024,  n = 16 (d = 64),  L/node = 24, bidirectional (non-causal)
  LLaMA  h = 8192,  n = 64 (d = 128), L/node = 8
  GPT    h = 12288, n = 96 (d = 128), L/node = 8
  FFN 4h GELU for all (reading R-5), bf16, b = 1.

The Llama variant (NEXT-3, readings R-GQA / R-SWIGLU) at the paper's LLaMA width:
  LLaMA-GQA  h = 8192, n = 64, n_kv = 8, SwiGLU F = 28672 (the Llama-2-70B block), L/node = 8
  Llama3-8B  h = 4096, n = 32, n_kv = 8, SwiGLU F = 14336, L/node = 32
(model FLOPs per token: 3 [2 (h (n + 2 n_kv) d + h^2 + 3 h F) + 2 s h] causal.)

Per model: (1) device-timed tokens/s of one layer fwd + bwd per strategy at a few
sequence lengths (the same kernels and C ABI as the 7B bench; CUDA events, L2 flushed);
(2) the OOM frontier of the L/node stack per uniform strategy, from the exact memory
model (pds_mem_bytes, Eq. 6 with reading R-22) against this device's free memory, each
confirmed by running the stack at the predicted maximum.

  python -m paper_2511_13198_b200.workloads --out profiles/x.json
"""
from __future__ import annotations

import argparse
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
MODELS = {
    "BERT": dict(h=1024, n=16, L=24, causal=0),
    "LLaMA": dict(h=8192, n=64, L=8, causal=1),
    "GPT": dict(h=12288, n=96, L=8, causal=1),
    "LLaMA-GQA": dict(h=8192, n=64, L=8, causal=1, n_kv=8, ffn=28672, act=1),
    "Llama3-8B": dict(h=4096, n=32, L=32, causal=1, n_kv=8, ffn=14336, act=1),
}


def layer_flops(cfg, s):
    """Model FLOPs of one layer fwd + bwd at length s (3 x forward; attention causal
    counts the lower triangle)."""
    h, n = cfg["h"], cfg["n"]
    nk, F = cfg.get("n_kv", n), cfg.get("ffn", 4 * h)
    lin = 2 * (h * (n + 2 * nk) * (h // n) + h * h + (3 if cfg.get("act") else 2) * h * F)
    att = (2 if cfg["causal"] else 4) * s * h
    return 3 * (lin + att) * s


def main():
    import torch
    from . import binding as B
    from .calibrate import make_layer_buffers
    from .frontier import predicted_bytes, run_stack
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", nargs="+", default=list(MODELS))
    ap.add_argument("--seqs", type=int, nargs="+", default=[4096, 16384])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--step", type=int, default=8192)
    ap.add_argument("--reserve-gb", type=float, default=4.0)
    ap.add_argument("--no-frontier", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    res = {"P": 1, "models": {}}
    for name in a.models:
        cfg = MODELS[name]
        h, n, L = cfg["h"], cfg["n"], cfg["L"]
        F = cfg.get("ffn", 4 * h)
        model = B.Model(h=h, n_heads=n, ffn=F, n_layers=L, causal=cfg["causal"], n_kv_heads=cfg.get("n_kv", 0),
                        ffn_act=cfg.get("act", 0))
        out = {"h": h, "n": n, "n_kv": cfg.get("n_kv", n), "ffn": F, "act": "swiglu" if cfg.get("act") else "gelu",
               "L_per_node": L, "causal": cfg["causal"], "layer": [], "frontier": {}}
        # (1) one layer fwd + bwd per strategy
        for s in a.seqs:
            w, gr, x, dy = make_layer_buffers(torch, model, 1, s, seed=3)
            W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
            G = B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))
            y, dx = torch.empty_like(x), torch.empty_like(x)
            ctx = B.Context(model)
            for pi, pname in ((0, "MegatronTS"), (1, "UlyssesZ"), (2, "METP")):
                times = []
                for r in range(a.reps + 1):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st.cuda_stream)
                    ctx.layer_bwd(pi, dy.data_ptr(), sv, W, G, dx.data_ptr(), st.cuda_stream)
                    e1.record(st)
                    e1.synchronize()
                    if r:
                        times.append(e0.elapsed_time(e1) / 1e3)
                t = min(times)
                flops = layer_flops(cfg, s)
                rec = {"s": s, "strategy": pname, "seconds": t, "tokens_per_s": s / t,
                       "model_tflops": flops / t / 1e12}
                out["layer"].append(rec)
                print(name, json.dumps(rec), flush=True)
            ctx.close()
            del w, gr, x, dy, y, dx
            torch.cuda.empty_cache()
        # (2) OOM frontier of the L/node stack, per uniform strategy
        if not a.no_frontier:
            ctx = B.Context(model)
            layers, keep = [], []
            for li in range(L):
                w, gr, _, _ = make_layer_buffers(torch, model, 1, 128, seed=li)
                keep.append((w, gr))
                layers.append((B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out",
                                                                          "g1", "g2"))),
                               B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out",
                                                                         "dg1", "dg2")))))
            torch.cuda.synchronize()
            free = torch.cuda.mem_get_info()[0]
            pers = L * B.mem_bytes(model, 1, 0, 1024)[2]
            cap = float(free) - a.reserve_gb * 2 ** 30 + pers
            for pi, pname in ((0, "MegatronTS"), (1, "UlyssesZ"), (2, "METP")):
                s, best = a.step, 0
                while s <= 1 << 20:
                    tot, ws = predicted_bytes(B, model, 1, [pi] * L, s)
                    if tot + ws >= cap:
                        break
                    best = s
                    s += a.step
                entry = {"predicted_max_s": best}
                if best:
                    try:
                        t = run_stack(torch, B, ctx, model, [pi] * L, best, layers)
                        entry["run_at_max"] = {"ok": True, "seconds": t, "tokens_per_s_per_layer": best * L / t}
                    except (B.PdsError, torch.OutOfMemoryError) as e:
                        entry["run_at_max"] = {"ok": False, "error": str(e)[:160]}
                        ctx.release_cache()
                        torch.cuda.empty_cache()
                out["frontier"][pname] = entry
                print(name, pname, json.dumps(entry), flush=True)
            ctx.close()
            del layers, keep
            torch.cuda.empty_cache()
        res["models"][name] = out
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
