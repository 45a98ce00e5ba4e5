"""OOM frontier of an L-layer stack: static strategies vs the adaptive plan.

BASELINE.json's metric has two halves: tokens/s and the "max seq len before OOM".
For each static strategy (uniform plan) and for the adaptive plan of pds_plan
(Algorithm 1 over the calibrated bundle and the exact memory model, Eq. 6), this
tool (1) predicts the largest s (multiple of `step`) whose plan satisfies Eq. 6
on this device, then (2) runs the full L-layer forward + backward through the C
ABI at that s (must succeed) and at s + step (must fail with PDS_ENOMEM — the
library maps cudaErrorMemoryAllocation to PDS_ENOMEM instead of crashing).

  python -m paper_2511_13198_b200.frontier --L 32 --step 4096 --out profiles/x.json
"""
from __future__ import annotations

import argparse
import json
import os
import time

HERE = os.path.dirname(os.path.abspath(__file__))


def predicted_bytes(B, model, P, plan, s):
    tot = 0
    ws = 0
    for pi in plan:
        sv, tr, pers = B.mem_bytes(model, P, pi, s)
        tot += sv + pers
        ws = max(ws, tr)
    return tot, ws


def run_stack(torch, B, ctx, model, plan, s, layers, timed=True, release=True):
    """fwd through len(plan) layers then bwd; returns seconds or raises PdsError.
    release=False keeps the library's workspace and cached saved blocks (the saved
    arena frees its cache and retries when cudaMalloc fails, so this never causes a
    false OOM)."""
    st = torch.cuda.current_stream()
    h = model.h
    acts = [torch.randn(s, h, device="cuda", dtype=torch.bfloat16)]
    saves = []
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st)
    try:
        for li, pi in enumerate(plan):
            W, _ = layers[li]
            y = torch.empty_like(acts[-1])
            saves.append(ctx.layer_fwd(pi, s, acts[-1].data_ptr(), W, y.data_ptr(), st.cuda_stream))
            acts.append(y)
        d = torch.randn_like(acts[-1])
        for li in reversed(range(len(plan))):
            W, G = layers[li]
            dx = torch.empty_like(d)
            ctx.layer_bwd(plan[li], d.data_ptr(), saves[li], W, G, dx.data_ptr(), st.cuda_stream)
            saves[li] = None
            d = dx
        t1.record(st)
        t1.synchronize()
        return t0.elapsed_time(t1) / 1e3
    finally:
        for sv in saves:
            if sv is not None:
                ctx.saved_release(sv)
        del acts
        torch.cuda.synchronize()
        if release:                 # keep both caches for an immediate rerun at the same length
            ctx.release_cache()
            torch.cuda.empty_cache()


def main():
    import torch
    from . import binding as B
    from .calibrate import make_layer_buffers
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--step", type=int, default=4096)
    ap.add_argument("--smax", type=int, default=262144)
    ap.add_argument("--reserve-gb", type=float, default=4.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-run", action="store_true")
    ap.add_argument("--metp-recompute", type=int, default=0, help="0 = ffn, 1 = full (Q/K/V recomputed too)")
    ap.add_argument("--plans", default="MegatronTS,UlyssesZ,METP,MegatronCZ,METP-full,adaptive")
    a = ap.parse_args()
    H, N, F = 4096, 32, 16384
    P = 1
    model = B.Model(h=H, n_heads=N, ffn=F, n_layers=a.L, metp_recompute=a.metp_recompute)
    ctx = B.Context(model)
    bundle = os.path.join(HERE, "bundles", f"h{H}_n{N}_f{F}_P{P}.txt")
    ctx.load_costs(bundle)
    # layer weights / grads (persistent, counted by the memory model)
    layers = []
    for li in range(a.L):
        w, gr, _, _ = make_layer_buffers(torch, model, P, 128, seed=li)
        W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
        G = B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))
        layers.append((W, G, w, gr))
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    # capacity the plan must stay under: what is free now, minus a reserve for the
    # rope table, torch's allocator and the boundary activations' rounding
    cap = float(free) - a.reserve_gb * 2 ** 30
    pers = sum(B.mem_bytes(model, P, 0, 1024)[2] for _ in range(a.L))
    ctx.set_capacity(cap + pers, 0.0)   # the planner's M includes persistent bytes
    res = {"device_total_bytes": total, "free_after_weights": free, "capacity_for_plan": cap + pers,
           "L": a.L, "P": P, "model": {"h": H, "n": N, "ffn": F, "metp_recompute": a.metp_recompute},
           "step": a.step, "plans": {}}
    lay = [(W, G) for W, G, _, _ in layers]
    candidates = {"MegatronTS": [0] * a.L, "UlyssesZ": [1] * a.L, "METP": [2] * a.L, "MegatronCZ": [3] * a.L,
                  "METP-full": [4] * a.L, "adaptive": None}
    for name, fixed in candidates.items():
        if name not in a.plans.split(","):
            continue
        best = None
        s = a.step
        while s <= a.smax:
            if fixed is None:
                plan, flags = ctx.plan(s, a.L)
                feas = not (flags & B.PLAN_INFEASIBLE)
            else:
                plan = fixed
                tot, ws = predicted_bytes(B, model, P, plan, s)
                feas = tot + ws < cap + pers
            if not feas:
                break
            best = (s, list(plan))
            s += a.step
        entry = {"predicted_max_s": best[0] if best else 0,
                 "plan_at_max": "".join("TUMCFR"[p] for p in best[1]) if best else None}
        if best and not a.no_run:
            s_ok, plan = best
            try:
                t = run_stack(torch, B, ctx, model, plan, s_ok, lay)
                entry["run_at_max"] = {"ok": True, "seconds": t, "tokens_per_s_per_layer": s_ok * a.L / t}
            except B.PdsError as e:
                entry["run_at_max"] = {"ok": False, "error": str(e)}
            torch.cuda.empty_cache()
            # one step above: the planner's own choice there (adaptive) or the same uniform plan
            s_hi = s_ok + a.step
            plan_hi = plan if fixed is not None else ctx.plan(s_hi, a.L)[0]
            try:
                run_stack(torch, B, ctx, model, plan_hi, s_hi, lay)
                entry["run_above"] = {"s": s_hi, "ok": True}
            except B.PdsError as e:
                entry["run_above"] = {"s": s_hi, "ok": False, "error": str(e)[:120]}
            except torch.OutOfMemoryError as e:
                entry["run_above"] = {"s": s_hi, "ok": False, "error": "torch OOM (boundary activations)"}
            torch.cuda.empty_cache()
        res["plans"][name] = entry
        print(name, json.dumps(entry), flush=True)
    ctx.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
    return res


if __name__ == "__main__":
    main()
