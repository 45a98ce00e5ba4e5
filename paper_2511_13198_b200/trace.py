"""Dynamic-length training trace (configs[4]; the protocol of Figure 3).

Lengths are drawn from a Table 3 histogram (readings R-29/R-30),
padded to a multiple of 128·P (R-15), curriculum-sorted short to long
(PAPER.md:336), and each sequence runs forward + backward through an L-layer
stack with the plan pds_plan returns for its length (adaptive), or with a fixed
uniform plan (static baselines).  Records per sequence: s, plan, device time,
OOM.  A static strategy's curve ends at its first OOM ("curve
termination indicates OOM failure").  Per Table 3 bucket: sum tokens / sum time.

  python -m paper_2511_13198_b200.trace --dataset grch38 --n 48 --L 32 --out profiles/t.json
"""
from __future__ import annotations

import argparse
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
BUCKET_EDGES = [0, 4096, 8192, 16384, 32768, 65536, 131072, 1 << 40]


def bucket_of(s):
    for i in range(len(BUCKET_EDGES) - 1):
        if BUCKET_EDGES[i] <= s < BUCKET_EDGES[i + 1]:
            return i
    return len(BUCKET_EDGES) - 2


def main():
    import sys
    sys.path.insert(0, ROOT)
    import torch
    from synth import pad_to, sample_lengths
    from . import binding as B
    from .calibrate import make_layer_buffers
    from .frontier import run_stack
    ap = argparse.ArgumentParser()
    ap.add_argument("--dataset", default="grch38")
    ap.add_argument("--n", type=int, default=48)
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--cap-s", type=int, default=131072, help="truncate sampled lengths (1 GPU)")
    ap.add_argument("--reserve-gb", type=float, default=4.0)
    ap.add_argument("--gamma", type=float, default=0.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    H, N, F, P = 4096, 32, 16384, 1
    model = B.Model(h=H, n_heads=N, ffn=F, n_layers=a.L)
    ctx = B.Context(model)
    ctx.load_costs(os.path.join(HERE, "bundles", f"h{H}_n{N}_f{F}_P{P}.txt"))
    layers = []
    keep = []
    for li in range(a.L):
        w, gr, _, _ = make_layer_buffers(torch, model, P, 128, seed=li)
        keep.append((w, gr))
        layers.append((B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2"))),
                       B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))))
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    pers = a.L * B.mem_bytes(model, P, 0, 1024)[2]
    ctx.set_capacity(float(free) - a.reserve_gb * 2 ** 30 + pers, max(a.gamma, 0.0) if a.gamma > 0 else 1e-9)
    lens = sample_lengths(a.dataset, a.n, seed=42)
    lens = sorted(min(int(pad_to(int(x), 128 * P)), a.cap_s) for x in lens)   # curriculum
    out = {"dataset": a.dataset, "n": a.n, "L": a.L, "P": P, "gamma": a.gamma, "lengths": lens, "runs": {}}
    for name, fixed in (("adaptive", None), ("MegatronTS", 0), ("METP", 2), ("UlyssesZ", 1)):
        recs, cum, oom_at = [], 0.0, None
        for s in lens:
            if fixed is None:
                plan, flags = ctx.plan(s, a.L)
                if flags & B.PLAN_INFEASIBLE:      # proactive OOM prediction
                    oom_at = s
                    recs.append({"s": s, "oom": True, "predicted": True})
                    break
            else:
                plan, flags = [fixed] * a.L, 0
            try:
                t = run_stack(torch, B, ctx, model, plan, s, layers)
            except (B.PdsError, torch.OutOfMemoryError) as e:
                oom_at = s
                recs.append({"s": s, "oom": True})
                break
            cum += t
            recs.append({"s": s, "plan": "".join("TUM"[p] for p in plan), "seconds": t, "cum": cum,
                         "flags": flags})
        per_bucket = {}
        for r in recs:
            if r.get("oom"):
                continue
            b = bucket_of(r["s"])
            tok, sec = per_bucket.get(b, (0, 0.0))
            per_bucket[b] = (tok + r["s"] * a.L, sec + r["seconds"])
        out["runs"][name] = {"records": recs, "cumulative_s": cum, "oom_at": oom_at,
                             "max_s_trained": max([r["s"] for r in recs if not r.get("oom")] + [0]),
                             "tokens_per_s_per_layer_by_bucket": {str(k): v[0] / v[1] for k, v in per_bucket.items()}}
        print(name, "cum %.1fs" % cum, "oom_at", oom_at, "max_s", out["runs"][name]["max_s_trained"], flush=True)
    ctx.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
