"""Dynamic-length training trace (configs[4]; the protocol of Figure 3)
and the ablation harness of Table 5.

Lengths are drawn from a Table 3 histogram (readings R-29/R-30),
padded to a multiple of 128·P (R-15), curriculum-sorted short to long
(PAPER.md:336), and each sequence runs forward + backward through an L-layer
stack with the plan pds_plan returns for its length (adaptive), or with a fixed
uniform plan (static baselines).  Records per sequence: s, plan, device time,
OOM.  A run ends at its first OOM ("curve termination indicates OOM
failure"); the adaptive planner stops *before* running when Eq. 6 has no
feasible plan (proactive OOM prediction).

--ablation runs ParaDySe (full) = all strategies, RF + PR cost model, smoothing
gamma = 0.05, and the variants w/o MegatronTS, w/o UlyssesZ, w/o
METP, w/o MegatronCZ (strategy set), w/o RF (PR everywhere: the bundle's s_profile_max set to 0,
Eq. 9), w/o Smoothing (gamma = 0), and reports Table 5's columns:
  Seq_len   = largest length trained before OOM,
  Time      = cumulative device time of the variant,
  Time_full = cumulative time of ParaDySe (full) up to that Seq_len,
  Saving    = (Time - Time_full) / Time.
"w/o METP" removes both METP variants (ffn and full recompute: one strategy of the
paper, two memory modes here).  Switching
statistics per run: plan changes between consecutive sequences and strategy
boundaries inside the plans.  --switch-cost measures a mixed plan's stack time
against the per-layer times of short uniform stacks at the same length.

--predict runs the same protocol WITHOUT a GPU on host-only planner contexts: every
sequence's per-layer times are the cost model's T_pi(s) (Eq. 9 on the committed bundle
of that P: measured at P = 1, modelled at P = 2, 4, 8 until an 8xB200 profile exists),
OOM is Eq. 6 on the library's exact memory plan against the bundle's per-GPU capacity,
and the output is labelled "predicted".  This is how the P > 1 rows of the north_star
(per-bucket tokens/s at 1/2/4/8 GPUs, the 624K adaptive frontier) are reported here.

  python -m paper_2511_13198_b200.trace --dataset grch38 --n 48 --L 32 --out profiles/t.json
  python -m paper_2511_13198_b200.trace --ablation --out profiles/ablation.json
  python -m paper_2511_13198_b200.trace --predict --P 8 --n 256 --gamma 0.05 --out profiles/p.json
"""
from __future__ import annotations

import argparse
import json
import os
import re
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
BUCKET_EDGES = [0, 4096, 8192, 16384, 32768, 65536, 131072, 1 << 40]


def bucket_of(s):
    for i in range(len(BUCKET_EDGES) - 1):
        if BUCKET_EDGES[i] <= s < BUCKET_EDGES[i + 1]:
            return i
    return len(BUCKET_EDGES) - 2


def pr_only_bundle(path):
    """Copy of a cost bundle whose Eq. 9 branch always takes the polynomial (w/o RF),
    in a temporary directory under the same file name (the name carries P)."""
    txt = open(path).read()
    txt = re.sub(r"s_profile_max [0-9.eE+-]+", "s_profile_max 0.0", txt)
    out = os.path.join(tempfile.mkdtemp(prefix="pds_pr_only_"), os.path.basename(path))
    with open(out, "w") as f:
        f.write(txt)
    return out


def switches(recs):
    plans = [r["plan"] for r in recs if "plan" in r]
    between = sum(1 for a, b in zip(plans, plans[1:]) if a != b)
    inside = sum(sum(1 for x, y in zip(p, p[1:]) if x != y) for p in plans)
    return {"plan_changes_between_sequences": between, "strategy_boundaries_inside_plans": inside}


def measure(torch, B, ctx, model, plan, s, layers, memo):
    """Device time of one fwd + bwd of the stack under `plan` at length s: an untimed
    warm-up pass (allocations of the saved arena / workspace at this length), then
    the timed pass.  Memoised on (s, plan): variants that choose the same plan for
    the same length share one measurement, so ablation deltas are not clock noise."""
    from .frontier import run_stack
    key = (s, tuple(plan))
    if key not in memo:
        run_stack(torch, B, ctx, model, plan, s, layers, release=False)
        memo[key] = run_stack(torch, B, ctx, model, plan, s, layers)
    return memo[key]


def run_trace(torch, B, ctx, model, lens, layers, L, fixed=None, memo=None):
    memo = {} if memo is None else memo
    recs, cum, oom_at = [], 0.0, None
    for s in lens:
        if fixed is None:
            plan, flags = ctx.plan(s, L)
            if flags & B.PLAN_INFEASIBLE:      # proactive OOM prediction
                oom_at = s
                recs.append({"s": s, "oom": True, "predicted": True})
                break
        else:
            plan, flags = [fixed] * L, 0
        try:
            t = measure(torch, B, ctx, model, plan, s, layers, memo)
        except (B.PdsError, torch.OutOfMemoryError):
            ctx.release_cache()
            torch.cuda.empty_cache()
            oom_at = s
            recs.append({"s": s, "oom": True})
            break
        cum += t
        recs.append({"s": s, "plan": "".join("TUMCFR"[p] for p in plan), "seconds": t, "cum": cum, "flags": flags})
    per_bucket = {}
    for r in recs:
        if r.get("oom"):
            continue
        b = bucket_of(r["s"])
        tok, sec = per_bucket.get(b, (0, 0.0))
        per_bucket[b] = (tok + r["s"] * L, sec + r["seconds"])
    return {"records": recs, "cumulative_s": cum, "oom_at": oom_at,
            "max_s_trained": max([r["s"] for r in recs if not r.get("oom")] + [0]),
            "tokens_per_s_per_layer_by_bucket": {str(k): v[0] / v[1] for k, v in per_bucket.items()},
            "switching": switches(recs)}


def common_bucket_table(runs, L):
    """Per Table 3 bucket, tokens/s per layer of every run over the sequences EVERY run
    completed (a static strategy that OOMs drops its longest sequences; comparing
    bucket rates over different sequence sets would favour it), and the adaptive
    plan's ratio to the best static strategy."""
    done = {n: {(i, r.get("real", r["s"])): r["seconds"] for i, r in enumerate(v["records"]) if "seconds" in r}
            for n, v in runs.items()}
    common = set.intersection(*[set(d) for d in done.values()])
    out = {}
    for b in sorted({bucket_of(k[1]) for k in common}):
        keys = [k for k in common if bucket_of(k[1]) == b]
        tps = {n: sum(k[1] for k in keys) * L / sum(done[n][k] for k in keys) for n in runs}
        statics = {n: v for n, v in tps.items() if n != "adaptive"}
        best = max(statics, key=statics.get)
        out[str(b)] = {"sequences": len(keys), "tokens_per_s_per_layer": tps, "best_static": best,
                       "adaptive_over_best_static": tps["adaptive"] / statics[best] if "adaptive" in tps else None}
    return out


def time_full_at(full, s_max):
    t = 0.0
    for r in full["records"]:
        if r.get("oom") or r["s"] > s_max:
            break
        t = r["cum"]
    return t


def switch_cost(torch, B, ctx, model, s, plan, layers, n_short=4):
    """Stack time of a mixed plan vs sum of per-layer times from short uniform stacks
    (every stack warmed up once at this length, then timed)."""
    memo = {}
    per_layer = {}
    for pi in sorted(set(plan)):
        t = measure(torch, B, ctx, model, [pi] * n_short, s, layers, memo)
        per_layer[pi] = t / n_short
    t_mixed = measure(torch, B, ctx, model, plan, s, layers, memo)
    pred = sum(per_layer[p] for p in plan)
    return {"s": s, "plan": "".join("TUMCFR"[p] for p in plan), "measured_s": t_mixed, "sum_of_layers_s": pred,
            "overhead": t_mixed / pred - 1.0,
            "per_layer_s": {"TUMCFR"[k]: v for k, v in per_layer.items()}}


STATIC = (("MegatronTS", 0), ("UlyssesZ", 1), ("METP", 2), ("MegatronCZ", 3), ("METP-full", 4), ("ColossalZ", 5))


def predict_trace(B, model, bundle, lens, L, gamma, fixed=None, real=None, mask=None):
    """The trace protocol on a host-only context: plan (adaptive) or the uniform plan
    (static), time = sum over layers of the bundle's T_pi(s), OOM = Eq. 6 infeasible.
    real[i]: the unpadded length of lens[i] (tokens/s counts real tokens, Q-15)."""
    real = lens if real is None else real
    ctx = B.Context(model, P=bundle_P(bundle), device=-1)
    ctx.load_costs(bundle)
    if fixed is not None:
        ctx.set_enabled(1 << fixed)
    elif mask is not None:
        ctx.set_enabled(mask)
    ctx.set_capacity(bundle_capacity(bundle), gamma if gamma > 0 else 1e-9)
    recs, cum, oom_at = [], 0.0, None
    for s, rs in zip(lens, real):
        try:
            plan, flags = ctx.plan(s, L)
        except B.PdsError as e:           # R-15: the strategy's divisibility does not hold at s
            recs.append({"s": s, "invalid": str(e)})
            continue
        if flags & B.PLAN_INFEASIBLE:
            oom_at = s
            recs.append({"s": s, "oom": True, "predicted": True})
            break
        t = ctx.cost_eval(s)[0]
        sec = sum(t[p] for p in plan)
        cum += sec
        recs.append({"s": s, "real": int(rs), "plan": "".join("TUMCFR"[p] for p in plan), "seconds": sec, "cum": cum,
                     "flags": flags})
    ctx.close()
    per_bucket = {}
    for r in recs:
        if "seconds" not in r:
            continue
        b = bucket_of(r["real"])
        tok, sec = per_bucket.get(b, (0, 0.0))
        per_bucket[b] = (tok + r["real"] * L, sec + r["seconds"])
    return {"records": recs, "cumulative_s": cum, "oom_at": oom_at,
            "max_s_trained": max([r["s"] for r in recs if "seconds" in r] + [0]),
            "tokens_per_s_per_layer_by_bucket": {str(k): v[0] / v[1] for k, v in per_bucket.items()},
            "switching": switches(recs)}


def predict_frontier(B, model, bundle, L, unit, fixed=None, s_max=1 << 20):
    """Largest multiple of `unit` up to s_max for which Eq. 6 has a feasible plan (the
    adaptive plan, or the uniform plan of strategy `fixed`): bisection, feasibility
    being monotone in s."""
    ctx = B.Context(model, P=bundle_P(bundle), device=-1)
    ctx.load_costs(bundle)
    if fixed is not None:
        ctx.set_enabled(1 << fixed)

    def ok(k):
        try:
            return not ctx.plan(k * unit, L)[1] & B.PLAN_INFEASIBLE
        except B.PdsError:
            return False
    lo, hi = 0, s_max // unit
    if ok(hi):
        lo = hi
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if ok(mid):
            lo = mid
        else:
            hi = mid
    plan = "".join("TUMCFR"[p] for p in ctx.plan(lo * unit, L)[0]) if lo else None
    ctx.close()
    return {"s": lo * unit, "plan": plan}


def bundle_P(path):
    return int(re.search(r"_P(\d+)\.txt$", path).group(1))


def bundle_capacity(path):
    """The per-GPU capacity the bundle was calibrated with, minus its reserve (Eq. 6)."""
    txt = open(path).read()
    cap = float(re.search(r"\bcapacity ([0-9.eE+-]+)", txt).group(1))
    m = re.search(r"\breserve ([0-9.eE+-]+)", txt)
    return cap - (float(m.group(1)) if m else 0.0)


def predict_ablation(B, model, bundle, lens, real, L):
    """Table 5 on the cost model: ParaDySe (full, gamma = 0.05) and the
    variants without one strategy, without RF (PR everywhere) and without smoothing."""
    ALL = (1 << B.N_STRATEGIES) - 1
    variants = [("ParaDySe (full)", dict(gamma=0.05)), ("w/o MegatronTS", dict(mask=ALL & ~1, gamma=0.05)),
                ("w/o MegatronCZ", dict(mask=ALL & ~8, gamma=0.05)), ("w/o UlyssesZ", dict(mask=ALL & ~2, gamma=0.05)),
                ("w/o ColossalZ", dict(mask=ALL & ~32, gamma=0.05)),
                ("w/o METP", dict(mask=ALL & ~4 & ~16, gamma=0.05)), ("w/o RF", dict(gamma=0.05, pr_only=True)),
                ("w/o Smoothing", dict(gamma=0.0))]
    runs = {}
    for name, kw in variants:
        path = pr_only_bundle(bundle) if kw.get("pr_only") else bundle
        runs[name] = predict_trace(B, model, path, lens, L, kw["gamma"], real=real, mask=kw.get("mask"))
    full = runs["ParaDySe (full)"]
    table = []
    for name, _ in variants:
        r = runs[name]
        tf = time_full_at(full, r["max_s_trained"])
        table.append({"framework": name, "seq_len": r["max_s_trained"], "time_s": r["cumulative_s"], "time_full_s": tf,
                      "saving": None if name.endswith("(full)") or r["cumulative_s"] == 0
                      else (r["cumulative_s"] - tf) / r["cumulative_s"],
                      "switching": r["switching"]})
    return table


def predict_main(a):
    import sys
    sys.path.insert(0, ROOT)
    from synth import pad_to, sample_lengths
    from . import binding as B
    H, N, F = a.h, a.heads, a.ffn           # default configs[1]'s 7B layer; --h 12288 --heads 96 --ffn 49152 --L 8:
    model = B.Model(h=H, n_heads=N, ffn=F, n_layers=a.L,    # the paper's GPT of Table 4 / Table 5; --kv / --act:
                    n_kv_heads=a.kv, ffn_act=a.act)         # the Llama variant
    out = {"mode": "predicted (cost model + exact memory plan on host-only contexts; no device run)",
           "model": {"h": H, "n_heads": N, "ffn": F, "L": a.L, "n_kv": a.kv or N,
                     "act": "swiglu" if a.act else "gelu"},
           "dataset": a.dataset, "n": a.n, "L": a.L, "gamma": a.gamma, "by_P": {}}
    raw = sample_lengths(a.dataset, a.n, seed=42)
    for P in a.P:
        from .calibrate import bundle_name
        bundle = os.path.join(HERE, "bundles", bundle_name(H, N, F, P, a.kv, a.act))
        # pad to a multiple every strategy accepts (R-15; METP's c = P waves of 128 rows:
        # 128 P^2), curriculum order
        unit = max(128 * P * P, 256 * P)
        real = sorted(int(x) for x in raw)
        lens = [int(pad_to(x, unit)) for x in real]
        meta = json.load(open(bundle + ".json"))
        runs = {"adaptive": predict_trace(B, model, bundle, lens, a.L, a.gamma, real=real)}
        for name, pi in STATIC:
            runs[name] = predict_trace(B, model, bundle, lens, a.L, 0.0, fixed=pi, real=real)
        frontier = {"adaptive": predict_frontier(B, model, bundle, a.L, unit)}
        for name, pi in STATIC:
            frontier[name] = predict_frontier(B, model, bundle, a.L, unit, fixed=pi)
        entry = {"bundle": os.path.basename(bundle), "bundle_note": meta.get("note", "measured"),
                 "capacity_bytes": bundle_capacity(bundle), "pad_unit": unit, "lengths": lens, "runs": runs,
                 "bucket_common": common_bucket_table(runs, a.L),
                 "max_s_trained": {n: r["max_s_trained"] for n, r in runs.items()},
                 "frontier_L_stack": frontier}
        if a.ablation:
            entry["table5"] = predict_ablation(B, model, bundle, lens, real, a.L)
            for row in entry["table5"]:
                print("  ", {k: row[k] for k in ("framework", "seq_len", "time_s", "saving")}, flush=True)
        out["by_P"][str(P)] = entry
        print(f"P={P}", "max_s", entry["max_s_trained"], flush=True)
        print("  frontier", {n: v["s"] for n, v in frontier.items()}, flush=True)
        for b, row in entry["bucket_common"].items():
            print("  bucket", b, row["sequences"], "adaptive / best static (%s) = %.4f"
                  % (row["best_static"], row["adaptive_over_best_static"]), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
    return out


def main():
    import sys
    if "--predict" in sys.argv:
        ap = argparse.ArgumentParser()
        ap.add_argument("--predict", action="store_true")
        ap.add_argument("--dataset", default="grch38")
        ap.add_argument("--n", type=int, default=256)
        ap.add_argument("--L", type=int, default=32)
        ap.add_argument("--P", type=int, nargs="+", default=[1, 2, 4, 8])
        ap.add_argument("--gamma", type=float, default=0.0)
        ap.add_argument("--ablation", action="store_true")
        ap.add_argument("--h", type=int, default=4096)
        ap.add_argument("--heads", type=int, default=32)
        ap.add_argument("--ffn", type=int, default=16384)
        ap.add_argument("--kv", type=int, default=0)
        ap.add_argument("--act", type=int, default=0)
        ap.add_argument("--out", default=None)
        return predict_main(ap.parse_args())
    sys.path.insert(0, ROOT)
    import torch
    from synth import pad_to, sample_lengths
    from . import binding as B
    from .calibrate import make_layer_buffers
    ap = argparse.ArgumentParser()
    ap.add_argument("--dataset", default="grch38")
    ap.add_argument("--n", type=int, default=48)
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--cap-s", type=int, default=163840, help="truncate sampled lengths (1 GPU)")
    ap.add_argument("--reserve-gb", type=float, default=4.0)
    ap.add_argument("--gamma", type=float, default=0.0)
    ap.add_argument("--ablation", action="store_true")
    ap.add_argument("--switch-cost", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    H, N, F, P = 4096, 32, 16384, 1
    model = B.Model(h=H, n_heads=N, ffn=F, n_layers=a.L)
    bundle = os.path.join(HERE, "bundles", f"h{H}_n{N}_f{F}_P{P}.txt")
    layers, keep = [], []
    for li in range(a.L):
        w, gr, _, _ = make_layer_buffers(torch, model, P, 128, seed=li)
        keep.append((w, gr))
        layers.append((B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2"))),
                       B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))))
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    pers = a.L * B.mem_bytes(model, P, 0, 1024)[2]
    cap = float(free) - a.reserve_gb * 2 ** 30 + pers
    lens = sample_lengths(a.dataset, a.n, seed=42)
    # pad to what every strategy accepts (R-15: 128 | s/P; MegatronCZ's zigzag: 128 | s/(2P))
    lens = sorted(min(int(pad_to(int(x), 256 * P)), a.cap_s) for x in lens)   # curriculum
    out = {"dataset": a.dataset, "n": a.n, "L": a.L, "P": P, "lengths": lens, "capacity_for_plan": cap, "runs": {}}

    ALL = (1 << B.N_STRATEGIES) - 1

    def context(mask=ALL, gamma=0.0, pr_only=False):
        ctx = B.Context(model)
        ctx.load_costs(pr_only_bundle(bundle) if pr_only else bundle)
        ctx.set_enabled(mask)
        ctx.set_capacity(cap, gamma if gamma > 0 else 1e-9)
        return ctx

    out["timing"] = "per (s, plan): one untimed warm-up pass, then one timed fwd + bwd of the stack (memoised)"
    if a.ablation:
        variants = [("ParaDySe (full)", dict(gamma=0.05)), ("w/o MegatronTS", dict(mask=ALL & ~1, gamma=0.05)),
                    ("w/o MegatronCZ", dict(mask=ALL & ~8, gamma=0.05)),
                    ("w/o UlyssesZ", dict(mask=ALL & ~2, gamma=0.05)),
                    ("w/o METP", dict(mask=ALL & ~4 & ~16, gamma=0.05)),
                    ("w/o RF", dict(gamma=0.05, pr_only=True)), ("w/o Smoothing", dict(gamma=0.0))]
        out["gamma_full"] = 0.05
        memo = {}
        for name, kw in variants:
            ctx = context(**kw)
            out["runs"][name] = run_trace(torch, B, ctx, model, lens, layers, a.L, memo=memo)
            ctx.close()
            r = out["runs"][name]
            print(name, "cum %.1fs" % r["cumulative_s"], "max_s", r["max_s_trained"], r["switching"], flush=True)
        full = out["runs"]["ParaDySe (full)"]
        table = []
        for name, _ in variants:
            r = out["runs"][name]
            tf = time_full_at(full, r["max_s_trained"])
            table.append({"framework": name, "seq_len": r["max_s_trained"], "time_s": r["cumulative_s"],
                          "time_full_s": tf,
                          "saving": None if name.endswith("(full)") or r["cumulative_s"] == 0
                          else (r["cumulative_s"] - tf) / r["cumulative_s"]})
        out["table5"] = table
        for row in table:
            print(row, flush=True)
    else:
        memo = {}
        for name, fixed in (("adaptive", None), ("MegatronTS", 0), ("METP", 2), ("UlyssesZ", 1), ("MegatronCZ", 3),
                            ("METP-full", 4)):
            ctx = context(mask=ALL if fixed is None else 1 << fixed, gamma=a.gamma)
            out["runs"][name] = run_trace(torch, B, ctx, model, lens, layers, a.L, fixed, memo=memo)
            ctx.close()
            r = out["runs"][name]
            print(name, "cum %.1fs" % r["cumulative_s"], "oom_at", r["oom_at"], "max_s", r["max_s_trained"],
                  flush=True)
    if not a.ablation:
        out["bucket_common"] = common_bucket_table(out["runs"], a.L)
        for b, row in out["bucket_common"].items():
            print("bucket", b, row["sequences"], "adaptive / best static (%s) = %.4f"
                  % (row["best_static"], row["adaptive_over_best_static"]), flush=True)
    if a.switch_cost:
        ctx = context()
        mixed = None
        for s in reversed(lens):
            plan, flags = ctx.plan(s, a.L)
            if not flags & B.PLAN_INFEASIBLE and len(set(plan)) > 1:
                mixed = (s, plan)
                break
        if mixed:
            out["switch_cost"] = switch_cost(torch, B, ctx, model, mixed[0], mixed[1], layers)
            print("switch cost", out["switch_cost"], flush=True)
        ctx.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
