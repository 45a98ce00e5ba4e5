"""Cost-model calibration: profile -> fit -> export bundle.

1. Profile: device-timed fwd+bwd of ONE layer (R-31) per strategy over a
   geometric grid of sequence lengths, CUDA events on the launching stream,
   median of `reps` after warm-up, through the C ABI (pds_layer_fwd/bwd).
2. Fit per strategy: a RandomForestRegressor (n_estimators=50,
   max_depth=10, random_state=42) on features
   one-hot(strategy) + normalised (h, n, L) + normalised s, and a polynomial of
   degree 1..3 chosen by AIC in x = s / s_max (R-26).
3. Export the "pds_bundle 1" text file read by pds_load_costs (Eq. 9 dispatch:
   RF iff s <= s_profile_max, else PR).

For P > 1 on a single-GPU box the profile is MODELLED: the per-rank compute of
each strategy is measured on one GPU at the per-rank shapes through the
loopback group, and the collective time is its byte count (oracle-independent
formula of DESIGN.md §Comm) over the measured NVLink peer bandwidth (770 GB/s,
B200_PROFILING.md), minus what the tile-overlapped MegatronTS / METP collectives
hide under their GEMMs.  The bundle header records which.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BUNDLES = os.path.join(HERE, "bundles")
ALL = (0, 1, 2, 3, 4, 5)    # TS, UZ, METP, CZ, METP-full, ColossalZ (include/paradyse.h)


def fits(torch, B, model, pi, s, P=1):
    """One layer of strategy pi at length s fits on this device (ColossalZ's quadratic
    score matrix limits its profiled range; the other strategies fit the whole grid)."""
    try:
        sv, ws, pers = B.mem_bytes(model, P, pi, s)
    except B.PdsError:                 # not valid at this length (R-15 divisibility)
        return False
    free, _ = torch.cuda.mem_get_info()
    return sv + ws + pers < 0.85 * free


S_EXTRAP_MAX = float(1 << 20)    # longest length the bundles extrapolate to (> 624K, Q-16)


def monotone(c, x0, x1):
    """The polynomial (numpy order) is non-decreasing on [x0, x1]: derivative >= 0 at
    both ends and at every real critical point of the derivative inside."""
    d = np.polyder(c)
    pts = [x0, x1] + [float(r.real) for r in np.roots(np.polyder(d)) if abs(r.imag) < 1e-12 and x0 < r.real < x1] \
        if len(d) > 1 else [x0, x1]
    return all(np.polyval(d, t) >= 0 for t in pts)


PR_DEGREES = (1, 2)


def aic_poly(s, y, degrees=PR_DEGREES):
    """Least squares in x = s / s_max, degree by AIC = n ln(max(RSS/n, 1e-12 var y)) + 2k.
    Reading R-26b: of the paper's optional orders 1..3 only those up to
    the layer's complexity order are candidates (time is O(s^2); O-7:
    72h^2 s + 6hs^2 flops), and a fit that is not non-decreasing on [min s,
    S_EXTRAP_MAX] is not admissible (a layer cannot get faster as s grows; PR only
    extrapolates).  If no degree is admissible, the line with its slope clamped at 0."""
    s = np.asarray(s, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    scale = float(s.max())
    x = s / scale
    best = None
    for deg in degrees:
        if len(np.unique(x)) < deg + 1:
            continue
        c = np.polyfit(x, y, deg)
        if not monotone(c, float(x.min()), S_EXTRAP_MAX / scale):
            continue
        rss = float(np.sum((np.polyval(c, x) - y) ** 2))
        n = len(y)
        floor = 1e-12 * float(np.var(y)) if np.var(y) > 0 else 1e-300
        a = n * math.log(max(rss / n, floor)) + 2 * (deg + 1)
        if best is None or a < best[0] - 1e-12:
            best = (a, deg, c)
    if best is None:
        c = np.polyfit(x, y, 1)
        c[0] = max(c[0], 0.0)
        best = (None, 1, c)
    return best[1], best[2], scale


def fit_and_export(path, P, h, n, ffn, L, records, capacity, reserve, note="", n_kv=0, act=0):
    """records: {strategy: [(s, seconds), ...]} -> bundle file."""
    from sklearn.ensemble import RandomForestRegressor
    strategies = sorted(k for k in records if len(records[k]) >= 2)   # profiled (fits the device)
    all_s = [s for st in strategies for s, _ in records[st]]
    norm = [(h, h), (n, n), (L, L), (float(min(all_s)), float(max(all_s)))]

    def feats(pi, s):
        oh = [1.0 if e == pi else 0.0 for e in strategies]
        def nz(v, a, b):
            return 0.0 if a == b else (v - a) / (b - a)
        return oh + [nz(h, *norm[0]), nz(n, *norm[1]), nz(L, *norm[2]), nz(s, *norm[3])]

    variant = f" kv {n_kv} act {act}" if (n_kv and n_kv != n) or act else ""   # Llama variant only
    lines = ["pds_bundle 1",
             f"P {P} h {h} n {n} ffn {ffn} L {L} capacity {capacity!r} reserve {reserve!r}{variant}",
             "norm " + " ".join(f"{float(a)!r} {float(b)!r}" for a, b in norm),
             f"n_strat {len(strategies)}"]
    for pi in strategies:
        ss = np.array([s for s, _ in records[pi]], dtype=np.float64)
        ts = np.array([t for _, t in records[pi]], dtype=np.float64)
        X = np.array([feats(pi, s) for s in ss])
        rf = RandomForestRegressor(n_estimators=50, max_depth=10, random_state=42).fit(X, ts)
        deg, coef, scale = aic_poly(ss, ts)
        lines.append(f"strategy {pi} s_profile_max {float(ss.max())!r} poly {deg} {scale!r} "
                     + " ".join(repr(float(c)) for c in coef))
        lines.append(f"trees {len(rf.estimators_)}")
        for est in rf.estimators_:
            tr = est.tree_
            lines.append(f"tree {tr.node_count}")
            for i in range(tr.node_count):
                lines.append(f"{int(tr.feature[i])} {float(tr.threshold[i])!r} {int(tr.children_left[i])} "
                             f"{int(tr.children_right[i])} {float(tr.value[i].ravel()[0])!r}")
    lines.append("end")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(path + ".json", "w") as f:
        json.dump({"P": P, "h": h, "n": n, "ffn": ffn, "L": L, "n_kv": n_kv, "act": act, "note": note,
                   "records": {str(k): v for k, v in records.items()}}, f, indent=1)
    return path


def refit(path):
    """Re-export a bundle from the profile records stored beside it (no GPU): the RF
    (seed 42) and the PR fit are deterministic functions of the records."""
    import re
    meta = json.load(open(path + ".json"))
    hdr = open(path).readline() and open(path).read().splitlines()[1]
    cap = float(re.search(r"capacity ([0-9.eE+-]+)", hdr).group(1))
    res = float(re.search(r"reserve ([0-9.eE+-]+)", hdr).group(1))
    records = {int(k): [tuple(r) for r in v] for k, v in meta["records"].items()}
    return fit_and_export(path, meta["P"], meta["h"], meta["n"], meta["ffn"], meta["L"], records, cap, res,
                          note=meta.get("note", ""), n_kv=meta.get("n_kv", 0), act=meta.get("act", 0))


# ------------------------------------------------------------------ profiling (GPU)
def make_layer_buffers(torch, model, P, s, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    h, F = model.h, model.ffn
    sl = s // P
    def rn(*shape, std=1.0):
        return (torch.randn(*shape, generator=g, device="cuda") * std).to(torch.bfloat16)
    n, nk = model.n_heads, (getattr(model, "n_kv_heads", 0) or model.n_heads)
    qrows = (n + 2 * nk) * (h // n) // P                      # GQA: (n + 2 n_kv) d / P
    frows = (2 if getattr(model, "ffn_act", 0) == 1 else 1) * F // P   # SwiGLU: [gate | up]
    w = dict(w_qkv_t=rn(qrows, h, std=h ** -0.5), w_proj=rn(h // P, h, std=h ** -0.5),
             w_in_t=rn(frows, h, std=h ** -0.5), w_out=rn(F // P, h, std=F ** -0.5),
             g1=(1 + 0.1 * torch.randn(h, generator=g, device="cuda")).to(torch.bfloat16),
             g2=(1 + 0.1 * torch.randn(h, generator=g, device="cuda")).to(torch.bfloat16))
    gr = {k: torch.zeros(v.shape, dtype=torch.float32, device="cuda") for k, v in
          (("dw_qkv_t", w["w_qkv_t"]), ("dw_proj", w["w_proj"]), ("dw_in_t", w["w_in_t"]),
           ("dw_out", w["w_out"]), ("dg1", w["g1"]), ("dg2", w["g2"]))}
    x = rn(sl, h)
    dy = rn(sl, h)
    return w, gr, x, dy


def time_layer(torch, B, ctx, pi, s, w, gr, x, dy, reps=5, warm=2):
    st = torch.cuda.current_stream()
    W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
    G = B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    ts = []
    for i in range(warm + reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        sv = ctx.layer_fwd(pi, s, x.data_ptr(), W, y.data_ptr(), st.cuda_stream)
        ctx.layer_bwd(pi, dy.data_ptr(), sv, W, G, dx.data_ptr(), st.cuda_stream)
        b.record(st)
        b.synchronize()
        if i >= warm:
            ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def comm_bytes_per_rank(pi, h, F, s, P, n=None, n_kv=None, act=0):
    """Bytes each rank moves per layer fwd+bwd (ring payload (P-1)/P x full).  Llama variant:
    GQA narrows the K / V blocks to n_kv d (Q|K|V width h + 2 n_kv d), SwiGLU weighs 3hF."""
    if P == 1:
        return 0.0
    fr = (P - 1) / P
    act_b = s * h * 2
    hk = h if not n or not n_kv else n_kv * (h // n)
    qw = h + 2 * hk
    if pi in (0, 2):
        return 10 * fr * act_b + 2 * fr * 8 * h
    if pi == 4:              # METP-full: TS bytes + one more AG(u) for the Q/K/V recompute
        return 11 * fr * act_b + 2 * fr * 8 * h
    wb = qw * h + h * h + (3 if act else 2) * h * F
    if pi == 3:              # CZ (R-CZ): zigzag exchanges + K/V ring (bf16) + dK/dV ring (fp32), ZeRO3 weights
        return cz_zig_bytes(h, s, P, qw) + cz_ring_bytes(hk, s, P) + fr * wb * (2 + 2 + 4) + 2 * fr * 8 * h
    if pi == 5:              # ColossalZ (RSA): K, V rings fwd + V, K rings bwd (bf16), dV, dK rings (fp32)
        kb = (s // P) * hk
        return 4 * (P - 1) * kb * 2 + 2 * P * kb * 4 + fr * wb * (2 + 2 + 4) + 2 * fr * 8 * h
    a2a = 2 * fr * (s // P) * (qw + h) * 2
    return a2a + fr * wb * (2 + 2 + 4) + 2 * fr * 8 * h


def cz_zig_bytes(h, s, P, qw=None):
    """MegatronCZ's boundary <-> zigzag point-to-point exchanges per rank per layer (mean):
    QKV and O (fwd), O, dO and dQKV (bwd); a half-chunk moves unless its zigzag owner is
    its boundary owner (layer.cpp zig_exchange).  qw: the Q|K|V width (3h for MHA)."""
    qw = 3 * h if qw is None else qw
    moved = sum(1 for j in range(2 * P) if (j if j < P else 2 * P - 1 - j) != j // 2)
    return moved * (s // (2 * P)) * (2 * qw + 3 * h) * 2 / P


def cz_ring_bytes(hk, s, P):
    """K/V ring passes (P - 1 fwd, P - 1 bwd, bf16) and the dK/dV accumulator ring (P, fp32);
    hk = the K (V) width (h for MHA)."""
    kv = (s // P) * 2 * hk
    return 2 * (P - 1) * kv * 2 + P * kv * 4


def class_seconds(torch, B, ctx, pi, s, w, gr, x, dy, classes):
    """Device time of the kernels of the given profiler classes (0 GEMM, 1 attention
    fwd, 2 attention bwd, 3 norm / elementwise) in one layer fwd + bwd."""
    ctx.profile(True)
    ctx.profile_reset()
    time_layer(torch, B, ctx, pi, s, w, gr, x, dy, reps=1, warm=0)
    ms = sum(ctx.profile_read(k)["ms"] for k in classes)
    ctx.profile(False)
    return ms / 1e3


def bundle_name(h, n, ffn, P, n_kv=0, act=0):
    var = (f"_kv{n_kv}" if n_kv and n_kv != n else "") + ("_swiglu" if act else "")
    return f"h{h}_n{n}{var}_f{ffn}_P{P}.txt"


def profile(P_target, h, n, ffn, L, grid, out_dir=BUNDLES, reps=5, link_gbs=770.0, n_kv=0, act=0):
    import torch
    from . import binding as B
    model = B.Model(h=h, n_heads=n, ffn=ffn, n_layers=L, n_kv_heads=n_kv, ffn_act=act)
    records = {pi: [] for pi in ALL}
    if P_target == 1:
        ctx = B.Context(model)
        for s in grid:
            w, gr, x, dy = make_layer_buffers(torch, model, 1, s)
            run = [pi for pi in ALL if fits(torch, B, model, pi, s)]
            # strategies interleaved rep by rep (one warm-up pass each first), so slow drift
            # of the power-capped clock does not favour whichever strategy runs last
            for pi in run:
                time_layer(torch, B, ctx, pi, s, w, gr, x, dy, reps=1, warm=1)
                ctx.release_cache()
            ts = {pi: [] for pi in run}
            for _ in range(reps):
                for pi in run:
                    ts[pi].append(time_layer(torch, B, ctx, pi, s, w, gr, x, dy, reps=1, warm=0))
            for pi in run:
                t = float(np.median(ts[pi]))
                records[pi].append((int(s), t))
                print(f"P=1 s={s} pi={pi} t={t * 1e3:.3f} ms", flush=True)
            del w, gr, x, dy
            torch.cuda.empty_cache()
        ctx.close()
        note = "measured: device-timed one-layer fwd+bwd on 1 B200"
    else:
        # modelled: per-rank compute measured at the per-rank shapes (TS: s tokens for
        # the column/row-parallel GEMMs; UZ: s/P local tokens + full-s attention over
        # n/P heads; METP: TS compute + waves) on a 1-rank context whose layer runs the
        # same kernels, then collective bytes / link bandwidth added.
        ctx = B.Context(model)
        ctx_m = B.Context(B.Model(h=h, n_heads=n, ffn=ffn, n_layers=L, metp_chunks=P_target, n_kv_heads=n_kv,
                                  ffn_act=act))
        for s in grid:
            t_unit, t_gemm = {}, {}
            t_att = 0.0
            for pi in [q for q in ALL if fits(torch, B, ctx_m.model if q in (2, 4) else model, q, s)]:
                w, gr, x, dy = make_layer_buffers(torch, model, 1, s)
                cx = ctx_m if pi in (2, 4) else ctx
                t1 = time_layer(torch, B, cx, pi, s, w, gr, x, dy, reps=reps)
                t_unit[pi] = t1
                t_gemm[pi] = class_seconds(torch, B, cx, pi, s, w, gr, x, dy, (0,))
                if pi == 3:
                    t_att = class_seconds(torch, B, ctx, pi, s, w, gr, x, dy, (1, 2))
                del w, gr, x, dy
                cx.release_cache()
            torch.cuda.empty_cache()
            for pi in t_unit:
                comp = t_unit[pi] / P              # CZ: zigzag placement, every rank 1/P of the attention
                comm = comm_bytes_per_rank(pi, h, ffn, s, P, n, n_kv, act) / (link_gbs * 1e9)
                if pi == 3:
                    # the K/V ring passes run on the side stream under the ring step's
                    # attention (P steps of 1/P^2 of it each); the rest stays exposed
                    hk = h if not n_kv else n_kv * (h // n)
                    ring = 2 * (P - 1) * (s // P) * 2 * hk * 2 / (link_gbs * 1e9)
                    comm -= min(ring, t_att / P * (P - 1) / P)
                if pi in (0, 2, 4):
                    # tile-overlapped AG / RS: each runs under the GEMM that
                    # consumes / produces it (those GEMMs carry 48h^2 of the 72h^2 GEMM
                    # flops per token); at least one chunk per collective stays exposed
                    comm = max(comm / P, comm - (2.0 / 3.0) * t_gemm[pi] / P)
                extra = (2 * P - 1) * 8e-6 * (P if pi in (2, 4) else 1)   # collective launch latency
                if pi in (3, 5):
                    extra += 6 * 8e-6 * (P - 1)                           # part-wise weight AG / RS
                records[pi].append((int(s), comp + comm + extra))
        ctx.close()
        ctx_m.close()
        note = (f"modelled for P={P_target}: P=1 device time / P + comm bytes / {link_gbs} GB/s "
                "(+ per-collective latency; TS / METP: minus the share hidden under the tile-overlapped "
                "GEMMs, at least one chunk per collective exposed; CZ: zigzag-balanced ring attention, its K/V "
                "ring passes hidden under the ring steps' attention); replace with a measured profile on an "
                "8xB200 box")
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, bundle_name(h, n, ffn, P_target, n_kv, act))
    cap = float(torch.cuda.get_device_properties(0).total_memory)
    fit_and_export(path, P_target, h, n, ffn, L, records, capacity=cap, reserve=8.0 * 2 ** 30, note=note,
                   n_kv=n_kv, act=act)
    return path


def profile_measured(h, n, ffn, L, grid, out_dir=BUNDLES, reps=3):
    """P > 1 MEASURED: run under torchrun with one rank per GPU (WORLD_SIZE = P), e.g.
      python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \
          -m paper_2511_13198_b200.calibrate --measured
    Every rank runs the strategy's layer fwd + bwd on its [s/P, h] shard over NCCL;
    the layer time is the max over ranks of the device-timed median (CUDA events on
    the launching stream).  Rank 0 fits and exports the bundle."""
    import torch
    import torch.distributed as dist
    from . import binding as B
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [B.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    model = B.Model(h=h, n_heads=n, ffn=ffn, n_layers=L)
    ctx = B.Context(model, P=P, rank=rank, device=local, uid=obj[0])
    records = {pi: [] for pi in ALL}
    for s in grid:
        if s % (P * 128) or (s // P) % (P * 128):
            continue                                  # METP waves need s/(P c) % 128 == 0, c = P
        w, gr, x, dy = make_layer_buffers(torch, model, P, s, seed=1 + rank)
        ok = torch.tensor([1.0 if fits(torch, B, model, pi, s, P) else 0.0 for pi in ALL], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)            # every rank runs the same set
        run = [pi for i, pi in enumerate(ALL) if ok[i] > 0]
        for pi in run:
            time_layer(torch, B, ctx, pi, s, w, gr, x, dy, reps=1, warm=1)
            ctx.release_cache()
        ts = {pi: [] for pi in run}
        for _ in range(reps):
            for pi in run:
                ts[pi].append(time_layer(torch, B, ctx, pi, s, w, gr, x, dy, reps=1, warm=0))
        med = torch.tensor([float(np.median(ts[pi])) for pi in run], dtype=torch.float64, device="cuda")
        dist.all_reduce(med, op=dist.ReduceOp.MAX)
        for i, pi in enumerate(run):
            records[pi].append((int(s), float(med[i])))
        if rank == 0:
            print(f"P={P} s={s} " + " ".join(f"pi{pi}={float(med[i]) * 1e3:.3f}ms" for i, pi in enumerate(run)),
                  flush=True)
        del w, gr, x, dy
        torch.cuda.empty_cache()
    ctx.close()
    path = None
    if rank == 0:
        os.makedirs(out_dir, exist_ok=True)
        path = os.path.join(out_dir, f"h{h}_n{n}_f{ffn}_P{P}.txt")
        cap = float(torch.cuda.get_device_properties(local).total_memory)
        fit_and_export(path, P, h, n, ffn, L, records, capacity=cap, reserve=8.0 * 2 ** 30,
                       note=f"measured: device-timed one-layer fwd+bwd on {P} B200 over NCCL, max over ranks")
    dist.barrier()
    dist.destroy_process_group()
    return path


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, nargs="+", default=[1])
    ap.add_argument("--h", type=int, default=4096)
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--ffn", type=int, default=16384)
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--kv", type=int, default=0, help="GQA key/value heads (Llama variant; 0: MHA)")
    ap.add_argument("--act", type=int, default=0, help="1: SwiGLU FFN (Llama variant)")
    # four lengths per octave, 1K..64K, multiples of 256 (every strategy valid at P = 1):
    # the random forest interpolates between profiled lengths only (Eq. 9), and with one
    # point per octave its piecewise-constant predictions misranked near-equal strategies
    ap.add_argument("--grid", type=int, nargs="+",
                    default=sorted({int(round(1024 * 2 ** (i / 4) / 256)) * 256 for i in range(25)}))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--measured", action="store_true", help="P = WORLD_SIZE ranks under torchrun, over NCCL")
    ap.add_argument("--refit", action="store_true", help="re-fit the committed bundles from their stored records (CPU)")
    a = ap.parse_args()
    if a.refit:
        for P in a.P:
            print(refit(os.path.join(BUNDLES, bundle_name(a.h, a.n, a.ffn, P, a.kv, a.act))))
        raise SystemExit(0)
    if a.measured:
        grid = a.grid if a.grid != ap.get_default("grid") else [8192, 16384, 32768, 65536, 131072]
        print(profile_measured(a.h, a.n, a.ffn, a.L, grid, reps=a.reps))
        raise SystemExit(0)
    for P in a.P:
        t0 = time.time()
        print(profile(P, a.h, a.n, a.ffn, a.L, a.grid, reps=a.reps, n_kv=a.kv, act=a.act), f"{time.time() - t0:.1f}s")
