#!/usr/bin/env python
"""ParaDySe hot-path benchmark (driver contract).

Metric (BASELINE.json): tokens/s per layer, fwd+bwd, vs sequence length.
Workload at N = 1: configs[1] — Llama-style 7B layer (h=4096, n=32, d=128,
F=16384), bf16, seq 4K-32K.  One step = for each s in {4096, 8192, 16384, 32768}:
pds_plan(s) (Algorithm 1 on the calibrated bundle) + one layer fwd + bwd with
the planned strategy, through the C ABI.  value = sum tokens / sum device time
(max over ranks).  At N > 1 (torchrun) every rank holds an [s/N, 1, h] shard
and the layer runs with P = N over NCCL ("weak" in tokens per GPU is not the
case here: total work is fixed per s -> "strong").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, N_HEADS, FFN, L_STACK = 4096, 32, 16384, 32
SEQS = [4096, 8192, 16384, 32768]
METRIC = "tokens/s per layer fwd+bwd (7B layer, seq 4K-32K)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, idx):
        self.idx = idx
        self.p = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                out = ""
            for line in out.strip().splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9:
                    self.rows.append(f)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(sample_s=1024, d=None):
    """The fp64 oracle, as it stands, on this host's cores: one 7B layer fwd+bwd at
    s = sample_s (a bounded sample of the workload), tokens/s = s / seconds.
    `d` = pre-generated inputs (the seeded generator is not part of the timing)."""
    import numpy as np
    from oracle import layer as OL
    from synth import layer_inputs
    if d is None:
        d = layer_inputs(H, N_HEADS, FFN, sample_s, 1, seed=42)
    t0 = time.perf_counter()
    y, c = OL.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], n=N_HEADS)
    OL.layer_bwd(d["dy"], c, d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], n=N_HEADS)
    dt = time.perf_counter() - t0
    cores, blas = os.cpu_count(), "unknown"
    try:
        from threadpoolctl import threadpool_info
        info = [i for i in threadpool_info() if i.get("user_api") == "blas"] or threadpool_info()
        cores = max([i.get("num_threads", 0) for i in info] + [1])
        blas = ", ".join(f"{i.get('internal_api')} {i.get('version')} ({i.get('architecture')})" for i in info)
    except Exception:
        pass
    cpu = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"value": sample_s / dt, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"numpy fp64 oracle, one 7B layer (h={H}, n={N_HEADS}, F={FFN}) fwd+bwd at s={sample_s}, "
                      f"{dt:.2f} s", "seconds": dt,
            "cpu_model": cpu, "affinity_cores": aff, "os_cpu_count": os.cpu_count(), "blas": blas}


def run_reference(args, rank, world):
    """--impl reference: the oracle timed as the reference arm (bounded samples)."""
    if rank != 0:
        return
    from synth import layer_inputs
    d = layer_inputs(H, N_HEADS, FFN, 512, 1, seed=42)      # generated once, reused by every step
    cb = None
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(sample_s=512, d=d)
        if i >= args.warmup:
            vals.append(r["seconds"])
        cb = r
    tot = sum(vals)
    v = 512 * len(vals) / tot
    cb["value"] = v
    out = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(vals), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": "configs[1]: Llama-style 7B layer, seq 4K-32K (oracle sample s=512)",
                      "h": H, "n_heads": N_HEADS, "ffn": FFN, "seq_lens": [512]},
           "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                               "affinity_cores", "os_cpu_count", "blas")},
           "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def self_launch(n):
    """`python bench.py --gpus N` without torchrun: start N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 with this same command line, and exit with its code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seqs", type=int, nargs="+", default=SEQS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strategy", type=int, default=-1, help="force a static strategy (default: pds_plan)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    P = world
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2511_13198_b200 import binding as B
    from paper_2511_13198_b200.calibrate import make_layer_buffers

    uid = None
    if P > 1:
        obj = [B.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    model = B.Model(h=H, n_heads=N_HEADS, ffn=FFN, n_layers=L_STACK)
    ctx = B.Context(model, P=P, rank=rank, device=local, uid=uid)
    bundle = os.path.join(ROOT, "paper_2511_13198_b200", "bundles", f"h{H}_n{N_HEADS}_f{FFN}_P{P}.txt")
    have_bundle = os.path.exists(bundle)
    if have_bundle:
        ctx.load_costs(bundle)
    # workspace for the strategies the runs will use (the plan of every s; ColossalZ's
    # quadratic workspace at 32K alone would exceed the device)
    if args.strategy >= 0:
        mask = 1 << args.strategy
    elif have_bundle:
        mask = 0
        for s in args.seqs:
            for q in ctx.plan(s, L_STACK)[0]:
                mask |= 1 << q
    else:
        mask = 1
    ctx.reserve(max(args.seqs), mask)

    st = torch.cuda.current_stream()
    bufs = {}
    for s in args.seqs:
        w, gr, x, dy = make_layer_buffers(torch, model, P, s, seed=1 + rank)
        W = B.Weights(*(w[k].data_ptr() for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")))
        G = B.Grads(*(gr[k].data_ptr() for k in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")))
        bufs[s] = dict(w=w, gr=gr, x=x, dy=dy, W=W, G=G, y=torch.empty_like(x), dx=torch.empty_like(x))
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    plans = {}

    def choose(s):
        if args.strategy >= 0:
            return args.strategy
        if have_bundle:
            plan, _ = ctx.plan(s, L_STACK)
            plans[s] = plan
            return plan[0]
        return 0

    def step(s, timed_events=None):
        b = bufs[s]
        pi = choose(s)
        sv = ctx.layer_fwd(pi, s, b["x"].data_ptr(), b["W"], b["y"].data_ptr(), st.cuda_stream)
        ctx.layer_bwd(pi, b["dy"].data_ptr(), sv, b["W"], b["G"], b["dx"].data_ptr(), st.cuda_stream)
        return pi

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up
    for _ in range(args.warmup):
        for s in args.seqs:
            step(s)
    barrier()

    # timed: each (step, s) bracketed by events; L2 flushed between timed iterations
    ctx.profile(True)
    ctx.profile_reset()
    per_s = {s: 0.0 for s in args.seqs}
    used = {}
    with Clocks(local) as clk:
        barrier()
        for k in range(args.steps):
            for s in args.seqs:
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                a.record(st)
                used[s] = step(s)
                e.record(st)
                e.synchronize()
                per_s[s] += a.elapsed_time(e)
        barrier()
    prof = {k: ctx.profile_read(k) for k in range(5)}
    ctx.profile(False)
    total_ms = sum(per_s.values())
    if world > 1:
        t = torch.tensor([total_ms] + [per_s[s] for s in args.seqs], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
        for i, s in enumerate(args.seqs):
            per_s[s] = float(t[i + 1])
    tokens = sum(args.seqs) * args.steps
    value = tokens / (total_ms / 1e3)

    # end-to-end through the C ABI with HOST buffers (pinned): pds_layer_step_host uploads x, dy and
    # downloads y, dx of every step inside the timed region
    host = {s: dict(x=bufs[s]["x"].cpu().pin_memory(), dy=bufs[s]["dy"].cpu().pin_memory(),
                    y=torch.empty_like(bufs[s]["x"], device="cpu").pin_memory(),
                    dx=torch.empty_like(bufs[s]["x"], device="cpu").pin_memory()) for s in args.seqs}
    # one warm-up pass of the host path (staging allocation), then K steps back to back:
    # the library pipelines each call's transfers against its neighbours' compute, and
    # the timed region ends after pds_host_drain, i.e. after the last dx download
    for s in args.seqs:
        b, hb = bufs[s], host[s]
        ctx.layer_step_host(choose(s), s, hb["x"].data_ptr(), hb["dy"].data_ptr(), b["W"], b["G"],
                            hb["y"].data_ptr(), hb["dx"].data_ptr(), st.cuda_stream)
    ctx.host_drain(st.cuda_stream)
    barrier()
    a = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for k in range(max(1, args.steps)):
        for s in args.seqs:
            b, hb = bufs[s], host[s]
            pi = choose(s)
            ctx.layer_step_host(pi, s, hb["x"].data_ptr(), hb["dy"].data_ptr(), b["W"], b["G"],
                                hb["y"].data_ptr(), hb["dx"].data_ptr(), st.cuda_stream)
    ctx.host_drain(st.cuda_stream)
    e.record(st)
    e.synchronize()
    e2e_ms = a.elapsed_time(e)
    nb = lambda t: t.numel() * t.element_size()
    h2d = sum(nb(host[s]["x"]) + nb(host[s]["dy"]) for s in args.seqs)
    d2h = sum(nb(host[s]["y"]) + nb(host[s]["dx"]) for s in args.seqs)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    e2e_val = sum(args.seqs) * max(1, args.steps) / (e2e_ms / 1e3)

    burst, sustained, hbm, src = peaks()
    g = prof[0]
    gemm_tf = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0
    launches = sum(prof[k]["launches"] for k in range(4))
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    attn = {k: (prof[k]["flops"] / (prof[k]["ms"] / 1e3) / 1e12 if prof[k]["ms"] > 0 else 0.0) for k in (1, 2)}
    model_flops = sum((72 * H * H + 6 * s * H) * s for s in args.seqs) * args.steps / P

    # the metric's second half, "max seq len before OOM": the longest s (a multiple of
    # 1024 P, reading R-15) whose adaptive plan for the L = 32 stack satisfies Eq. 6 on
    # this device (exact memory model; confirmed by running it in profiles/*oom_frontier*)
    frontier = None
    if have_bundle and args.strategy < 0:
        step_s = 1024 * P

        def feasible(sv):
            plan, flags = ctx.plan(sv, L_STACK)
            return not (flags & B.PLAN_INFEASIBLE), plan
        lo, hi = 0, step_s
        while feasible(hi)[0] and hi < (1 << 24):
            lo, hi = hi, hi * 2
        while hi - lo > step_s:
            mid = (lo + hi) // 2 // step_s * step_s
            if feasible(mid)[0]:
                lo = mid
            else:
                hi = mid
        if lo:
            frontier = {"s": lo, "layers": L_STACK, "plan": "".join("TUMCFR"[q] for q in feasible(lo)[1]),
                        "source": "pds_plan (Algorithm 1, Eq. 6 on the exact memory plan, device capacity "
                                  "minus the bundle's reserve); measured frontiers in profiles/"}
    out = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "configs[1]: Llama-style 7B layer (h=4096, n=32, d=128, F=16384 GELU), bf16, "
                               "one layer fwd+bwd per s, planned by pds_plan",
                   "seq_lens": args.seqs, "batch": 1, "parallelism": f"sp{P}",
                   "strategy_used": {str(s): used.get(s) for s in args.seqs},
                   "plan_source": "calibrated bundle" if have_bundle else "no bundle: MegatronTS",
                   "l2": "flushed (256 MB write) between timed iterations; weights 403 MB > L2",
                   "per_seq_tokens_per_s": {str(s): s * args.steps / (per_s[s] / 1e3) for s in args.seqs},
                   "model_tflops_per_gpu": model_flops / (total_ms / 1e3) / 1e12,
                   "max_seq_len_before_oom": frontier},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMM (gemm2_tc_kernel CTA pair / gemm_tc_kernel)",
                     "achieved": gemm_tf,
                     "peak": sustained, "unit": "TFLOP/s", "frac": gemm_tf / sustained,
                     "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a long step)",
                     "traffic": traffic,
                     "algorithmic_bytes_per_launch": g["bytes"] / g["launches"] if g["launches"] else None,
                     "launches": g["launches"], "gemm_ms": g["ms"],
                     "step_share": g["ms"] / total_ms if total_ms else None,
                     "attn_fwd_tflops": attn[1], "attn_bwd_tflops": attn[2],
                     "norm_ms": prof[3]["ms"], "norm_gbs": (prof[3]["bytes"] / (prof[3]["ms"] / 1e3) / 1e9
                                                             if prof[3]["ms"] > 0 else None)},
    }
    if world > 1:
        # collective bus bandwidth at this run's message sizes (torch.distributed's NCCL,
        # nccl-tests convention), the NVLink side of the roofline
        from paper_2511_13198_b200.nccl_bw import measure
        bw = measure(torch, dist, world, h=H, seqs=(max(args.seqs),), reps=5, warm=2)
        out["nccl_busbw"] = {"unit": "GB/s", "peak_per_direction": 900.0,
                             "results": [{k: r[k] for k in ("op", "what", "bytes", "busbw_gbs")} for r in bw]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline()
        out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                  "affinity_cores", "os_cpu_count", "blas")}
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
