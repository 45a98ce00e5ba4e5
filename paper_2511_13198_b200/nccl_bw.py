"""NCCL bus bandwidth of the collectives the strategies issue, at their message sizes
("collectives: bus GB/s vs 900 GB/s per direction"), one process per GPU
under torchrun.  nccl-tests convention: algbw = bytes / time; busbw = algbw (P-1)/P for
AllGather / ReduceScatter / AllToAll (bytes = the full gathered tensor), 2 (P-1)/P for
AllReduce.  Device-timed with CUDA events on the issuing stream, median of `reps`, max
over ranks.

  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
      -m paper_2511_13198_b200.nccl_bw [--out profiles/r02_nccl_busbw_P8.json]
"""
from __future__ import annotations

import argparse
import json
import os


def measure(torch, dist, P, h=4096, seqs=(4096, 32768, 131072), reps=10, warm=3):
    """Message sizes: TS / METP AG and RS of u = [s/P, h] bf16 per rank (full tensor s h 2 B),
    UlyssesZ A2A of the packed QKV (s/P x 3h bf16 per rank), the ZeRO3 weight AG (12 h^2 bf16)."""
    st = torch.cuda.current_stream()
    out = []

    def timed(fn):
        for _ in range(warm):
            fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        t = torch.tensor([sorted(ts)[len(ts) // 2]], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    fr = (P - 1) / P
    for s in seqs:
        n = s // P * h
        src = torch.randn(n, device="cuda").to(torch.bfloat16)
        full = torch.empty(n * P, dtype=torch.bfloat16, device="cuda")
        t = timed(lambda: dist.all_gather_into_tensor(full, src))
        out.append(dict(op="AllGather", what=f"u [s/P, h], s={s}", bytes=full.numel() * 2, seconds=t,
                        algbw_gbs=full.numel() * 2 / t / 1e9, busbw_gbs=full.numel() * 2 / t / 1e9 * fr))
        t = timed(lambda: dist.reduce_scatter_tensor(src, full))
        out.append(dict(op="ReduceScatter", what=f"partial [s, h] -> [s/P, h], s={s}", bytes=full.numel() * 2,
                        seconds=t, algbw_gbs=full.numel() * 2 / t / 1e9, busbw_gbs=full.numel() * 2 / t / 1e9 * fr))
        a2a_in = torch.randn(3 * n, device="cuda").to(torch.bfloat16)
        a2a_out = torch.empty_like(a2a_in)
        t = timed(lambda: dist.all_to_all_single(a2a_out, a2a_in))
        tot = a2a_in.numel() * 2 * P
        out.append(dict(op="AllToAll", what=f"packed QKV [s/P, 3h] per rank, s={s}", bytes=tot, seconds=t,
                        algbw_gbs=tot / t / 1e9, busbw_gbs=tot / t / 1e9 * fr))
        del src, full, a2a_in, a2a_out
    wsh = torch.randn(12 * h * h // P, device="cuda").to(torch.bfloat16)
    wfull = torch.empty(12 * h * h, dtype=torch.bfloat16, device="cuda")
    t = timed(lambda: dist.all_gather_into_tensor(wfull, wsh))
    out.append(dict(op="AllGather", what="ZeRO3 weights 12 h^2 bf16", bytes=wfull.numel() * 2, seconds=t,
                    algbw_gbs=wfull.numel() * 2 / t / 1e9, busbw_gbs=wfull.numel() * 2 / t / 1e9 * fr))
    g = torch.randn(2 * h, device="cuda")
    t = timed(lambda: dist.all_reduce(g))
    out.append(dict(op="AllReduce", what="dgamma 2h fp32", bytes=g.numel() * 4, seconds=t,
                    algbw_gbs=g.numel() * 4 / t / 1e9, busbw_gbs=g.numel() * 4 / t / 1e9 * 2 * fr))
    return out


def main():
    import torch
    import torch.distributed as dist
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = measure(torch, dist, P)
    if rank == 0:
        doc = {"P": P, "peak_gbs_per_direction": 900.0, "results": res,
               "device": torch.cuda.get_device_name(local), "nccl": ".".join(map(str, torch.cuda.nccl.version()))}
        txt = json.dumps(doc, indent=1)
        print(txt)
        if a.out:
            with open(a.out, "w") as f:
                f.write(txt)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
