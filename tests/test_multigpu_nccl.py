"""Every strategy at P = 2 / 4 / 8 REAL ranks (one process per GPU, NCCL over NVLink)
against the fp64 oracle, with the tile-overlapped collectives off and on.

Two ways to run it:
* pytest -m gpu on a box with >= 2 GPUs: the test below launches this file under
  torch.distributed.run with P = min(8, #GPUs) ranks (and P = 2 when more are there),
  under a watchdog (a hung collective fails the test instead of hanging the box);
  with one GPU it is skipped (the loopback group of tests/test_gpu_layer.py covers
  P > 1 on one device);
* directly: python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1
  tests/test_multigpu_nccl.py  (exit code 0 = every check passed).

Checks per rank (north_star tolerance 1e-2, shard indexing per O-4): y, dx, O, Z of
the rank's [s/P, h] rows vs the oracle's slice; every weight-gradient shard vs the
oracle's rank-r shard; overlapped == in-order bit for bit.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

TOL = 1e-2
CASES = [  # h, n, F, s, metp_chunks, n_kv, act, varlen lens: C1, a d = 128 shape with 2 METP waves,
           # the Llama variant (GQA 16 -> 8, SwiGLU) and varlen packing (TS / UZ / METP / METP-full)
    (256, 4, 1024, 512, 0, None, "gelu", None),
    (1024, 8, 4096, 2048, 2, None, "gelu", None),
    (2048, 16, 2048, 2048, 2, 8, "swiglu", None),
    (1024, 8, 2048, 2048, 2, None, "gelu", [512, 1024, 512]),
]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_rank():
    import faulthandler

    import torch
    import torch.distributed as dist

    from oracle import layer as OL
    from oracle import shard as OS
    from paper_2511_13198_b200 import binding as B
    from synth import bf16_bits, layer_inputs

    faulthandler.dump_traceback_later(int(os.environ.get("PDS_WATCHDOG_S", "600")), exit=True)
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def dev(a):
        return torch.from_numpy(bf16_bits(np.ascontiguousarray(a)).view(np.int16)).cuda().view(torch.bfloat16)

    def host(t):
        return t.float().cpu().numpy().astype(np.float64)

    failures = []
    for (h, n, F, s, chunks, n_kv, act, lens) in CASES:
        if n % P or (n_kv or n) % P or (s // P) % 128 or (chunks and (s // P // chunks) % 128):
            continue
        d = layer_inputs(h, n, F, s, 1, seed=21, n_kv=n_kv, act=act)
        wargs = (d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"])
        kw = dict(n=n, n_kv=n_kv, act=act)
        if lens:
            y_ref, cs = OL.layer_fwd_varlen(d["x"], lens, *wargs, **kw)
            g_ref = OL.layer_bwd_varlen(d["dy"], cs, lens, *wargs, **kw)
            c = dict(o=np.concatenate([q["o"] for q in cs]), z=np.concatenate([q["z"] for q in cs]))
        else:
            y_ref, c = OL.layer_fwd(d["x"], *wargs, **kw)
            g_ref = OL.layer_bwd(d["dy"], c, *wargs, **kw)
        W = OS.shard_weights(d, n, P, n_kv=n_kv, act=act)
        ref_sh = OS.shard_weights(dict(w_qkv=g_ref["dw_qkv"], w_proj=g_ref["dw_proj"], w_in=g_ref["dw_in"],
                                       w_out=g_ref["dw_out"], g1=g_ref["dg1"], g2=g_ref["dg2"]), n, P,
                                  n_kv=n_kv, act=act)
        sl = s // P
        rows = slice(rank * sl, (rank + 1) * sl)
        obj = [B.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = B.Context(B.Model(h=h, n_heads=n, ffn=F, metp_chunks=chunks, n_kv_heads=n_kv or 0,
                                ffn_act=1 if act == "swiglu" else 0), P=P, rank=rank, device=local, uid=obj[0])
        if lens:
            ctx.set_varlen(lens)
        st = torch.cuda.current_stream().cuda_stream
        keys = ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")
        w = {k: dev(W[k][rank]) for k in keys}
        Wp = B.Weights(*(w[k].data_ptr() for k in keys))
        x = dev(d["x"][rows, 0])
        dy = dev(d["dy"][rows, 0])
        for pi in ((0, 1, 2, 4) if lens else range(B.N_STRATEGIES)):
            if pi == 3 and (s // P) % 256:
                continue                       # MegatronCZ's zigzag half-chunks (R-CZ)
            res = []
            for ov in (0, 1):
                ctx.set_overlap(ov)
                gr = {k: torch.zeros(w[k].shape, dtype=torch.float32, device="cuda") for k in keys}
                G = B.Grads(*(gr[k].data_ptr() for k in keys))
                y, dx, o, z = (torch.empty_like(x) for _ in range(4))
                ctx.debug_taps(o.data_ptr(), z.data_ptr())
                sv = ctx.layer_fwd(pi, s, x.data_ptr(), Wp, y.data_ptr(), st)
                ctx.layer_bwd(pi, dy.data_ptr(), sv, Wp, G, dx.data_ptr(), st)
                torch.cuda.synchronize()
                res.append((host(y), host(dx), host(o), host(z), {k: host(v) for k, v in gr.items()}))
            (y0, dx0, o0, z0, g0), (y1, dx1, o1, z1, g1) = res
            chk = dict(y=_rel(y0, y_ref[rows, 0]), dx=_rel(dx0, g_ref["dx"][rows, 0]), o=_rel(o0, c["o"][rows, 0]),
                       z=_rel(z0, c["z"][rows, 0]))
            for k in keys:
                chk["d" + k] = _rel(g0[k], ref_sh[k][rank])
            bad = {k: v for k, v in chk.items() if not v < TOL}
            same = all(np.array_equal(a, b) for a, b in ((y0, y1), (dx0, dx1), (o0, o1), (z0, z1))) and \
                all(np.array_equal(g0[k], g1[k]) for k in keys)
            tag = f"P={P} rank={rank} h={h} s={s} pi={pi} kv={n_kv} {act} varlen={lens}"
            if bad or not same:
                failures.append(f"{tag}: bad={bad} overlap_bitwise={same}")
            elif rank == 0:
                print(f"ok {tag} y={chk['y']:.2e} dx={chk['dx']:.2e}", flush=True)
        ctx.close()
    dist.barrier()
    dist.destroy_process_group()
    for f in failures:
        print("FAIL", f, flush=True)
    return 1 if failures else 0


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_strategies_real_ranks(P):
    if _ngpu() < P:
        pytest.skip(f"needs {P} GPUs (this box has {_ngpu()}); P > 1 on one GPU: tests/test_gpu_layer.py loopback")
    # P = 1: one rank with a one-rank NCCL communicator (validates this harness on a 1-GPU box)
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
    env = dict(os.environ, PDS_WATCHDOG_S="540")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


if __name__ == "__main__":
    raise SystemExit(run_rank())
