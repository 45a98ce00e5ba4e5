"""world_size-2 CPU tests (gloo) of the N > 1 host path.

The library's strategies assume NCCL's collective conventions: AllGather
concatenates in rank order (in place: rank r's send buffer is slot r of the
receive buffer), ReduceScatter hands chunk r of the sum to rank r (in place:
the output is slot r of the input), All-to-All sends block j to rank j and
receives rank j's block in slot j.  These tests run the MegatronTS, UlyssesZ and
MegatronCZ forward dataflow of csrc/layer.cpp in two / four real processes with torch.distributed
(gloo, fp64) using exactly those conventions, and compare with the oracle's
unsharded layer, and the pairwise-step schedule of the tile-overlapped AG / RS
(comm.cpp) against the plain collectives.  They also cover the bench's host logic: NCCL-uid broadcast via
broadcast_object_list, max-over-ranks timing, and that every rank's planner
returns the same plan (Algorithm 1 is deterministic).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import layer as OL
from oracle import shard as OS
from synth import layer_inputs

H, N, F, S = 32, 4, 128, 32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ag(local, P):
    out = [torch.empty_like(local) for _ in range(P)]
    dist.all_gather(out, local)
    return torch.cat(out, 0)


def _rs(full, P):
    # gloo lacks reduce_scatter: all_reduce then keep chunk r (NCCL RS semantics)
    t = full.clone()
    dist.all_reduce(t)
    return t.chunk(P, 0)[dist.get_rank()].clone()


def _a2a(send_blocks):
    """send_blocks[j] goes to rank j; returns received blocks in source order."""
    P = len(send_blocks)
    r = dist.get_rank()
    recv = [None] * P
    for j in range(P):
        # scatter from source j: rank i receives source j's block i
        out = torch.empty_like(send_blocks[0])
        dist.scatter(out, [b.contiguous() for b in send_blocks] if j == r else None, src=j)
        recv[j] = out
    return recv


def _rmsnorm(x, g, eps=1e-5):
    r = torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)
    return x * r * g


def _attn(qkv, nl, d, positions):
    s = qkv.shape[0]
    hl = nl * d
    out = torch.empty(s, hl, dtype=qkv.dtype)
    inv = 10000.0 ** (-2 * torch.arange(d // 2, dtype=torch.float64) / d)
    ang = positions.double()[:, None] * inv[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)

    def rot(t):
        a, b = t[:, :d // 2], t[:, d // 2:]
        return torch.cat([a * cos - b * sin, a * sin + b * cos], -1)
    for hh in range(nl):
        q = rot(qkv[:, hh * d:(hh + 1) * d])
        k = rot(qkv[:, hl + hh * d:hl + (hh + 1) * d])
        v = qkv[:, 2 * hl + hh * d:2 * hl + (hh + 1) * d]
        out[:, hh * d:(hh + 1) * d] = torch.nn.functional.scaled_dot_product_attention(
            q[None], k[None], v[None], is_causal=True)[0]
    return out


def _rope_qk(qkv, n, d, positions):
    """RoPE on the Q and K column blocks of [rows, 3 n d] at the given global positions."""
    h = n * d
    inv = 10000.0 ** (-2 * torch.arange(d // 2, dtype=torch.float64) / d)
    ang = positions.double()[:, None] * inv[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)
    out = qkv.clone()
    for blk in (0, 1):
        for hh in range(n):
            t = qkv[:, blk * h + hh * d:blk * h + (hh + 1) * d]
            a, b = t[:, :d // 2], t[:, d // 2:]
            out[:, blk * h + hh * d:blk * h + (hh + 1) * d] = torch.cat([a * cos - b * sin, a * sin + b * cos], -1)
    return out


def _attn_keys(q, kv, pq, pk, n, d):
    """Causal softmax attention of queries (post-RoPE, positions pq) over the keys of kv
    [K | V] (positions pk) alone: (O [rows, n d], LSE [n, rows], -inf without keys)."""
    h = n * d
    o = torch.zeros(q.shape[0], h, dtype=q.dtype)
    lse = torch.full((n, q.shape[0]), -float("inf"), dtype=q.dtype)
    mask = pk[None, :] > pq[:, None]
    for hh in range(n):
        sc = q[:, hh * d:(hh + 1) * d] @ kv[:, hh * d:(hh + 1) * d].T / d ** 0.5
        sc = sc.masked_fill(mask, -float("inf"))
        l = torch.logsumexp(sc, dim=1)
        p = torch.exp(sc - l[:, None]).nan_to_num(0.0)
        o[:, hh * d:(hh + 1) * d] = p @ kv[:, h + hh * d:h + (hh + 1) * d]
        lse[hh] = l
    return o, lse


def _exchange(blocks, sends, recvs):
    """Point-to-point sends of blocks[i] to (peer, tag) = sends[i]; receives (peer, tag)
    = recvs[j] into blocks of the same shape, concatenated in recvs order (comm.cpp p2p:
    a transfer to this rank itself is a copy)."""
    rank = dist.get_rank()
    out = [torch.empty_like(blocks[0]) for _ in recvs]
    reqs = []
    for (peer, tag), blk in zip(sends, blocks):
        if peer == rank:
            out[[i for i, r in enumerate(recvs) if r == (rank, tag)][0]].copy_(blk)
        else:
            reqs.append(dist.isend(blk.contiguous(), peer, tag=tag))
    for i, (peer, tag) in enumerate(recvs):
        if peer != rank:
            reqs.append(dist.irecv(out[i], peer, tag=tag))
    for r in reqs:
        r.wait()
    return torch.cat(out, 0)


def _worker(rank, P, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        d = layer_inputs(H, N, F, S, 1, seed=3)
        W = OS.shard_weights(d, N, P)
        T = lambda a: torch.tensor(a, dtype=torch.float64)
        x = T(OS.shard_act(d["x"], P)[rank][:, 0])
        g1, g2 = T(d["g1"]), T(d["g2"])
        wq, wp, wi, wo = (T(W[k][rank]) for k in ("w_qkv_t", "w_proj", "w_in_t", "w_out"))
        sl, nl, d_, hl = S // P, N // P, H // N, H // P
        gelu = torch.nn.functional.gelu
        # ---- MegatronTS forward (csrc/layer.cpp ts_fwd)
        U = _ag(_rmsnorm(x, g1), P)                             # in-place AG: slot r = local u
        qkv = U @ wq.T
        a = _attn(qkv, nl, d_, torch.arange(S))
        o = _rs(a @ wp, P)
        x1 = x + o
        V = _ag(_rmsnorm(x1, g2), P)
        z = _rs(gelu(V @ wi.T) @ wo, P)
        y_ts = x1 + z
        # ---- UlyssesZ forward (csrc/layer.cpp uz_fwd)
        wqf, wpf, wif, wof = _ag(wq, P), _ag(wp, P), _ag(wi, P), _ag(wo, P)
        u = _rmsnorm(x, g1)
        qkv_loc = u @ wqf.T                                     # head-group-major columns
        blocks = list(qkv_loc.split(3 * hl, dim=1))             # pack: block j -> rank j
        qkv_h = torch.cat(_a2a(blocks), 0)                      # [s, 3h/P], positions in order
        a_h = _attn(qkv_h, nl, d_, torch.arange(S))
        back = _a2a(list(a_h.split(sl, dim=0)))                 # row block j -> rank j
        afull = torch.cat(back, 1)                              # unpack: slot j = group j columns
        x1u = x + afull @ wpf
        y_uz = x1u + gelu(_rmsnorm(x1u, g2) @ wif.T) @ wof
        # ---- MegatronCZ forward (csrc/layer.cpp cz_fwd, reading R-CZ): W_qkv^T gathered
        # part by part into [Q all; K all; V all], local QKV with RoPE at global positions,
        # point-to-point exchange to the zigzag rows (half-chunks r, 2P-1-r), P ring steps
        # of K/V with log-sum-exp merges, the reverse exchange of O
        wq_all = torch.cat([_ag(wq[i * hl:(i + 1) * hl].contiguous(), P) for i in range(3)], 0)
        qkv_b = _rope_qk(_rmsnorm(x, g1) @ wq_all.T, N, d_, torch.arange(rank * sl, (rank + 1) * sl))
        c = sl // 2
        zz = lambda j: j if j < P else 2 * P - 1 - j
        zig = (rank, 2 * P - 1 - rank)
        qkvz = _exchange([qkv_b[:c], qkv_b[c:]], [(zz(2 * rank), 2 * rank), (zz(2 * rank + 1), 2 * rank + 1)],
                         [(j // 2, j) for j in zig])
        pos = torch.cat([torch.arange(j * c, (j + 1) * c) for j in zig])
        kv, kv_pos = qkvz[:, H:].contiguous(), pos
        o_acc = torch.zeros(sl, H, dtype=torch.float64)
        l_acc = torch.full((N, sl), -float("inf"), dtype=torch.float64)
        for k in range(P):
            o_p, l_p = _attn_keys(qkvz[:, :H], kv, pos, kv_pos, N, d_)
            l_new = torch.logaddexp(l_acc, l_p)
            wa = torch.exp(l_acc - l_new).nan_to_num(0.0)
            wpr = torch.exp(l_p - l_new).nan_to_num(0.0)
            o_acc = (o_acc.view(sl, N, d_) * wa.T[..., None] + o_p.view(sl, N, d_) * wpr.T[..., None]).view(sl, H)
            l_acc = l_new
            if k < P - 1:                                     # ring: K/V (and positions) to rank + 1
                kv = _exchange([kv], [((rank + 1) % P, 0)], [((rank - 1) % P, 0)])
                kv_pos = _exchange([kv_pos.double()[:, None]], [((rank + 1) % P, 1)],
                                   [((rank - 1) % P, 1)])[:, 0].long()
        a_c = _exchange([o_acc[:c], o_acc[c:]], [(j // 2, j) for j in zig],
                        [(zz(2 * rank), 2 * rank), (zz(2 * rank + 1), 2 * rank + 1)])
        x1c = x + a_c @ wpf
        y_cz = x1c + gelu(_rmsnorm(x1c, g2) @ wif.T) @ wof
        # ---- tile-overlapped TS collectives (comm.cpp all_gather_flagged /
        # reduce_scatter_gated): P - 1 pairwise steps; AG step k sends the own chunk to
        # rank - k and receives chunk rank + k; RS step k sends chunk rank + k to its
        # owner and receives this rank's chunk from rank - k; then the rank-order sum
        u_loc = _rmsnorm(x, g1)
        ag = [None] * P
        ag[rank] = u_loc
        for k in range(1, P):
            frm, to = (rank + k) % P, (rank - k) % P
            buf = torch.empty_like(u_loc)
            reqs = [dist.isend(u_loc.contiguous(), to), dist.irecv(buf, frm)]
            for rq in reqs:
                rq.wait()
            ag[frm] = buf
        ag_ok = torch.equal(torch.cat(ag, 0), U)
        part = (a @ wp).contiguous()                            # [P][sl][h] partials
        recv = [None] * P
        for k in range(1, P):
            to, frm = (rank + k) % P, (rank - k) % P
            buf = torch.empty(sl, H, dtype=part.dtype)
            reqs = [dist.isend(part[to * sl:(to + 1) * sl].contiguous(), to), dist.irecv(buf, frm)]
            for rq in reqs:
                rq.wait()
            recv[frm] = buf
        recv[rank] = part[rank * sl:(rank + 1) * sl]
        rs_sum = recv[0].clone()
        for j in range(1, P):
            rs_sum += recv[j]
        rs_ok = torch.allclose(rs_sum, o, rtol=0, atol=1e-12)
        # ---- bench host logic: uid broadcast, max over ranks, plan agreement
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        from paper_2511_13198_b200 import binding as B
        plan, _ = B.plan_ex(32, [1.0, 1.5, 3.0], [5.0, 4.0, 1.0], [1, 1, 1], 100.0)
        plans = [None] * P
        dist.all_gather_object(plans, plan)
        q.put((rank, y_ts.numpy(), y_uz.numpy(), obj[0], float(t), plans, y_cz.numpy(), ag_ok, rs_ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 4])
def test_two_process_strategies_and_host_logic(P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(P)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = layer_inputs(H, N, F, S, 1, seed=3)
    y_ref, _ = OL.layer_fwd(d["x"], d["w_qkv"], d["w_proj"], d["w_in"], d["w_out"], d["g1"], d["g2"], n=N)
    y_ts = np.concatenate([r[1] for r in res])
    y_uz = np.concatenate([r[2] for r in res])
    assert np.max(np.abs(y_ts - y_ref[:, 0])) < 1e-10
    assert np.max(np.abs(y_uz - y_ref[:, 0])) < 1e-10
    y_cz = np.concatenate([r[6] for r in res])
    assert np.max(np.abs(y_cz - y_ref[:, 0])) < 1e-10
    for r in res:
        assert r[7] and r[8]                      # pairwise-step AG / RS = the collectives
        assert r[3] == bytes(range(128))          # NCCL uid broadcast
        assert r[4] == float(P)                   # max over ranks
        assert r[5][0] == r[5][1]                 # identical plans on every rank
