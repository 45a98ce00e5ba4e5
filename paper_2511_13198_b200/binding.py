"""ctypes binding of include/paradyse.h (same names, argument marshalling only).

Device buffers are passed as integer device addresses (e.g. ``tensor.data_ptr()``)
and streams as ``torch.cuda.Stream.cuda_stream`` integers; torch is plumbing
(memory, streams, process groups), never on the compute path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDS_LIB") or os.path.join(HERE, "libparadyse.so")   # PDS_LIB: A/B builds

TS, UZ, METP, CZ, METP_FULL, COLOSSAL_Z = 0, 1, 2, 3, 4, 5
STRATEGIES = {TS: "MegatronTS", UZ: "UlyssesZ", METP: "METP", CZ: "MegatronCZ", METP_FULL: "METP-full",
              COLOSSAL_Z: "ColossalZ"}
N_STRATEGIES = 6
LETTERS = "TUMCFR"          # plan strings: T, U, M(ETP), C(Z), F(ull METP), R(ing self-attention: ColossalZ)

STATUS = {0: "PDS_OK", -1: "PDS_EINVAL", -2: "PDS_EDIVISIBILITY", -3: "PDS_ESTRATEGY", -4: "PDS_ENOMEM",
          -5: "PDS_ECUDA", -6: "PDS_ENCCL", -7: "PDS_ESTATE", -8: "PDS_ENOCOSTS", -9: "PDS_ENOTIMPL"}
PLAN_INFEASIBLE, PLAN_CACHED, PLAN_EARLY, PLAN_SMOOTHED = 1, 2, 4, 8


class PdsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class _Model(C.Structure):
    _fields_ = [("h", C.c_int32), ("n_heads", C.c_int32), ("ffn", C.c_int32), ("n_layers", C.c_int32),
                ("batch", C.c_int32), ("norm_eps", C.c_float), ("rope_theta", C.c_double),
                ("causal", C.c_int32), ("metp_chunks", C.c_int32), ("metp_recompute", C.c_int32),
                ("n_kv_heads", C.c_int32), ("ffn_act", C.c_int32)]


class _Weights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("w_qkv_t", "w_proj", "w_in_t", "w_out", "g1", "g2")]


class _Grads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("dw_qkv_t", "dw_proj", "dw_in_t", "dw_out", "dg1", "dg2")]


@dataclass
class Model:
    h: int
    n_heads: int
    ffn: int
    n_layers: int = 1
    batch: int = 1
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0
    causal: int = 1
    metp_chunks: int = 0
    metp_recompute: int = 0
    n_kv_heads: int = 0          # GQA key/value heads (0: n_heads)
    ffn_act: int = 0             # 0 GELU, 1 SwiGLU (Llama variant)

    def c(self):
        return _Model(self.h, self.n_heads, self.ffn, self.n_layers, self.batch, self.norm_eps,
                      self.rope_theta, self.causal, self.metp_chunks, self.metp_recompute,
                      self.n_kv_heads, self.ffn_act)


@dataclass
class Weights:
    w_qkv_t: int
    w_proj: int
    w_in_t: int
    w_out: int
    g1: int
    g2: int

    def c(self):
        return _Weights(self.w_qkv_t, self.w_proj, self.w_in_t, self.w_out, self.g1, self.g2)


@dataclass
class Grads:
    dw_qkv_t: int
    dw_proj: int
    dw_in_t: int
    dw_out: int
    dg1: int
    dg2: int

    def c(self):
        return _Grads(self.dw_qkv_t, self.dw_proj, self.dw_in_t, self.dw_out, self.dg1, self.dg2)


_lib = None

_SIGS = {
    "pds_nccl_unique_id": [C.c_void_p],
    "pds_create": [C.POINTER(_Model), C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)],
    "pds_group_create": [C.c_int32, C.POINTER(C.c_void_p)],
    "pds_group_destroy": [C.c_void_p],
    "pds_create_loopback": [C.POINTER(_Model), C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)],
    "pds_destroy": [C.c_void_p],
    "pds_reserve": [C.c_void_p, C.c_int64, C.c_uint32],
    "pds_release_cache": [C.c_void_p],
    "pds_load_costs": [C.c_void_p, C.c_char_p],
    "pds_set_capacity": [C.c_void_p, C.c_double, C.c_double],
    "pds_set_enabled": [C.c_void_p, C.c_uint32],
    "pds_plan": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.POINTER(C.c_uint32)],
    "pds_plan_ex": [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                    C.c_double, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32), C.c_void_p],
    "pds_cost_eval": [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p],
    "pds_mem_bytes": [C.POINTER(_Model), C.c_int32, C.c_uint8, C.c_int64, C.POINTER(C.c_int64),
                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "pds_layer_fwd": [C.c_void_p, C.c_uint8, C.c_int64, C.c_void_p, C.POINTER(_Weights), C.c_void_p,
                      C.POINTER(C.c_void_p), C.c_void_p],
    "pds_layer_bwd": [C.c_void_p, C.c_uint8, C.c_void_p, C.c_void_p, C.POINTER(_Weights),
                      C.POINTER(_Grads), C.c_void_p, C.c_void_p],
    "pds_layer_step_host": [C.c_void_p, C.c_uint8, C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(_Weights),
                            C.POINTER(_Grads), C.c_void_p, C.c_void_p, C.c_void_p],
    "pds_host_drain": [C.c_void_p, C.c_void_p],
    "pds_debug_trace": [C.c_void_p, C.c_int32],
    "pds_saved_release": [C.c_void_p, C.c_void_p],
    "pds_debug_taps": [C.c_void_p, C.c_void_p, C.c_void_p],
    "pds_k_gemm_sync": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                        C.c_void_p, C.c_int64, C.c_void_p, C.c_uint32, C.c_void_p, C.c_int64, C.c_int64,
                        C.c_int32, C.c_void_p],
    "pds_k_stream_write32": [C.c_void_p, C.c_void_p, C.c_uint32],
    "pds_k_stream_wait32": [C.c_void_p, C.c_void_p, C.c_uint32],
    "pds_set_overlap": [C.c_void_p, C.c_int32],
    "pds_set_varlen": [C.c_void_p, C.c_int32, C.POINTER(C.c_int64)],
    "pds_comm_log": [C.c_void_p, C.c_int32],
    "pds_comm_log_read": [C.c_void_p, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)],
    "pds_profile_enable": [C.c_void_p, C.c_int32],
    "pds_profile_read": [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                         C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "pds_profile_reset": [C.c_void_p],
    "pds_k_gemm": [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                   C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
    "pds_k_gemm_rope": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                        C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                        C.c_int64, C.c_void_p],
    "pds_k_rope_table": [C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_void_p],
    "pds_k_rmsnorm_fwd": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_void_p,
                          C.c_void_p, C.c_void_p, C.c_void_p],
    "pds_k_rmsnorm_bwd": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                          C.c_void_p, C.c_void_p, C.c_void_p],
    "pds_k_attn_fwd": [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                       C.c_int64, C.c_void_p, C.c_void_p],
    "pds_k_attn_bwd": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32,
                       C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p],
    "pds_k_attn_fwd_rows": [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                            C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p],
    "pds_k_attn_bwd_rows": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32,
                            C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p],
    "pds_set_attn_bwd": [C.c_int32],
    "pds_k_attn_fwd_pair": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                            C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                            C.c_void_p],
    "pds_k_attn_bwd_pair": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                            C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                            C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p],
    "pds_k_attn_merge": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                         C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p],
    "pds_k_attn_dot": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p],
    "pds_k_attn_fwd_gqa": [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                           C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p],
    "pds_k_attn_bwd_gqa": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32,
                           C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p],
    "pds_k_gemm_swiglu": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                          C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                          C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
    "pds_k_gemm_rope_gqa": [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                            C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p],
    "pds_last_error": [],
    "pds_version": [],
}


def lib():
    """Load libparadyse.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run __graft_entry__.build() "
                              "(python paper_2511_13198_b200/build.py). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            if os.environ.get("PDS_LIB") and not hasattr(L, name):
                continue                  # an older A/B build may lack newer entry points
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_char_p if name in ("pds_last_error", "pds_version") else C.c_int
        _lib = L
    return _lib


def check(rc):
    if rc != 0:
        raise PdsError(rc, lib().pds_last_error().decode())
    return rc


def call(name, *args):
    return check(getattr(lib(), name)(*args))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    call("pds_nccl_unique_id", buf)
    return buf.raw


def mem_bytes(model: Model, P: int, strategy: int, s: int):
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    call("pds_mem_bytes", C.byref(model.c()), P, strategy, s, C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def plan_ex(L, t, m, enabled, capacity, gamma=0.0, prev=None, counters=False, w=None):
    n = len(t)
    ta = (C.c_double * n)(*t)
    ma = (C.c_double * n)(*m)
    wa = (C.c_double * n)(*w) if w is not None else None
    ea = (C.c_uint8 * n)(*[1 if e else 0 for e in enabled])
    out = (C.c_uint8 * L)()
    pv = (C.c_uint8 * L)(*prev) if prev is not None else None
    flags = C.c_uint32()
    ctr = (C.c_int64 * 3)()
    call("pds_plan_ex", L, n, ta, ma, wa, ea, capacity, gamma, pv, out, C.byref(flags), ctr)
    res = list(out), flags.value
    return (res + (list(ctr),)) if counters else res


class Group:
    """In-process loopback group: P virtual ranks on one device (single-GPU multi-rank tests)."""

    def __init__(self, P):
        h = C.c_void_p()
        call("pds_group_create", P, C.byref(h))
        self.h = h
        self.P = P

    def close(self):
        if self.h:
            lib().pds_group_destroy(self.h)
            self.h = None


class Context:
    def __init__(self, model: Model, P=1, rank=0, device=0, uid: bytes | None = None, group: Group | None = None):
        self.model, self.P, self.rank = model, P, rank
        h = C.c_void_p()
        self._m = model.c()
        if group is not None:
            call("pds_create_loopback", C.byref(self._m), group.h, rank, device, C.byref(h))
        else:
            ub = C.create_string_buffer(uid, 128) if uid else None
            call("pds_create", C.byref(self._m), P, rank, device, ub, C.byref(h))
        self.h = h

    def close(self):
        if self.h:
            lib().pds_destroy(self.h)
            self.h = None

    def reserve(self, max_seq_len, mask=(1 << N_STRATEGIES) - 1):
        call("pds_reserve", self.h, max_seq_len, mask)

    def release_cache(self):
        call("pds_release_cache", self.h)

    def load_costs(self, path):
        call("pds_load_costs", self.h, path.encode())

    def set_capacity(self, cap, gamma=0.0):
        call("pds_set_capacity", self.h, cap, gamma)

    def set_enabled(self, mask):
        call("pds_set_enabled", self.h, mask)

    def plan(self, s, L):
        out = (C.c_uint8 * L)()
        fl = C.c_uint32()
        call("pds_plan", self.h, s, out, L, C.byref(fl))
        return list(out), fl.value

    def cost_eval(self, s):
        t = (C.c_double * N_STRATEGIES)()
        m = (C.c_double * N_STRATEGIES)()
        b = (C.c_int32 * N_STRATEGIES)()
        call("pds_cost_eval", self.h, s, t, m, b)
        return list(t), list(m), list(b)

    def layer_fwd(self, strategy, s, x, w: Weights, y, stream=0, keep=True):
        sv = C.c_void_p()
        call("pds_layer_fwd", self.h, strategy, s, x, C.byref(w.c()), y, C.byref(sv) if keep else None, stream)
        return sv if keep else None

    def layer_bwd(self, strategy, dy, saved, w: Weights, g: Grads, dx, stream=0):
        call("pds_layer_bwd", self.h, strategy, dy, saved, C.byref(w.c()), C.byref(g.c()), dx, stream)

    def layer_step_host(self, strategy, seq_len, x_host, dy_host, w: Weights, g: Grads, y_host, dx_host,
                        stream=0):
        """One layer fwd + bwd on HOST buffers (pinned host pointers), asynchronous;
        results valid after host_drain(stream) and a sync.  pds_layer_step_host."""
        call("pds_layer_step_host", self.h, strategy, seq_len, x_host, dy_host, C.byref(w.c()), C.byref(g.c()),
             y_host, dx_host, stream)

    def host_drain(self, stream=0):
        """Orders `stream` after all pds_layer_step_host transfers (pds_host_drain)."""
        call("pds_host_drain", self.h, stream)

    def saved_release(self, saved):
        call("pds_saved_release", self.h, saved)

    def set_overlap(self, on):
        call("pds_set_overlap", self.h, 1 if on else 0)

    def comm_log(self, on=True):
        """Start (clearing) or stop the JSON-lines comm log of this rank."""
        call("pds_comm_log", self.h, 1 if on else 0)

    def read_comm_log(self):
        import json
        n = C.c_int64(0)
        call("pds_comm_log_read", self.h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        call("pds_comm_log_read", self.h, buf, n.value + 1, C.byref(n))
        return [json.loads(line) for line in buf.value.decode().splitlines() if line]

    def set_varlen(self, lens):
        """Pack len(lens) sequences into the following layer calls (R-VARLEN); [] = one."""
        arr = (C.c_int64 * max(1, len(lens)))(*[int(v) for v in lens])
        call("pds_set_varlen", self.h, len(lens), arr)

    def debug_taps(self, o=None, z=None):
        call("pds_debug_taps", self.h, o, z)

    def profile(self, on=True):
        call("pds_profile_enable", self.h, 1 if on else 0)

    def profile_read(self, klass):
        ms, n, fl, by = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        call("pds_profile_read", self.h, klass, C.byref(ms), C.byref(n), C.byref(fl), C.byref(by))
        return dict(ms=ms.value, launches=n.value, flops=fl.value, bytes=by.value)

    def profile_reset(self):
        call("pds_profile_reset", self.h)


# ------------------------------------------------------------------ kernel-level entry points
def k_gemm(A, lda, a_mn, B, ldb, b_mn, M, N, K, Cp, ldc, epi=0, aux_in=None, aux_out=None, ld_aux=0, stream=0):
    call("pds_k_gemm", A, lda, a_mn, B, ldb, b_mn, M, N, K, Cp, ldc, epi, aux_in, aux_out, ld_aux, stream)


def k_gemm_sync(A, lda, B, ldb, M, N, K, Cp, ldc, wait_flags=None, epoch=0, done_ctr=None, chunk_rows=0,
                m_rot_rows=0, sm_reserve=0, stream=0):
    call("pds_k_gemm_sync", A, lda, B, ldb, M, N, K, Cp, ldc, wait_flags, epoch, done_ctr, chunk_rows, m_rot_rows,
         sm_reserve, stream)


def k_stream_write32(stream, addr, value):
    call("pds_k_stream_write32", stream, addr, value)


def k_stream_wait32(stream, addr, value):
    call("pds_k_stream_wait32", stream, addr, value)


def k_gemm_rope(A, lda, B, ldb, M, N, K, Cp, ldc, rope, d, hq, seg=0, seg_stride=0, seg_base=0, stream=0):
    call("pds_k_gemm_rope", A, lda, B, ldb, M, N, K, Cp, ldc, rope, d, hq, seg, seg_stride, seg_base, stream)


def k_rope_table(t, n_pos, d, theta=10000.0, stream=0):
    call("pds_k_rope_table", t, n_pos, d, theta, stream)


def k_rmsnorm_fwd(x, res, g, rows, h, eps, x1, u, rstd, stream=0):
    call("pds_k_rmsnorm_fwd", x, res, g, rows, h, eps, x1, u, rstd, stream)


def k_rmsnorm_bwd(du, x, rstd, g, dres, rows, h, dx, dg, stream=0):
    call("pds_k_rmsnorm_bwd", du, x, rstd, g, dres, rows, h, dx, dg, stream)


def k_attn_fwd(qkv, ld, s, heads, d, causal, out, ld_out, lse, stream=0):
    call("pds_k_attn_fwd", qkv, ld, s, heads, d, causal, out, ld_out, lse, stream)


def k_attn_fwd_gqa(qkv, ld, s, heads, kv_heads, d, causal, out, ld_out, lse, stream=0):
    call("pds_k_attn_fwd_gqa", qkv, ld, s, heads, kv_heads, d, causal, out, ld_out, lse, stream)


def k_attn_bwd_gqa(qkv, ld, out, ld_out, lse, dout, s, heads, kv_heads, d, causal, dqkv, stream=0):
    call("pds_k_attn_bwd_gqa", qkv, ld, out, ld_out, lse, dout, s, heads, kv_heads, d, causal, dqkv, stream)


def k_gemm_swiglu(A, lda, B, ldb, M, N, K, bwd, Cp, ldc, h_in=None, ld_h=0, g_out=None, ld_g=0, c_t=None,
                  g_t=None, ld_t=0, stream=0):
    call("pds_k_gemm_swiglu", A, lda, B, ldb, M, N, K, bwd, Cp, ldc, h_in, ld_h, g_out, ld_g, c_t, g_t, ld_t, stream)


def k_gemm_rope_gqa(A, lda, B, ldb, M, N, K, Cp, ldc, rope, d, hq, hk, stream=0):
    call("pds_k_gemm_rope_gqa", A, lda, B, ldb, M, N, K, Cp, ldc, rope, d, hq, hk, stream)


def k_attn_bwd(qkv, ld, out, ld_out, lse, dout, s, heads, d, causal, dqkv, stream=0):
    call("pds_k_attn_bwd", qkv, ld, out, ld_out, lse, dout, s, heads, d, causal, dqkv, stream)


def k_attn_fwd_pair(q, ld_q, kv, ld_kv, kcol, vcol, sq, sk, heads, d, causal, out, ld_out, lse, stream=0):
    call("pds_k_attn_fwd_pair", q, ld_q, kv, ld_kv, kcol, vcol, sq, sk, heads, d, causal, out, ld_out, lse, stream)


def k_attn_bwd_pair(q, ld_q, kv, ld_kv, kcol, vcol, dout, ld_out, lse, dd, sq, sk, heads, d, causal, dq_acc, ld_dqa,
                    dkv_acc, ld_dkva, stream=0):
    call("pds_k_attn_bwd_pair", q, ld_q, kv, ld_kv, kcol, vcol, dout, ld_out, lse, dd, sq, sk, heads, d, causal,
         dq_acc, ld_dqa, dkv_acc, ld_dkva, stream)


def k_attn_merge(o_acc, ld_oacc, l_acc, lstride_acc, o_p, ld_op, l_p, lstride_p, rows, heads, d, first, out=None,
                 ld_out=0, stream=0):
    call("pds_k_attn_merge", o_acc, ld_oacc, l_acc, lstride_acc, o_p, ld_op, l_p, lstride_p, rows, heads, d, first,
         out, ld_out, stream)


def k_attn_dot(out, ld_out, dout, s, heads, d, dd, stream=0):
    call("pds_k_attn_dot", out, ld_out, dout, s, heads, d, dd, stream)


def set_attn_bwd(mode):
    """0 = split attention backward kernels (default), 1 = fused kernel where it applies (d = 128, causal)."""
    call("pds_set_attn_bwd", mode)


def k_attn_fwd_rows(qkv, ld, s, heads, d, causal, qlo, qn, out, ld_out, lse, stream=0):
    call("pds_k_attn_fwd_rows", qkv, ld, s, heads, d, causal, qlo, qn, out, ld_out, lse, stream)


def k_attn_bwd_rows(qkv, ld, out, ld_out, lse, dout, s, heads, d, causal, qlo, qn, dqkv, stream=0):
    call("pds_k_attn_bwd_rows", qkv, ld, out, ld_out, lse, dout, s, heads, d, causal, qlo, qn, dqkv, stream)
