// Kernel-level C-ABI entry points (per-stage parity) and the
// NCCL unique-id helper.  Thin argument checks + launch; no context.
#include <mutex>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "comm.hpp"
#include "internal.hpp"
#include "kernels/gemm.cuh"
#include "kernels/kernels.hpp"

using namespace pds;

static pds_status rc2s(int rc, const char* what) {
  if (rc == 0) return PDS_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString((cudaError_t)rc));
  return rc == (int)cudaErrorMemoryAllocation ? PDS_ENOMEM : (rc == (int)cudaErrorInvalidValue ? PDS_EINVAL : PDS_ECUDA);
}

extern "C" pds_status pds_nccl_unique_id(void* out128) {
  if (!out128) PDS_FAIL(PDS_EINVAL, "NULL out");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) PDS_FAIL(PDS_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memcpy(out128, &id, sizeof(id));
  return PDS_OK;
}

extern "C" pds_status pds_k_gemm(const void* A, int64_t lda, int32_t a_mn, const void* B, int64_t ldb,
                                 int32_t b_mn, int32_t M, int32_t N, int32_t K, void* C, int64_t ldc,
                                 int32_t epi, const void* aux_in, void* aux_out, int64_t ld_aux, void* stream) {
  if (!A || !B || !C) PDS_FAIL(PDS_EINVAL, "NULL operand");
  if (epi < 0 || epi > EPI_DGELU) PDS_FAIL(PDS_EINVAL, "bad epilogue");
  if ((epi == EPI_GELU && !aux_out) || (epi == EPI_DGELU && (!aux_in || !aux_out)))
    PDS_FAIL(PDS_EINVAL, "GELU epilogues need aux buffers");
  GemmArgs g;
  g.A = A; g.lda = lda; g.a_mn = a_mn; g.B = B; g.ldb = ldb; g.b_mn = b_mn;
  g.M = M; g.N = N; g.K = K; g.C = C; g.ldc = ldc; g.epi = epi;
  g.aux_in = aux_in; g.aux_out = aux_out; g.ld_aux = ld_aux;
  return rc2s(gemm_launch(g, static_cast<cudaStream_t>(stream)), "pds_k_gemm");
}

extern "C" pds_status pds_k_gemm_sync(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M,
                                      int32_t N, int32_t K, void* C, int64_t ldc, const uint32_t* wait_flags,
                                      uint32_t flag_epoch, uint32_t* done_ctr, int64_t chunk_rows,
                                      int64_t m_rot_rows, int32_t sm_reserve, void* stream) {
  if (!A || !B || !C) PDS_FAIL(PDS_EINVAL, "NULL operand");
  if ((wait_flags || done_ctr) && chunk_rows <= 0) PDS_FAIL(PDS_EINVAL, "chunk_rows must be > 0");
  GemmArgs g;
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.M = M; g.N = N; g.K = K; g.C = C; g.ldc = ldc;
  g.wait_flags = wait_flags; g.flag_epoch = flag_epoch; g.done_ctr = done_ctr;
  g.chunk_rows = chunk_rows; g.m_rot_rows = m_rot_rows; g.sm_reserve = sm_reserve;
  return rc2s(gemm_launch(g, static_cast<cudaStream_t>(stream)), "pds_k_gemm_sync");
}

extern "C" pds_status pds_k_stream_write32(void* stream, uint32_t* addr, uint32_t value) {
  if (!addr) PDS_FAIL(PDS_EINVAL, "NULL address");
  return stream_write32(static_cast<cudaStream_t>(stream), addr, value);
}

extern "C" pds_status pds_k_stream_wait32(void* stream, const uint32_t* addr, uint32_t value) {
  if (!addr) PDS_FAIL(PDS_EINVAL, "NULL address");
  return stream_wait32_geq(static_cast<cudaStream_t>(stream), addr, value);
}

extern "C" pds_status pds_k_gemm_rope(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M,
                                      int32_t N, int32_t K, void* C, int64_t ldc, const void* rope, int32_t d,
                                      int32_t hq, int64_t seg, int64_t seg_stride, int64_t seg_base,
                                      void* stream) {
  if (!A || !B || !C || !rope) PDS_FAIL(PDS_EINVAL, "NULL operand");
  if (hq <= 0 || N % (3 * hq)) PDS_FAIL(PDS_EINVAL, "N must be a multiple of 3*hq");
  GemmArgs g;
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.M = M; g.N = N; g.K = K; g.C = C; g.ldc = ldc;
  g.epi = EPI_ROPE; g.rope = reinterpret_cast<const float2*>(rope); g.rope_d = d; g.rope_hq = hq;
  g.seg = seg; g.seg_stride = seg_stride; g.seg_base = seg_base;
  return rc2s(gemm_launch(g, static_cast<cudaStream_t>(stream)), "pds_k_gemm_rope");
}

extern "C" pds_status pds_k_rope_table(void* table, int64_t n_pos, int32_t d, double theta, void* stream) {
  if (!table || n_pos <= 0 || d <= 0 || d % 2) PDS_FAIL(PDS_EINVAL, "bad rope table args");
  return rc2s(rope_table(table, n_pos, d, theta, static_cast<cudaStream_t>(stream)), "pds_k_rope_table");
}

extern "C" pds_status pds_k_rmsnorm_fwd(const void* x, const void* residual, const void* g, int64_t rows,
                                        int32_t h, float eps, void* x1_out, void* u_out, void* rstd_out,
                                        void* stream) {
  if (!x || !g || !u_out || !rstd_out || (residual && !x1_out)) PDS_FAIL(PDS_EINVAL, "NULL argument");
  return rc2s(rmsnorm_fwd(x, residual, g, rows, h, eps, x1_out, u_out, rstd_out, static_cast<cudaStream_t>(stream)),
              "pds_k_rmsnorm_fwd");
}

extern "C" pds_status pds_k_rmsnorm_bwd(const void* du, const void* x, const void* rstd, const void* g,
                                        const void* dres, int64_t rows, int32_t h, void* dx, void* dg,
                                        void* stream) {
  if (!du || !x || !rstd || !g || !dx || !dg) PDS_FAIL(PDS_EINVAL, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* part = nullptr;
  PDS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), (size_t)rmsnorm_bwd_grid(rows) * h * 4, st));
  pds_status r = rc2s(rmsnorm_bwd(du, x, rstd, g, dres, rows, h, dx, part, static_cast<float*>(dg), st),
                      "pds_k_rmsnorm_bwd");
  cudaFreeAsync(part, st);
  return r;
}

extern "C" pds_status pds_k_attn_fwd(const void* qkv, int64_t ld, int32_t s, int32_t heads, int32_t d,
                                     int32_t causal, void* out, int64_t ld_out, void* lse, void* stream) {
  if (!qkv || !out || !lse) PDS_FAIL(PDS_EINVAL, "NULL argument");
  return rc2s(attn_fwd(qkv, ld, s, heads, d, causal, out, ld_out, lse, static_cast<cudaStream_t>(stream)),
              "pds_k_attn_fwd");
}

extern "C" pds_status pds_k_attn_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out,
                                     const void* lse, const void* dout, int32_t s, int32_t heads, int32_t d,
                                     int32_t causal, void* dqkv, void* stream) {
  if (!qkv || !out || !lse || !dout || !dqkv) PDS_FAIL(PDS_EINVAL, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* dd = nullptr;
  PDS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dd), (size_t)heads * s * 4, st));
  // the fused backward's scratch (fp32 dQ accumulator + counters) is cached across calls
  // (grow-only, one per process): a stream-ordered allocation of hundreds of MB per call
  // would be re-mapped at every synchronisation and dominate the kernel's time
  static std::mutex mu;
  static void* scratch = nullptr;
  static size_t scratch_bytes = 0;
  float* acc = nullptr;
  int* ctr = nullptr;
  void* dsb = nullptr;
  int64_t dsb_bytes = 0;
  std::lock_guard<std::mutex> lk(mu);
  auto grow = [&](size_t need) -> pds_status {
    if (need > scratch_bytes) {
      PDS_CUDA(cudaStreamSynchronize(st));
      if (scratch) cudaFree(scratch);
      scratch = nullptr;
      scratch_bytes = 0;
      PDS_CUDA(cudaMalloc(&scratch, need));
      scratch_bytes = need;
    }
    return PDS_OK;
  };
  if (attn_bwd_fused_applies(d, causal) && s > 0) {
    const size_t acc_b = (size_t)heads * s * d * 4, need = acc_b + ((size_t)heads * (s / 128) + 1) * 4;
    PDS_TRY(grow(need));
    acc = static_cast<float*>(scratch);
    ctr = reinterpret_cast<int*>(static_cast<char*>(scratch) + acc_b);
  } else if (attn_bwd_mode() == 2 && (dsb_bytes = attn_ds_bytes(s, heads, heads, d, causal, kDsBudget)) > 0) {
    PDS_TRY(grow((size_t)dsb_bytes));               // dS through HBM
    dsb = scratch;
  }
  pds_status r = rc2s(attn_bwd(qkv, ld, out, ld_out, lse, dout, s, heads, d, causal, dqkv, nullptr, dd, st, acc, ctr,
                               0, nullptr, dsb, dsb_bytes), "pds_k_attn_bwd");
  cudaFreeAsync(dd, st);
  return r;
}

extern "C" pds_status pds_k_attn_fwd_gqa(const void* qkv, int64_t ld, int32_t s, int32_t heads, int32_t kv_heads,
                                         int32_t d, int32_t causal, void* out, int64_t ld_out, void* lse,
                                         void* stream) {
  if (!qkv || !out || !lse) PDS_FAIL(PDS_EINVAL, "NULL argument");
  if (kv_heads <= 0 || heads % kv_heads) PDS_FAIL(PDS_EINVAL, "kv_heads must divide heads");
  return rc2s(attn_fwd(qkv, ld, s, heads, d, causal, out, ld_out, lse, static_cast<cudaStream_t>(stream), kv_heads),
              "pds_k_attn_fwd_gqa");
}

extern "C" pds_status pds_k_attn_bwd_gqa(const void* qkv, int64_t ld, const void* out, int64_t ld_out,
                                         const void* lse, const void* dout, int32_t s, int32_t heads,
                                         int32_t kv_heads, int32_t d, int32_t causal, void* dqkv, void* stream) {
  if (!qkv || !out || !lse || !dout || !dqkv) PDS_FAIL(PDS_EINVAL, "NULL argument");
  if (kv_heads <= 0 || heads % kv_heads) PDS_FAIL(PDS_EINVAL, "kv_heads must divide heads");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* dd = nullptr;
  PDS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dd), (size_t)heads * s * 4, st));
  pds_status r = rc2s(attn_bwd(qkv, ld, out, ld_out, lse, dout, s, heads, d, causal, dqkv, nullptr, dd, st, nullptr,
                               nullptr, kv_heads), "pds_k_attn_bwd_gqa");
  cudaFreeAsync(dd, st);
  return r;
}

extern "C" pds_status pds_k_gemm_swiglu(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M, int32_t N,
                                        int32_t K, int32_t bwd, void* C, int64_t ldc, const void* h_in,
                                        int64_t ld_h, void* g_out, int64_t ld_g, void* c_t, void* g_t, int64_t ld_t,
                                        void* stream) {
  if (!A || !B || !C) PDS_FAIL(PDS_EINVAL, "NULL operand");
  if (!bwd && !g_out) PDS_FAIL(PDS_EINVAL, "SwiGLU forward needs g_out");
  if (bwd && !h_in) PDS_FAIL(PDS_EINVAL, "SwiGLU backward needs h_in");
  GemmArgs g;
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.M = M; g.N = N; g.K = K; g.C = C; g.ldc = ldc;
  g.epi = bwd ? EPI_DSWIGLU : EPI_SWIGLU;
  g.aux_in = h_in; g.ld_aux_in = ld_h; g.aux_out = g_out; g.ld_aux = ld_g;
  g.c_t = c_t; g.aux_t = g_t; g.ld_t = ld_t;
  return rc2s(gemm_launch(g, static_cast<cudaStream_t>(stream)), "pds_k_gemm_swiglu");
}

extern "C" pds_status pds_k_gemm_rope_gqa(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t M,
                                          int32_t N, int32_t K, void* C, int64_t ldc, const void* rope, int32_t d,
                                          int32_t hq, int32_t hk, void* stream) {
  if (!A || !B || !C || !rope) PDS_FAIL(PDS_EINVAL, "NULL operand");
  if (hq <= 0 || hk <= 0 || N % (hq + 2 * hk)) PDS_FAIL(PDS_EINVAL, "N must be a multiple of hq + 2 hk");
  GemmArgs g;
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.M = M; g.N = N; g.K = K; g.C = C; g.ldc = ldc;
  g.epi = EPI_ROPE; g.rope = reinterpret_cast<const float2*>(rope); g.rope_d = d; g.rope_hq = hq; g.rope_hk = hk;
  return rc2s(gemm_launch(g, static_cast<cudaStream_t>(stream)), "pds_k_gemm_rope_gqa");
}

extern "C" pds_status pds_k_attn_fwd_rows(const void* qkv, int64_t ld, int32_t s, int32_t heads, int32_t d,
                                          int32_t causal, int32_t qlo, int32_t qn, void* out, int64_t ld_out,
                                          void* lse, void* stream) {
  if (!qkv || !out || !lse) PDS_FAIL(PDS_EINVAL, "NULL argument");
  return rc2s(attn_fwd_rows(qkv, ld, s, heads, d, causal, qlo, qn, out, ld_out, lse,
                            static_cast<cudaStream_t>(stream)), "pds_k_attn_fwd_rows");
}

extern "C" pds_status pds_k_attn_bwd_rows(const void* qkv, int64_t ld, const void* out, int64_t ld_out,
                                          const void* lse, const void* dout, int32_t s, int32_t heads, int32_t d,
                                          int32_t causal, int32_t qlo, int32_t qn, void* dqkv, void* stream) {
  if (!qkv || !out || !lse || !dout || !dqkv) PDS_FAIL(PDS_EINVAL, "NULL argument");
  if (qn <= 0 || qn % 128) PDS_FAIL(PDS_EINVAL, "qn must be a positive multiple of 128");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* dd = nullptr;
  PDS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dd), (size_t)heads * qn * 4, st));
  pds_status r = rc2s(attn_bwd_rows(qkv, ld, out, ld_out, lse, dout, s, heads, d, causal, qlo, qn, dqkv, nullptr,
                                    dd, st), "pds_k_attn_bwd_rows");
  cudaFreeAsync(dd, st);
  return r;
}

extern "C" pds_status pds_k_attn_fwd_pair(const void* q, int64_t ld_q, const void* kv, int64_t ld_kv, int32_t kcol,
                                          int32_t vcol, int32_t sq, int32_t sk, int32_t heads, int32_t d,
                                          int32_t causal, void* out, int64_t ld_out, void* lse, void* stream) {
  if (!q || !kv || !out || !lse) PDS_FAIL(PDS_EINVAL, "NULL argument");
  return rc2s(attn_fwd_pair(q, ld_q, kv, ld_kv, kcol, vcol, sq, sk, heads, d, causal, out, ld_out, lse,
                            static_cast<cudaStream_t>(stream)), "pds_k_attn_fwd_pair");
}

extern "C" pds_status pds_k_attn_bwd_pair(const void* q, int64_t ld_q, const void* kv, int64_t ld_kv, int32_t kcol,
                                          int32_t vcol, const void* dout, int64_t ld_out, const void* lse,
                                          const void* Dd, int32_t sq, int32_t sk, int32_t heads, int32_t d,
                                          int32_t causal, void* dq_acc, int64_t ld_dqa, void* dkv_acc,
                                          int64_t ld_dkva, void* stream) {
  if (!q || !kv || !dout || !lse || !Dd || !dq_acc || !dkv_acc) PDS_FAIL(PDS_EINVAL, "NULL argument");
  return rc2s(attn_bwd_pair(q, ld_q, kv, ld_kv, kcol, vcol, dout, ld_out, lse, static_cast<const float*>(Dd), sq, sk,
                            heads, d, causal, static_cast<float*>(dq_acc), ld_dqa, static_cast<float*>(dkv_acc),
                            ld_dkva, static_cast<cudaStream_t>(stream)), "pds_k_attn_bwd_pair");
}

extern "C" pds_status pds_k_attn_merge(void* o_acc, int64_t ld_oacc, void* l_acc, int64_t lstride_acc,
                                       const void* o_p, int64_t ld_op, const void* l_p, int64_t lstride_p,
                                       int32_t rows, int32_t heads, int32_t d, int32_t first, void* out,
                                       int64_t ld_out, void* stream) {
  if (!o_acc || !l_acc || !o_p || !l_p) PDS_FAIL(PDS_EINVAL, "NULL argument");
  return rc2s(attn_merge(static_cast<float*>(o_acc), ld_oacc, static_cast<float*>(l_acc), lstride_acc, o_p, ld_op,
                         static_cast<const float*>(l_p), lstride_p, rows, heads, d, first, out, ld_out,
                         static_cast<cudaStream_t>(stream)), "pds_k_attn_merge");
}

extern "C" pds_status pds_k_attn_dot(const void* out, int64_t ld_out, const void* dout, int32_t s, int32_t heads,
                                     int32_t d, void* Dd, void* stream) {
  if (!out || !dout || !Dd) PDS_FAIL(PDS_EINVAL, "NULL argument");
  return rc2s(attn_dot(out, ld_out, dout, s, heads, d, static_cast<float*>(Dd), static_cast<cudaStream_t>(stream)),
              "pds_k_attn_dot");
}

extern "C" pds_status pds_set_attn_bwd(int32_t mode) {
  if (mode < 0 || mode > 2)
    PDS_FAIL(PDS_EINVAL, "attention backward mode must be 0 (split), 1 (fused) or 2 (dS through HBM)");
  set_attn_bwd_mode(mode);
  return PDS_OK;
}

extern "C" pds_status pds_debug_trace(int64_t* host_out, int32_t rows) {
  if (!host_out || rows <= 0 || rows > 4096) PDS_FAIL(PDS_EINVAL, "bad trace buffer");
  const int rc = attn_debug_trace(reinterpret_cast<long long*>(host_out), rows);
  if (rc < 0) PDS_FAIL(PDS_ENOTIMPL, "library built without PDS_TRACE");
  if (rc) PDS_FAIL(PDS_ECUDA, "trace copy failed");
  return PDS_OK;
}
