// Attention backward helper and dispatch (Eq. 2; causal per north_star,
// reading R-1).  The tcgen05 / TMEM kernels live in attn_tc.cu; this file holds
// D = rowsum(dO o O) (the one reduction the backward needs before its MMAs) and the
// entry points the layer calls.  The round-1 warp-level mma.sync FA2 kernels are no
// longer part of the product library: they moved to tools/fa2_sync_baseline.cu (an
// A/B baseline built separately, see its header).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

namespace pds {

// ------------------------------------------------------------------ backward: D = rowsum(dO o O)
// (also zeroes the fused backward's nctr turn / ticket counters, one per thread)
__global__ void attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ out, int64_t ld_out,
                                    const __nv_bfloat16* __restrict__ dout, int s, int heads, int d,
                                    float* __restrict__ Dd, int* __restrict__ ctr, int nctr) {
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi < nctr) ctr[gi] = 0;
  const int warp = gi >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= s * heads) return;
  const int row = warp / heads, head = warp % heads;
  const __nv_bfloat16* o = out + (int64_t)row * ld_out + head * d;
  const __nv_bfloat16* g = dout + (int64_t)row * ld_out + head * d;
  float acc = 0.f;
  for (int c = lane * 2; c < d; c += 64) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + c));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(g + c));
    acc += a.x * b.x + a.y * b.y;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, off);
  if (lane == 0) Dd[(int64_t)head * s + row] = acc;
}

int attn_fwd_tc(const void* qkv, int64_t ld, int s, int heads, int d, int causal, void* out, int64_t ld_out,
                void* lse, cudaStream_t st, int qlo = 0, int qn = -1, int kv_heads = 0,
                const int* segs = nullptr);

int attn_fwd(const void* qkv, int64_t ld, int s, int heads, int d, int causal, void* out,
             int64_t ld_out, void* lse, cudaStream_t st, int kv_heads, const int* segs) {
  return attn_fwd_tc(qkv, ld, s, heads, d, causal, out, ld_out, lse, st, 0, -1, kv_heads, segs);
}

int attn_bwd_tc(const void* qkv, int64_t ld, const void* dout, int64_t ld_out, const void* lse, const float* Dd,
                int s, int heads, int d, int causal, void* dqkv, const void* rope, cudaStream_t st, int qlo = 0,
                int qn = -1, int kv_heads = 0, const int* segs = nullptr);

int attn_bwd_fused_tc(const void* qkv, int64_t ld, const void* dout, int64_t ld_out, const void* lse, const float* Dd,
                      int s, int heads, void* dqkv, const void* rope, float* dqacc, int* ctr, cudaStream_t st);
int attn_bwd_ds_tc(const void* qkv, int64_t ld, const void* dout, int64_t ld_out, const void* lse, const float* Dd,
                   int s, int heads, int kv_heads, void* dqkv, const void* rope, void* dsbuf, int64_t ds_bytes,
                   cudaStream_t st);

int64_t attn_ds_bytes(int64_t s, int heads, int kv_heads, int d, int causal, int64_t budget) {
  if (d != 128 || !causal || s <= 0 || s % 128) return 0;
  if (kv_heads <= 0) kv_heads = heads;
  const int grp = heads / kv_heads;
  const int64_t per = s * s * 2;
  int64_t G = std::min<int64_t>(heads, budget / per);
  G -= G % grp;
  return G >= 1 ? G * per : 0;
}

// 0: split dK/dV + dQ kernels (default), 1: fused kernel where it applies, 2: dS through HBM
// for the kernel-level entry points (pds_set_attn_bwd; the layer path picks dS by its plan).
// The fused kernel executes 5 matmuls instead of 7 but adds 64 KB of fp32 dQ reduction per
// (key block, query block) pair through L2, which B200's L2 reduction throughput cannot
// sustain at this tile shape: measured slower.
static int g_bwd_mode = 0;
void set_attn_bwd_mode(int mode) { g_bwd_mode = mode; }
bool attn_bwd_fused_applies(int d, int causal) { return g_bwd_mode == 1 && d == 128 && causal; }
int attn_bwd_mode() { return g_bwd_mode; }

int attn_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* lse,
             const void* dout, int s, int heads, int d, int causal, void* dqkv, const void* rope,
             float* Dd, cudaStream_t st, float* dqacc, int* ctr, int kv_heads, const int* segs, void* dsbuf,
             int64_t ds_bytes) {
  if (s % 128) return (int)cudaErrorInvalidValue;
  if (kv_heads <= 0) kv_heads = heads;
  const bool dspath = dsbuf && !segs && d == 128 && causal && ds_bytes >= (int64_t)s * s * 2 * (heads / kv_heads);
  const bool fused = dqacc && ctr && attn_bwd_fused_applies(d, causal) && kv_heads == heads && !segs;
  const int nctr = fused ? heads * (s / 128) + 1 : 0;
  const int nblk = (s * heads + 7) / 8;
  if (nctr > nblk * 256) return (int)cudaErrorInvalidValue;
  attn_bwd_dot_kernel<<<nblk, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(out), ld_out,
                                            reinterpret_cast<const __nv_bfloat16*>(dout), s, heads, d, Dd, ctr,
                                            nctr);
  if (fused) return attn_bwd_fused_tc(qkv, ld, dout, ld_out, lse, Dd, s, heads, dqkv, rope, dqacc, ctr, st);
  if (dspath) return attn_bwd_ds_tc(qkv, ld, dout, ld_out, lse, Dd, s, heads, kv_heads, dqkv, rope, dsbuf, ds_bytes, st);
  return attn_bwd_tc(qkv, ld, dout, ld_out, lse, Dd, s, heads, d, causal, dqkv, rope, st, 0, -1, kv_heads, segs);
}

// Context parallelism (MegatronCZ): queries [qlo, qlo + qn) of the s positions against
// all keys of qkv [s][ld]; out [qn][ld_out], lse / Dd [heads][qn] local.  Backward:
// dQ rows [qlo, qlo + qn) and the dK / dV contributions of those queries to every key
// row into dqkv [s][ld] (key blocks past the last query, causal, are not written).
int attn_fwd_rows(const void* qkv, int64_t ld, int s, int heads, int d, int causal, int qlo, int qn, void* out,
                  int64_t ld_out, void* lse, cudaStream_t st) {
  return attn_fwd_tc(qkv, ld, s, heads, d, causal, out, ld_out, lse, st, qlo, qn);
}

int attn_bwd_rows(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* lse,
                  const void* dout, int s, int heads, int d, int causal, int qlo, int qn, void* dqkv,
                  const void* rope, float* Dd, cudaStream_t st) {
  if (qn % 128 || qn <= 0) return (int)cudaErrorInvalidValue;
  attn_bwd_dot_kernel<<<(qn * heads + 7) / 8, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(out), ld_out,
                                                           reinterpret_cast<const __nv_bfloat16*>(dout), qn, heads,
                                                           d, Dd, nullptr, 0);
  return attn_bwd_tc(qkv, ld, dout, ld_out, lse, Dd, s, heads, d, causal, dqkv, rope, st, qlo, qn);
}

// ------------------------------------------------------------------ ring attention helpers
// Log-sum-exp merge of a pair's partial attention (o_p bf16 [rows][ld_op], l_p fp32
// [heads][lstride_p]) into the running result (o_acc fp32 [rows][ld_oacc], l_acc fp32
// [heads][lstride_acc]): L = log(e^La + e^Lp), O = e^(La-L) O_acc + e^(Lp-L) O_p.
// first: the accumulator is empty (copy).  out (nullable): also write bf16 O.
// Thread = (row, head, 8 columns); d / 8 threads per (row, head).
__global__ void attn_merge_kernel(float* __restrict__ o_acc, int64_t ld_oacc, float* __restrict__ l_acc,
                                  int64_t lstride_acc, const __nv_bfloat16* __restrict__ o_p, int64_t ld_op,
                                  const float* __restrict__ l_p, int64_t lstride_p, int rows, int heads, int d,
                                  int first, __nv_bfloat16* __restrict__ out, int64_t ld_out) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = d / 8;
  if (gi >= (int64_t)rows * heads * per) return;
  const int g = (int)(gi % per), head = (int)((gi / per) % heads), row = (int)(gi / ((int64_t)per * heads));
  const float lp = l_p[(int64_t)head * lstride_p + row];
  float* la_p = l_acc + (int64_t)head * lstride_acc + row;
  const float la = first ? -INFINITY : *la_p;
  const float m = fmaxf(la, lp);
  float wa = 0.f, wp = 0.f, L = -INFINITY;
  if (m > -INFINITY) {
    const float ea = expf(la - m), ep = expf(lp - m);
    L = m + logf(ea + ep);
    wa = ea / (ea + ep);
    wp = ep / (ea + ep);
  }
  float* oa = o_acc + (int64_t)row * ld_oacc + head * d + 8 * g;
  const __nv_bfloat16* op = o_p + (int64_t)row * ld_op + head * d + 8 * g;
  const uint4 pv = *reinterpret_cast<const uint4*>(op);
  const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&pv);
  float v[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(p2[i]);
    v[2 * i] = f.x * wp;
    v[2 * i + 1] = f.y * wp;
  }
  if (!first) {
    const float4 a0 = reinterpret_cast<const float4*>(oa)[0], a1 = reinterpret_cast<const float4*>(oa)[1];
    v[0] += a0.x * wa; v[1] += a0.y * wa; v[2] += a0.z * wa; v[3] += a0.w * wa;
    v[4] += a1.x * wa; v[5] += a1.y * wa; v[6] += a1.z * wa; v[7] += a1.w * wa;
  }
  reinterpret_cast<float4*>(oa)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(oa)[1] = make_float4(v[4], v[5], v[6], v[7]);
  if (out) {
    __nv_bfloat162 b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(out + (int64_t)row * ld_out + head * d + 8 * g) = *reinterpret_cast<const uint4*>(b);
  }
  if (g == 0) *la_p = L;
}

int attn_merge(float* o_acc, int64_t ld_oacc, float* l_acc, int64_t lstride_acc, const void* o_p, int64_t ld_op,
               const float* l_p, int64_t lstride_p, int rows, int heads, int d, int first, void* out, int64_t ld_out,
               cudaStream_t st) {
  if (d % 8 || ld_oacc % 4 || ld_op % 8 || (out && ld_out % 8)) return (int)cudaErrorInvalidValue;
  const int64_t n = (int64_t)rows * heads * (d / 8);
  if (n == 0) return 0;
  attn_merge_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      o_acc, ld_oacc, l_acc, lstride_acc, reinterpret_cast<const __nv_bfloat16*>(o_p), ld_op, l_p, lstride_p, rows,
      heads, d, first, reinterpret_cast<__nv_bfloat16*>(out), ld_out);
  return (int)cudaGetLastError();
}

// fp32 [rows][ld_src] -> bf16 [rows][ld_dst], `cols` columns; rope (nullable): RoPE^T on
// every head's (k, k + d/2) pairs at position pos(row) = (row < half ? base0 : base1) +
// (row % half) / b  (two position runs: a zigzag pair of half-chunks of b sequences).
// Thread = (row, one pair column k of one head) -> columns k and k + d/2.
__global__ void rope_t_f32_bf16_kernel(const float* __restrict__ src, int64_t ld_src, int rows, int cols, int d,
                                       const float2* __restrict__ rope, int64_t base0, int64_t base1, int half,
                                       int b, __nv_bfloat16* __restrict__ dst, int64_t ld_dst) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int pairs = cols / 2;
  if (gi >= (int64_t)rows * pairs) return;
  const int row = (int)(gi / pairs), pc = (int)(gi % pairs);
  const int head = pc / (d / 2), k = pc % (d / 2);
  const float* s = src + (int64_t)row * ld_src + head * d;
  float x = s[k], y = s[k + d / 2];
  if (rope) {
    const int64_t pos = (row < half ? base0 : base1) + (row % half) / b;
    const float2 cs = rope[pos * (d / 2) + k];
    const float nx = x * cs.x + y * cs.y;
    y = -x * cs.y + y * cs.x;
    x = nx;
  }
  __nv_bfloat16* o = dst + (int64_t)row * ld_dst + head * d;
  o[k] = __float2bfloat16_rn(x);
  o[k + d / 2] = __float2bfloat16_rn(y);
}

int rope_t_f32_bf16(const float* src, int64_t ld_src, int rows, int cols, int d, const void* rope, int64_t base0,
                    int64_t base1, int half, int b, void* dst, int64_t ld_dst, cudaStream_t st) {
  if (cols % d || d % 2 || half <= 0 || b <= 0) return (int)cudaErrorInvalidValue;
  const int64_t n = (int64_t)rows * (cols / 2);
  if (n == 0) return 0;
  rope_t_f32_bf16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      src, ld_src, rows, cols, d, reinterpret_cast<const float2*>(rope), base0, base1, half, b,
      reinterpret_cast<__nv_bfloat16*>(dst), ld_dst);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ Ring Self-Attention (ColossalZ)
// Row softmax of materialised scores (R-COL): p[row][c] = exp(scale S - max) / sum over
// the visible columns (causal: c <= pos(row), pos(row) = pos0 + row % rows_per_head),
// bf16 out.  One warp per row.
__global__ void rsa_softmax_kernel(const float* __restrict__ S, int64_t lds, int rows, int cols, int rows_per_head,
                                   int64_t pos0, int causal, float scale, __nv_bfloat16* __restrict__ Pr,
                                   int64_t ldp) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float* srow = S + (int64_t)warp * lds;
  __nv_bfloat16* prow = Pr + (int64_t)warp * ldp;
  const int64_t last = causal ? pos0 + warp % rows_per_head : (int64_t)cols - 1;   // last visible column
  const int nv = (int)(last + 1 < cols ? last + 1 : cols);
  float m = -INFINITY;
  for (int c = lane; c < nv; c += 32) m = fmaxf(m, srow[c] * scale);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
  float l = 0.f;
  for (int c = lane; c < nv; c += 32) l += expf(srow[c] * scale - m);
#pragma unroll
  for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffff, l, o);
  const float inv = 1.0f / l;
  for (int c = lane; c < cols; c += 32)
    prow[c] = __float2bfloat16_rn(c < nv ? expf(srow[c] * scale - m) * inv : 0.f);
}

int rsa_softmax(const float* S, int64_t lds, int rows, int cols, int rows_per_head, int64_t pos0, int causal,
                float scale, void* Pr, int64_t ldp, cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || rows_per_head <= 0) return (int)cudaErrorInvalidValue;
  rsa_softmax_kernel<<<(rows + 7) / 8, 256, 0, st>>>(S, lds, rows, cols, rows_per_head, pos0, causal, scale,
                                                     reinterpret_cast<__nv_bfloat16*>(Pr), ldp);
  return (int)cudaGetLastError();
}

// dS = scale * P o (dP - D[row]) (bf16), P bf16, dP fp32, D fp32 [rows]
__global__ void rsa_dsoftmax_kernel(const __nv_bfloat16* __restrict__ Pr, int64_t ldp, const float* __restrict__ dP,
                                    int64_t lddp, const float* __restrict__ D, int rows, int cols, float scale,
                                    __nv_bfloat16* __restrict__ dS, int64_t ldds) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = cols / 8;
  if (gi >= (int64_t)rows * per) return;
  const int row = (int)(gi / per), c = (int)(gi % per) * 8;
  const uint4 pv = *reinterpret_cast<const uint4*>(Pr + (int64_t)row * ldp + c);
  const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&pv);
  const float4 a = *reinterpret_cast<const float4*>(dP + (int64_t)row * lddp + c);
  const float4 b = *reinterpret_cast<const float4*>(dP + (int64_t)row * lddp + c + 4);
  const float dd = D[row];
  const float dp[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  __nv_bfloat162 o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 p = __bfloat1622float2(p2[i]);
    o[i] = __floats2bfloat162_rn(scale * p.x * (dp[2 * i] - dd), scale * p.y * (dp[2 * i + 1] - dd));
  }
  *reinterpret_cast<uint4*>(dS + (int64_t)row * ldds + c) = *reinterpret_cast<const uint4*>(o);
}

int rsa_dsoftmax(const void* Pr, int64_t ldp, const float* dP, int64_t lddp, const float* D, int rows, int cols,
                 float scale, void* dS, int64_t ldds, cudaStream_t st) {
  if (cols % 8 || ldp % 8 || lddp % 4 || ldds % 8) return (int)cudaErrorInvalidValue;
  const int64_t n = (int64_t)rows * (cols / 8);
  if (n == 0) return 0;
  rsa_dsoftmax_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(Pr), ldp, dP, lddp, D, rows, cols, scale,
      reinterpret_cast<__nv_bfloat16*>(dS), ldds);
  return (int)cudaGetLastError();
}

// D = rowsum(dO o O) alone (ring attention: once per layer on the zigzag rows)
int attn_dot(const void* out, int64_t ld_out, const void* dout, int s, int heads, int d, float* Dd, cudaStream_t st) {
  attn_bwd_dot_kernel<<<(s * heads + 7) / 8, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(out), ld_out,
                                                          reinterpret_cast<const __nv_bfloat16*>(dout), s, heads, d,
                                                          Dd, nullptr, 0);
  return (int)cudaGetLastError();
}

}  // namespace pds
