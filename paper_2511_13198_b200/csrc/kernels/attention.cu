// Attention backward helper and dispatch (Eq. 2; causal per north_star,
// reading R-1).  The tcgen05 / TMEM kernels live in attn_tc.cu; this file holds
// D = rowsum(dO o O) (the one reduction the backward needs before its MMAs) and the
// entry points the layer calls.  The round-1 warp-level mma.sync FA2 kernels are no
// longer part of the product library: they moved to tools/fa2_sync_baseline.cu (an
// A/B baseline built separately, see its header).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
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
                void* lse, cudaStream_t st, int qlo = 0, int qn = -1);

int attn_fwd(const void* qkv, int64_t ld, int s, int heads, int d, int causal, void* out,
             int64_t ld_out, void* lse, cudaStream_t st) {
  return attn_fwd_tc(qkv, ld, s, heads, d, causal, out, ld_out, lse, st);
}

int attn_bwd_tc(const void* qkv, int64_t ld, const void* dout, int64_t ld_out, const void* lse, const float* Dd,
                int s, int heads, int d, int causal, void* dqkv, const void* rope, cudaStream_t st, int qlo = 0,
                int qn = -1);

int attn_bwd_fused_tc(const void* qkv, int64_t ld, const void* dout, int64_t ld_out, const void* lse, const float* Dd,
                      int s, int heads, void* dqkv, const void* rope, float* dqacc, int* ctr, cudaStream_t st);

// 0: split dK/dV + dQ kernels (default), 1: fused kernel where it applies (pds_set_attn_bwd).
// The fused kernel executes 5 matmuls instead of 7 but adds 64 KB of fp32 dQ reduction per
// (key block, query block) pair through L2, which B200's L2 reduction throughput cannot
// sustain at this tile shape: measured slower.
static int g_bwd_mode = 0;
void set_attn_bwd_mode(int mode) { g_bwd_mode = mode; }
bool attn_bwd_fused_applies(int d, int causal) { return g_bwd_mode == 1 && d == 128 && causal; }

int attn_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* lse,
             const void* dout, int s, int heads, int d, int causal, void* dqkv, const void* rope,
             float* Dd, cudaStream_t st, float* dqacc, int* ctr) {
  if (s % 128) return (int)cudaErrorInvalidValue;
  const bool fused = dqacc && ctr && attn_bwd_fused_applies(d, causal);
  const int nctr = fused ? heads * (s / 128) + 1 : 0;
  const int nblk = (s * heads + 7) / 8;
  if (nctr > nblk * 256) return (int)cudaErrorInvalidValue;
  attn_bwd_dot_kernel<<<nblk, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(out), ld_out,
                                            reinterpret_cast<const __nv_bfloat16*>(dout), s, heads, d, Dd, ctr,
                                            nctr);
  if (fused) return attn_bwd_fused_tc(qkv, ld, dout, ld_out, lse, Dd, s, heads, dqkv, rope, dqacc, ctr, st);
  return attn_bwd_tc(qkv, ld, dout, ld_out, lse, Dd, s, heads, d, causal, dqkv, rope, st);
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

}  // namespace pds
