// Persistent, warp-specialised tcgen05 GEMMs for sm_100a with fused epilogues.
//
// The dense contractions of the layer (Eqs. 1, 3, 4 and their
// gradients) all run here:  C[M,N] = A[M,K] * B[N,K]^T, bf16 operands staged by
// TMA (SWIZZLE_128B) into a shared-memory ring, one elected thread issuing
// tcgen05.mma into a double-buffered TMEM accumulator, epilogue warps draining
// TMEM with tcgen05.ld while the next tile accumulates.  Two kernels:
//
//   gemm_tc_kernel   1 CTA, M = 128, N = BN (128 / 256) per MMA, 4-6 stages;
//                    warps 4..7 epilogue (TMEM lanes 32*(warp%4) .. +31, one
//                    output row per thread)
//   gemm2_tc_kernel  CTA pair (cluster of 2, cta_group::2): M = 256, N = 256 per
//                    MMA, each CTA stages half of A and half of B (6 x 32 KB),
//                    TMA completion on the leader's mbarrier, commits multicast to
//                    both CTAs; warps 4..11 epilogue, two warpgroups splitting the
//                    256 accumulator columns
//
//   warp 0      TMA producer (one elected lane)
//   warp 1      MMA issuer   (one elected lane; the leader CTA's in the pair kernel)
//   warp 2      TMEM allocator
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "gemm.cuh"
#include "ptx.cuh"

namespace pds {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int GROUP_M = 16;

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

struct EpiParams {
  int M, N;
  void* C;
  int64_t ldc;
  int epi;
  int blk_w;
  int64_t blk_stride;
  const __nv_bfloat16* aux_in;
  __nv_bfloat16* aux_out;
  int64_t ld_aux, ld_aux_in;
  const float2* rope;
  int rope_d, rope_hq, rope_hk, rope_b;
  const int* rope_segs;
  int64_t seg, seg_stride, seg_base;
  int64_t c_seg, c_stride, c_base;
  __nv_bfloat16* c_t;      // transposed copies (dGELU epilogue): [N][ld_t]
  __nv_bfloat16* aux_t;
  int64_t ld_t;
  // collective overlap (gemm.cuh): chunk flags / counters, tile rotation in M blocks
  const uint32_t* wait_flags;
  uint32_t flag_epoch;
  uint32_t* done_ctr;
  int chunk_rows;
  int rot_mb;
  int chunk_cols;      // > 0: done_ctr counts per column block instead of per row chunk
  int rot_nb;
  // batched / causal-K problems (gemm.cuh)
  int batch;
  int64_t a_boff, b_boff, c_boff;
  int b_grp;
  int k_causal;
  float epi_scale;
};

// AG -> GEMM: wait until every chunk overlapping rows [r0, r0 + n) has landed.  The
// flag is written by the collective's stream (after its copy) with release semantics;
// the acquire load plus a generic -> async proxy fence make the landed rows visible to
// the TMA loads that follow.  A chunk that never lands is a bug: trap after > 30 s
// instead of hanging the device.
__device__ __forceinline__ void wait_chunks(const EpiParams& ep, int r0, int n) {
  if (!ep.wait_flags || n <= 0) return;
  const int c0 = r0 / ep.chunk_rows, c1 = (r0 + n - 1) / ep.chunk_rows;
  for (int c = c0; c <= c1; ++c) {
    uint32_t spins = 0;
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ep.wait_flags + c) : "memory");
      if ((int32_t)(v - ep.flag_epoch) >= 0) break;
      __nanosleep(128);
      if (++spins > (1u << 28)) __trap();
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// GEMM -> RS / A2A: one epilogue warp has stored its 32 rows x `ncols` columns; count
// them, in units of 8 elements (N and the column blocks are multiples of 8, and the
// unit keeps a chunk's per-call growth far below 2^31), into the chunk's counter once
// every lane's stores are ordered before the add.
__device__ __forceinline__ void count_stored(const EpiParams& ep, int warp_row0, bool row_ok, int n0, int ncols) {
  if (!ep.done_ctr) return;
  const unsigned vm = __ballot_sync(0xffffffffu, row_ok);
  __threadfence();
  __syncwarp();
  if ((threadIdx.x & 31) == 0 && vm && ncols > 0) {
    const uint32_t nrows = __popc(vm);
    if (ep.chunk_cols > 0) {            // column blocks (All-to-All): split the range over blocks
      for (int c = n0; c < n0 + ncols;) {
        const int blk = c / ep.chunk_cols;
        const int end = min(n0 + ncols, (blk + 1) * ep.chunk_cols);
        atomicAdd(ep.done_ctr + blk, nrows * (uint32_t)((end - c) >> 3));
        c = end;
      }
    } else {
      atomicAdd(ep.done_ctr + warp_row0 / ep.chunk_rows, nrows * (uint32_t)(ncols >> 3));
    }
  }
}

struct RowMap {
  int64_t seg, stride, base;
  __device__ __forceinline__ int map(int r) const {
    return (int)((r / seg) * stride + base + (r % seg));
  }
};

// Phi(x) (standard normal CDF) and phi(x) sharing one exponential: erf(|x|/sqrt 2) by
// Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7, far below the bf16 rounding of the
// outputs), e^{-x^2/2} serving both the erf tail and the density.
__device__ __forceinline__ void normal_cdf_pdf(float x, float& cdf, float& pdf) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = __fdividef(1.0f, fmaf(0.3275911f, z, 1.0f));
  float poly = fmaf(1.061405429f, t, -1.453152027f);
  poly = fmaf(poly, t, 1.421413741f);
  poly = fmaf(poly, t, -0.284496736f);
  poly = fmaf(poly, t, 0.254829592f);
  poly *= t;
  const float e = __expf(-0.5f * x * x);
  const float erf_abs = fmaf(-poly, e, 1.0f);
  cdf = 0.5f + 0.5f * copysignf(erf_abs, x);
  pdf = 0.39894228040143268f * e;
}
__device__ __forceinline__ float gelu_f(float x) {
  float cdf, pdf;
  normal_cdf_pdf(x, cdf, pdf);
  return x * cdf;
}
__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}
// SiLU(x) = x sigma(x) and sigma(x) (R-SWIGLU)
__device__ __forceinline__ float sigmoid_f(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

__device__ __forceinline__ int rot_block(int mb, int mt, int rot) {
  return rot ? (mb + rot) % mt : mb;
}

__device__ __forceinline__ void tile_coords(int t, int mt, int nt, int& mb, int& nb, int group_m = GROUP_M) {
  const int band = t / (group_m * nt);
  const int first = band * group_m;
  const int gm = min(group_m, mt - first);
  const int idx = t - band * group_m * nt;
  mb = first + idx % gm;
  nb = idx / gm;
}

// transposed store: element (row, col + i) -> dst[(col + i) * ld + row]; the 32 lanes
// of a warp hold 32 consecutive rows, so each column is one 64-byte segment
__device__ __forceinline__ void store_col32_bf16(__nv_bfloat16* dst, int64_t ld, int row, int col, const float* v,
                                                 int valid) {
  __nv_bfloat16* p = dst + (int64_t)col * ld + row;
  if (valid == 32) {                           // full chunk: no predicates, one pointer walk
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const __nv_bfloat162 b = __floats2bfloat162_rn(v[i], v[i + 1]);
      p[0] = b.x;
      p[ld] = b.y;
      p += 2 * ld;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < valid) p[(int64_t)i * ld] = __float2bfloat16_rn(v[i]);
  }
}

// store 32 consecutive bf16 values of one row
__device__ __forceinline__ void store_row32_bf16(__nv_bfloat16* dst, const float* v, int valid) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q * 8 < valid) {
      uint4 w;
      w.x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
      w.y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
      w.z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
      w.w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
      d4[q] = w;
    }
  }
}
__device__ __forceinline__ void load_row32_bf16(const __nv_bfloat16* src, float* v, int valid) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 w = make_uint4(0, 0, 0, 0);
    if (q * 8 < valid) w = s4[q];
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(b[e]);
      v[q * 8 + 2 * e] = f.x;
      v[q * 8 + 2 * e + 1] = f.y;
    }
  }
}

__device__ __forceinline__ int64_t out_offset(const EpiParams& p, int row_l, int col) {
  const int64_t row = (row_l / p.c_seg) * p.c_stride + p.c_base + (row_l % p.c_seg);
  if (p.blk_w > 0) {
    const int blk = col / p.blk_w;
    return (int64_t)blk * p.blk_stride + (int64_t)row * p.ldc + (col - blk * p.blk_w);
  }
  return (int64_t)row * p.ldc + col;
}

// Drain one accumulator tile (this thread's row, BN columns at TMEM address tbase)
// through the fused epilogue.  Called by the four epilogue warps (warp-collective
// tcgen05.ld, so every lane executes every load).
template <int BN>
__device__ __forceinline__ void epilogue_tile(const EpiParams& ep, uint32_t tbase, int row, bool row_ok,
                                              int n0, int N, int bz = 0) {
  if (ep.epi == EPI_ROPE_T) {
    // RoPE^T (rotation by -angle) of the scaled accumulator, d = BN = 128 (one head per tile)
    constexpr int D2 = BN / 2;
    __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(ep.C) + (int64_t)bz * ep.c_boff;
    for (int j0 = 0; j0 < D2; j0 += 32) {
      uint32_t r1[32], r2[32];
      tmem_ld32(tbase + j0, r1);
      tmem_ld32(tbase + j0 + D2, r2);
      tmem_ld_wait();
      if (row_ok) {
        const float2* cs = ep.rope ? ep.rope + (int64_t)row * D2 + j0 : nullptr;   // NULL: no rotation
        float v1[32], v2[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float2 c = cs ? cs[i] : make_float2(1.0f, 0.0f);
          const float a = __uint_as_float(r1[i]) * ep.epi_scale, b = __uint_as_float(r2[i]) * ep.epi_scale;
          v1[i] = a * c.x + b * c.y;
          v2[i] = -a * c.y + b * c.x;
        }
        store_row32_bf16(C + (int64_t)row * ep.ldc + j0, v1, 32);
        store_row32_bf16(C + (int64_t)row * ep.ldc + j0 + D2, v2, 32);
      }
      __syncwarp();
    }
  } else if (ep.epi == EPI_ROPE) {
    const int d = ep.rope_d, d2 = d >> 1;
    int64_t pos = 0;
    if (row_ok) {
      const int64_t r = row;
      pos = ((r / ep.seg) * ep.seg_stride + ep.seg_base + (r % ep.seg)) / ep.rope_b;
      if (ep.rope_segs) pos -= (int64_t)ep.rope_segs[2 * (pos >> 7)] * 128;   // position in its sequence
    }
    for (int hs = 0; hs < BN; hs += d) {
      for (int j0 = 0; j0 < d2; j0 += 32) {
        uint32_t r1[32], r2[32];
        tmem_ld32(tbase + hs + j0, r1);
        tmem_ld32(tbase + hs + j0 + d2, r2);
        tmem_ld_wait();
        const int c1 = n0 + hs + j0;
        if (row_ok && c1 < N) {
        float v1[32], v2[32];
        const int within = (n0 + hs) % (ep.rope_hq + 2 * ep.rope_hk);
        if (within < ep.rope_hq + ep.rope_hk) {
          const float2* cs = ep.rope + pos * d2 + j0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float2 c = cs[i];
            const float a = __uint_as_float(r1[i]), b = __uint_as_float(r2[i]);
            v1[i] = a * c.x - b * c.y;
            v2[i] = a * c.y + b * c.x;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v1[i] = __uint_as_float(r1[i]);
            v2[i] = __uint_as_float(r2[i]);
          }
        }
        __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(ep.C);
        store_row32_bf16(C + out_offset(ep, row, c1), v1, 32);
        store_row32_bf16(C + out_offset(ep, row, c1 + d2), v2, 32);
        }
        __syncwarp();
      }
    }
  } else if (ep.epi == EPI_SWIGLU) {
    // each 128-column group of the tile is one (gate_j | up_j) pair of 64-column blocks
    for (int g0 = 0; g0 < BN; g0 += 128) {
      for (int cc = 0; cc < 64; cc += 32) {
        uint32_t rg[32], ru[32];
        tmem_ld32(tbase + g0 + cc, rg);
        tmem_ld32(tbase + g0 + 64 + cc, ru);
        tmem_ld_wait();
        const int col = n0 + g0 + cc;
        if (row_ok && col < N) {
          float vg[32], vu[32], g[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            vg[i] = __uint_as_float(rg[i]);
            vu[i] = __uint_as_float(ru[i]);
            const float x = bf16_round(vg[i]);
            g[i] = x * sigmoid_f(x) * bf16_round(vu[i]);
          }
          __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(ep.C);
          store_row32_bf16(C + out_offset(ep, row, col), vg, 32);
          store_row32_bf16(C + out_offset(ep, row, col + 64), vu, 32);
          store_row32_bf16(ep.aux_out + (int64_t)row * ep.ld_aux + (n0 + g0) / 2 + cc, g, 32);
        }
        __syncwarp();
      }
    }
  } else if (ep.epi == EPI_DSWIGLU) {
    for (int cc = 0; cc < BN; cc += 32) {
      uint32_t r[32];
      tmem_ld32(tbase + cc, r);
      tmem_ld_wait();
      const int col = n0 + cc;                           // FFN column of dG
      if (row_ok && col < N) {
        const int valid = min(32, N - col);
        const int hc = (col >> 6) * 128 + (col & 63);    // its gate column in H / dH
        float gt[32], up[32], dgt[32], dup[32], g[32];
        const __nv_bfloat16* hrow = ep.aux_in + (int64_t)row * ep.ld_aux_in;
        load_row32_bf16(hrow + hc, gt, valid);
        load_row32_bf16(hrow + hc + 64, up, valid);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float dg = __uint_as_float(r[i]);
          const float sg = sigmoid_f(gt[i]);
          const float si = gt[i] * sg;
          g[i] = si * up[i];
          dup[i] = dg * si;
          dgt[i] = dg * up[i] * sg * fmaf(gt[i], 1.0f - sg, 1.0f);
        }
        __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(ep.C);
        store_row32_bf16(C + out_offset(ep, row, hc), dgt, valid);
        store_row32_bf16(C + out_offset(ep, row, hc + 64), dup, valid);
        if (ep.aux_out) store_row32_bf16(ep.aux_out + (int64_t)row * ep.ld_aux + col, g, valid);
        if (ep.c_t) {
          store_col32_bf16(ep.c_t, ep.ld_t, row, hc, dgt, valid);
          store_col32_bf16(ep.c_t, ep.ld_t, row, hc + 64, dup, valid);
        }
        if (ep.aux_t) store_col32_bf16(ep.aux_t, ep.ld_t, row, col, g, valid);
      }
      __syncwarp();
    }
  } else {
    for (int cc = 0; cc < BN; cc += 32) {
      uint32_t r[32];
      tmem_ld32(tbase + cc, r);
      tmem_ld_wait();
      const int col = n0 + cc;
      if (row_ok && col < N) {
      const int valid = min(32, N - col);
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
      if (ep.epi == EPI_BF16) {
        store_row32_bf16(reinterpret_cast<__nv_bfloat16*>(ep.C) + out_offset(ep, row, col), v,
                         valid);
      } else if (ep.epi == EPI_F32_ACC || ep.epi == EPI_F32) {
        float4* c4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.C) + out_offset(ep, row, col));
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e * 4 < valid) {
            float4 o = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
            if (ep.epi == EPI_F32_ACC) {
              const float4 old = c4[e];
              o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
            }
            c4[e] = o;
          }
        }
      } else if (ep.epi == EPI_GELU) {
        float g[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) g[i] = gelu_f(bf16_round(v[i]));
        store_row32_bf16(reinterpret_cast<__nv_bfloat16*>(ep.C) + out_offset(ep, row, col), v,
                         valid);
        store_row32_bf16(ep.aux_out + (int64_t)row * ep.ld_aux + col, g, valid);
      } else if (ep.epi == EPI_DGELU) {
        float hh[32], g[32];
        load_row32_bf16(ep.aux_in + (int64_t)row * ep.ld_aux + col, hh, valid);
#pragma unroll
        for (int i = 0; i < 32; ++i) {        // G = x Phi(x), G' = Phi(x) + x phi(x)
          const float x = hh[i];
          float cdf, pdf;
          normal_cdf_pdf(x, cdf, pdf);
          g[i] = x * cdf;
          v[i] = v[i] * fmaf(x, pdf, cdf);
        }
        store_row32_bf16(reinterpret_cast<__nv_bfloat16*>(ep.C) + out_offset(ep, row, col), v,
                         valid);
        if (ep.aux_out) store_row32_bf16(ep.aux_out + (int64_t)row * ep.ld_aux + col, g, valid);
        if (ep.c_t) store_col32_bf16(ep.c_t, ep.ld_t, row, col, v, valid);
        if (ep.aux_t) store_col32_bf16(ep.aux_t, ep.ld_t, row, col, g, valid);
      }
      }
      __syncwarp();
    }
  }
}

template <int BN, int A_MN, int B_MN>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, RowMap amap, RowMap bmap, EpiParams ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mt = (M + BM - 1) / BM;
  const int nt = (N + BN - 1) / BN;
  const int per = mt * nt;                       // tiles per problem (batch: ep.batch problems)
  const int ntiles = per * ep.batch;
  const int nkb_all = (K + BK - 1) / BK;
  // tile t -> (problem z, m block, n block); a causal-K problem visits its heaviest
  // (last) m blocks first so the persistent schedule ends balanced
  auto coords = [&](int t, int& z, int& mb, int& nb) {
    if (ep.batch > 1 || ep.k_causal) {
      const int u = t % per;
      z = t / per;
      mb = mt - 1 - u / nt;                      // descending m: longest K first
      nb = u % nt;
      if (!ep.k_causal) mb = mt - 1 - mb;
    } else {
      z = 0;
      tile_coords(t, mt, nt, mb, nb);
      mb = rot_block(mb, mt, ep.rot_mb);
      nb = rot_block(nb, nt, ep.rot_nb);
    }
  };
  auto kblocks = [&](int mb) { return ep.k_causal ? min(nkb_all, (mb * BM + BM + BK - 1) / BK) : nkb_all; };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int z, mb, nb;
        coords(t, z, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        const int nkb = kblocks(mb);
        wait_chunks(ep, m0, min(BM, M - m0));
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
          if (A_MN) {
            const int kr = amap.map(k0) + (int)(z * ep.a_boff);
            tma_load_2d(sa, &tmA, &full_bar[stage], m0, kr);
            tma_load_2d(sa + 8192, &tmA, &full_bar[stage], m0 + 64, kr);
          } else {
            tma_load_2d(sa, &tmA, &full_bar[stage], k0, amap.map(m0) + (int)(z * ep.a_boff));
          }
          if (B_MN) {
            const int kr = bmap.map(k0);
            const int nz = n0 + (int)((z / ep.b_grp) * ep.b_boff);
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d(sb + i * 8192, &tmB, &full_bar[stage], nz + 64 * i, kr);
          } else {
            tma_load_2d(sb, &tmB, &full_bar[stage], k0, bmap.map(n0) + (int)((z / ep.b_grp) * ep.b_boff));
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int z, mb, nb;
      coords(t, z, mb, nb);
      const int nkb = kblocks(mb);
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad, bd;
            if (A_MN) ad = umma_desc_sw128(sa + k * 2048, 8192, 1024);
            else      ad = umma_desc_sw128(sa + k * 32, 16, 1024);
            if (B_MN) bd = umma_desc_sw128(sb + k * 2048, 8192, 1024);
            else      bd = umma_desc_sw128(sb + k * 32, 16, 1024);
            umma_f16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty_bar[stage]);
          if (kb == nkb - 1) umma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int z, mb, nb;
      coords(t, z, mb, nb);
      const int m0 = mb * BM, n0 = nb * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < M;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      epilogue_tile<BN>(ep, tbase, row, row_ok, n0, N, z);
      count_stored(ep, m0 + q * 32, row_ok, n0, min(BN, N - n0));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ CTA-pair variant
// cta_group::2: a cluster of two CTAs on one TPC computes a 256 x 256 tile with one
// tcgen05.mma (M = 256, N = 256, K = 16) issued by the leader.  Each CTA stages only
// its half of A (128 rows) and its half of B (128 rows of N) per k-block, so every SM
// reads 32 KB per stage instead of 48 KB for the same MMA work; each CTA's TMEM holds
// its 128 rows of the accumulator and its own epilogue warps drain them.
template <int A_MN, int B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    gemm2_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    int M, int N, int K, RowMap amap, RowMap bmap, EpiParams ep, int group_m) {
  constexpr int STAGES = 6;
  constexpr int HALF = 128 * BK * 2;           // 16 KB: one operand half per stage
  constexpr int STAGE = 2 * HALF;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int mt = (M + 255) / 256;
  const int nt = (N + 255) / 256;
  const int ntiles = mt * nt;
  const int nkb = (K + BK - 1) / BK;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 16);      // 8 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        int mb, nb;
        tile_coords(t, mt, nt, mb, nb, group_m);
        mb = rot_block(mb, mt, ep.rot_mb);
        nb = rot_block(nb, nt, ep.rot_nb);
        const int m0 = mb * 256 + rank * 128, n0 = nb * 256 + rank * 128;
        wait_chunks(ep, m0, min(128, M - m0));
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE;
          uint8_t* sb = sa + HALF;
          const uint32_t fb = mapa_u32(&full_bar[stage], 0);    // the leader's barrier
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * STAGE);
          const int k0 = kb * BK;
          if (A_MN) {   // one 3-D box = both 64-wide MN groups (dims: elem, K row, MN group)
            tma_load_3d_2sm(sa, &tmA, fb, 0, amap.map(k0), m0 >> 6);
          } else {
            tma_load_2d_2sm(sa, &tmA, fb, k0, amap.map(m0));
          }
          if (B_MN) {
            tma_load_3d_2sm(sb, &tmB, fb, 0, bmap.map(k0), n0 >> 6);
          } else {
            tma_load_2d_2sm(sb, &tmB, fb, k0, bmap.map(n0));
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, 256, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(smem + stage * STAGE);
            const uint32_t sb = sa + HALF;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              uint64_t ad, bd;
              if (A_MN) ad = umma_desc_sw128(sa + k * 2048, 8192, 1024);
              else      ad = umma_desc_sw128(sa + k * 32, 16, 1024);
              if (B_MN) bd = umma_desc_sw128(sb + k * 2048, 8192, 1024);
              else      bd = umma_desc_sw128(sb + k * 32, 16, 1024);
              umma_f16_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
            umma_commit_2sm_mc(&empty_bar[stage], 0x3);
            if (kb == nkb - 1) umma_commit_2sm_mc(&tfull_bar[acc], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // two epilogue warpgroups, one per 128-column half of the accumulator, so heavy
    // epilogues (dGELU with transposed copies, RoPE) stay under the mainloop time
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cid; t < ntiles; t += ncl) {
      int mb, nb;
      tile_coords(t, mt, nt, mb, nb, group_m);
      mb = rot_block(mb, mt, ep.rot_mb);
      nb = rot_block(nb, nt, ep.rot_nb);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mb * 256 + rank * 128 + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256 + half * 128;
      epilogue_tile<128>(ep, tbase, row, row < M, nb * 256 + half * 128, N);
      count_stored(ep, row - lane, row < M, nb * 256 + half * 128, min(128, N - (nb * 256 + half * 128)));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_u32(&tempty_bar[acc], 0));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor map: inner (contiguous) dim `inner`, outer dim `outer`, row stride in elements
static int make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t ld, uint32_t box_inner, uint32_t box_outer) {
  auto enc = get_encode();
  if (!enc) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// 3-D view of an MN-major operand: (64 elements, K rows, MN/64 groups), box (64, 64, 2)
static int make_map_mn3(CUtensorMap* m, const void* base, uint64_t mn, uint64_t rows, uint64_t ld) {
  auto enc = get_encode();
  if (!enc) return (int)cudaErrorNotSupported;
  cuuint64_t dims[3] = {64, rows, mn / 64};
  cuuint64_t strides[2] = {ld * 2, 128};
  cuuint32_t box[3] = {64, 64, 2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

int gemm_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int BN, int A_MN, int B_MN>
static int launch_t(const GemmArgs& g, const EpiParams& ep, cudaStream_t st) {
  using Cfg = GemmCfg<BN>;
  CUtensorMap ta, tb;
  int rc;
  const int64_t a_rows = g.a_rows > 0 ? g.a_rows : (A_MN ? g.K : g.M);
  const int64_t b_rows = g.b_rows > 0 ? g.b_rows : (B_MN ? g.K : g.N);
  if (A_MN) rc = make_map(&ta, g.A, g.M, a_rows, g.lda, 64, 64);
  else      rc = make_map(&ta, g.A, g.K, a_rows, g.lda, 64, BM);
  if (rc) return rc;
  if (B_MN) rc = make_map(&tb, g.B, g.b_cols > 0 ? g.b_cols : g.N, b_rows, g.ldb, 64, 64);
  else      rc = make_map(&tb, g.B, g.K, b_rows, g.ldb, 64, BN);
  if (rc) return rc;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr_set = true;
  }
  const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN) * (g.batch > 0 ? g.batch : 1);
  const int sms = gemm_num_sms() - g.sm_reserve;
  const int grid = tiles < sms ? tiles : sms;
  RowMap am{g.a_seg > 0 ? g.a_seg : (int64_t)1 << 40, g.a_stride, g.a_base};
  RowMap bm{g.b_seg > 0 ? g.b_seg : (int64_t)1 << 40, g.b_stride, g.b_base};
  kern<<<grid, 256, Cfg::SMEM, st>>>(ta, tb, g.M, g.N, g.K, am, bm, ep);
  return (int)cudaGetLastError();
}

template <int A_MN, int B_MN>
static int launch2_t(const GemmArgs& g, const EpiParams& ep, cudaStream_t st) {
  constexpr int SMEM = 6 * 32768 + 1024 + 256;
  CUtensorMap ta, tb;
  int rc;
  const int64_t a_rows = g.a_rows > 0 ? g.a_rows : (A_MN ? g.K : g.M);
  const int64_t b_rows = g.b_rows > 0 ? g.b_rows : (B_MN ? g.K : g.N);
  if (A_MN) rc = make_map_mn3(&ta, g.A, g.M, a_rows, g.lda);
  else      rc = make_map(&ta, g.A, g.K, a_rows, g.lda, 64, 128);
  if (rc) return rc;
  if (B_MN) rc = make_map_mn3(&tb, g.B, g.N, b_rows, g.ldb);
  else      rc = make_map(&tb, g.B, g.K, b_rows, g.ldb, 64, 128);
  if (rc) return rc;
  auto kern = gemm2_tc_kernel<A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr_set = true;
  }
  const int tiles = ((g.M + 255) / 256) * ((g.N + 255) / 256);
  const int ncl = std::min(tiles, (gemm_num_sms() - g.sm_reserve) / 2);
  RowMap am{g.a_seg > 0 ? g.a_seg : (int64_t)1 << 40, g.a_stride, g.a_base};
  RowMap bm{g.b_seg > 0 ? g.b_seg : (int64_t)1 << 40, g.b_stride, g.b_base};
  static const int env_gm = [] { const char* e = getenv("PDS_GEMM_GM"); return e ? atoi(e) : 0; }();
  static const int env_short = [] { const char* e = getenv("PDS_GEMM_GM_SHORT"); return e ? atoi(e) : 0; }();
  // CTA-pair raster band: 8 m-blocks (2048 rows).  At fixed clocks 16 was best, but
  // under the 1000 W power cap 8 reads less DRAM and won 5 of 6 interleaved whole-bench
  // rounds (+0.7 %, profiles/round1_ab_gemm_group_m*.txt); 32 lost 4 % (raw_r02/gm_*).
  // Short-K GEMMs (K <= 4096: QKV, proj, FC1, dG, dA) read the least DRAM with a band of
  // 16 (fixed clocks, s = 16K FC1 shape: 1.68 GB vs 2.68 GB at 8, same time); long-K
  // GEMMs keep 8.  PDS_GEMM_GM overrides both, PDS_GEMM_GM_SHORT the short-K band.
  const int group_m = env_gm > 0 ? env_gm : (g.K <= 4096 ? (env_short > 0 ? env_short : 16) : 8);
  kern<<<2 * ncl, 384, SMEM, st>>>(ta, tb, g.M, g.N, g.K, am, bm, ep, group_m);
  return (int)cudaGetLastError();
}

static int pair_mode() {
  static int v = [] {
    const char* e = getenv("PDS_GEMM_PAIR");
    return e ? atoi(e) : 1;
  }();
  return v;
}

int gemm_launch(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return 0;
  if (g.N % 8 || (g.blk_w % 32)) return (int)cudaErrorInvalidValue;
  EpiParams ep;
  ep.M = g.M; ep.N = g.N; ep.C = g.C; ep.ldc = g.ldc; ep.epi = g.epi;
  ep.blk_w = g.blk_w; ep.blk_stride = g.blk_stride;
  ep.aux_in = reinterpret_cast<const __nv_bfloat16*>(g.aux_in);
  ep.aux_out = reinterpret_cast<__nv_bfloat16*>(g.aux_out);
  ep.ld_aux = g.ld_aux;
  ep.ld_aux_in = g.ld_aux_in > 0 ? g.ld_aux_in : g.ld_aux;
  ep.c_t = reinterpret_cast<__nv_bfloat16*>(g.c_t);
  ep.aux_t = reinterpret_cast<__nv_bfloat16*>(g.aux_t);
  ep.ld_t = g.ld_t;
  ep.rope = g.rope; ep.rope_d = g.rope_d; ep.rope_hq = g.rope_hq; ep.rope_b = g.rope_b > 0 ? g.rope_b : 1;
  ep.rope_hk = g.rope_hk > 0 ? g.rope_hk : g.rope_hq;
  ep.rope_segs = g.rope_segs;
  ep.seg = g.seg > 0 ? g.seg : (int64_t)1 << 40;
  ep.seg_stride = g.seg_stride; ep.seg_base = g.seg_base;
  ep.c_seg = g.c_seg > 0 ? g.c_seg : (int64_t)1 << 40;
  ep.c_stride = g.c_stride; ep.c_base = g.c_base;
  ep.wait_flags = g.wait_flags; ep.flag_epoch = g.flag_epoch;
  ep.done_ctr = g.done_ctr; ep.chunk_rows = (int)g.chunk_rows; ep.rot_mb = 0;
  ep.chunk_cols = (int)g.chunk_cols; ep.rot_nb = 0;
  ep.batch = g.batch > 0 ? g.batch : 1;
  ep.a_boff = g.a_boff; ep.b_boff = g.b_boff; ep.c_boff = g.c_boff;
  ep.b_grp = g.b_grp > 0 ? g.b_grp : 1;
  ep.k_causal = g.k_causal; ep.epi_scale = g.epi_scale;
  const bool plain1 = ep.batch > 1 || g.k_causal || g.epi == EPI_ROPE_T;   // 1-CTA kernel, BN = 128
  if (plain1 && (g.wait_flags || g.done_ctr || g.blk_w || g.a_seg || g.b_seg || g.c_seg || g.m_rot_rows ||
                 g.n_rot_cols))
    return (int)cudaErrorInvalidValue;
  if (g.epi == EPI_ROPE_T && g.N != 128) return (int)cudaErrorInvalidValue;
  if (g.wait_flags || (g.done_ctr && g.chunk_cols <= 0)) {
    if (g.chunk_rows <= 0 || g.chunk_rows % 32 || g.M % g.chunk_rows) return (int)cudaErrorInvalidValue;
    if (g.wait_flags && (g.a_mn || g.a_seg)) return (int)cudaErrorInvalidValue;
    if (g.done_ctr && (g.c_seg || g.blk_w)) return (int)cudaErrorInvalidValue;
  }
  if (g.chunk_cols < 0 || (g.chunk_cols > 0 && (!g.done_ctr || g.N % g.chunk_cols || g.chunk_cols % 8)))
    return (int)cudaErrorInvalidValue;
  if (g.sm_reserve < 0 || g.sm_reserve > gemm_num_sms() - 2) return (int)cudaErrorInvalidValue;
  // a tile must not straddle a remap segment
  if (g.a_seg > 0 && g.a_seg % (g.a_mn ? 64 : BM)) return (int)cudaErrorInvalidValue;
  if (g.b_seg > 0 && g.b_seg % (g.b_mn ? 64 : 256)) return (int)cudaErrorInvalidValue;
  // BN = 256 when N is large enough to fill the machine, else 128 (more tiles)
  const int64_t tiles256 = (int64_t)((g.M + BM - 1) / BM) * ((g.N + 255) / 256);
  bool use256 = (g.N % 256 == 0 || g.N > 1024) && tiles256 >= gemm_num_sms();
  if (g.epi == EPI_ROPE && (g.rope_d % 64 || 128 % g.rope_d)) return (int)cudaErrorInvalidValue;
  if (g.epi == EPI_ROPE && g.rope_hk > 0 && g.rope_hk % g.rope_d) return (int)cudaErrorInvalidValue;
  // SwiGLU: whole (gate, up) 64-column pairs per 128 output columns; no column blocking
  if ((g.epi == EPI_SWIGLU || g.epi == EPI_DSWIGLU) && (g.blk_w || g.chunk_cols)) return (int)cudaErrorInvalidValue;
  if (g.epi == EPI_SWIGLU && (g.N % 128 || !g.aux_out)) return (int)cudaErrorInvalidValue;
  if (g.epi == EPI_DSWIGLU && (g.N % 64 || !g.aux_in)) return (int)cudaErrorInvalidValue;
  const int64_t pair_tiles = (int64_t)((g.M + 255) / 256) * ((g.N + 255) / 256);
  if (plain1) use256 = false;
  const bool pair_ok = !plain1 && pair_mode() && g.M >= 256 && (g.N % 256 == 0 || g.N > 1024) &&
                       pair_tiles >= gemm_num_sms() / 2 && (g.a_seg == 0 || g.a_seg % 128 == 0) &&
                       (!g.a_mn || g.M % 64 == 0) && (!g.b_mn || g.N % 64 == 0) &&
                       (g.b_seg == 0 || g.b_seg % 128 == 0);
  if (g.m_rot_rows) ep.rot_mb = (int)(g.m_rot_rows / (pair_ok ? 256 : BM));
  if (g.n_rot_cols) ep.rot_nb = (int)(g.n_rot_cols / (pair_ok || use256 ? 256 : 128));
  if (pair_ok) {
    switch ((g.a_mn ? 2 : 0) | (g.b_mn ? 1 : 0)) {
      case 0: return launch2_t<0, 0>(g, ep, st);
      case 1: return launch2_t<0, 1>(g, ep, st);
      case 2: return launch2_t<1, 0>(g, ep, st);
      default: return launch2_t<1, 1>(g, ep, st);
    }
  }
  const int key = (use256 ? 4 : 0) | (g.a_mn ? 2 : 0) | (g.b_mn ? 1 : 0);
  switch (key) {
    case 0: return launch_t<128, 0, 0>(g, ep, st);
    case 1: return launch_t<128, 0, 1>(g, ep, st);
    case 2: return launch_t<128, 1, 0>(g, ep, st);
    case 3: return launch_t<128, 1, 1>(g, ep, st);
    case 4: return launch_t<256, 0, 0>(g, ep, st);
    case 5: return launch_t<256, 0, 1>(g, ep, st);
    case 6: return launch_t<256, 1, 0>(g, ep, st);
    default: return launch_t<256, 1, 1>(g, ep, st);
  }
}

}  // namespace pds
