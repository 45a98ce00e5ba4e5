// tcgen05 / TMEM causal flash attention (Eq. 2; causal R-1) for
// sm_100a, forward and backward.  Every kernel: warp 0 = TMA producer, warp 1 = the
// single-thread MMA issuer, warp 2 = TMEM allocator (512 columns), warps 4.. =
// elementwise warpgroups (thread = TMEM lane = one row of the 128-row tile; two
// warpgroups in the forward and dQ kernels, four in dK/dV, splitting the columns).
//
//   attn_fwd_tc_kernel     CTA = two 128-query tiles x one head; S = Q K^T per
//                          128-key block into TMEM, online softmax with lazy
//                          rescale, P written back into TMEM (packed bf16) and
//                          used as the A operand of O += P V.
//   attn_bwd_dkdv4_kernel  CTA = 128 keys x one head, loop over 128-query blocks:
//                          S^T, dP^T in TMEM; P^T, dS^T written back into TMEM
//                          as A operands of dV += P^T dO, dK += dS^T Q.
//   attn_bwd_dq4_kernel    CTA = 128 queries x one head (Q, dO resident in TMEM as
//                          A operands), loop over 128-key blocks: S, dP, dS into
//                          TMEM, dQ += dS K.
// dQ and dK leave through RoPE^T (gradients w.r.t. the pre-rotation Q, K) and the
// softmax scale; D = rowsum(dO o O) comes from attn_bwd_dot_kernel (attention.cu).
//
// Operand layouts: every smem tile is a TMA box of 64 columns x 128 rows of the
// row-major [s][3*heads*d] QKV (or [s][heads*d] dO) buffer, SWIZZLE_128B; a tile is
// read K-major when the contraction runs over d and MN-major when it runs over rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <string>
#include <type_traits>

#include "ptx.cuh"
#include "gemm.cuh"

namespace pds {

namespace attn_tc {

[[maybe_unused]] constexpr int BM = 128;  // queries per tile
constexpr int BN = 128;  // keys per block
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;


}  // namespace attn_tc

using namespace attn_tc;

// K-major SW128 descriptor of k-step kk (16 elements) in a [rows][64*atoms] tile whose
// 64-column atoms are `atom` bytes apart (rows * 128)
__device__ __forceinline__ uint64_t kmaj_desc(uint32_t tile, int kk, uint32_t atom = 16384) {
  return umma_desc_sw128(tile + (kk >> 2) * atom + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 descriptor: the tile's rows are K, 64-wide MN groups `atom` bytes
// apart (LBO), k-step kk = 16 rows (2 x 8-row groups, SBO = 1024)
__device__ __forceinline__ uint64_t mnmaj_desc(uint32_t tile, int kk, uint32_t atom = 16384) {
  return umma_desc_sw128(tile + kk * 2048, atom, 1024);
}

// 2^x on the MUFU unit, flush-to-zero (P is rounded to bf16 anyway)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for x <= 0 on the FMA pipe (Cody-Waite split + degree-3 minimax on [-0.5, 0.5],
// max relative error 7.5e-5 — far below the bf16 rounding of P).  Used for a share of
// the softmax exponentials so the MUFU (ex2) unit is not the bottleneck.
__device__ __forceinline__ float exp2_fma(float x) {
  x = fmaxf(x, -125.0f);
  const float t = x + 12582912.0f;             // 1.5 * 2^23: round to nearest integer
  const float f = x - (t - 12582912.0f);       // [-0.5, 0.5]
  float p = fmaf(0.05517161f, f, 0.24261112f);
  p = fmaf(p, f, 0.693261f);
  p = fmaf(p, f, 0.99992807f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Packed fp32 pair arithmetic (sm_100 FFMA2 / FADD2 / FMUL2): one instruction per
// two elements for the softmax / dS elementwise work, which is issue-bound.
struct f2 { float x, y; };
__device__ __forceinline__ uint64_t f2u(f2 a) {
  return (uint64_t)__float_as_uint(a.x) | ((uint64_t)__float_as_uint(a.y) << 32);
}
__device__ __forceinline__ f2 u2f(uint64_t v) { return f2{__uint_as_float((uint32_t)v), __uint_as_float((uint32_t)(v >> 32))}; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
// exp2_fma on a pair: the same Cody-Waite split and polynomial with packed arithmetic
__device__ __forceinline__ f2 exp2_fma2(f2 x) {
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const f2 big{12582912.0f, 12582912.0f};
  const f2 t = add2(x, big);
  const f2 f = sub2(x, sub2(t, big));
  f2 p = fma2(f2{0.05517161f, 0.05517161f}, f, f2{0.24261112f, 0.24261112f});
  p = fma2(p, f, f2{0.693261f, 0.693261f});
  p = fma2(p, f, f2{0.99992807f, 0.99992807f});
  return f2{__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
            __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23))};
}

// Which element pairs take exp2 on the FMA pipe: bit (pair index mod 8) of the mask.
// 0x88 = 1 pair in 4 (25 %).  MUFU ex2 runs 16 / clk / SM, the FFMA2 emulation costs
// issue slots instead; the best split depends on the kernel's other work.
#ifndef PDS_EMU_MASK
#define PDS_EMU_MASK 0x88
#endif
__host__ __device__ constexpr bool emu_pair(int pair) { return (PDS_EMU_MASK >> (pair & 7)) & 1; }

// Optional timeline trace of one CTA (build with -DPDS_TRACE=1 for the dQ kernel, =2 for
// dK/dV; read with pds_debug_trace): clock64 stamps per block, see the kernels.
#ifdef PDS_TRACE
__device__ long long g_trace[4096][8];
#define PDS_TR_(j, k) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 4096) g_trace[j][k] = clock64();
#else
#define PDS_TR_(j, k)
#endif
#if defined(PDS_TRACE) && PDS_TRACE == 1
#define PDS_TR(j, k) PDS_TR_(j, k)
#else
#define PDS_TR(j, k)
#endif
#if defined(PDS_TRACE) && PDS_TRACE == 2
#define PDS_TR2(j, k) PDS_TR_(j, k)
#else
#define PDS_TR2(j, k)
#endif

// 16-byte chunk store into a K-major SW128 tile: row r, 16-byte chunk c of atom a
__device__ __forceinline__ void st_sw128(uint8_t* tile, uint32_t atom, int r, int a, int c, uint4 v) {
  *reinterpret_cast<uint4*>(tile + a * atom + r * 128 + ((c ^ (r & 7)) << 4)) = v;
}

// Forward, two 128-row query tiles per CTA (rows [q0, q0+128) and [q0+128, q0+256))
// sharing every K/V tile.  TMEM: S0 | S1 | O0 | O1 (128 columns each).  MMA order per
// KV block j:  PV0_{j-1}? ... S0_j, S1_j, PV0_j, S0_{j+1}, PV1_j, S1_{j+1}, ...  so the
// softmax of one tile overlaps the other tile's MMAs.  P_t is written back as packed
// bf16 into the first 64 columns of S_t and consumed with the A operand in TMEM;
// because tcgen05 MMAs of one thread execute in issue order, S_t(j+1) (issued after
// PV_t(j)) completing implies PV_t(j) completed, so the softmax may rescale O_t and
// overwrite P_t as soon as S_t(j+1) is ready.
template <int D>
struct Fwd2Cfg {
  static constexpr int TILE = 128 * D * 2;
  static constexpr int Q_OFF = 0;                 // Q0, Q1
  static constexpr int K_OFF = 2 * TILE;          // [2 stages]
  static constexpr int V_OFF = K_OFF + 2 * TILE;  // [2 stages]
  static constexpr int BAR_OFF = V_OFF + 2 * TILE;
  static constexpr int RED_OFF = BAR_OFF + 256;           // NS = 2: row-max / row-sum exchange
  static constexpr int SMEM = RED_OFF + 2 * 2 * 2 * 128 * 4 + 1024;
};

// RP (register pass, the default; PDS_ATTN_FWD=2pass: off): the producer / MMA warpgroup gives
// registers up (setmaxnreg.dec 56) and each softmax warpgroup takes 224, so a thread
// holds its whole 128-key S row in registers: one TMEM read per block instead of two.
// NS (softmax warpgroups per query tile, opt-in PDS_ATTN_FWD=split for NS = 2): with two,
// each warpgroup owns half of the 128 keys of a block (threads of both hold the same rows,
// TMEM lanes), the row max and the final row sum are exchanged through shared memory
// under a named barrier per tile, and the half-0 warpgroup alone releases the first PV
// half: a tile's softmax latency per block is halved.
template <int D, bool RP = false, int NS = 1>
__global__ void __launch_bounds__(128 + 256 * NS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmq, int s,
                       int heads, int causal, __nv_bfloat16* __restrict__ out, int64_t ld_out, float* __restrict__ lse,
                       float scale_log2, int qlo, int qn, int kcol, int vcol, int grp,
                       const int* __restrict__ segs) {
  using C = Fwd2Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;    // [2]
  uint64_t* kv_empty = bar + 3;   // [2]
  uint64_t* s_full = bar + 5;     // [2] per tile
  uint64_t* p_full = bar + 7;     // [2] per tile
  uint64_t* o_done = bar + 9;     // [2] per tile
  uint64_t* p_half = bar + 12;    // [2] per tile: P columns of keys 0..63 written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // query rows [qlo, qlo + qn) of the s positions (context parallelism; default all):
  // out / lse are indexed by the local row (row - qlo)
  const int nqb = (qn + 255) / 256;
  const int qb = causal ? (nqb - 1 - (int)blockIdx.x) : (int)blockIdx.x;
  const int head = blockIdx.y;
  const int kvh = head / grp;           // GQA: the key / value head of this query head
  const int q0 = qlo + qb * 256;
  // varlen packing (R-VARLEN): the keys of this query block's own sequence only, key
  // blocks [kb0, kb0 + nkv); segs[2 blk], segs[2 blk + 1] = its sequence's block range
  const int kb0 = segs ? segs[2 * (q0 / 128)] : 0;
  const int nkv = (causal ? min(s, q0 + 256) / BN : (segs ? segs[2 * (q0 / 128) + 1] : s / BN)) - kb0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    tma_prefetch(&tmq);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4 * NS);
      mbar_init(&p_half[i], 4);
      mbar_init(&o_done[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
   if (RP) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
   if (warp == 0) {
    if (elect_one()) {
      mbar_arrive_expect_tx(q_full, 2 * C::TILE);
      for (int t = 0; t < 2; ++t)
        for (int a = 0; a < D / 64; ++a)
          tma_load_2d(sm + C::Q_OFF + t * C::TILE + a * 16384, &tmq, q_full, head * D + a * 64, q0 + 128 * t);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(&kv_empty[st], ((j >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * C::TILE);
        for (int a = 0; a < D / 64; ++a) {
          tma_load_2d(sm + C::K_OFF + st * C::TILE + a * 16384, &tm, &kv_full[st], kcol + kvh * D + a * 64,
                      (kb0 + j) * BN);
          tma_load_2d(sm + C::V_OFF + st * C::TILE + a * 16384, &tm, &kv_full[st], vcol + kvh * D + a * 64,
                      (kb0 + j) * BN);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, BN, 0, 0);
    constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, 0, 1);
    const uint32_t sq = smem_u32(sm + C::Q_OFF);
    mbar_wait(q_full, 0);
    auto issue_s = [&](int t, int j) {
      if (elect_one()) {
        const uint32_t sk = smem_u32(sm + C::K_OFF + (j & 1) * C::TILE);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16(tmem + t * 128, kmaj_desc(sq + t * C::TILE, kk), kmaj_desc(sk, kk), idesc_s, kk > 0);
        umma_commit(&s_full[t]);
      }
      __syncwarp();
    };
    // O_t += P_t V in two halves of keys: the first as soon as the softmax has written
    // P for keys 0..63, overlapping the exponentials of keys 64..127
    auto issue_pv = [&](int t, int j) {
      const uint32_t sv = smem_u32(sm + C::V_OFF + (j & 1) * C::TILE);
      mbar_wait(&p_half[t], j & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < BN / 32; ++kk)
          umma_f16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mnmaj_desc(sv, kk), idesc_o, (j | kk) != 0);
      }
      __syncwarp();
      mbar_wait(&p_full[t], j & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = BN / 32; kk < BN / 16; ++kk)
          umma_f16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mnmaj_desc(sv, kk), idesc_o, 1);
      }
      __syncwarp();
    };
    mbar_wait(&kv_full[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    for (int j = 0; j < nkv; ++j) {
      issue_pv(0, j);
      if (j + 1 < nkv) {
        mbar_wait(&kv_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
        tc_fence_after();
        issue_s(0, j + 1);
      } else if (elect_one()) {
        umma_commit(&o_done[0]);
      }
      __syncwarp();
      issue_pv(1, j);
      if (elect_one()) umma_commit(&kv_empty[j & 1]);
      __syncwarp();
      if (j + 1 < nkv) issue_s(1, j + 1);
      else if (elect_one()) umma_commit(&o_done[1]);
      __syncwarp();
    }
   }
  } else {
    // the pool is the CTA's launch allocation (threads x compiled count: 384 x 168 / 640 x 96),
    // so the increase is what WG0's decrease frees: 224 (NS = 1), 104 (NS = 2)
    if (RP) {
      if (NS == 1) asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
      else asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
    }
    constexpr int KC = BN / NS;              // keys (S columns) per softmax warpgroup
    constexpr int OC = D / NS;               // O columns per softmax warpgroup
    const int wgi = (warp - 4) >> 2;
    const int tile = wgi / NS;               // NS = 1: 0 = warps 4-7, 1 = warps 8-11
    const int half = wgi % NS;               // NS = 2: keys [half KC, (half + 1) KC)
    const int q = warp & 3;
    const int tr = q * 32 + lane;            // row within the tile = TMEM lane
    const int row = q0 + tile * 128 + tr;
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t s_col = tile * 128 + half * KC, o_col = 256 + tile * 128 + half * OC;
    float* red = reinterpret_cast<float*>(sm + C::RED_OFF);   // [2 parity][2 tiles][2 halves][128]
    auto tile_sync = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + tile) : "memory"); };
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(&s_full[tile], j & 1);
      tc_fence_after();
      const int k0 = (kb0 + j) * BN + half * KC;      // this warpgroup's first key
      const bool mask = causal && (k0 + KC - 1 > q0 + tile * 128);
      auto block = [&](auto mask_c) {
        constexpr bool MASK = decltype(mask_c)::value;
      // pass 1: row max; 16-column TMEM loads software-pipelined (next chunk in flight)
      float mxa[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      uint32_t srow[RP ? KC : 1];                // RP: the whole S row, read once
      if constexpr (RP) {
#pragma unroll
        for (int c = 0; c < KC / 32; ++c)
          tmem_ld32(lb + s_col + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&srow[c * 32]));
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < KC; ++i) {
          float v = __uint_as_float(srow[i]);
          if (MASK && k0 + i > row) v = -INFINITY;
          mxa[i & 3] = fmaxf(mxa[i & 3], v);
        }
      } else {
        uint32_t cur[16], nxt[16];
        tmem_ld16(lb + s_col, cur);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < KC / 16; ++c) {
          if (c + 1 < KC / 16) tmem_ld16(lb + s_col + (c + 1) * 16, nxt);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float v = __uint_as_float(cur[i]);
            if (MASK && k0 + c * 16 + i > row) v = -INFINITY;
            mxa[i & 3] = fmaxf(mxa[i & 3], v);
          }
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) cur[i] = nxt[i];
        }
      }
      float mx = fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3]));
      if constexpr (NS == 2) {                 // the row max over both halves of the keys
        float* rb = red + ((j & 1) * 4 + tile * 2) * 128;
        rb[half * 128 + tr] = mx;
        tile_sync();
        mx = fmaxf(mx, rb[(half ^ 1) * 128 + tr]);
      }
      const float m_new = mx * scale_log2;
      const bool need = m_new > m_used + 8.0f;
      if (j > 0 && __any_sync(0xffffffff, need)) {
        const float f = need ? ex2(m_used - m_new) : 1.0f;
#pragma unroll
        for (int c = 0; c < OC / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(lb + o_col + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
          tmem_st16(lb + o_col + c * 32, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
          tmem_st16(lb + o_col + c * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&r[16]));
        }
        if (need) l *= f;
      }
      if (need) m_used = m_new;
      // pass 2: p = exp2(s scale - m) (1 in 4 on the FMA pipe), bf16-packed P written
      // back into the consumed S columns (chunk c of 16 keys -> 8 packed columns at 8c)
      f2 rs2[2] = {f2{0.f, 0.f}, f2{0.f, 0.f}};
      const f2 nm2{-m_used, -m_used}, sl2{scale_log2, scale_log2};
      {
        uint32_t cur[16], nxt[16];
        if constexpr (!RP) {
          tmem_ld16(lb + s_col, cur);
          tmem_ld_wait();
        }
#pragma unroll
        for (int c = 0; c < KC / 16; ++c) {
          if constexpr (RP) {
#pragma unroll
            for (int i = 0; i < 16; ++i) cur[i] = srow[c * 16 + i];
          } else {
            if (c + 1 < KC / 16) tmem_ld16(lb + s_col + (c + 1) * 16, nxt);
          }
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const f2 x = fma2(f2{__uint_as_float(cur[i]), __uint_as_float(cur[i + 1])}, sl2, nm2);
            f2 p;
            if (emu_pair(i >> 1)) {
              p = exp2_fma2(x);                  // share of the pairs on the FMA pipe
            } else {
              p.x = ex2(x.x);
              p.y = ex2(x.y);
            }
            if (MASK) {
              if (k0 + c * 16 + i > row) p.x = 0.f;
              if (k0 + c * 16 + i + 1 > row) p.y = 0.f;
            }
            rs2[(i >> 1) & 1] = add2(rs2[(i >> 1) & 1], p);
            pk[i >> 1] = pack_bf16(p.x, p.y);
          }
          tmem_st8(lb + tile * 128 + (half * KC) / 2 + c * 8, pk);   // packed P of keys half KC + 16c..
          if (half * KC + (c + 1) * 16 == BN / 2) {   // P of keys 0..63 complete: release the first PV half
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_half[tile]);
          }
          if constexpr (!RP) {
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) cur[i] = nxt[i];
          }
        }
      }
        const f2 rs = add2(rs2[0], rs2[1]);
        l += rs.x + rs.y;
      };
      if (mask) block(std::true_type{});
      else block(std::false_type{});
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[tile]);
    }
    mbar_wait(&o_done[tile], 0);
    tc_fence_after();
    if constexpr (NS == 2) {                   // the row sum over both halves of the keys
      float* rb = red + ((nkv & 1) * 4 + tile * 2) * 128;   // the parity buffer block nkv - 2 used
      rb[half * 128 + tr] = l;
      tile_sync();
      l += rb[(half ^ 1) * 128 + tr];
    }
    const float inv = 1.0f / l;
    const bool ok = row < qlo + qn;
    __nv_bfloat16* o = out + (int64_t)(row - qlo) * ld_out + head * D + half * OC;
#pragma unroll
    for (int c = 0; c < OC / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(lb + o_col + c * 32, r);
      tmem_ld_wait();
      if (ok) {
        uint4* d4 = reinterpret_cast<uint4*>(o + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          d4[e] = make_uint4(pack_bf16(__uint_as_float(r[8 * e]) * inv, __uint_as_float(r[8 * e + 1]) * inv),
                             pack_bf16(__uint_as_float(r[8 * e + 2]) * inv, __uint_as_float(r[8 * e + 3]) * inv),
                             pack_bf16(__uint_as_float(r[8 * e + 4]) * inv, __uint_as_float(r[8 * e + 5]) * inv),
                             pack_bf16(__uint_as_float(r[8 * e + 6]) * inv, __uint_as_float(r[8 * e + 7]) * inv));
      }
    }
    if (ok && half == 0) lse[(int64_t)head * qn + (row - qlo)] = (m_used + log2f(l)) * LN2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================ forward, CTA pair
// The forward above reads 192 KB of operands per 128-key block from shared memory
// (S0 and S1 each stream Q_t and K, PV0 and PV1 each stream V) plus the 64 KB TMA
// refill: ~125 B/clk at the tensor peak, the shared-memory limit.  Here a cluster of
// two CTAs issues every MMA as cta_group::2 (M = 256: CTA c's 128 query rows of tile t
// in its own TMEM), and each CTA stages only HALF of every B operand — K rows
// [64c, 64c+64) of the key block for S = Q K^T, V columns [64c, 64c+64) for O += P V —
// so per CTA the operand stream is 128 KB per key block and the refill 32 KB.
// The pair covers 512 query rows: tile t of CTA c = rows base + 256 t + 128 c, so the
// pair MMA t needs the key blocks up to (base + 256 t + 255) / 128 (per-tile nkv).
// The leader (rank 0) issues all MMAs and owns q_full / kv_full / p_half / p_full
// (both CTAs' TMA bytes and softmax arrivals land on the leader's barriers); the
// commits multicast s_full / o_done / kv_empty to both CTAs.  Everything else (online
// softmax, lazy rescale, P in TMEM, epilogue) is the single-CTA kernel's, per CTA.
struct FwdPairCfg {
  static constexpr int D = 128;
  static constexpr int TILE = 128 * D * 2;        // one Q tile [128][128] bf16
  static constexpr int KH = 64 * D * 2;           // K half [64 keys][128]
  static constexpr int VH = 128 * 64 * 2;         // V half [128 keys][64]
  static constexpr int NST = 3;
  static constexpr int Q_OFF = 0;                 // Q0, Q1
  static constexpr int K_OFF = 2 * TILE;          // [NST]
  static constexpr int V_OFF = K_OFF + NST * KH;  // [NST]
  static constexpr int BAR_OFF = V_OFF + NST * VH;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    attn_fwd_pair_tc_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                            const __grid_constant__ CUtensorMap tmv, int s, int heads, int causal,
                            __nv_bfloat16* __restrict__ out, int64_t ld_out, float* __restrict__ lse,
                            float scale_log2, int qlo, int qn, int kcol, int vcol) {
  using C = FwdPairCfg;
  constexpr int D = C::D, NST = C::NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;             // [NST] (leader)
  uint64_t* kv_empty = bar + 1 + NST;      // [NST] (both, multicast commit)
  uint64_t* s_full = bar + 1 + 2 * NST;    // [2] per tile (both)
  uint64_t* p_full = bar + 3 + 2 * NST;    // [2] (leader, 8 arrivals)
  uint64_t* o_done = bar + 5 + 2 * NST;    // [2] (both)
  uint64_t* p_half = bar + 7 + 2 * NST;    // [2] (leader, 8 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 9 + 2 * NST);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int npb = (qn + 511) / 512;
  const int pb = causal ? (npb - 1 - (int)(blockIdx.x >> 1)) : (int)(blockIdx.x >> 1);
  const int head = blockIdx.y;
  const int base = qlo + pb * 512;
  // per pair-MMA t: key blocks up to the last query row of tile t of CTA 1
  int nkv_t[2];
  for (int t = 0; t < 2; ++t)
    nkv_t[t] = causal ? (min(s, base + 256 * t + 256) + BN - 1) / BN : s / BN;
  const int nkv = max(nkv_t[0], nkv_t[1]);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmq);
    tma_prefetch(&tmk);
    tma_prefetch(&tmv);
    mbar_init(q_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
      mbar_init(&p_half[i], 8);
      mbar_init(&o_done[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint32_t qf = mapa_u32(q_full, 0);
      if (rank == 0) mbar_arrive_expect_tx(q_full, 2 * 2 * C::TILE);
      for (int t = 0; t < 2; ++t)
        for (int a = 0; a < D / 64; ++a)
          tma_load_2d_2sm(sm + C::Q_OFF + t * C::TILE + a * 16384, &tmq, qf, head * D + a * 64,
                          base + 256 * t + 128 * rank);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % NST;
        if (j >= NST) mbar_wait(&kv_empty[st], ((j / NST) - 1) & 1);
        const uint32_t kf = mapa_u32(&kv_full[st], 0);
        if (rank == 0) mbar_arrive_expect_tx(&kv_full[st], 2 * (C::KH + C::VH));
        for (int a = 0; a < D / 64; ++a)
          tma_load_2d_2sm(sm + C::K_OFF + st * C::KH + a * 8192, &tmk, kf, kcol + head * D + a * 64,
                          j * BN + 64 * rank);
        tma_load_2d_2sm(sm + C::V_OFF + st * C::VH, &tmv, kf, vcol + head * D + 64 * rank, j * BN);
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(256, BN, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(256, D, 0, 1);
      const uint32_t sq = smem_u32(sm + C::Q_OFF);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int t, int j) {
        if (elect_one()) {
          const uint32_t sk = smem_u32(sm + C::K_OFF + (j % NST) * C::KH);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            umma_f16_2sm(tmem + t * 128, kmaj_desc(sq + t * C::TILE, kk), kmaj_desc(sk, kk, 8192), idesc_s, kk > 0);
          umma_commit_2sm_mc(&s_full[t], 0x3);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j) {
        const uint32_t sv = smem_u32(sm + C::V_OFF + (j % NST) * C::VH);
        mbar_wait(&p_half[t], j & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BN / 32; ++kk)
            umma_f16_ts_2sm(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mnmaj_desc(sv, kk), idesc_o, (j | kk) != 0);
        }
        __syncwarp();
        mbar_wait(&p_full[t], j & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = BN / 32; kk < BN / 16; ++kk)
            umma_f16_ts_2sm(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, mnmaj_desc(sv, kk), idesc_o, 1);
        }
        __syncwarp();
      };
      auto wait_kv = [&](int j) {
        mbar_wait(&kv_full[j % NST], (j / NST) & 1);
        tc_fence_after();
      };
      wait_kv(0);
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < nkv; ++j) {
        const bool a0 = j < nkv_t[0];
        if (a0) {
          issue_pv(0, j);
          if (j + 1 < nkv_t[0]) {
            wait_kv(j + 1);
            issue_s(0, j + 1);
          } else if (elect_one()) {
            umma_commit_2sm_mc(&o_done[0], 0x3);
          }
          __syncwarp();
        }
        issue_pv(1, j);
        if (elect_one()) umma_commit_2sm_mc(&kv_empty[j % NST], 0x3);
        __syncwarp();
        if (j + 1 < nkv_t[1]) {
          if (!(j + 1 < nkv_t[0])) wait_kv(j + 1);
          issue_s(1, j + 1);
        } else if (elect_one()) {
          umma_commit_2sm_mc(&o_done[1], 0x3);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int tile = (warp - 4) >> 2;        // 0: warps 4-7, 1: warps 8-11
    const int q = warp & 3;
    const int tr = q * 32 + lane;            // row within the tile = TMEM lane
    const int q0 = base + 256 * tile + 128 * (int)rank;   // this CTA's tile rows
    const int row = q0 + tr;
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t s_col = tile * 128, o_col = 256 + tile * 128;
    const uint32_t ph_lead = mapa_u32(&p_half[tile], 0), pf_lead = mapa_u32(&p_full[tile], 0);
    const int my_nkv = nkv_t[tile];
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < my_nkv; ++j) {
      mbar_wait(&s_full[tile], j & 1);
      tc_fence_after();
      const int k0 = j * BN;
      const bool mask = causal && (k0 + BN - 1 > q0);
      auto block = [&](auto mask_c) {
        constexpr bool MASK = decltype(mask_c)::value;
        float mxa[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        {
          uint32_t cur[16], nxt[16];
          tmem_ld16(lb + s_col, cur);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < BN / 16; ++c) {
            if (c + 1 < BN / 16) tmem_ld16(lb + s_col + (c + 1) * 16, nxt);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float v = __uint_as_float(cur[i]);
              if (MASK && k0 + c * 16 + i > row) v = -INFINITY;
              mxa[i & 3] = fmaxf(mxa[i & 3], v);
            }
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) cur[i] = nxt[i];
          }
        }
        const float mx = fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3]));
        const float m_new = mx * scale_log2;
        const bool need = m_new > m_used + 8.0f;
        if (j > 0 && __any_sync(0xffffffff, need)) {
          const float f = need ? ex2(m_used - m_new) : 1.0f;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(lb + o_col + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
            tmem_st16(lb + o_col + c * 32, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
            tmem_st16(lb + o_col + c * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&r[16]));
          }
          if (need) l *= f;
        }
        if (need) m_used = m_new;
        f2 rs2[2] = {f2{0.f, 0.f}, f2{0.f, 0.f}};
        const f2 nm2{-m_used, -m_used}, sl2{scale_log2, scale_log2};
        {
          uint32_t cur[16], nxt[16];
          tmem_ld16(lb + s_col, cur);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < BN / 16; ++c) {
            if (c + 1 < BN / 16) tmem_ld16(lb + s_col + (c + 1) * 16, nxt);
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const f2 x = fma2(f2{__uint_as_float(cur[i]), __uint_as_float(cur[i + 1])}, sl2, nm2);
              f2 p;
              if (emu_pair(i >> 1)) {
                p = exp2_fma2(x);
              } else {
                p.x = ex2(x.x);
                p.y = ex2(x.y);
              }
              if (MASK) {
                if (k0 + c * 16 + i > row) p.x = 0.f;
                if (k0 + c * 16 + i + 1 > row) p.y = 0.f;
              }
              rs2[(i >> 1) & 1] = add2(rs2[(i >> 1) & 1], p);
              pk[i >> 1] = pack_bf16(p.x, p.y);
            }
            tmem_st8(lb + s_col + c * 8, pk);
            if (c == BN / 32 - 1) {
              tmem_st_wait();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(ph_lead);
            }
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) cur[i] = nxt[i];
          }
        }
        const f2 rs = add2(rs2[0], rs2[1]);
        l += rs.x + rs.y;
      };
      if (mask) block(std::true_type{});
      else block(std::false_type{});
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(pf_lead);
    }
    mbar_wait(&o_done[tile], 0);
    tc_fence_after();
    const float inv = 1.0f / l;
    const bool ok = row < qlo + qn;
    __nv_bfloat16* o = out + (int64_t)(row - qlo) * ld_out + head * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(lb + o_col + c * 32, r);
      tmem_ld_wait();
      if (ok) {
        uint4* d4 = reinterpret_cast<uint4*>(o + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          d4[e] = make_uint4(pack_bf16(__uint_as_float(r[8 * e]) * inv, __uint_as_float(r[8 * e + 1]) * inv),
                             pack_bf16(__uint_as_float(r[8 * e + 2]) * inv, __uint_as_float(r[8 * e + 3]) * inv),
                             pack_bf16(__uint_as_float(r[8 * e + 4]) * inv, __uint_as_float(r[8 * e + 5]) * inv),
                             pack_bf16(__uint_as_float(r[8 * e + 6]) * inv, __uint_as_float(r[8 * e + 7]) * inv));
      }
    }
    if (ok) lse[(int64_t)head * qn + (row - qlo)] = (m_used + log2f(l)) * LN2;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}

// ================================================================== backward
// RoPE^T + scale on one accumulator row held as chunk pairs (cols c*32.. and c*32 + D/2..)
template <int D>
__device__ __forceinline__ void rope_t_rows(float* a, float* b, const float2* rope, int64_t pos, int k0, float sc) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float x = a[i] * sc, y = b[i] * sc;
    if (rope) {
      const float2 cs = rope[pos * (D / 2) + k0 + i];
      const float nx = x * cs.x + y * cs.y;
      y = -x * cs.y + y * cs.x;
      x = nx;
    }
    a[i] = x;
    b[i] = y;
  }
}

__device__ __forceinline__ void store32_bf16(__nv_bfloat16* dst, const float* v) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int e = 0; e < 4; ++e)
    d4[e] = make_uint4(pack_bf16(v[8 * e], v[8 * e + 1]), pack_bf16(v[8 * e + 2], v[8 * e + 3]),
                       pack_bf16(v[8 * e + 4], v[8 * e + 5]), pack_bf16(v[8 * e + 6], v[8 * e + 7]));
}

template <int D>
__device__ __forceinline__ void row_to_tmem(uint32_t lb, uint32_t col, const __nv_bfloat16* src, bool ok) {
#pragma unroll
  for (int c = 0; c < D / 64; ++c) {
    uint32_t r[32];
    const uint4* s4 = reinterpret_cast<const uint4*>(src + c * 64);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 v = ok ? __ldg(s4 + q) : make_uint4(0, 0, 0, 0);
      r[4 * q] = v.x; r[4 * q + 1] = v.y; r[4 * q + 2] = v.z; r[4 * q + 3] = v.w;
    }
    tmem_st32(lb + col + c * 32, r);
  }
}

// ============================================================ backward v4
// 128 x 128 blocks everywhere: every MMA has N = 128 (tcgen05 MMAs with N = 64 run
// at 2/3 of the tensor peak, tools/mma_probe.cu).  The elementwise results P^T / dS^T
// (dK/dV kernel) and dS (dQ kernel) are written back into TMEM as packed bf16 and
// used as the A operand of the next MMA, so no shared-memory round trip and no
// generic->async proxy fence sits on the critical path.  Two elementwise
// warpgroups split the 128 columns of a block: warpgroup w owns columns
// [64w, 64w + 64) and writes its packed half into TMEM columns [64w, 64w + 32) of
// the same region, so the A operand's k-step kk lives at column acol(kk).
// (warpgroup w of NWG owns CW = 128 / NWG columns and writes their packed half into
// columns [CW w, CW w + CW / 2))
template <int NWG>
__device__ __forceinline__ uint32_t acol(int kk) {
  constexpr int CW = 128 / NWG, KPW = CW / 16;    // k-steps (16 columns) per warpgroup
  return (kk / KPW) * CW + (kk % KPW) * 8;
}

__device__ __forceinline__ float4 lds4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

template <int D>
struct BwdKV4Cfg {
  static constexpr int T = 128 * D * 2;      // one [128][D] bf16 tile
  static constexpr int NST = D == 128 ? 2 : 3;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = T;
  static constexpr int Q_OFF = 2 * T;        // [NST]
  static constexpr int O_OFF = Q_OFF + NST * T;
  static constexpr int L_OFF = O_OFF + NST * T;    // lse [NST][128], then D [NST][128]
  static constexpr int BAR_OFF = L_OFF + 2 * NST * 512;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
};

// dK / dV.  CTA = (128-key block kb, head); loop over 128-query blocks i.
//   MMA order:  S^T_0 dP^T_0 | dV_0 S^T_1 | dK_0 dP^T_1 | dV_1 S^T_2 | dK_1 dP^T_2 ...
//   S^T = K Q^T (TMEM cols 0..127), dP^T = V dO^T (cols 128..255),
//   P^T (bf16) overwrites S^T, dS^T = P^T (dP^T - D) overwrites dP^T;
//   dV += P^T dO (cols 256..), dK += dS^T Q (cols 256 + D..).
// A later MMA that overwrites a region is issued after the MMA that reads it, and
// tcgen05 MMAs of one thread execute in order.
template <int D, int NWG>
__global__ void __launch_bounds__(128 + 128 * NWG, 1)
    attn_bwd_dkdv4_kernel(const __grid_constant__ CUtensorMap tkv, const __grid_constant__ CUtensorMap tq,
                          const __grid_constant__ CUtensorMap tdo, const float* __restrict__ lse,
                          const float* __restrict__ Dd, int s, int heads, int causal, __nv_bfloat16* __restrict__ dqkv,
                          int64_t ld, const float2* __restrict__ rope, float scale, float scale_log2, int qlo,
                          int qn, int kcol, int vcol, float* __restrict__ acc, int64_t ld_acc, int grp,
                          const int* __restrict__ segs, __nv_bfloat16* __restrict__ ds_out, int64_t ds_ld,
                          int64_t ds_hstride, int head0) {
  using C = BwdKV4Cfg<D>;
  constexpr int NST = C::NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* q_full = bar + 0;             // [NST]
  uint64_t* q_empty = bar + NST;          // [NST]
  uint64_t* kv_full = bar + 2 * NST;
  uint64_t* s_full = bar + 2 * NST + 1;
  uint64_t* dp_full = bar + 2 * NST + 2;
  uint64_t* p_full = bar + 2 * NST + 3;
  uint64_t* ds_full = bar + 2 * NST + 4;
  uint64_t* fin = bar + 2 * NST + 5;
  uint64_t* p_half = bar + 2 * NST + 6;   // first half of every warpgroup's P^T columns written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2 * NST + 7);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // GQA: CTA = (key block, key / value head); its grp query heads run one after the
  // other through the same loop (iteration i = query head g = i / nqh, query block
  // qstart + i % nqh), so dK / dV accumulate over the group in TMEM
  // ds_out (dS through HBM): also store dS^T = P^T o (dP^T - D) of every
  // (key block, query block) as bf16 rows [query head - head0 * grp][key][query]; the dQ
  // kernel is then replaced by one batched causal GEMM dQ = dS K
  const int kb = blockIdx.x, head = head0 + blockIdx.y;
  const int k0 = kb * 128;
  // only the query blocks of [qlo, qlo + qn) contribute (dO, LSE, D are local to them);
  // the launch covers only key blocks that have at least one
  // varlen packing: only the queries of the key block's own sequence
  const int qstart = max(causal ? kb : (segs ? segs[2 * kb] : 0), qlo / 128);
  const int nqh = (segs ? min((qlo + qn) / 128, segs[2 * kb + 1]) : (qlo + qn) / 128) - qstart;
  const int nq = nqh * grp;
  constexpr int ST_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 256 + D;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tkv);
    tma_prefetch(&tq);
    tma_prefetch(&tdo);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&q_full[i], 1);
      // the dK MMA's commit plus every elementwise warp (done reading the stage's LSE / D
      // rows: an explicit edge for the bulk copy that overwrites them)
      mbar_init(&q_empty[i], 1 + 4 * NWG);
    }
    mbar_init(kv_full, 1);
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_full, 4 * NWG);
    mbar_init(p_half, 4 * NWG);
    mbar_init(ds_full, 4 * NWG);
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      mbar_arrive_expect_tx(kv_full, 2 * C::T);
      for (int a = 0; a < D / 64; ++a) {
        tma_load_2d(sm + C::K_OFF + a * 16384, &tkv, kv_full, kcol + head * D + a * 64, k0);
        tma_load_2d(sm + C::V_OFF + a * 16384, &tkv, kv_full, vcol + head * D + a * 64, k0);
      }
      for (int i = 0; i < nq; ++i) {
        const int b = i % NST, q0 = (qstart + i % nqh) * 128, qh = head * grp + i / nqh;
        if (i >= NST) mbar_wait(&q_empty[b], ((i / NST) - 1) & 1);
        mbar_arrive_expect_tx(&q_full[b], 2 * C::T + 1024);
        for (int a = 0; a < D / 64; ++a) {
          tma_load_2d(sm + C::Q_OFF + b * C::T + a * 16384, &tq, &q_full[b], qh * D + a * 64, q0);
          tma_load_2d(sm + C::O_OFF + b * C::T + a * 16384, &tdo, &q_full[b], qh * D + a * 64, q0 - qlo);
        }
        bulk_load(sm + C::L_OFF + b * 512, lse + (int64_t)qh * qn + (q0 - qlo), 512, &q_full[b]);
        bulk_load(sm + C::L_OFF + (NST + b) * 512, Dd + (int64_t)qh * qn + (q0 - qlo), 512, &q_full[b]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idesc_acc = umma_idesc_bf16(128, D, 0, 1);
    const uint32_t sk = smem_u32(sm + C::K_OFF), sv = smem_u32(sm + C::V_OFF);
    auto qtile = [&](int i) { return smem_u32(sm + C::Q_OFF + (i % NST) * C::T); };
    auto otile = [&](int i) { return smem_u32(sm + C::O_OFF + (i % NST) * C::T); };
    auto issue_s = [&](int i) {
      mbar_wait(&q_full[i % NST], (i / NST) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sq = qtile(i);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16(tmem + ST_COL, kmaj_desc(sk, kk), kmaj_desc(sq, kk), idesc_s, kk > 0);
        umma_commit(s_full);
      }
      __syncwarp();
    };
    auto issue_dp = [&](int i) {
      if (elect_one()) {
        const uint32_t so = otile(i);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16(tmem + DP_COL, kmaj_desc(sv, kk), kmaj_desc(so, kk), idesc_s, kk > 0);
        umma_commit(dp_full);
      }
      __syncwarp();
    };
    mbar_wait(kv_full, 0);
    issue_s(0);
    issue_dp(0);
    for (int i = 0; i < nq; ++i) {
      if (lane == 0) PDS_TR2(i, 7);
      // dV += P^T dO in two halves: the k-steps of every warpgroup's first half of
      // columns as soon as those are written, overlapping the second half's exponentials
      constexpr int KPW = 8 / NWG;            // k-steps (16 queries) per warpgroup
      mbar_wait(p_half, i & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t so = otile(i);
#pragma unroll
        for (int w = 0; w < NWG; ++w)
#pragma unroll
          for (int jj = 0; jj < KPW / 2; ++jj) {
            const int kk = w * KPW + jj;
            umma_f16_ts(tmem + DV_COL, tmem + ST_COL + acol<NWG>(kk), mnmaj_desc(so, kk), idesc_acc, (i | kk) != 0);
          }
      }
      __syncwarp();
      mbar_wait(p_full, i & 1);
      if (lane == 0) PDS_TR2(i, 0);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t so = otile(i);
#pragma unroll
        for (int w = 0; w < NWG; ++w)
#pragma unroll
          for (int jj = KPW / 2; jj < KPW; ++jj) {
            const int kk = w * KPW + jj;
            umma_f16_ts(tmem + DV_COL, tmem + ST_COL + acol<NWG>(kk), mnmaj_desc(so, kk), idesc_acc, 1);
          }
      }
      __syncwarp();
      if (i + 1 < nq) issue_s(i + 1);
      mbar_wait(ds_full, i & 1);
      if (lane == 0) PDS_TR2(i, 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sq = qtile(i);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_f16_ts(tmem + DK_COL, tmem + DP_COL + acol<NWG>(kk), mnmaj_desc(sq, kk), idesc_acc, (i | kk) != 0);
        umma_commit(&q_empty[i % NST]);
      }
      __syncwarp();
      if (i + 1 < nq) issue_dp(i + 1);
    }
    if (elect_one()) umma_commit(fin);
    __syncwarp();
  } else if (warp >= 4) {
    constexpr int CW = 128 / NWG;             // query columns per warpgroup
    const int wg = (warp - 4) >> 2;          // query columns [CW wg, CW wg + CW)
    const int q = warp & 3;
    const int t = q * 32 + lane;             // key row (TMEM lane)
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t c_s = lb + ST_COL + CW * wg, c_d = lb + DP_COL + CW * wg;
    for (int i = 0; i < nq; ++i) {
      const int b = i % NST;
      const uint32_t lsm = smem_u32(sm + C::L_OFF + b * 512) + wg * CW * 4;
      const uint32_t dsm = smem_u32(sm + C::L_OFF + (NST + b) * 512) + wg * CW * 4;
      const bool diag = causal && qstart + i % nqh == kb;   // the query block on the key block's diagonal
      float p[CW];
      {
        uint32_t sr[CW / 32][32];
        mbar_wait(s_full, i & 1);
        if (warp == 4 && lane == 0) PDS_TR2(i, 2);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < CW / 32; ++h) tmem_ld32(c_s + 32 * h, sr[h]);
        tmem_ld_wait();
        if (warp == 4 && lane == 0) PDS_TR2(i, 3);
        const f2 sl2{scale_log2, scale_log2}, nlog2e{-LOG2E, -LOG2E};
        // two halves of CW / 2 columns; the first releases its dV MMAs early (p_half)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
          for (int e = hf * CW / 2; e < (hf + 1) * CW / 2; e += 4) {
            const float4 L = lds4(lsm + e * 4);
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
              const f2 sv{__uint_as_float(sr[(e + u) / 32][(e + u) % 32]),
                          __uint_as_float(sr[(e + u + 1) / 32][(e + u + 1) % 32])};
              const f2 nl = mul2(u ? f2{L.z, L.w} : f2{L.x, L.y}, nlog2e);
              const f2 x = fma2(sv, sl2, nl);
              f2 pp;
              if (emu_pair((e + u) >> 1)) {
                pp = exp2_fma2(x);               // share of the pairs on the FMA pipe
              } else {
                pp.x = ex2(x.x);
                pp.y = ex2(x.y);
              }
              p[e + u] = pp.x;
              p[e + u + 1] = pp.y;
            }
          }
          if (diag) {
#pragma unroll
            for (int e = hf * CW / 2; e < (hf + 1) * CW / 2; ++e)
              if (t > CW * wg + e) p[e] = 0.f;
          }
          uint32_t pk[CW / 4];
#pragma unroll
          for (int e = 0; e < CW / 4; ++e) pk[e] = pack_bf16(p[hf * CW / 2 + 2 * e], p[hf * CW / 2 + 2 * e + 1]);
          if (CW == 64) tmem_st16(c_s + hf * CW / 4, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
          else tmem_st8(c_s + hf * CW / 4, *reinterpret_cast<uint32_t(*)[8]>(&pk[0]));
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0 && hf == 0) mbar_arrive(p_half);
        }
        if (lane == 0) mbar_arrive(p_full);
        if (warp == 4 && lane == 0) PDS_TR2(i, 4);
      }
      {
        mbar_wait(dp_full, i & 1);
        if (warp == 4 && lane == 0) PDS_TR2(i, 5);
        tc_fence_after();
        uint32_t pk[CW / 2];
#pragma unroll
        for (int h = 0; h < CW / 32; ++h) {
          uint32_t dv[32];
          tmem_ld32(c_d + 32 * h, dv);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 Dq = lds4(dsm + (32 * h + e) * 4);
            const f2 d0 = mul2(f2{p[32 * h + e], p[32 * h + e + 1]},
                               sub2(f2{__uint_as_float(dv[e]), __uint_as_float(dv[e + 1])}, f2{Dq.x, Dq.y}));
            const f2 d1 = mul2(f2{p[32 * h + e + 2], p[32 * h + e + 3]},
                               sub2(f2{__uint_as_float(dv[e + 2]), __uint_as_float(dv[e + 3])}, f2{Dq.z, Dq.w}));
            pk[16 * h + e / 2] = pack_bf16(d0.x, d0.y);
            pk[16 * h + e / 2 + 1] = pack_bf16(d1.x, d1.y);
          }
        }
        if (CW == 64) tmem_st32(c_d, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
        else tmem_st16(c_d, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
        if (ds_out) {                          // this key row's CW dS values, one contiguous run
          const int qh = i / nqh;               // query head within the group (launch-local)
          const int qcol = (qstart + i % nqh) * 128 + CW * wg;
          uint4* dst = reinterpret_cast<uint4*>(ds_out + ((int64_t)(blockIdx.y * grp + qh)) * ds_hstride +
                                                (int64_t)(k0 + t) * ds_ld + qcol);
#pragma unroll
          for (int e = 0; e < CW / 8; ++e)
            dst[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(ds_full);
          mbar_arrive(&q_empty[b]);
        }
        if (warp == 4 && lane == 0) PDS_TR2(i, 6);
      }
    }
    mbar_wait(fin, 0);
    tc_fence_after();
    const int key = k0 + t;
    if (acc) {
      // accumulate mode (ring attention): dK (scaled, no RoPE^T) at columns head*D and
      // dV at kv_heads*D + head*D of the fp32 row (head = the key / value head), added
      // to what is there
      float* arow = acc + (int64_t)key * ld_acc + head * D;
      for (int task = wg; task < 2 * (D / 32); task += NWG) {
        const int kv = task / (D / 32), c = task % (D / 32);
        uint32_t r[32];
        tmem_ld32(lb + (kv ? DV_COL : DK_COL) + c * 32, r);
        tmem_ld_wait();
        const float sc = kv ? 1.0f : scale;
        float4* d4 = reinterpret_cast<float4*>(arow + kv * (heads / grp) * D + c * 32);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float4 v = d4[e];
          v.x += __uint_as_float(r[4 * e]) * sc;
          v.y += __uint_as_float(r[4 * e + 1]) * sc;
          v.z += __uint_as_float(r[4 * e + 2]) * sc;
          v.w += __uint_as_float(r[4 * e + 3]) * sc;
          d4[e] = v;
        }
      }
    } else {
    __nv_bfloat16* rowp = dqkv + (int64_t)key * ld + head * D;
    // epilogue tasks: D/64 RoPE^T chunk pairs of dK, then D/32 chunks of dV
    for (int task = wg; task < D / 64 + D / 32; task += NWG) {
      if (task < D / 64) {
        const int c = task;
        uint32_t ra[32], rb[32];
        tmem_ld32(lb + DK_COL + c * 32, ra);
        tmem_ld32(lb + DK_COL + c * 32 + D / 2, rb);
        tmem_ld_wait();
        float a[32], bb[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) { a[j] = __uint_as_float(ra[j]); bb[j] = __uint_as_float(rb[j]); }
        rope_t_rows<D>(a, bb, rope, segs ? key - segs[2 * (key / 128)] * 128 : key, c * 32, scale);
        store32_bf16(rowp + kcol + c * 32, a);          // dK at kcol + head * D
        store32_bf16(rowp + kcol + c * 32 + D / 2, bb);
      } else {
        const int c = task - D / 64;
        uint32_t r[32];
        tmem_ld32(lb + DV_COL + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        store32_bf16(rowp + vcol + c * 32, v);          // dV at vcol + head * D
      }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
struct BwdQ4Cfg {
  static constexpr int T = 128 * D * 2;     // K or V [128][D]
  static constexpr int NST = D == 128 ? 3 : 4;
  static constexpr int K_OFF = 0;           // [NST]
  static constexpr int V_OFF = NST * T;     // [NST]
  static constexpr int BAR_OFF = 2 * NST * T;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
};

// dQ.  CTA = (128-query block, head); loop over 128-key blocks j.  Q, dO (the fixed
// A operands) live in TMEM; S = Q K^T (cols 128..255), dP = dO V^T (cols 256..383),
// dS = P (dP - D) overwrites dP as packed bf16, dQ += dS K (cols 384..).
//   MMA order:  S_0 dP_0 | S_1 | dQ_0 dP_1 | S_2 | dQ_1 dP_2 ...
// S_{j+1} is issued as soon as the elementwise warps have read S_j.
template <int D, int NWG>
__global__ void __launch_bounds__(128 + 128 * NWG, 1)
    attn_bwd_dq4_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld, const __nv_bfloat16* __restrict__ dout,
                        int64_t ld_out, const __grid_constant__ CUtensorMap tkv, const float* __restrict__ lse,
                        const float* __restrict__ Dd, int s, int heads, int causal, __nv_bfloat16* __restrict__ dqkv,
                        const float2* __restrict__ rope, float scale, float scale_log2, int qlo, int qn, int kcol,
                        int vcol, int64_t ld_dq, float* __restrict__ acc, int64_t ld_acc, int grp,
                        const int* __restrict__ segs) {
  using C = BwdQ4Cfg<D>;
  constexpr int NST = C::NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* kv_full = bar + 0;            // [NST]
  uint64_t* kv_empty = bar + NST;         // [NST]
  uint64_t* s_full = bar + 2 * NST;
  uint64_t* s_free = bar + 2 * NST + 1;
  uint64_t* dp_full = bar + 2 * NST + 2;
  uint64_t* ds_full = bar + 2 * NST + 3;
  uint64_t* q_ready = bar + 2 * NST + 4;
  uint64_t* fin = bar + 2 * NST + 5;
  uint64_t* ds_half = bar + 2 * NST + 6;  // first half of every warpgroup's dS columns written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2 * NST + 7);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = qn / 128;                 // local query blocks of [qlo, qlo + qn)
  const int qb = qlo / 128 + (causal ? (nqb - 1 - (int)blockIdx.x) : (int)blockIdx.x);
  const int head = blockIdx.y;
  const int q0 = qb * 128;
  // varlen packing: key blocks [kb0, kb0 + nkv) of the query block's own sequence
  const int kb0 = segs ? segs[2 * qb] : 0;
  const int nkv = (causal ? qb + 1 : (segs ? segs[2 * qb + 1] : s / 128)) - kb0;
  constexpr int Q_COL = 0, O_COL = 64, S_COL = 128, DP_COL = 256, DQ_COL = 384;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tkv);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4 * NWG);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 4 * NWG);
    mbar_init(ds_half, 4 * NWG);
    mbar_init(q_ready, 8);
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      for (int j = 0; j < nkv; ++j) {
        const int b = j % NST;
        if (j >= NST) mbar_wait(&kv_empty[b], ((j / NST) - 1) & 1);
        mbar_arrive_expect_tx(&kv_full[b], 2 * C::T);
        for (int a = 0; a < D / 64; ++a) {
          tma_load_2d(sm + C::K_OFF + b * C::T + a * 16384, &tkv, &kv_full[b], kcol + (head / grp) * D + a * 64,
                      (kb0 + j) * 128);
          tma_load_2d(sm + C::V_OFF + b * C::T + a * 16384, &tkv, &kv_full[b], vcol + (head / grp) * D + a * 64,
                      (kb0 + j) * 128);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idesc_q = umma_idesc_bf16(128, D, 0, 1);
    auto ktile = [&](int j) { return smem_u32(sm + C::K_OFF + (j % NST) * C::T); };
    auto vtile = [&](int j) { return smem_u32(sm + C::V_OFF + (j % NST) * C::T); };
    auto issue_s = [&](int j) {
      mbar_wait(&kv_full[j % NST], (j / NST) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sk = ktile(j);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ts(tmem + S_COL, tmem + Q_COL + kk * 8, kmaj_desc(sk, kk), idesc_s, kk > 0);
        umma_commit(s_full);
      }
      __syncwarp();
    };
    auto issue_dp = [&](int j) {
      if (elect_one()) {
        const uint32_t sv = vtile(j);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          umma_f16_ts(tmem + DP_COL, tmem + O_COL + kk * 8, kmaj_desc(sv, kk), idesc_s, kk > 0);
        umma_commit(dp_full);
      }
      __syncwarp();
    };
    mbar_wait(q_ready, 0);
    tc_fence_after();
    issue_s(0);
    issue_dp(0);
    for (int j = 0; j < nkv; ++j) {
      if (lane == 0) PDS_TR(j, 7);
      if (j + 1 < nkv) {
        mbar_wait(s_free, j & 1);
        if (lane == 0) PDS_TR(j, 0);
        tc_fence_after();
        issue_s(j + 1);
      }
      // dQ += dS K in two halves: every warpgroup's first half of dS columns is released
      // while it computes the second
      constexpr int KPW = 8 / NWG;
      mbar_wait(ds_half, j & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sk = ktile(j);
#pragma unroll
        for (int w = 0; w < NWG; ++w)
#pragma unroll
          for (int jj = 0; jj < KPW / 2; ++jj) {
            const int kk = w * KPW + jj;
            umma_f16_ts(tmem + DQ_COL, tmem + DP_COL + acol<NWG>(kk), mnmaj_desc(sk, kk), idesc_q, (j | kk) != 0);
          }
      }
      __syncwarp();
      mbar_wait(ds_full, j & 1);
      if (lane == 0) PDS_TR(j, 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sk = ktile(j);
#pragma unroll
        for (int w = 0; w < NWG; ++w)
#pragma unroll
          for (int jj = KPW / 2; jj < KPW; ++jj) {
            const int kk = w * KPW + jj;
            umma_f16_ts(tmem + DQ_COL, tmem + DP_COL + acol<NWG>(kk), mnmaj_desc(sk, kk), idesc_q, 1);
          }
        umma_commit(&kv_empty[j % NST]);
      }
      __syncwarp();
      if (j + 1 < nkv) issue_dp(j + 1);
    }
    if (elect_one()) umma_commit(fin);
    __syncwarp();
  } else if (warp >= 4) {
    constexpr int CW = 128 / NWG;             // key columns per warpgroup
    const int wg = (warp - 4) >> 2;          // key columns [CW wg, CW wg + CW) of each block
    const int q = warp & 3;
    const int t = q * 32 + lane;
    const int row = q0 + t;
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
    if (wg == 0) row_to_tmem<D>(lb, Q_COL, qkv + (int64_t)row * ld + head * D, true);
    else if (wg == 1) row_to_tmem<D>(lb, O_COL, dout + (int64_t)(row - qlo) * ld_out + head * D, true);
    if (wg < 2) {
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_ready);
    }
    const float nl2 = -lse[(int64_t)head * qn + (row - qlo)] * LOG2E;
    const float dd = Dd[(int64_t)head * qn + (row - qlo)];
    const uint32_t c_s = lb + S_COL + CW * wg, c_d = lb + DP_COL + CW * wg;
    for (int j = 0; j < nkv; ++j) {
      const bool diag = causal && j == nkv - 1;
      float p[CW];
      {
        uint32_t sr[CW / 32][32];
        mbar_wait(s_full, j & 1);
        if (warp == 4 && lane == 0) PDS_TR(j, 2);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < CW / 32; ++h) tmem_ld32(c_s + 32 * h, sr[h]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
        if (warp == 4 && lane == 0) PDS_TR(j, 3);
        const f2 sl2{scale_log2, scale_log2}, nl{nl2, nl2};
#pragma unroll
        for (int e = 0; e < CW; e += 2) {
          const f2 x = fma2(f2{__uint_as_float(sr[e / 32][e % 32]), __uint_as_float(sr[(e + 1) / 32][(e + 1) % 32])},
                            sl2, nl);
          f2 pp;
          if (emu_pair(e >> 1)) {
            pp = exp2_fma2(x);                   // share of the pairs on the FMA pipe
          } else {
            pp.x = ex2(x.x);
            pp.y = ex2(x.y);
          }
          p[e] = pp.x;
          p[e + 1] = pp.y;
        }
        if (diag) {
#pragma unroll
          for (int e = 0; e < CW; ++e)
            if (CW * wg + e > t) p[e] = 0.f;
        }
      }
      if (warp == 4 && lane == 0) PDS_TR(j, 4);
      mbar_wait(dp_full, j & 1);
      if (warp == 4 && lane == 0) PDS_TR(j, 5);
      tc_fence_after();
      // two halves of CW / 2 columns; the first releases its dQ MMAs early (ds_half)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        constexpr int HW = CW / 2;
        uint32_t dv[HW];
        if (HW == 32) tmem_ld32(c_d + hf * HW, *reinterpret_cast<uint32_t(*)[32]>(&dv[0]));
        else tmem_ld16(c_d + hf * HW, *reinterpret_cast<uint32_t(*)[16]>(&dv[0]));
        tmem_ld_wait();
        uint32_t pk[HW / 2];
#pragma unroll
        for (int e = 0; e < HW; e += 2) {
          const f2 d = mul2(f2{p[hf * HW + e], p[hf * HW + e + 1]},
                            sub2(f2{__uint_as_float(dv[e]), __uint_as_float(dv[e + 1])}, f2{dd, dd}));
          pk[e / 2] = pack_bf16(d.x, d.y);
        }
        if (HW == 32) tmem_st16(c_d + hf * HW / 2, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
        else tmem_st8(c_d + hf * HW / 2, *reinterpret_cast<uint32_t(*)[8]>(&pk[0]));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(hf == 0 ? ds_half : ds_full);
      }
      if (warp == 4 && lane == 0) PDS_TR(j, 6);
    }
    mbar_wait(fin, 0);
    tc_fence_after();
    if (acc) {                               // accumulate mode: dQ (scaled, no RoPE^T) into fp32
      float* arow = acc + (int64_t)(row - qlo) * ld_acc + head * D;
      for (int c = wg; c < D / 32; c += NWG) {
        uint32_t r[32];
        tmem_ld32(lb + DQ_COL + c * 32, r);
        tmem_ld_wait();
        float4* d4 = reinterpret_cast<float4*>(arow + c * 32);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float4 v = d4[e];
          v.x += __uint_as_float(r[4 * e]) * scale;
          v.y += __uint_as_float(r[4 * e + 1]) * scale;
          v.z += __uint_as_float(r[4 * e + 2]) * scale;
          v.w += __uint_as_float(r[4 * e + 3]) * scale;
          d4[e] = v;
        }
      }
    } else {
    __nv_bfloat16* rowp = dqkv + (int64_t)row * ld_dq + head * D;
    for (int c = wg; c < D / 64; c += NWG) {
      uint32_t ra[32], rb[32];
      tmem_ld32(lb + DQ_COL + c * 32, ra);
      tmem_ld32(lb + DQ_COL + c * 32 + D / 2, rb);
      tmem_ld_wait();
      float a[32], bb[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) { a[i] = __uint_as_float(ra[i]); bb[i] = __uint_as_float(rb[i]); }
      rope_t_rows<D>(a, bb, rope, segs ? row - kb0 * 128 : row, c * 32, scale);
      store32_bf16(rowp + c * 32, a);
      store32_bf16(rowp + c * 32 + D / 2, bb);
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================ fused backward (d = 128, causal)
// One kernel for dQ, dK and dV: 5 matmuls per (key block, query block) pair instead of
// the split kernels' 7 (the dQ kernel above recomputes S and dP).  CTA = (128-key block
// kb, head), loop over the query blocks qb = kb, kb+1, ... (causal, all s positions):
//   S^T = K Q^T (TMEM cols 0..127) -> P^T (packed bf16, same cols), dV += P^T dO
//   dP^T = V dO^T (cols 128..255) -> dS^T (packed bf16, same cols), dK += dS^T Q
//   dS (bf16) also stored to shared memory (into the dO slot, free once dV and dP^T
//   have read it) and dQ_partial = dS K into cols 128..255 (after dK has read dS^T).
// TMEM is full (S^T | dP^T | dV | dK), so dQ_partial reuses the dP^T region and is read
// out by a dedicated warpgroup before the next dP^T is issued:
//   MMA cycle:  dK_i  dQ_i | dV_{i+1}  dP^T_{i+1}  S^T_{i+2}
// so the readout (and the exponentials of block i+1) overlap dK_i / dQ_i / dV_{i+1}.
//
// dQ across key blocks, deterministically: the partial of key block kb for query block qb
// is added into an fp32 accumulator [heads][qb][32 col-chunks][128 rows][4] in a FIXED
// order kb = qb, qb-1, ..., 0 (a per-(head, qb) counter, acquire / release at gpu scope):
// the diagonal block stores, later ones red.add, and key block 0 (the last) adds its own
// partial, applies RoPE^T and the scale, and writes bf16 dQ.  Key block kb+1 reaches
// query block qb one iteration before key block kb does, so with CTAs of a head claimed
// in the order kb = nkb-1 .. 0 (a ticket counter, not blockIdx, so a CTA only ever waits
// for a CTA that is already running) the order costs no waiting in steady state.
// Head-major claiming keeps one head's accumulator (16 MB at s = 32K) hot in L2.
// ctr: [heads * nkb] turn counters + [1] ticket, zeroed before the launch.
template <int NWG>
struct BwdFCfg {
  static constexpr int D = 128;
  static constexpr int T = 128 * D * 2;      // one [128][128] bf16 tile
  static constexpr int NST = 2;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = T;
  static constexpr int Q_OFF = 2 * T;        // [NST]
  static constexpr int O_OFF = Q_OFF + NST * T;    // [NST] dO, then dS of the same query block
  static constexpr int L_OFF = O_OFF + NST * T;    // lse [NST][128], then D [NST][128]
  static constexpr int BAR_OFF = L_OFF + 2 * NST * 512;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int THREADS = 128 + 128 * NWG + 128;
};
static_assert(BwdFCfg<2>::SMEM <= 232448, "fused backward exceeds 227 KB of shared memory");

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ float4 ld_cg4(const float* p) {
  float4 v;
  asm volatile("ld.relaxed.gpu.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_cg4(float* p, float4 v) {
  asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
template <int R>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R));
}
template <int R>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R));
}

template <int NWG>
__global__ void __launch_bounds__(BwdFCfg<NWG>::THREADS, 1)
    attn_bwd_fused_kernel(const __grid_constant__ CUtensorMap tkv, const __grid_constant__ CUtensorMap tdo,
                          const float* __restrict__ lse, const float* __restrict__ Dd, int s, int heads,
                          __nv_bfloat16* __restrict__ dqkv, int64_t ld, const float2* __restrict__ rope, float scale,
                          float scale_log2, float* __restrict__ dqacc, int* __restrict__ ctr) {
  using C = BwdFCfg<NWG>;
  constexpr int D = 128, NST = C::NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* q_full = bar + 0;             // [NST] Q + LSE
  uint64_t* q_empty = bar + NST;          // [NST]
  uint64_t* o_full = bar + 2 * NST;       // [NST] dO + D
  uint64_t* o_empty = bar + 3 * NST;      // [NST]
  uint64_t* kv_full = bar + 4 * NST;
  uint64_t* s_full = bar + 4 * NST + 1;
  uint64_t* dp_full = bar + 4 * NST + 2;
  uint64_t* p_full = bar + 4 * NST + 3;
  uint64_t* ds_full = bar + 4 * NST + 4;
  uint64_t* fin = bar + 4 * NST + 5;
  uint64_t* p_half = bar + 4 * NST + 6;
  uint64_t* dq_full = bar + 4 * NST + 7;
  uint64_t* dq_free = bar + 4 * NST + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 4 * NST + 9);
  int* tick = reinterpret_cast<int*>(bar + 4 * NST + 10);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = s / 128;
  const int hq = heads * D;
  constexpr int ST_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 256 + D;
  constexpr int DQ_WARP0 = 4 + 4 * NWG;

  if (threadIdx.x == 0) {
    *tick = atomicAdd(ctr + heads * nkb, 1);
    tma_prefetch(&tkv);
    tma_prefetch(&tdo);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1 + 4 * NWG);     // dK commit + elementwise warps done with LSE
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 1 + 4 * NWG);     // dQ commit + elementwise warps done with D
    }
    mbar_init(kv_full, 1);
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_full, 4 * NWG);
    mbar_init(p_half, 4 * NWG);
    mbar_init(ds_full, 4 * NWG);
    mbar_init(fin, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int tk = *tick;
  const int head = tk / nkb;
  const int kb = nkb - 1 - tk % nkb;          // short key blocks first within a head
  const int k0 = kb * 128;
  const int nq = nkb - kb;                    // query blocks kb .. nkb-1

  if (warp < 4) {
    reg_dealloc<72>();
    if (warp == 0) {
      if (elect_one()) {
        mbar_arrive_expect_tx(kv_full, 2 * C::T);
        for (int a = 0; a < D / 64; ++a) {
          tma_load_2d(sm + C::K_OFF + a * 16384, &tkv, kv_full, hq + head * D + a * 64, k0);
          tma_load_2d(sm + C::V_OFF + a * 16384, &tkv, kv_full, 2 * hq + head * D + a * 64, k0);
        }
        for (int i = 0; i < nq; ++i) {
          const int b = i % NST, q0 = (kb + i) * 128;
          if (i >= NST) mbar_wait(&q_empty[b], ((i / NST) - 1) & 1);
          mbar_arrive_expect_tx(&q_full[b], C::T + 512);
          for (int a = 0; a < D / 64; ++a)
            tma_load_2d(sm + C::Q_OFF + b * C::T + a * 16384, &tkv, &q_full[b], head * D + a * 64, q0);
          bulk_load(sm + C::L_OFF + b * 512, lse + (int64_t)head * s + q0, 512, &q_full[b]);
          if (i >= NST) mbar_wait(&o_empty[b], ((i / NST) - 1) & 1);
          mbar_arrive_expect_tx(&o_full[b], C::T + 512);
          for (int a = 0; a < D / 64; ++a)
            tma_load_2d(sm + C::O_OFF + b * C::T + a * 16384, &tdo, &o_full[b], head * D + a * 64, q0);
          bulk_load(sm + C::L_OFF + (NST + b) * 512, Dd + (int64_t)head * s + q0, 512, &o_full[b]);
        }
      }
    } else if (warp == 1) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_acc = umma_idesc_bf16(128, D, 0, 1);
      constexpr uint32_t idesc_dq = umma_idesc_bf16(128, D, 1, 1);
      const uint32_t sk = smem_u32(sm + C::K_OFF), sv = smem_u32(sm + C::V_OFF);
      auto qtile = [&](int i) { return smem_u32(sm + C::Q_OFF + (i % NST) * C::T); };
      auto otile = [&](int i) { return smem_u32(sm + C::O_OFF + (i % NST) * C::T); };
      auto issue_s = [&](int i) {
        mbar_wait(&q_full[i % NST], (i / NST) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sq = qtile(i);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            umma_f16(tmem + ST_COL, kmaj_desc(sk, kk), kmaj_desc(sq, kk), idesc_s, kk > 0);
          umma_commit(s_full);
        }
        __syncwarp();
      };
      auto issue_dp = [&](int i) {
        if (elect_one()) {
          const uint32_t so = otile(i);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            umma_f16(tmem + DP_COL, kmaj_desc(sv, kk), kmaj_desc(so, kk), idesc_s, kk > 0);
          umma_commit(dp_full);
        }
        __syncwarp();
      };
      // dV += P^T dO in two halves (every warpgroup's first half of P^T columns first)
      auto issue_dv = [&](int i) {
        constexpr int KPW = 8 / NWG;
        mbar_wait(&o_full[i % NST], (i / NST) & 1);
        mbar_wait(p_half, i & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t so = otile(i);
#pragma unroll
          for (int w = 0; w < NWG; ++w)
#pragma unroll
            for (int jj = 0; jj < KPW / 2; ++jj) {
              const int kk = w * KPW + jj;
              umma_f16_ts(tmem + DV_COL, tmem + ST_COL + acol<NWG>(kk), mnmaj_desc(so, kk), idesc_acc, (i | kk) != 0);
            }
        }
        __syncwarp();
        mbar_wait(p_full, i & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t so = otile(i);
#pragma unroll
          for (int w = 0; w < NWG; ++w)
#pragma unroll
            for (int jj = KPW / 2; jj < KPW; ++jj) {
              const int kk = w * KPW + jj;
              umma_f16_ts(tmem + DV_COL, tmem + ST_COL + acol<NWG>(kk), mnmaj_desc(so, kk), idesc_acc, 1);
            }
        }
        __syncwarp();
      };
      mbar_wait(kv_full, 0);
      issue_s(0);
      issue_dv(0);
      issue_dp(0);
      if (nq > 1) issue_s(1);
      for (int i = 0; i < nq; ++i) {
        mbar_wait(ds_full, i & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sq = qtile(i), sd = otile(i);
          // dQ_partial = dS K: A = dS [queries x keys] (the smem tile read MN-major), B = K
          // (MN-major), into the dP^T region (the elementwise warps have read dP^T)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_f16(tmem + DP_COL, mnmaj_desc(sd, kk), mnmaj_desc(sk, kk), idesc_dq, kk > 0);
          umma_commit(dq_full);
          // dK += dS^T Q: A = dS^T [keys x queries] (the same tile read K-major)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_f16(tmem + DK_COL, kmaj_desc(sd, kk), mnmaj_desc(sq, kk), idesc_acc, (i | kk) != 0);
          umma_commit(&q_empty[i % NST]);
          umma_commit(&o_empty[i % NST]);
        }
        __syncwarp();
        if (i + 1 < nq) {
          issue_dv(i + 1);
          mbar_wait(dq_free, i & 1);          // dQ_i read out of the dP^T region
          tc_fence_after();
          issue_dp(i + 1);
          if (i + 2 < nq) issue_s(i + 2);
        }
      }
      if (elect_one()) umma_commit(fin);
      __syncwarp();
    }
  } else if (warp < DQ_WARP0) {
    reg_alloc<168>();
    constexpr int CW = 128 / NWG;             // query columns per warpgroup
    const int wg = (warp - 4) >> 2;
    const int q = warp & 3;
    const int t = q * 32 + lane;             // key row (TMEM lane)
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t c_s = lb + ST_COL + CW * wg, c_d = lb + DP_COL + CW * wg;
    for (int i = 0; i < nq; ++i) {
      const int b = i % NST;
      const uint32_t lsm = smem_u32(sm + C::L_OFF + b * 512) + wg * CW * 4;
      const uint32_t dsm = smem_u32(sm + C::L_OFF + (NST + b) * 512) + wg * CW * 4;
      const bool diag = i == 0;
      float p[CW];
      {
        uint32_t sr[CW / 32][32];
        mbar_wait(s_full, i & 1);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < CW / 32; ++h) tmem_ld32(c_s + 32 * h, sr[h]);
        tmem_ld_wait();
        const f2 sl2{scale_log2, scale_log2}, nlog2e{-LOG2E, -LOG2E};
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
          for (int e = hf * CW / 2; e < (hf + 1) * CW / 2; e += 4) {
            const float4 L = lds4(lsm + e * 4);
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
              const f2 sv{__uint_as_float(sr[(e + u) / 32][(e + u) % 32]),
                          __uint_as_float(sr[(e + u + 1) / 32][(e + u + 1) % 32])};
              const f2 nl = mul2(u ? f2{L.z, L.w} : f2{L.x, L.y}, nlog2e);
              const f2 x = fma2(sv, sl2, nl);
              f2 pp;
              if (emu_pair((e + u) >> 1)) {
                pp = exp2_fma2(x);
              } else {
                pp.x = ex2(x.x);
                pp.y = ex2(x.y);
              }
              p[e + u] = pp.x;
              p[e + u + 1] = pp.y;
            }
          }
          if (diag) {
#pragma unroll
            for (int e = hf * CW / 2; e < (hf + 1) * CW / 2; ++e)
              if (t > CW * wg + e) p[e] = 0.f;
          }
          uint32_t pk[CW / 4];
#pragma unroll
          for (int e = 0; e < CW / 4; ++e) pk[e] = pack_bf16(p[hf * CW / 2 + 2 * e], p[hf * CW / 2 + 2 * e + 1]);
          if (CW == 64) tmem_st16(c_s + hf * CW / 4, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
          else tmem_st8(c_s + hf * CW / 4, *reinterpret_cast<uint32_t(*)[8]>(&pk[0]));
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0 && hf == 0) mbar_arrive(p_half);
        }
        if (lane == 0) {
          mbar_arrive(p_full);
          mbar_arrive(&q_empty[b]);
        }
      }
      {
        mbar_wait(dp_full, i & 1);
        tc_fence_after();
        uint32_t pk[CW / 2];
#pragma unroll
        for (int h = 0; h < CW / 32; ++h) {
          uint32_t dv[32];
          tmem_ld32(c_d + 32 * h, dv);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 Dq = lds4(dsm + (32 * h + e) * 4);
            const f2 d0 = mul2(f2{p[32 * h + e], p[32 * h + e + 1]},
                               sub2(f2{__uint_as_float(dv[e]), __uint_as_float(dv[e + 1])}, f2{Dq.x, Dq.y}));
            const f2 d1 = mul2(f2{p[32 * h + e + 2], p[32 * h + e + 3]},
                               sub2(f2{__uint_as_float(dv[e + 2]), __uint_as_float(dv[e + 3])}, f2{Dq.z, Dq.w}));
            pk[16 * h + e / 2] = pack_bf16(d0.x, d0.y);
            pk[16 * h + e / 2 + 1] = pack_bf16(d1.x, d1.y);
          }
        }
        // dS row (key t, this warpgroup's CW queries) into the dO slot: the MN-major A
        // operand of dQ and the K-major A operand of dK; 64-query atom (CW wg) / 64,
        // 16-byte chunks from (CW wg % 64) / 8
        {
          uint8_t* dst = sm + C::O_OFF + b * C::T;
          const int atom = (CW * wg) / 64, c0 = ((CW * wg) % 64) / 8;
#pragma unroll
          for (int c = 0; c < CW / 8; ++c)
            st_sw128(dst, 16384, t, atom, c0 + c, make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(ds_full);
          mbar_arrive(&o_empty[b]);
        }
      }
    }
    mbar_wait(fin, 0);
    tc_fence_after();
    const int key = k0 + t;
    __nv_bfloat16* rowp = dqkv + (int64_t)key * ld + head * D;
    for (int task = wg; task < D / 64 + D / 32; task += NWG) {
      if (task < D / 64) {
        const int c = task;
        uint32_t ra[32], rb[32];
        tmem_ld32(lb + DK_COL + c * 32, ra);
        tmem_ld32(lb + DK_COL + c * 32 + D / 2, rb);
        tmem_ld_wait();
        float a[32], bb[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) { a[j] = __uint_as_float(ra[j]); bb[j] = __uint_as_float(rb[j]); }
        rope_t_rows<D>(a, bb, rope, key, c * 32, scale);
        store32_bf16(rowp + hq + c * 32, a);
        store32_bf16(rowp + hq + c * 32 + D / 2, bb);
      } else {
        const int c = task - D / 64;
        uint32_t r[32];
        tmem_ld32(lb + DV_COL + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        store32_bf16(rowp + 2 * hq + c * 32, v);
      }
    }
  } else {
    // dQ warpgroup: dQ_partial out of TMEM (query row t = TMEM lane) in 16-column chunks,
    // added to the fp32 accumulator [head][s][128] with red.global.add.v4.f32 straight
    // from registers, every thread along its own 512-byte row (no shared-memory staging:
    // the staging stores plus bulk reductions cost more shared-memory bandwidth than the
    // kernel has to spare; per-thread rows are the fastest register red pattern,
    // tools/l2_reduce_probe.cu), in key-block order (the turn counter).
    reg_dealloc<104>();
    const int q = warp & 3;
    const int t = q * 32 + lane;
    const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
    for (int i = 0; i < nq; ++i) {
      const int qb = kb + i;
      int* turn = ctr + head * nkb + qb;
      float* acc = dqacc + ((int64_t)head * s + qb * 128 + t) * 128;
      mbar_wait(dq_full, i & 1);
      tc_fence_after();
      if (i > 0) {                           // not the diagonal block: key block kb+1 first
        if (t == 0) {
          int ns = 32;
          while (ld_acquire_gpu(turn) < i) {
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
          }
        }
        named_bar(1, 128);
      }
      uint32_t r[2][16];
      tmem_ld16(lb + DP_COL, r[0]);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        tmem_ld_wait();
        if (c + 1 < 8) {
          tmem_ld16(lb + DP_COL + 16 * (c + 1), r[(c + 1) & 1]);
        } else {                             // the dP^T region may be overwritten
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dq_free);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t* v = &r[c & 1][4 * j];
          float* pp = acc + 16 * c + 4 * j;
          if (i == 0) st_cg4(pp, make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]),
                                             __uint_as_float(v[3])));
          else red_add_v4(pp, __uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]),
                          __uint_as_float(v[3]));
        }
      }
      if (kb > 0) {                          // hand the turn to key block kb-1
        __threadfence();
        named_bar(1, 128);
        if (t == 0) st_release_gpu(turn, i + 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// dQ = RoPE^T(scale * accumulator) in bf16 (the fused kernel's fp32 dQ, [heads][s][128]).
// Thread = (row, 8-column group g): columns 8g..8g+7 and their RoPE partners 64+8g.. .
__global__ void __launch_bounds__(256) attn_dq_finish_kernel(const float* __restrict__ dqacc, int s, int heads,
                                                           __nv_bfloat16* __restrict__ dqkv, int64_t ld,
                                                           const float2* __restrict__ rope, float scale) {
  const int rl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t rb = blockIdx.x;                 // 32-row band of one head
  const int head = (int)(rb / (s / 32));
  const int row = (int)(rb % (s / 32)) * 32 + rl;
  const float* acc = dqacc + ((int64_t)head * s + row) * 128;
  const float4 a0 = __ldcs(reinterpret_cast<const float4*>(acc + 8 * g));
  const float4 a1 = __ldcs(reinterpret_cast<const float4*>(acc + 8 * g + 4));
  const float4 b0 = __ldcs(reinterpret_cast<const float4*>(acc + 64 + 8 * g));
  const float4 b1 = __ldcs(reinterpret_cast<const float4*>(acc + 68 + 8 * g));
  float a[8], b[8];
  a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
  b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w; b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
  uint32_t pa[4], pb[4];
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    float x0 = a[i] * scale, y0 = b[i] * scale, x1 = a[i + 1] * scale, y1 = b[i + 1] * scale;
    if (rope) {
      const float4 cs = *reinterpret_cast<const float4*>(rope + (int64_t)row * 64 + 8 * g + i);
      const float n0 = x0 * cs.x + y0 * cs.y, n1 = x1 * cs.z + y1 * cs.w;
      y0 = -x0 * cs.y + y0 * cs.x;
      y1 = -x1 * cs.w + y1 * cs.z;
      x0 = n0;
      x1 = n1;
    }
    pa[i / 2] = pack_bf16(x0, x1);
    pb[i / 2] = pack_bf16(y0, y1);
  }
  __nv_bfloat16* o = dqkv + (int64_t)row * ld + head * 128 + 8 * g;
  *reinterpret_cast<uint4*>(o) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
  *reinterpret_cast<uint4*>(o + 64) = make_uint4(pb[0], pb[1], pb[2], pb[3]);
}

// ------------------------------------------------------------------ host
int attn_debug_trace(long long* host_out, int rows) {
#ifdef PDS_TRACE
  return (int)cudaMemcpyFromSymbol(host_out, g_trace, (size_t)rows * 8 * sizeof(long long));
#else
  (void)host_out;
  (void)rows;
  return -1;
#endif
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_map_rows(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld,
                  uint32_t box_rows = 128) {
  auto enc = encode_fn();
  if (!enc) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// q: queries [rows of the q map][ld_q] (head i at column i*D); kv: keys at column kcol
// and values at vcol (head i at + i*D) of [s][ld_kv]; q == kv with kcol = heads*D, vcol =
// 2*heads*D is the packed [Q | K | V] buffer.  Query rows [qlo, qlo + qn) of the q map.
// PDS_ATTN_FWD=pair selects the CTA-pair forward (opt-in): measured slower than the
// single-CTA kernel (s = 32K: 1010 vs 1341 TF/s; ncu at 16K: tensor pipe 47.5 %, the
// softmax warps wait on S — every P half-release of either CTA reaches the leader's MMA
// thread through a cluster-scope remote arrive, which lengthens the S -> softmax -> PV
// -> S chain more than the halved operand traffic saves; profiles/r02_attn_fwd_pair.md)
static int fwd_pair_mode() {
  static const int v = [] {
    const char* e = getenv("PDS_ATTN_FWD");
    return (e && std::string(e) == "pair") ? 1 : 0;
  }();
  return v;
}

static int fwd_pair(const void* q, int64_t ld_q, uint64_t q_rows, const void* kv, int64_t ld_kv, int kcol, int vcol,
                    int s, int heads, int causal, void* out, int64_t ld_out, void* lse, int qlo, int qn,
                    cudaStream_t st) {
  constexpr int D = 128;
  CUtensorMap tmq, tmk, tmv;
  int rc = make_map_rows(&tmq, q, (uint64_t)heads * D, q_rows, (uint64_t)ld_q, 128);
  rc |= make_map_rows(&tmk, kv, (uint64_t)vcol + heads * D, (uint64_t)s, (uint64_t)ld_kv, 64);
  rc |= make_map_rows(&tmv, kv, (uint64_t)vcol + heads * D, (uint64_t)s, (uint64_t)ld_kv, 128);
  if (rc) return (int)cudaErrorInvalidValue;
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(attn_fwd_pair_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdPairCfg::SMEM);
    once = true;
  }
  const float scale_log2 = (1.0f / sqrtf((float)D)) * LOG2E;
  attn_fwd_pair_tc_kernel<<<dim3(2 * ((qn + 511) / 512), heads), 384, FwdPairCfg::SMEM, st>>>(
      tmq, tmk, tmv, s, heads, causal, reinterpret_cast<__nv_bfloat16*>(out), ld_out, reinterpret_cast<float*>(lse),
      scale_log2, qlo, qn, kcol, vcol);
  return (int)cudaGetLastError();
}

template <int D>
static int fwd_tc_t(const void* q, int64_t ld_q, uint64_t q_rows, const void* kv, int64_t ld_kv, int kcol, int vcol,
                    int s, int heads, int causal, void* out, int64_t ld_out, void* lse, int qlo, int qn,
                    cudaStream_t st, int grp = 1, const int* segs = nullptr) {
  if (D == 128 && fwd_pair_mode() && grp == 1 && !segs)
    return fwd_pair(q, ld_q, q_rows, kv, ld_kv, kcol, vcol, s, heads, causal, out, ld_out, lse, qlo, qn, st);
  CUtensorMap tm, tmq;
  int rc = make_map_rows(&tm, kv, (uint64_t)vcol + heads / grp * D, (uint64_t)s, (uint64_t)ld_kv);
  rc |= make_map_rows(&tmq, q, (uint64_t)heads * D, q_rows, (uint64_t)ld_q);
  if (rc) return (int)cudaErrorInvalidValue;
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(attn_fwd_tc_kernel<D, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Fwd2Cfg<D>::SMEM);
    cudaFuncSetAttribute(attn_fwd_tc_kernel<D, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Fwd2Cfg<D>::SMEM);
    once = true;
  }
  // register pass by default: bit-identical to the two-pass softmax, 0.3 % faster at fixed
  // clocks, ~1 % event-timed (profiles/raw_r02/ab_fwd_*); PDS_ATTN_FWD=2pass selects the latter
  static const int fmode = [] {               // 0: two-pass, 1: register pass, 2: split (NS = 2)
    const char* e = getenv("PDS_ATTN_FWD");
    if (e && std::string(e) == "2pass") return 0;
    if (e && std::string(e) == "split") return 2;
    return 1;
  }();
  static bool once2 = false;
  if (!once2) {
    cudaFuncSetAttribute(attn_fwd_tc_kernel<D, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Fwd2Cfg<D>::SMEM);
    once2 = true;
  }
  const float scale_log2 = (1.0f / sqrtf((float)D)) * LOG2E;
  auto kern = fmode == 2 ? attn_fwd_tc_kernel<D, true, 2>
                         : fmode == 1 ? attn_fwd_tc_kernel<D, true, 1> : attn_fwd_tc_kernel<D, false, 1>;
  const int nthr = fmode == 2 ? 128 + 512 : 384;
  kern<<<dim3((qn + 255) / 256, heads), nthr, Fwd2Cfg<D>::SMEM, st>>>(
      tm, tmq, s, heads, causal, reinterpret_cast<__nv_bfloat16*>(out), ld_out, reinterpret_cast<float*>(lse),
      scale_log2, qlo, qn, kcol, vcol, grp, segs);
  return (int)cudaGetLastError();
}

// packed [Q (heads) | K (kv_heads) | V (kv_heads)] rows; kv_heads = 0: heads (MHA)
int attn_fwd_tc(const void* qkv, int64_t ld, int s, int heads, int d, int causal, void* out, int64_t ld_out,
                void* lse, cudaStream_t st, int qlo, int qn, int kv_heads, const int* segs) {
  if (qn < 0) qn = s;
  if (segs && (qlo != 0 || qn != s)) return (int)cudaErrorInvalidValue;
  if (kv_heads <= 0) kv_heads = heads;
  if (s % 128 || (ld % 8) || qlo % 128 || qn % 128 || qn <= 0 || qlo + qn > s || heads % kv_heads)
    return (int)cudaErrorInvalidValue;
  const int hq = heads * d, hk = kv_heads * d, grp = heads / kv_heads;
  if (d == 128)
    return fwd_tc_t<128>(qkv, ld, s, qkv, ld, hq, hq + hk, s, heads, causal, out, ld_out, lse, qlo, qn, st, grp, segs);
  if (d == 64)
    return fwd_tc_t<64>(qkv, ld, s, qkv, ld, hq, hq + hk, s, heads, causal, out, ld_out, lse, qlo, qn, st, grp, segs);
  return (int)cudaErrorInvalidValue;
}

// One (query block, key block) pair of ring attention: queries q [sq][ld_q] against keys /
// values of kv [sk][ld_kv] (columns kcol / vcol); causal = the diagonal pair (sq == sk,
// aligned positions), else every key is visible.  out / lse as attn_fwd_tc (the pair's
// own softmax; pairs merge by log-sum-exp).
int attn_fwd_pair(const void* q, int64_t ld_q, const void* kv, int64_t ld_kv, int kcol, int vcol, int sq, int sk,
                  int heads, int d, int causal, void* out, int64_t ld_out, void* lse, cudaStream_t st, int kv_heads) {
  if (kv_heads <= 0) kv_heads = heads;
  if (sq % 128 || sk % 128 || sq <= 0 || sk <= 0 || ld_q % 8 || ld_kv % 8 || kcol % 8 || vcol % 8 ||
      (causal && sq != sk) || heads % kv_heads)
    return (int)cudaErrorInvalidValue;
  const int grp = heads / kv_heads;
  if (d == 128)
    return fwd_tc_t<128>(q, ld_q, sq, kv, ld_kv, kcol, vcol, sk, heads, causal, out, ld_out, lse, 0, sq, st, grp);
  if (d == 64)
    return fwd_tc_t<64>(q, ld_q, sq, kv, ld_kv, kcol, vcol, sk, heads, causal, out, ld_out, lse, 0, sq, st, grp);
  return (int)cudaErrorInvalidValue;
}

}  // namespace pds

namespace pds {
// q / kv as fwd_tc_t.  dqkv != NULL: bf16 dQ (RoPE^T) into dqkv [q rows][ld] at columns
// head*D and dK / dV into dqkv at kcol / vcol of the key rows (the packed-buffer layout:
// q == kv == the QKV buffer).  dqkv == NULL: accumulate mode — dQ (scaled) added into
// dq_acc [qn][heads*D] fp32, dK (scaled) / dV into dkv_acc [s][2*heads*D] fp32, no RoPE^T.
template <int D>
static int bwd_tc_t(const void* q, int64_t ld_q, uint64_t q_rows, const void* kv, int64_t ld_kv, int kcol, int vcol,
                    const void* dout, int64_t ld_out, const void* lse, const float* Dd, int s, int heads, int causal,
                    void* dqkv, int64_t ld, const void* rope, int qlo, int qn, float* dq_acc, int64_t ld_dqa,
                    float* dkv_acc, int64_t ld_dkva, cudaStream_t st, int grp = 1, const int* segs = nullptr,
                    __nv_bfloat16* ds_out = nullptr, int64_t ds_ld = 0, int64_t ds_hstride = 0, int head0 = 0,
                    int kv_launch = 0) {
  CUtensorMap kv128, q128, do128;
  int rc = make_map_rows(&kv128, kv, (uint64_t)vcol + heads / grp * D, s, ld_kv, 128);
  rc |= make_map_rows(&q128, q, (uint64_t)heads * D, q_rows, ld_q, 128);
  rc |= make_map_rows(&do128, dout, (uint64_t)heads * D, qn, ld_out, 128);
  if (rc) return (int)cudaErrorInvalidValue;
  // Elementwise warpgroups per CTA, measured under fixed clocks (ncu --clock-control
  // base, s = 16384): dK/dV 4 (4766 us vs 4792 with 2), dQ 2 (3408 us vs 3484 with 4).
  // PDS_BWD_NWG=2|4 forces both (A/B).
  static const int force = [] {
    const char* e = getenv("PDS_BWD_NWG");
    return e ? atoi(e) : 0;
  }();
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(attn_bwd_dkdv4_kernel<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdKV4Cfg<D>::SMEM);
    cudaFuncSetAttribute(attn_bwd_dq4_kernel<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdQ4Cfg<D>::SMEM);
    cudaFuncSetAttribute(attn_bwd_dkdv4_kernel<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdKV4Cfg<D>::SMEM);
    cudaFuncSetAttribute(attn_bwd_dq4_kernel<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdQ4Cfg<D>::SMEM);
    once = true;
  }
  const float scale = 1.0f / sqrtf((float)D);
  const float scale_log2 = scale * LOG2E;
  auto dkdv = [&](auto nw) {
    constexpr int NW = decltype(nw)::value;
    // the Q map is the K/V map (same buffer, same box): only the column offset differs
    // causal: key blocks past the last local query get nothing (the caller zeroes them)
    const int nkb = causal ? (qlo + qn) / 128 : s / 128;
    attn_bwd_dkdv4_kernel<D, NW><<<dim3(nkb, kv_launch > 0 ? kv_launch : heads / grp), 128 + 128 * NW,
                                    BwdKV4Cfg<D>::SMEM, st>>>(
        kv128, q128, do128, reinterpret_cast<const float*>(lse), Dd, s, heads, causal,
        reinterpret_cast<__nv_bfloat16*>(dqkv), ld, reinterpret_cast<const float2*>(rope), scale, scale_log2,
        qlo, qn, kcol, vcol, dkv_acc, ld_dkva, grp, segs, ds_out, ds_ld, ds_hstride, head0);
  };
  auto dq = [&](auto nw) {
    constexpr int NW = decltype(nw)::value;
    attn_bwd_dq4_kernel<D, NW><<<dim3(qn / 128, heads), 128 + 128 * NW, BwdQ4Cfg<D>::SMEM, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(q), ld_q, reinterpret_cast<const __nv_bfloat16*>(dout), ld_out, kv128,
        reinterpret_cast<const float*>(lse), Dd, s, heads, causal, reinterpret_cast<__nv_bfloat16*>(dqkv),
        reinterpret_cast<const float2*>(rope), scale, scale_log2, qlo, qn, kcol, vcol, ld, dq_acc, ld_dqa, grp,
        segs);
  };
  if (force == 2) dkdv(std::integral_constant<int, 2>{});
  else dkdv(std::integral_constant<int, 4>{});
  if (ds_out) return (int)cudaGetLastError();        // dQ by the caller's GEMM from dS
  if (force == 4) dq(std::integral_constant<int, 4>{});
  else dq(std::integral_constant<int, 2>{});
  return (int)cudaGetLastError();
}

// Fused backward (d = 128, causal, all s query positions): dqacc holds heads * s * 128
// fp32, ctr heads * (s / 128) + 1 ints that must be zero at launch.
int attn_bwd_fused_tc(const void* qkv, int64_t ld, const void* dout, int64_t ld_out, const void* lse, const float* Dd,
                      int s, int heads, void* dqkv, const void* rope, float* dqacc, int* ctr, cudaStream_t st) {
  if (s % 128 || ld % 8 || ld_out % 8 || !dqacc || !ctr) return (int)cudaErrorInvalidValue;
  constexpr int NWG = 2;
  using C = BwdFCfg<NWG>;
  CUtensorMap kv128, do128;
  int rc = make_map_rows(&kv128, qkv, (uint64_t)3 * heads * 128, s, ld, 128);
  rc |= make_map_rows(&do128, dout, (uint64_t)heads * 128, s, ld_out, 128);
  if (rc) return (int)cudaErrorInvalidValue;
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(attn_bwd_fused_kernel<NWG>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    once = true;
  }
  const float scale = 1.0f / sqrtf(128.0f);
  attn_bwd_fused_kernel<NWG><<<(s / 128) * heads, C::THREADS, C::SMEM, st>>>(
      kv128, do128, reinterpret_cast<const float*>(lse), Dd, s, heads, reinterpret_cast<__nv_bfloat16*>(dqkv), ld,
      reinterpret_cast<const float2*>(rope), scale, scale * LOG2E, dqacc, ctr);
  attn_dq_finish_kernel<<<(s / 32) * heads, 256, 0, st>>>(dqacc, s, heads, reinterpret_cast<__nv_bfloat16*>(dqkv),
                                                          ld, reinterpret_cast<const float2*>(rope), scale);
  return (int)cudaGetLastError();
}

// dQ, dK, dV into dqkv (same [s][ld] layout as qkv); Dd = rowsum(dO o O) precomputed
int attn_bwd_tc(const void* qkv, int64_t ld, const void* dout, int64_t ld_out, const void* lse, const float* Dd,
                int s, int heads, int d, int causal, void* dqkv, const void* rope, cudaStream_t st, int qlo, int qn,
                int kv_heads, const int* segs) {
  if (qn < 0) qn = s;
  if (kv_heads <= 0) kv_heads = heads;
  if (s % 128 || ld % 8 || ld_out % 8 || qlo % 128 || qn % 128 || qn <= 0 || qlo + qn > s || heads % kv_heads)
    return (int)cudaErrorInvalidValue;
  if (segs && (qlo != 0 || qn != s)) return (int)cudaErrorInvalidValue;
  const int hq = heads * d, hk = kv_heads * d, grp = heads / kv_heads;
  if (d == 128)
    return bwd_tc_t<128>(qkv, ld, s, qkv, ld, hq, hq + hk, dout, ld_out, lse, Dd, s, heads, causal, dqkv, ld, rope,
                         qlo, qn, nullptr, 0, nullptr, 0, st, grp, segs);
  if (d == 64)
    return bwd_tc_t<64>(qkv, ld, s, qkv, ld, hq, hq + hk, dout, ld_out, lse, Dd, s, heads, causal, dqkv, ld, rope, qlo,
                        qn, nullptr, 0, nullptr, 0, st, grp, segs);
  return (int)cudaErrorInvalidValue;
}

// dS through HBM (reading of the 5-matmul backward): per group of G query
// heads, the dK/dV kernel also writes dS^T [G][s][s] (bf16, causal blocks only) into
// dsbuf, and one batched causal tcgen05 GEMM dQ = scale * dS K (A = dS^T MN-major, B =
// the K columns MN-major, K extent per query block = its causal prefix) applies RoPE^T
// in its epilogue.  Executes 5 matmuls instead of 7; dS costs 2 s^2 B per head of HBM
// traffic (written once, read once).  d = 128, causal, packed [Q | K | V] rows, no
// varlen; G = ds_bytes / (2 s^2) rounded down to whole KV groups (>= 1 required).
int attn_bwd_ds_tc(const void* qkv, int64_t ld, const void* dout, int64_t ld_out, const void* lse, const float* Dd,
                   int s, int heads, int kv_heads, void* dqkv, const void* rope, void* dsbuf, int64_t ds_bytes,
                   cudaStream_t st) {
  constexpr int D = 128;
  if (kv_heads <= 0) kv_heads = heads;
  const int grp = heads / kv_heads;
  const int64_t per = (int64_t)s * s * 2;
  int G = (int)std::min<int64_t>(heads, ds_bytes / per);
  G -= G % grp;
  if (s % 128 || G < 1 || !dsbuf) return (int)cudaErrorInvalidValue;
  const int hq = heads * D, hk = kv_heads * D;
  for (int h0 = 0; h0 < heads; h0 += G) {
    const int g = std::min(G, heads - h0);
    int rc = bwd_tc_t<D>(qkv, ld, s, qkv, ld, hq, hq + hk, dout, ld_out, lse, Dd, s, heads, 1, dqkv, ld, rope, 0, s,
                         nullptr, 0, nullptr, 0, st, grp, nullptr, static_cast<__nv_bfloat16*>(dsbuf), s,
                         (int64_t)s * s, h0 / grp, g / grp);
    if (rc) return rc;
    GemmArgs ga;
    ga.A = dsbuf; ga.lda = s; ga.a_mn = 1; ga.a_rows = (int64_t)g * s;
    ga.B = static_cast<const __nv_bfloat16*>(qkv) + hq + (h0 / grp) * D; ga.ldb = ld; ga.b_mn = 1;
    ga.b_rows = s; ga.b_cols = (int64_t)(kv_heads - h0 / grp) * D;
    ga.M = s; ga.N = D; ga.K = s;
    ga.C = static_cast<__nv_bfloat16*>(dqkv) + h0 * D; ga.ldc = ld;
    ga.epi = EPI_ROPE_T; ga.rope = reinterpret_cast<const float2*>(rope); ga.rope_d = D;
    ga.epi_scale = 1.0f / sqrtf((float)D);
    ga.batch = g; ga.a_boff = s; ga.b_boff = D; ga.b_grp = grp; ga.c_boff = D; ga.k_causal = 1;
    rc = gemm_launch(ga, st);
    if (rc) return rc;
  }
  return 0;
}

// Backward of one ring-attention pair (attn_fwd_pair): lse / Dd [heads][sq] are the
// MERGED row statistics; dQ (scaled) accumulates into dq_acc [sq][heads*d] fp32, dK
// (scaled) / dV into dkv_acc [sk][2*heads*d] fp32; RoPE^T is the caller's.
int attn_bwd_pair(const void* q, int64_t ld_q, const void* kv, int64_t ld_kv, int kcol, int vcol, const void* dout,
                  int64_t ld_out, const void* lse, const float* Dd, int sq, int sk, int heads, int d, int causal,
                  float* dq_acc, int64_t ld_dqa, float* dkv_acc, int64_t ld_dkva, cudaStream_t st, int kv_heads) {
  if (kv_heads <= 0) kv_heads = heads;
  if (sq % 128 || sk % 128 || sq <= 0 || sk <= 0 || ld_q % 8 || ld_kv % 8 || ld_out % 8 || kcol % 8 || vcol % 8 ||
      ld_dqa % 4 || ld_dkva % 4 || (causal && sq != sk) || !dq_acc || !dkv_acc || heads % kv_heads)
    return (int)cudaErrorInvalidValue;
  const int grp = heads / kv_heads;
  if (d == 128)
    return bwd_tc_t<128>(q, ld_q, sq, kv, ld_kv, kcol, vcol, dout, ld_out, lse, Dd, sk, heads, causal, nullptr, 0,
                         nullptr, 0, sq, dq_acc, ld_dqa, dkv_acc, ld_dkva, st, grp);
  if (d == 64)
    return bwd_tc_t<64>(q, ld_q, sq, kv, ld_kv, kcol, vcol, dout, ld_out, lse, Dd, sk, heads, causal, nullptr, 0,
                        nullptr, 0, sq, dq_acc, ld_dqa, dkv_acc, ld_dkva, st, grp);
  return (int)cudaErrorInvalidValue;
}
}  // namespace pds
