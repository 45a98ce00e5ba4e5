// Causal flash attention forward / backward (Eq. 2; causal per
// north_star, reading R-1) on the head-sharded [s][ld] QKV buffer every strategy
// produces (TS after the QKV GEMM, UZ after the sequence->head All-to-All, METP
// after its waves).  Online softmax in fp32 with exp2; LSE stored (natural log)
// for the backward.
//
// ROUND-1 BASELINE (not in the product library): FA2-style warp-level mma.sync.m16n8k16 (bf16 -> fp32)
// with cp.async double-buffered K/V tiles and XOR-swizzled shared memory.  This
// is the correctness baseline the tcgen05/TMEM version replaces.
//
// Backward = three kernels: D = rowsum(dO o O); dK/dV per 128-key block (each
// warp owns 16 keys, computes S^T / dP^T directly so no cross-warp exchange);
// dQ per 128-query block (no atomics).  RoPE^T (reading R-3) and the softmax
// scale are applied to dQ / dK in registers before the bf16 store.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

// Build (A/B only; nothing in the product loads it):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC \
//        -o tools/libfa2_baseline.so tools/fa2_sync_baseline.cu
// It exports pds_fa2_fwd / pds_fa2_bwd with the argument lists of pds_k_attn_fwd /
// pds_k_attn_bwd (+ a caller-provided fp32 D scratch [heads][s]).
namespace pds {
__global__ void attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ out, int64_t ld_out,
                                    const __nv_bfloat16* __restrict__ dout, int s, int heads, int d,
                                    float* __restrict__ Dd) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
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


__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(su32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(su32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pk(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// swizzled tile address: [row][D] bf16, 16-byte chunk c stored at c ^ (row & 7)
template <int D>
__device__ __forceinline__ char* tile_ptr(char* base, int row, int col) {
  const int c = col >> 3;
  return base + row * (D * 2) + (((c ^ (row & 7)) << 4) | ((col & 7) << 1));
}

template <int D, int ROWS, int NT>
__device__ __forceinline__ void load_tile(char* s, const __nv_bfloat16* g, int64_t ld, int tid) {
  constexpr int CH = D / 8;
#pragma unroll
  for (int i = tid; i < ROWS * CH; i += NT) {
    const int r = i / CH, c = i % CH;
    cp_async16(s + r * (D * 2) + ((c ^ (r & 7)) << 4), g + (int64_t)r * ld + c * 8);
  }
}

// A-operand fragments (16 rows x 16 k) of rows [r0, r0+16) at k offset k0
template <int D>
__device__ __forceinline__ void lda_frag(uint32_t (&a)[4], char* s, int r0, int k0, int lane) {
  ldsm_x4(a, tile_ptr<D>(s, r0 + (lane & 15), k0 + ((lane >> 4) << 3)));
}
// B-operand (n = tile rows, k = tile cols, "row.col" non-trans): two n-tiles [n0, n0+16) at k0
// r[0], r[1] = b0, b1 of n-tile n0 ; r[2], r[3] = b0, b1 of n-tile n0 + 8
template <int D>
__device__ __forceinline__ void ldb_frag(uint32_t (&r)[4], char* s, int n0, int k0, int lane) {
  ldsm_x4(r, tile_ptr<D>(s, n0 + (lane & 7) + ((lane >> 4) << 3), k0 + (((lane >> 3) & 1) << 3)));
}
// B-operand from a k-major tile (k = tile rows, n = tile cols) via ldmatrix.trans
template <int D>
__device__ __forceinline__ void ldb_frag_t(uint32_t (&r)[4], char* s, int k0, int n0, int lane) {
  ldsm_x4_t(r, tile_ptr<D>(s, k0 + (lane & 7) + (((lane >> 3) & 1) << 3), n0 + ((lane >> 4) << 3)));
}

constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// ------------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(256, 1)
    attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld, int s, int heads,
                    int causal, __nv_bfloat16* __restrict__ out, int64_t ld_out,
                    float* __restrict__ lse, float scale_log2) {
  constexpr int BM = 128, BN = 64;
  extern __shared__ __align__(128) char sm[];
  char* sQ = sm;
  char* sK = sQ + BM * D * 2;
  char* sV = sK + 2 * BN * D * 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nqb = s / BM;
  const int qb = causal ? (nqb - 1 - blockIdx.x) : blockIdx.x;   // heavy blocks first
  const int head = blockIdx.y;
  const int hq = heads * D;
  const int q0 = qb * BM;
  const __nv_bfloat16* Qg = qkv + (int64_t)q0 * ld + head * D;
  const __nv_bfloat16* Kg = qkv + hq + head * D;
  const __nv_bfloat16* Vg = qkv + 2 * hq + head * D;

  load_tile<D, BM, 256>(sQ, Qg, ld, tid);
  load_tile<D, BN, 256>(sK, Kg, ld, tid);
  load_tile<D, BN, 256>(sV, Vg, ld, tid);
  cp_commit();
  const int nkb = causal ? (q0 + BM) / BN : s / BN;

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  uint32_t qf[D / 16][4];
  const int wr0 = q0 + warp * 16;     // first query row of this warp

  for (int j = 0; j < nkb; ++j) {
    if (j + 1 < nkb) {
      const int b = (j + 1) & 1;
      load_tile<D, BN, 256>(sK + b * BN * D * 2, Kg + (int64_t)(j + 1) * BN * ld, ld, tid);
      load_tile<D, BN, 256>(sV + b * BN * D * 2, Vg + (int64_t)(j + 1) * BN * ld, ld, tid);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) lda_frag<D>(qf[kk], sQ, warp * 16, kk * 16, lane);
    }
    char* cK = sK + (j & 1) * BN * D * 2;
    char* cV = sV + (j & 1) * BN * D * 2;
    const int k0 = j * BN;
    if (!causal || k0 <= wr0 + 15) {
      float sc[BN / 8][4];
#pragma unroll
      for (int i = 0; i < BN / 8; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int np = 0; np < BN / 16; ++np) {
          uint32_t b[4];
          ldb_frag<D>(b, cK, np * 16, kk * 16, lane);
          mma16816(sc[2 * np], qf[kk], b[0], b[1]);
          mma16816(sc[2 * np + 1], qf[kk], b[2], b[3]);
        }
      }
      const bool need_mask = causal && (k0 + BN - 1 > wr0);
      float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = sc[nt][e] * scale_log2;
          if (need_mask) {
            const int row = wr0 + (lane >> 2) + ((e >> 1) << 3);
            const int col = k0 + nt * 8 + ((lane & 3) << 1) + (e & 1);
            if (col > row) v = -INFINITY;
          }
          sc[nt][e] = v;
          mx[e >> 1] = fmaxf(mx[e >> 1], v);
        }
      }
      float corr[2];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        mx[h2] = fmaxf(mx[h2], __shfl_xor_sync(0xffffffff, mx[h2], 1));
        mx[h2] = fmaxf(mx[h2], __shfl_xor_sync(0xffffffff, mx[h2], 2));
        const float mn = fmaxf(m[h2], mx[h2]);
        corr[h2] = exp2f(m[h2] - mn);
        m[h2] = mn;
      }
      float rs[2] = {0.f, 0.f};
#pragma unroll
      for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p = exp2f(sc[nt][e] - m[e >> 1]);
          sc[nt][e] = p;
          rs[e >> 1] += p;
        }
      }
      l[0] = l[0] * corr[0] + rs[0];
      l[1] = l[1] * corr[1] + rs[1];
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        o[i][0] *= corr[0]; o[i][1] *= corr[0];
        o[i][2] *= corr[1]; o[i][3] *= corr[1];
      }
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        uint32_t a[4];
        a[0] = pk(sc[2 * kk][0], sc[2 * kk][1]);
        a[1] = pk(sc[2 * kk][2], sc[2 * kk][3]);
        a[2] = pk(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
        a[3] = pk(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
        for (int np = 0; np < D / 16; ++np) {
          uint32_t b[4];
          ldb_frag_t<D>(b, cV, kk * 16, np * 16, lane);
          mma16816(o[2 * np], a, b[0], b[1]);
          mma16816(o[2 * np + 1], a, b[2], b[3]);
        }
      }
    }
    __syncthreads();
  }
  // epilogue: normalise, stage through sQ (own 16 rows), coalesced store
  float inv[2];
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) {
    l[h2] += __shfl_xor_sync(0xffffffff, l[h2], 1);
    l[h2] += __shfl_xor_sync(0xffffffff, l[h2], 2);
    inv[h2] = 1.f / l[h2];
  }
#pragma unroll
  for (int nt = 0; nt < D / 8; ++nt) {
    const int col = nt * 8 + ((lane & 3) << 1);
    const int r = warp * 16 + (lane >> 2);
    *reinterpret_cast<uint32_t*>(tile_ptr<D>(sQ, r, col)) = pk(o[nt][0] * inv[0], o[nt][1] * inv[0]);
    *reinterpret_cast<uint32_t*>(tile_ptr<D>(sQ, r + 8, col)) = pk(o[nt][2] * inv[1], o[nt][3] * inv[1]);
  }
  if ((lane & 3) == 0) {
    const int r = wr0 + (lane >> 2);
    lse[(int64_t)head * s + r] = (m[0] + log2f(l[0])) * LN2;
    lse[(int64_t)head * s + r + 8] = (m[1] + log2f(l[1])) * LN2;
  }
  __syncwarp();
  constexpr int CH = D / 8;
  for (int i = lane; i < 16 * CH; i += 32) {
    const int r = warp * 16 + i / CH, c = i % CH;
    const uint4 v = *reinterpret_cast<const uint4*>(sQ + r * (D * 2) + ((c ^ (r & 7)) << 4));
    *reinterpret_cast<uint4*>(out + (int64_t)(q0 + r) * ld_out + head * D + c * 8) = v;
  }
}


// RoPE^T on a 16 x D accumulator tile held as acc[D/8][4] (partner column +D/2 is
// n-tile nt + D/16 in the same thread); rows r_lo = row of e in {0,1}, r_hi = +8
template <int D>
__device__ __forceinline__ void rope_t_acc(float (&acc)[D / 8][4], const float2* rope, int r_lo,
                                           int lane) {
  if (!rope) return;
#pragma unroll
  for (int nt = 0; nt < D / 16; ++nt) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int row = r_lo + ((e >> 1) << 3);
      const int k = nt * 8 + ((lane & 3) << 1) + (e & 1);
      const float2 cs = rope[(int64_t)row * (D / 2) + k];
      const float a = acc[nt][e], b = acc[nt + D / 16][e];
      acc[nt][e] = a * cs.x + b * cs.y;
      acc[nt + D / 16][e] = -a * cs.y + b * cs.x;
    }
  }
}

// ------------------------------------------------------------------ backward: dK, dV
template <int D>
__global__ void __launch_bounds__(256, 1)
    attn_bwd_dkdv_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld,
                         const __nv_bfloat16* __restrict__ dout, int64_t ld_out,
                         const float* __restrict__ lse, const float* __restrict__ Dd, int s,
                         int heads, int causal, __nv_bfloat16* __restrict__ dqkv,
                         const float2* __restrict__ rope, float scale, float scale_log2) {
  constexpr int BN = 128, BM = 64;   // 128 keys per CTA (16 per warp), 64-query blocks
  extern __shared__ __align__(128) char sm[];
  char* sK = sm;
  char* sV = sK + BN * D * 2;
  char* sQ = sV + BN * D * 2;                 // [2][BM][D]
  char* sO = sQ + 2 * BM * D * 2;             // dO [2][BM][D]
  float* sL = reinterpret_cast<float*>(sO + 2 * BM * D * 2);   // [2][BM] lse*log2e
  float* sD = sL + 2 * BM;                                     // [2][BM]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kb = blockIdx.x, head = blockIdx.y;
  const int hq = heads * D;
  const int k0 = kb * BN;
  load_tile<D, BN, 256>(sK, qkv + (int64_t)k0 * ld + hq + head * D, ld, tid);
  load_tile<D, BN, 256>(sV, qkv + (int64_t)k0 * ld + 2 * hq + head * D, ld, tid);
  const int qstart = causal ? k0 / BM : 0;
  const int nqb = s / BM;
  auto load_q = [&](int qi, int b) {
    load_tile<D, BM, 256>(sQ + b * BM * D * 2, qkv + (int64_t)qi * BM * ld + head * D, ld, tid);
    load_tile<D, BM, 256>(sO + b * BM * D * 2, dout + (int64_t)qi * BM * ld_out + head * D, ld_out, tid);
    if (tid < BM) {
      sL[b * BM + tid] = lse[(int64_t)head * s + qi * BM + tid] * LOG2E;
      sD[b * BM + tid] = Dd[(int64_t)head * s + qi * BM + tid];
    }
  };
  load_q(qstart, 0);
  cp_commit();
  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int wk0 = k0 + warp * 16;   // first key of this warp
  for (int qi = qstart; qi < nqb; ++qi) {
    const int b = (qi - qstart) & 1;
    if (qi + 1 < nqb) load_q(qi + 1, b ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    char* cQ = sQ + b * BM * D * 2;
    char* cO = sO + b * BM * D * 2;
    const float* cL = sL + b * BM;
    const float* cD = sD + b * BM;
    const int q0 = qi * BM;
    if (!causal || q0 + BM - 1 >= wk0) {
      // S^T = K_w Q^T  (16 keys x 64 queries)
      float st[BM / 8][4], dpt[BM / 8][4];
#pragma unroll
      for (int i = 0; i < BM / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        uint32_t a[4], av[4];
        lda_frag<D>(a, sK, warp * 16, kk * 16, lane);
        lda_frag<D>(av, sV, warp * 16, kk * 16, lane);
#pragma unroll
        for (int np = 0; np < BM / 16; ++np) {
          uint32_t bq[4], bo[4];
          ldb_frag<D>(bq, cQ, np * 16, kk * 16, lane);
          mma16816(st[2 * np], a, bq[0], bq[1]);
          mma16816(st[2 * np + 1], a, bq[2], bq[3]);
          ldb_frag<D>(bo, cO, np * 16, kk * 16, lane);
          mma16816(dpt[2 * np], av, bo[0], bo[1]);
          mma16816(dpt[2 * np + 1], av, bo[2], bo[3]);
        }
      }
      // P^T = exp2(S^T * scale_log2 - lse2[q]); dS^T = P^T (dP^T - D[q])
#pragma unroll
      for (int nt = 0; nt < BM / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = wk0 + (lane >> 2) + ((e >> 1) << 3);
          const int ql = nt * 8 + ((lane & 3) << 1) + (e & 1);
          float p = exp2f(st[nt][e] * scale_log2 - cL[ql]);
          if (causal && key > q0 + ql) p = 0.f;
          st[nt][e] = p;
          dpt[nt][e] = p * (dpt[nt][e] - cD[ql]);
        }
      }
      // dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
      for (int kk = 0; kk < BM / 16; ++kk) {
        uint32_t ap[4], ad[4];
        ap[0] = pk(st[2 * kk][0], st[2 * kk][1]);
        ap[1] = pk(st[2 * kk][2], st[2 * kk][3]);
        ap[2] = pk(st[2 * kk + 1][0], st[2 * kk + 1][1]);
        ap[3] = pk(st[2 * kk + 1][2], st[2 * kk + 1][3]);
        ad[0] = pk(dpt[2 * kk][0], dpt[2 * kk][1]);
        ad[1] = pk(dpt[2 * kk][2], dpt[2 * kk][3]);
        ad[2] = pk(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]);
        ad[3] = pk(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3]);
#pragma unroll
        for (int np = 0; np < D / 16; ++np) {
          uint32_t bo[4], bq[4];
          ldb_frag_t<D>(bo, cO, kk * 16, np * 16, lane);
          mma16816(dv[2 * np], ap, bo[0], bo[1]);
          mma16816(dv[2 * np + 1], ap, bo[2], bo[3]);
          ldb_frag_t<D>(bq, cQ, kk * 16, np * 16, lane);
          mma16816(dk[2 * np], ad, bq[0], bq[1]);
          mma16816(dk[2 * np + 1], ad, bq[2], bq[3]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] *= scale;
  rope_t_acc<D>(dk, rope, wk0 + (lane >> 2), lane);
#pragma unroll
  for (int nt = 0; nt < D / 8; ++nt) {
    const int col = nt * 8 + ((lane & 3) << 1);
    const int r = wk0 + (lane >> 2);
    __nv_bfloat16* pk_ = dqkv + (int64_t)r * ld + hq + head * D + col;
    __nv_bfloat16* pv_ = dqkv + (int64_t)r * ld + 2 * hq + head * D + col;
    *reinterpret_cast<uint32_t*>(pk_) = pk(dk[nt][0], dk[nt][1]);
    *reinterpret_cast<uint32_t*>(pk_ + 8 * ld) = pk(dk[nt][2], dk[nt][3]);
    *reinterpret_cast<uint32_t*>(pv_) = pk(dv[nt][0], dv[nt][1]);
    *reinterpret_cast<uint32_t*>(pv_ + 8 * ld) = pk(dv[nt][2], dv[nt][3]);
  }
}

// ------------------------------------------------------------------ backward: dQ
template <int D>
__global__ void __launch_bounds__(256, 1)
    attn_bwd_dq_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld,
                       const __nv_bfloat16* __restrict__ dout, int64_t ld_out,
                       const float* __restrict__ lse, const float* __restrict__ Dd, int s,
                       int heads, int causal, __nv_bfloat16* __restrict__ dqkv,
                       const float2* __restrict__ rope, float scale, float scale_log2) {
  constexpr int BM = 128, BN = 64;
  extern __shared__ __align__(128) char sm[];
  char* sQ = sm;
  char* sO = sQ + BM * D * 2;
  char* sK = sO + BM * D * 2;      // [2][BN][D]
  char* sV = sK + 2 * BN * D * 2;  // [2][BN][D]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nqb = s / BM;
  const int qb = causal ? (nqb - 1 - blockIdx.x) : blockIdx.x;
  const int head = blockIdx.y;
  const int hq = heads * D;
  const int q0 = qb * BM;
  const __nv_bfloat16* Kg = qkv + hq + head * D;
  const __nv_bfloat16* Vg = qkv + 2 * hq + head * D;
  load_tile<D, BM, 256>(sQ, qkv + (int64_t)q0 * ld + head * D, ld, tid);
  load_tile<D, BM, 256>(sO, dout + (int64_t)q0 * ld_out + head * D, ld_out, tid);
  load_tile<D, BN, 256>(sK, Kg, ld, tid);
  load_tile<D, BN, 256>(sV, Vg, ld, tid);
  cp_commit();
  const int wr0 = q0 + warp * 16;
  const float l2lo = lse[(int64_t)head * s + wr0 + (lane >> 2)] * LOG2E;
  const float l2hi = lse[(int64_t)head * s + wr0 + (lane >> 2) + 8] * LOG2E;
  const float dlo = Dd[(int64_t)head * s + wr0 + (lane >> 2)];
  const float dhi = Dd[(int64_t)head * s + wr0 + (lane >> 2) + 8];
  const int nkb = causal ? (q0 + BM) / BN : s / BN;
  float dq[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
  uint32_t qf[D / 16][4], of[D / 16][4];
  for (int j = 0; j < nkb; ++j) {
    if (j + 1 < nkb) {
      const int b = (j + 1) & 1;
      load_tile<D, BN, 256>(sK + b * BN * D * 2, Kg + (int64_t)(j + 1) * BN * ld, ld, tid);
      load_tile<D, BN, 256>(sV + b * BN * D * 2, Vg + (int64_t)(j + 1) * BN * ld, ld, tid);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        lda_frag<D>(qf[kk], sQ, warp * 16, kk * 16, lane);
        lda_frag<D>(of[kk], sO, warp * 16, kk * 16, lane);
      }
    }
    char* cK = sK + (j & 1) * BN * D * 2;
    char* cV = sV + (j & 1) * BN * D * 2;
    const int k0 = j * BN;
    if (!causal || k0 <= wr0 + 15) {
      float sc[BN / 8][4], dp[BN / 8][4];
#pragma unroll
      for (int i = 0; i < BN / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[i][e] = dp[i][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int np = 0; np < BN / 16; ++np) {
          uint32_t b[4], bv[4];
          ldb_frag<D>(b, cK, np * 16, kk * 16, lane);
          mma16816(sc[2 * np], qf[kk], b[0], b[1]);
          mma16816(sc[2 * np + 1], qf[kk], b[2], b[3]);
          ldb_frag<D>(bv, cV, np * 16, kk * 16, lane);
          mma16816(dp[2 * np], of[kk], bv[0], bv[1]);
          mma16816(dp[2 * np + 1], of[kk], bv[2], bv[3]);
        }
      }
#pragma unroll
      for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = wr0 + (lane >> 2) + ((e >> 1) << 3);
          const int col = k0 + nt * 8 + ((lane & 3) << 1) + (e & 1);
          float p = exp2f(sc[nt][e] * scale_log2 - ((e >> 1) ? l2hi : l2lo));
          if (causal && col > row) p = 0.f;
          dp[nt][e] = p * (dp[nt][e] - ((e >> 1) ? dhi : dlo));
        }
      }
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        uint32_t a[4];
        a[0] = pk(dp[2 * kk][0], dp[2 * kk][1]);
        a[1] = pk(dp[2 * kk][2], dp[2 * kk][3]);
        a[2] = pk(dp[2 * kk + 1][0], dp[2 * kk + 1][1]);
        a[3] = pk(dp[2 * kk + 1][2], dp[2 * kk + 1][3]);
#pragma unroll
        for (int np = 0; np < D / 16; ++np) {
          uint32_t b[4];
          ldb_frag_t<D>(b, cK, kk * 16, np * 16, lane);
          mma16816(dq[2 * np], a, b[0], b[1]);
          mma16816(dq[2 * np + 1], a, b[2], b[3]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dq[i][e] *= scale;
  rope_t_acc<D>(dq, rope, wr0 + (lane >> 2), lane);
#pragma unroll
  for (int nt = 0; nt < D / 8; ++nt) {
    const int col = nt * 8 + ((lane & 3) << 1);
    __nv_bfloat16* p = dqkv + (int64_t)(wr0 + (lane >> 2)) * ld + head * D + col;
    *reinterpret_cast<uint32_t*>(p) = pk(dq[nt][0], dq[nt][1]);
    *reinterpret_cast<uint32_t*>(p + 8 * ld) = pk(dq[nt][2], dq[nt][3]);
  }
}

// ------------------------------------------------------------------ launchers
template <int D>
static int fwd_t(const void* qkv, int64_t ld, int s, int heads, int causal, void* out,
                 int64_t ld_out, void* lse, cudaStream_t st) {
  constexpr int SMEM = (128 + 4 * 64) * D * 2;
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    once = true;
  }
  const float scale_log2 = (1.0f / sqrtf((float)D)) * LOG2E;
  dim3 grid(s / 128, heads);
  attn_fwd_kernel<D><<<grid, 256, SMEM, st>>>(reinterpret_cast<const __nv_bfloat16*>(qkv), ld, s,
                                              heads, causal, reinterpret_cast<__nv_bfloat16*>(out),
                                              ld_out, reinterpret_cast<float*>(lse), scale_log2);
  return (int)cudaGetLastError();
}

// warp-level mma.sync FA2 forward (round-1 baseline, kept for A/B: PDS_ATTN_FWD=sync)
int attn_fwd_sync(const void* qkv, int64_t ld, int s, int heads, int d, int causal, void* out,
                  int64_t ld_out, void* lse, cudaStream_t st) {
  if (s % 128) return (int)cudaErrorInvalidValue;
  if (d == 128) return fwd_t<128>(qkv, ld, s, heads, causal, out, ld_out, lse, st);
  if (d == 64) return fwd_t<64>(qkv, ld, s, heads, causal, out, ld_out, lse, st);
  return (int)cudaErrorInvalidValue;
}

template <int D>
static int bwd_t(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* lse,
                 const void* dout, int s, int heads, int causal, void* dqkv, const void* rope,
                 float* Dd, cudaStream_t st) {
  const float scale = 1.0f / sqrtf((float)D);
  const float scale_log2 = scale * LOG2E;
  {
    const int warps = s * heads;
    attn_bwd_dot_kernel<<<(warps + 7) / 8, 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(out), ld_out,
        reinterpret_cast<const __nv_bfloat16*>(dout), s, heads, D, Dd);
  }
  constexpr int SM_KV = (2 * 128 + 4 * 64) * D * 2 + 4 * 64 * 4;
  constexpr int SM_Q = (2 * 128 + 4 * 64) * D * 2;
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(attn_bwd_dkdv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_KV);
    cudaFuncSetAttribute(attn_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_Q);
    once = true;
  }
  attn_bwd_dkdv_kernel<D><<<dim3(s / 128, heads), 256, SM_KV, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), ld, reinterpret_cast<const __nv_bfloat16*>(dout),
      ld_out, reinterpret_cast<const float*>(lse), Dd, s, heads, causal,
      reinterpret_cast<__nv_bfloat16*>(dqkv), reinterpret_cast<const float2*>(rope), scale, scale_log2);
  attn_bwd_dq_kernel<D><<<dim3(s / 128, heads), 256, SM_Q, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), ld, reinterpret_cast<const __nv_bfloat16*>(dout),
      ld_out, reinterpret_cast<const float*>(lse), Dd, s, heads, causal,
      reinterpret_cast<__nv_bfloat16*>(dqkv), reinterpret_cast<const float2*>(rope), scale, scale_log2);
  return (int)cudaGetLastError();
}

// Dd: fp32 scratch [heads][s]
int attn_bwd_sync(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* lse,
             const void* dout, int s, int heads, int d, int causal, void* dqkv, const void* rope,
             float* Dd, cudaStream_t st) {
  if (s % 128) return (int)cudaErrorInvalidValue;
  if (d == 128) return bwd_t<128>(qkv, ld, out, ld_out, lse, dout, s, heads, causal, dqkv, rope, Dd, st);
  if (d == 64) return bwd_t<64>(qkv, ld, out, ld_out, lse, dout, s, heads, causal, dqkv, rope, Dd, st);
  return (int)cudaErrorInvalidValue;
}

}  // namespace pds

extern "C" int pds_fa2_fwd(const void* qkv, int64_t ld, int s, int heads, int d, int causal, void* out,
                           int64_t ld_out, void* lse, void* st) {
  return pds::attn_fwd_sync(qkv, ld, s, heads, d, causal, out, ld_out, lse, (cudaStream_t)st);
}
extern "C" int pds_fa2_bwd(const void* qkv, int64_t ld, const void* out, int64_t ld_out, const void* lse,
                           const void* dout, int s, int heads, int d, int causal, void* dqkv, const void* rope,
                           float* Dd, void* st) {
  return pds::attn_bwd_sync(qkv, ld, out, ld_out, lse, dout, s, heads, d, causal, dqkv, rope, Dd,
                            (cudaStream_t)st);
}
