// HBM-bound elementwise kernels of the layer: fused residual-add + RMSNorm
// forward / backward (reading R-2: pre-norm Llama block, fp32 statistics),
// the RoPE cos/sin table (reading R-3: angles formed in fp64), recompute of a
// normalised activation from its saved input + rstd, and bf16 add / copy.
//
// Norm kernels: one block per row (fwd) / grid-stride rows (bwd), 16-byte vector
// loads/stores, each byte read once; the other kernels: one warp per row.  Algorithmic bytes per element: fwd 8 B with a
// residual (x, res in; x1, u out), bwd 8 B (du, x, dres in; dx out).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace pds {

__device__ __forceinline__ void unpack8(const uint4& w, float* f) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __bfloat1622float2(b[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 w;
  uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat162 v = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
    u[e] = *reinterpret_cast<uint32_t*>(&v);
  }
  return w;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}

// Block-per-row layout for the norm kernels: NT threads (min(h/8, 256) for h <= 4096,
// 512 above), each owning VPT = ceil(h / (8 NT)) 16-byte vectors of the row (8 bf16
// columns per vector; the last one predicated when NT does not divide h/8), so a row
// is one fully coalesced pass and the only cross-thread step is the row sum (warp
// shuffle + one shared-memory exchange).  Any h that is a multiple of 256 up to 16384.
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

template <int VPT, int NT, bool TAIL>
__global__ void __launch_bounds__(NT)
    rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ res,
                       const __nv_bfloat16* __restrict__ g, int64_t rows, int h, float eps,
                       __nv_bfloat16* __restrict__ x1_out, __nv_bfloat16* __restrict__ u_out,
                       float* __restrict__ rstd_out) {
  __shared__ float red[16];
  const int64_t row = blockIdx.x;
  const int nvec = h >> 3;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * h);
  const uint4* rr = reinterpret_cast<const uint4*>(res + row * h);
  uint4 w[VPT], rw[VPT];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    w[k] = make_uint4(0, 0, 0, 0);
    rw[k] = make_uint4(0, 0, 0, 0);
    if (!TAIL || c < nvec) {
      w[k] = __ldcs(xr + c);
      if (res) rw[k] = __ldcs(rr + c);
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    float v[8];
    unpack8(w[k], v);
    if (res) {
      float r[8];
      unpack8(rw[k], r);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] += r[e];
      w[k] = pack8(v);                         // x1 = bf16(x + res)
      unpack8(w[k], v);
      if (!TAIL || c < nvec) reinterpret_cast<uint4*>(x1_out + row * h)[c] = w[k];
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) ss += v[e] * v[e];
  }
  ss = block_sum(ss, red);
  const float r = rsqrtf(ss / (float)h + eps);
  if (threadIdx.x == 0) rstd_out[row] = r;
  const uint4* gr = reinterpret_cast<const uint4*>(g);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    if (TAIL && c >= nvec) continue;
    float v[8], gg[8], o[8];
    unpack8(w[k], v);
    unpack8(__ldg(gr + c), gg);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = v[e] * r * gg[e];
    reinterpret_cast<uint4*>(u_out + row * h)[c] = pack8(o);
  }
}

// dx = r (a - xhat mean(a xhat)) + dres, a = du g, xhat = x r;  dg_part[block][:] =
// sum over the block's rows of du xhat (each thread keeps its columns' partials in
// registers across the grid-stride row loop).
template <int VPT, int NT, bool TAIL>
__global__ void __launch_bounds__(NT, NT == 256 ? 3 : 1)
    rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ du, const __nv_bfloat16* __restrict__ x,
                       const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ g,
                       const __nv_bfloat16* __restrict__ dres, int64_t rows, int h,
                       __nv_bfloat16* __restrict__ dx, float* __restrict__ dg_part) {
  __shared__ float red[2][16];
  const int nvec = h >> 3;
  uint4 gw[VPT];
  float dga[VPT][8];
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    gw[k] = (!TAIL || c < nvec) ? __ldg(reinterpret_cast<const uint4*>(g) + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int e = 0; e < 8; ++e) dga[k][e] = 0.f;
  }
  int par = 0;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x, par ^= 1) {
    const float r = rstd[row];
    uint4 xw[VPT], dw[VPT], rw[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = threadIdx.x + k * blockDim.x;
      if (!TAIL || c < nvec) {
        xw[k] = __ldcs(reinterpret_cast<const uint4*>(x + row * h) + c);
        dw[k] = __ldcs(reinterpret_cast<const uint4*>(du + row * h) + c);
        if (dres) rw[k] = __ldcs(reinterpret_cast<const uint4*>(dres + row * h) + c);
      } else {
        xw[k] = dw[k] = rw[k] = make_uint4(0, 0, 0, 0);
      }
    }
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      float xh[8], d8[8], gg[8];
      unpack8(xw[k], xh);
      unpack8(dw[k], d8);
      unpack8(gw[k], gg);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xh[e] *= r;
        dot += d8[e] * gg[e] * xh[e];
        dga[k][e] += d8[e] * xh[e];
      }
    }
    dot = block_sum(dot, red[par]) / (float)h;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int c = threadIdx.x + k * blockDim.x;
      if (TAIL && c >= nvec) continue;
      float xh[8], d8[8], dr[8], o[8], gg[8];
      unpack8(xw[k], xh);
      unpack8(dw[k], d8);
      unpack8(gw[k], gg);
      if (dres) unpack8(rw[k], dr);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = r * (d8[e] * gg[e] - xh[e] * r * dot) + (dres ? dr[e] : 0.f);
      reinterpret_cast<uint4*>(dx + row * h)[c] = pack8(o);
    }
  }
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    if (TAIL && c >= nvec) continue;
    float4* o = reinterpret_cast<float4*>(dg_part + (int64_t)blockIdx.x * h + 8 * c);
    o[0] = make_float4(dga[k][0], dga[k][1], dga[k][2], dga[k][3]);
    o[1] = make_float4(dga[k][4], dga[k][5], dga[k][6], dga[k][7]);
  }
}

// out[i] += sum_p part[p][i]: 32 columns per block, 8 row groups, smem tree
__global__ void __launch_bounds__(256)
    reduce_rows_add_kernel(const float* __restrict__ part, int nparts, int h, float* __restrict__ out) {
  __shared__ float red[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int g = threadIdx.x >> 5;
  float acc = 0.f;
  if (c < h)
    for (int p = g; p < nparts; p += 8) acc += part[(int64_t)p * h + c];
  red[g][threadIdx.x & 31] = acc;
  __syncthreads();
  if (g == 0 && c < h) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    out[c] += t;
  }
}

// u = x * rstd * g  (recompute of a normalised activation from saved x, rstd)
template <int VPT, int NT, bool TAIL>
__global__ void __launch_bounds__(NT)
    apply_norm_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ rstd,
                      const __nv_bfloat16* __restrict__ g, int64_t rows, int h,
                      __nv_bfloat16* __restrict__ u) {
  const int64_t row = blockIdx.x;
  const int nvec = h >> 3;
  const float r = rstd[row];
  const uint4* gr = reinterpret_cast<const uint4*>(g);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    if (TAIL && c >= nvec) continue;
    float v[8], gg[8];
    unpack8(__ldcs(reinterpret_cast<const uint4*>(x + row * h) + c), v);
    unpack8(__ldg(gr + c), gg);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = v[e] * r * gg[e];
    reinterpret_cast<uint4*>(u + row * h)[c] = pack8(v);
  }
}

__global__ void add_bf16_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                uint4* __restrict__ c, int64_t n8) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x[8], y[8];
    unpack8(__ldcs(a + i), x);
    unpack8(__ldcs(b + i), y);
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] += y[e];
    c[i] = pack8(x);
  }
}

// sum of P buffers (loopback reduce-scatter / all-reduce), fp32 accumulation in rank order
struct Ptrs8 {
  const void* p[8];
};
__global__ void sum_bf16_kernel(Ptrs8 srcs, int P, uint4* __restrict__ dst, int64_t n8) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc[8], t[8];
    unpack8(reinterpret_cast<const uint4*>(srcs.p[0])[i], acc);
    for (int p = 1; p < P; ++p) {
      unpack8(reinterpret_cast<const uint4*>(srcs.p[p])[i], t);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += t[e];
    }
    dst[i] = pack8(acc);
  }
}
__global__ void sum_f32_kernel(Ptrs8 srcs, int P, float* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = reinterpret_cast<const float*>(srcs.p[0])[i];
    for (int p = 1; p < P; ++p) acc += reinterpret_cast<const float*>(srcs.p[p])[i];
    dst[i] = acc;
  }
}
__global__ void add_f32_kernel(const float4* __restrict__ a, float4* __restrict__ acc, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 x = acc[i];
    const float4 y = a[i];
    x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
    acc[i] = x;
  }
}

// dst[t][j*cw + c] = src[j][t][c]; 16-byte vectors (cw % 8 == 0)
__global__ void unpack_blocks_kernel(const uint4* __restrict__ src, int P, int64_t rows, int64_t cw8,
                                     uint4* __restrict__ dst, int64_t ld8) {
  const int64_t n = (int64_t)P * rows * cw8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % cw8;
    const int64_t t = (i / cw8) % rows;
    const int64_t j = i / (cw8 * rows);
    dst[t * ld8 + j * cw8 + c] = __ldcs(src + i);
  }
}

// dst[c][r] = src[map(r)][c] for r < rows, c < cols (bf16); 64 x 64 tiles through
// shared memory, 16-byte global loads and stores.  map(r) = (r / seg) * stride + base + r % seg
// (METP waves read position-ordered buffers).  HBM-bound: 4 B per element.
__global__ void __launch_bounds__(256)
    transpose_bf16_kernel(const uint16_t* __restrict__ src, int64_t ld_src, int64_t rows, int64_t cols,
                          uint16_t* __restrict__ dst, int64_t ld_dst, int64_t seg, int64_t stride, int64_t base) {
  // Two 64 x 64 tiles (source rows r0 .. r0 + 127) as 32-bit words (column pairs), row
  // stride 33 words: the 16-byte loads are stored as 4 conflict-free 32-bit words; the
  // transposed reads hit <= 2 banks per word; two output vectors per thread are
  // assembled with byte permutes.  All four loads of a thread are issued first.
  __shared__ uint32_t tile[128][33];
  const int64_t r0 = (int64_t)blockIdx.y * 128, c0 = (int64_t)blockIdx.x * 64;
  const int t = threadIdx.x;
  const bool remap = seg < rows || base != 0;     // one segment with an offset is a remap too
  uint4 x[4];
#pragma unroll
  for (int h4 = 0; h4 < 4; ++h4) {
    const int rr = (t >> 3) + 32 * h4, v = t & 7;
    const int64_t r = r0 + rr;
    x[h4] = make_uint4(0, 0, 0, 0);
    if (r < rows && c0 + v * 8 < cols) {
      const int64_t sr = remap ? (r / seg) * stride + base + (r % seg) : r;
      x[h4] = __ldcs(reinterpret_cast<const uint4*>(src + sr * ld_src + c0 + v * 8));
    }
  }
#pragma unroll
  for (int h4 = 0; h4 < 4; ++h4) {
    const int rr = (t >> 3) + 32 * h4, v = t & 7;
    tile[rr][v * 4 + 0] = x[h4].x;
    tile[rr][v * 4 + 1] = x[h4].y;
    tile[rr][v * 4 + 2] = x[h4].z;
    tile[rr][v * 4 + 3] = x[h4].w;
  }
  __syncthreads();
  // thread -> column pair cp (dst rows c0 + 2cp, +1), source rows rb*8 .. +7 of each half
  const int cp = t >> 3, rb = t & 7;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = tile[half * 64 + rb * 8 + i][cp];
    uint4 lo, hi;
    lo.x = __byte_perm(w[0], w[1], 0x5410); hi.x = __byte_perm(w[0], w[1], 0x7632);
    lo.y = __byte_perm(w[2], w[3], 0x5410); hi.y = __byte_perm(w[2], w[3], 0x7632);
    lo.z = __byte_perm(w[4], w[5], 0x5410); hi.z = __byte_perm(w[4], w[5], 0x7632);
    lo.w = __byte_perm(w[6], w[7], 0x5410); hi.w = __byte_perm(w[6], w[7], 0x7632);
    const int64_t c = c0 + 2 * cp, rr0 = r0 + half * 64 + rb * 8;
    if (rr0 < rows) {
      if (c < cols) *reinterpret_cast<uint4*>(dst + c * ld_dst + rr0) = lo;
      if (c + 1 < cols) *reinterpret_cast<uint4*>(dst + (c + 1) * ld_dst + rr0) = hi;
    }
  }
}

__global__ void rope_table_kernel(float2* __restrict__ t, int64_t n_pos, int d, double theta) {
  const int d2 = d / 2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pos * d2) return;
  const int64_t pos = i / d2;
  const int k = (int)(i % d2);
  const double inv = pow(theta, -2.0 * (double)k / (double)d);
  const double ang = (double)pos * inv;        // fp64 angle, fp64 range reduction in sincos
  double s, c;
  sincos(ang, &s, &c);
  t[i] = make_float2((float)c, (float)s);
}

// ------------------------------------------------------------------ launchers
// NT x VPT dispatch of the block-per-row kernels (see the layout note above)
static bool h_ok(int h) { return h % 256 == 0 && h >= 256 && h <= 16384; }
static int row_threads(int h) { return h <= 4096 ? (h / 8 < 256 ? h / 8 : 256) : 512; }
#define PDS_ROW_DISPATCH(h, KERN, GRID, SMEM, ST, ...)                                    \
  do {                                                                                 \
    const int nt_ = row_threads(h), vpt_ = (h / 8 + nt_ - 1) / nt_;                    \
    const bool tail_ = vpt_ * nt_ != h / 8;                                            \
    if (nt_ <= 256 && vpt_ == 1) {                                                     \
      KERN<1, 256, false><<<GRID, nt_, SMEM, ST>>>(__VA_ARGS__);                       \
    } else if (nt_ <= 256) {                                                           \
      if (tail_) KERN<2, 256, true><<<GRID, nt_, SMEM, ST>>>(__VA_ARGS__);             \
      else KERN<2, 256, false><<<GRID, nt_, SMEM, ST>>>(__VA_ARGS__);                  \
    } else if (vpt_ == 2) {                                                            \
      if (tail_) KERN<2, 512, true><<<GRID, nt_, SMEM, ST>>>(__VA_ARGS__);             \
      else KERN<2, 512, false><<<GRID, nt_, SMEM, ST>>>(__VA_ARGS__);                  \
    } else if (vpt_ == 3) {                                                            \
      if (tail_) KERN<3, 512, true><<<GRID, nt_, SMEM, ST>>>(__VA_ARGS__);             \
      else KERN<3, 512, false><<<GRID, nt_, SMEM, ST>>>(__VA_ARGS__);                  \
    } else {                                                                           \
      KERN<4, 512, true><<<GRID, nt_, SMEM, ST>>>(__VA_ARGS__);                        \
    }                                                                                  \
  } while (0)

int rmsnorm_fwd(const void* x, const void* res, const void* g, int64_t rows, int h, float eps,
                void* x1_out, void* u_out, void* rstd, cudaStream_t st) {
  if (!h_ok(h)) return (int)cudaErrorInvalidValue;
  if (rows <= 0) return 0;
  auto X = reinterpret_cast<const __nv_bfloat16*>(x);
  auto R = reinterpret_cast<const __nv_bfloat16*>(res);
  auto G = reinterpret_cast<const __nv_bfloat16*>(g);
  auto X1 = reinterpret_cast<__nv_bfloat16*>(x1_out);
  auto U = reinterpret_cast<__nv_bfloat16*>(u_out);
  auto RS = reinterpret_cast<float*>(rstd);
  PDS_ROW_DISPATCH(h, rmsnorm_fwd_kernel, (unsigned)rows, 0, st, X, R, G, rows, h, eps, X1, U, RS);
  return (int)cudaGetLastError();
}

int rmsnorm_bwd_grid(int64_t rows) {
  int64_t b = (rows + 3) / 4;
  return (int)(b < 444 ? b : 444);   // 148 SMs x 3 resident blocks (all resident: one wave)
}

// dg_part: fp32 scratch [rmsnorm_bwd_grid(rows)][h]; dg (fp32 [h]) += reduced partials
int rmsnorm_bwd(const void* du, const void* x, const void* rstd, const void* g, const void* dres,
                int64_t rows, int h, void* dx, float* dg_part, float* dg, cudaStream_t st) {
  if (!h_ok(h)) return (int)cudaErrorInvalidValue;
  if (rows <= 0) return 0;
  const int grid = rmsnorm_bwd_grid(rows);
  auto DU = reinterpret_cast<const __nv_bfloat16*>(du);
  auto X = reinterpret_cast<const __nv_bfloat16*>(x);
  auto RS = reinterpret_cast<const float*>(rstd);
  auto G = reinterpret_cast<const __nv_bfloat16*>(g);
  auto DR = reinterpret_cast<const __nv_bfloat16*>(dres);
  auto DX = reinterpret_cast<__nv_bfloat16*>(dx);
  PDS_ROW_DISPATCH(h, rmsnorm_bwd_kernel, grid, 0, st, DU, X, RS, G, DR, rows, h, DX, dg_part);
  int rc = (int)cudaGetLastError();
  if (rc) return rc;
  reduce_rows_add_kernel<<<(h + 31) / 32, 256, 0, st>>>(dg_part, grid, h, dg);
  return (int)cudaGetLastError();
}

int apply_norm(const void* x, const void* rstd, const void* g, int64_t rows, int h, void* u,
               cudaStream_t st) {
  if (!h_ok(h)) return (int)cudaErrorInvalidValue;
  if (rows <= 0) return 0;
  auto X = reinterpret_cast<const __nv_bfloat16*>(x);
  auto RS = reinterpret_cast<const float*>(rstd);
  auto G = reinterpret_cast<const __nv_bfloat16*>(g);
  auto U = reinterpret_cast<__nv_bfloat16*>(u);
  PDS_ROW_DISPATCH(h, apply_norm_kernel, (unsigned)rows, 0, st, X, RS, G, rows, h, U);
  return (int)cudaGetLastError();
}

static unsigned ew_grid(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (unsigned)(b < 148 * 16 ? b : 148 * 16);
}

int add_bf16(const void* a, const void* b, void* c, int64_t n, cudaStream_t st) {
  if (n % 8) return (int)cudaErrorInvalidValue;
  add_bf16_kernel<<<ew_grid(n / 8), 256, 0, st>>>(reinterpret_cast<const uint4*>(a),
                                                  reinterpret_cast<const uint4*>(b),
                                                  reinterpret_cast<uint4*>(c), n / 8);
  return (int)cudaGetLastError();
}
int sum_bf16_p(const void* const* srcs, int P, void* dst, int64_t n, cudaStream_t st) {
  if (n % 8 || P > 8) return (int)cudaErrorInvalidValue;
  Ptrs8 p{};
  for (int i = 0; i < P; ++i) p.p[i] = srcs[i];
  sum_bf16_kernel<<<ew_grid(n / 8), 256, 0, st>>>(p, P, reinterpret_cast<uint4*>(dst), n / 8);
  return (int)cudaGetLastError();
}
int sum_f32_p(const void* const* srcs, int P, void* dst, int64_t n, cudaStream_t st) {
  if (P > 8) return (int)cudaErrorInvalidValue;
  Ptrs8 p{};
  for (int i = 0; i < P; ++i) p.p[i] = srcs[i];
  sum_f32_kernel<<<ew_grid(n), 256, 0, st>>>(p, P, reinterpret_cast<float*>(dst), n);
  return (int)cudaGetLastError();
}
int add_f32(const void* a, void* acc, int64_t n, cudaStream_t st) {
  if (n % 4) return (int)cudaErrorInvalidValue;
  add_f32_kernel<<<ew_grid(n / 4), 256, 0, st>>>(reinterpret_cast<const float4*>(a),
                                                 reinterpret_cast<float4*>(acc), n / 4);
  return (int)cudaGetLastError();
}

int unpack_blocks(const void* src, int P, int64_t rows, int64_t cw, void* dst, int64_t ld_dst,
                  cudaStream_t st) {
  if (cw % 8 || ld_dst % 8) return (int)cudaErrorInvalidValue;
  const int64_t n = (int64_t)P * rows * cw / 8;
  unpack_blocks_kernel<<<ew_grid(n), 256, 0, st>>>(reinterpret_cast<const uint4*>(src), P, rows, cw / 8,
                                                   reinterpret_cast<uint4*>(dst), ld_dst / 8);
  return (int)cudaGetLastError();
}

int transpose_bf16(const void* src, int64_t ld_src, int64_t rows, int64_t cols, void* dst, int64_t ld_dst,
                   int64_t seg, int64_t stride, int64_t base, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return 0;
  if (rows % 8 || cols % 8 || ld_src % 8 || ld_dst % 8) return (int)cudaErrorInvalidValue;
  dim3 grid((unsigned)((cols + 63) / 64), (unsigned)((rows + 127) / 128));
  transpose_bf16_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint16_t*>(src), ld_src, rows, cols,
                                               reinterpret_cast<uint16_t*>(dst), ld_dst,
                                               seg > 0 ? seg : ((int64_t)1 << 40), stride, base);
  return (int)cudaGetLastError();
}

int rope_table(void* t, int64_t n_pos, int d, double theta, cudaStream_t st) {
  const int64_t n = n_pos * (d / 2);
  rope_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(reinterpret_cast<float2*>(t), n_pos,
                                                                  d, theta);
  return (int)cudaGetLastError();
}

}  // namespace pds
