// Microbenchmark: tcgen05.mma kind::f16 throughput per SM for the operand
// majors / shapes the attention kernels use (SS vs TS, K-major vs MN-major).
// One CTA per SM, operands resident in SMEM/TMEM, one thread issues `iters`
// x 4 MMAs (K = 16 each) into one TMEM accumulator; reports flop/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_13198_b200/csrc/kernels tools/mma_probe.cu -o /tmp/mma_probe -lcuda
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace pds;

__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) { return umma_desc_sw128(base + kk * 32, 16, 1024); }
__device__ __forceinline__ uint64_t mdesc(uint32_t base, int kk, uint32_t atom) { return umma_desc_sw128(base + kk * 2048, atom, 1024); }

template <int N, int AMN, int BMN, int TS>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (128 + 256) * 64 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u ^ i, 0x3f003f00u, 0x3e803e80u + i, 0x3c003c00u);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 128 * 128);
    constexpr uint32_t idesc = umma_idesc_bf16(128, N, AMN, BMN);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bd = BMN ? mdesc(sb, kk, N >= 128 ? 8192 : 8192) : kdesc(sb, kk);
        if (TS) umma_f16_ts(tmem + 256, tmem + kk * 8, bd, idesc, 1);
        else umma_f16(tmem + 256, AMN ? mdesc(sa, kk, 8192) : kdesc(sa, kk), bd, idesc, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, int AMN, int BMN, int TS>
void run(const char* name) {
  const int iters = 20000, grid = 148;
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  auto k = probe<N, AMN, BMN, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<grid, 128, 100 * 1024>>>(200, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 128, 100 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
  double fl = 2.0 * 128 * N * 16 * 4 * (double)iters;
  printf("%-18s N=%3d  %7.0f flop/clk/SM  (%.1f%% of 8192)  %7.1f TF/s  %s\n", name, N, fl / avg, 100 * fl / avg / 8192,
         fl * grid / ms / 1e9, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<256, 0, 0, 0>("SS  A-K  B-K");
  run<128, 0, 0, 0>("SS  A-K  B-K");
  run<64, 0, 0, 0>("SS  A-K  B-K");
  run<128, 0, 1, 0>("SS  A-K  B-MN");
  run<64, 0, 1, 0>("SS  A-K  B-MN");
  run<128, 1, 0, 0>("SS  A-MN B-K");
  run<128, 1, 1, 0>("SS  A-MN B-MN");
  run<256, 0, 1, 0>("SS  A-K  B-MN");
  run<256, 0, 0, 1>("TS  A-tm B-K");
  run<128, 0, 0, 1>("TS  A-tm B-K");
  run<64, 0, 0, 1>("TS  A-tm B-K");
  run<128, 0, 1, 1>("TS  A-tm B-MN");
  run<64, 0, 1, 1>("TS  A-tm B-MN");
  return 0;
}
