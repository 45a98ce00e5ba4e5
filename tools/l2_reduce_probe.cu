// L2 reduction-throughput probe (design input for a fused attention backward that
// accumulates dQ partials in fp32 global memory): every CTA repeatedly adds a 64 KB
// fp32 tile (one 128 x 128 dQ partial) into a rotating slot of a dst region that fits
// in L2, three ways:
//   mode 0: red.global.add.v4.f32, thread = one 512-byte row (a TMEM 32x32b readout)
//   mode 1: red.global.add.v4.f32, consecutive threads on consecutive 16 B (coalesced)
//   mode 2: cp.reduce.async.bulk.global.shared::cta.add.f32 of the tile from smem
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_reduce_probe tools/l2_reduce_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(128) probe(float* dst, int slots, int iters, int mode) {
  extern __shared__ __align__(128) float tile[];     // 64 KB
  const int t = threadIdx.x;
  for (int i = t; i < 16384; i += 128) tile[i] = 1.0f;
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    const int slot = (blockIdx.x * 7 + it) % slots;
    float* d = dst + (size_t)slot * 16384;
    if (mode == 0) {
      float* row = d + t * 128;
#pragma unroll 8
      for (int c = 0; c < 128; c += 4)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + c), "f"(1.f), "f"(1.f), "f"(1.f),
                     "f"(1.f) : "memory");
    } else if (mode == 1) {
#pragma unroll 8
      for (int c = 0; c < 128; ++c) {
        float* p = d + (c * 128 + t) * 4 / 4 * 1;   // 128 threads x 16 B = 2 KB per step
        p = d + c * 512 + t * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f),
                     "f"(1.f) : "memory");
      }
    } else {
      if (t == 0) {
        uint32_t s = (uint32_t)__cvta_generic_to_shared(tile);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(d), "r"(s),
                     "r"(65536) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncthreads();
    }
  }
  if (mode == 2 && t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int slots = 256;           // 16 MB destination (one head's dQ at s = 32K)
  float* dst;
  cudaMalloc(&dst, (size_t)slots * 65536);
  cudaMemset(dst, 0, (size_t)slots * 65536);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 200;
  for (int grid : {148, 296}) {
    for (int mode = 0; mode < 3; ++mode) {
      probe<<<grid, 128, 65536>>>(dst, slots, 10, mode);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      probe<<<grid, 128, 65536>>>(dst, slots, iters, mode);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)grid * iters * 65536;
      printf("grid %d mode %d: %.3f ms, %.1f GB/s of fp32 reductions (%.2f us per 64 KB tile per CTA)\n", grid, mode,
             ms, bytes / ms / 1e6, ms * 1e3 / iters * (grid > 148 ? 148.0 / grid : 1.0));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
