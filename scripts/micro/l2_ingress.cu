// Microbenchmark: L2 -> shared memory bulk-copy throughput vs number of CTAs (is the limit per
// SM ingress or aggregate L2?).  Each CTA streams `iters` x 48 KB through a 4-deep ring with
// cp.async.bulk from a 4 MB L2-resident region (distinct offsets per CTA).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2301_12443_b200/csrc/kernels/sm100.cuh"
using namespace pbdk;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int CHUNK>
__global__ void __launch_bounds__(32, 1) ingress(const uint8_t* src, int iters, size_t region) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int st = i & 3;
      if (i >= 4) mbar_wait(&bar[st], ((i >> 2) - 1) & 1);
      mbar_arrive_expect_tx(&bar[st], CHUNK);
      const size_t off = (static_cast<size_t>(blockIdx.x) * 7919 + i) * CHUNK % (region - CHUNK);
      bulk_g2s(smem + st * CHUNK, src + (off & ~size_t(127)), CHUNK, &bar[st]);
    }
    for (int i = iters; i < iters + 4; ++i) mbar_wait(&bar[i & 3], ((i >> 2) - 1) & 1);
  }
}

int main() {
  const size_t region = 4 << 20;
  uint8_t* src;
  cudaMalloc(&src, region);
  cudaMemset(src, 1, region);
  constexpr int CHUNK = 48 * 1024;
  cudaFuncSetAttribute(ingress<CHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * CHUNK + 1024);
  const int iters = 400;
  for (int ctas : {16, 32, 64, 96, 128, 148}) {
    ingress<CHUNK><<<ctas, 32, 4 * CHUNK + 1024>>>(src, iters, region);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ingress<CHUNK><<<ctas, 32, 4 * CHUNK + 1024>>>(src, iters, region);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(ctas) * iters * CHUNK;
    printf("ctas=%3d  aggregate %.2f TB/s  per-SM %.1f GB/s (err=%s)\n", ctas, bytes / ms / 1e9,
           bytes / ctas / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
