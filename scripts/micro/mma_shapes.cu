// Microbenchmark: tcgen05.mma kind::f16 issue rate for the operand placements a 64-output-channel
// conv could use.  SS = both operands in shared memory (the halo conv today: 128x64x16, smem-port
// bound); TS = A from TMEM (only B crosses the shared-memory port).  M = 64 tiles would put the
// 64 output channels on M and pixels on N (filter = A in TMEM, image window = B in smem).
// One CTA per SM, one thread issues `iters` MMAs into one accumulator; cycles per MMA and the
// MAC rate relative to 128x64x16 SS are printed.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2301_12443_b200/csrc/kernels/sm100.cuh"
using namespace pbdk;

__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <int M, int N, bool TS, int ACC = 1>
__global__ void __launch_bounds__(128, 1) loop(int iters, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(M, N, 0, 0);
    const uint32_t sa = smem_u32(smem);
    const uint32_t sb = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      const uint32_t d = tmem + (ACC > 1 ? (i % ACC) * N : 0);
      if (TS)
        umma_bf16_ts(d, tmem + 256 + kk * 8, umma_smem_desc(sb + kk * 32, 16, 1024, 2), idesc, i > 0);
      else
        umma_bf16(d, umma_smem_desc(sa + (ACC > 1 ? (i % ACC) * 16384 : 0) + kk * 32, 16, 1024, 2),
                  umma_smem_desc(sb + kk * 32, 16, 1024, 2), idesc, i >= ACC);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int M, int N, bool TS, int ACC = 1>
void run() {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(loop<M, N, TS, ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 8192;
  for (int r = 0; r < 2; ++r) loop<M, N, TS, ACC><<<148, 128, smem>>>(iters, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  loop<M, N, TS, ACC><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double cpm = double(cyc) / iters;
  const double rel = (double(M) * N / cpm) / (128.0 * 64 / 48.0);
  printf("acc=%d %s M=%3d N=%3d: %6.1f cycles/MMA  %5.0f TFLOP/s  MAC rate x%.2f of SS 128x64 @48cyc  (err=%s)\n",
         ACC, TS ? "TS" : "SS", M, N, cpm, 2.0 * M * N * 16 * iters * 148 / (ms * 1e-3) / 1e12, rel,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<128, 64, false>();
  run<128, 128, false>();
  run<128, 256, false>();
  run<64, 64, false>();
  run<64, 128, false>();
  run<64, 256, false>();
  run<128, 64, true>();
  run<128, 128, true>();
  run<128, 256, true>();
  run<64, 128, true>();
  run<64, 256, true>();
  run<128, 64, false, 2>();
  run<128, 64, false, 4>();
  run<128, 32, false, 2>();
  run<128, 32, false, 4>();
  run<128, 64, true, 2>();
  run<128, 128, false, 2>();
  return 0;
}
