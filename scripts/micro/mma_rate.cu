// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, SS) issue rate vs N, and the cost of
// non-1024-aligned A start addresses (halo conv row offsets).  One CTA per SM, lane 0 of warp 0
// issues `iters` MMAs back to back into one TMEM accumulator, commit + wait at the end.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2301_12443_b200/csrc/kernels/sm100.cuh"
using namespace pbdk;

template <int N>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, int a_row_offset, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, N < 32 ? 32 : N);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
    const uint32_t sa = smem_u32(smem) + a_row_offset * 128;
    const uint32_t sb = smem_u32(smem + 32768);
    long long t0 = clock64();
    if (a_row_offset >= 0) {
      for (int i = 0; i < iters; ++i) {
        const int kk = i & 3;
        umma_bf16(tmem, umma_smem_desc(sa + kk * 32, 16, 1024, 2), umma_smem_desc(sb + kk * 32, 16, 1024, 2), idesc, i > 0);
      }
    } else {  // halo pattern: 9 taps x 4 kk, A at row offset r*34+s, B tap tile t*N*128
      const uint64_t a0 = umma_smem_desc(smem_u32(smem), 16, 1024, 2);
      const uint64_t b0 = umma_smem_desc(smem_u32(smem + 32768), 16, 1024, 2);
      for (int i = 0; i < iters; i += 36) {
#pragma unroll
        for (int t = 0; t < 9; ++t)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(tmem, a0 + (((t / 3) * 34 + (t % 3)) * 128 + kk * 32) / 16, b0 + (t * N * 128 / 9 / 128 * 128 + kk * 32) / 16, idesc, (i | t | kk) > 0);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, N < 32 ? 32 : N); }
}

template <int N>
void run(int off) {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_loop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int iters = 4096;
  mma_loop<N><<<148, 128, 80 * 1024>>>(iters, off, d);
  mma_loop<N><<<148, 128, 80 * 1024>>>(iters, off, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<N><<<148, 128, 80 * 1024>>>(iters, off, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double flops = 2.0 * 128 * N * 16 * iters * 148;
  printf("N=%3d a_off=%d rows: %.2f cycles/MMA, %.0f TFLOP/s (err=%s)\n", N, off, double(cyc) / iters,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<32>(0); run<64>(0); run<128>(0); run<256>(0);
  run<64>(1); run<64>(3); run<64>(35); run<256>(3);
  run<64>(-1); run<32>(-1); run<128>(-1);
  return 0;
}
