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
  __shared__ uint64_t bar2[2];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2[0], 1); mbar_init(&bar2[1], 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, N < 32 ? 64 : 2 * N);
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
    } else if (a_row_offset <= -2) {  // halo pattern + per-tile commit (-2), + acc alternation (-3), + acc reset (-4)
      const int mode = -a_row_offset;
      const uint64_t a0 = umma_smem_desc(smem_u32(smem), 16, 1024, 2);
      const uint64_t b0 = umma_smem_desc(smem_u32(smem + 32768), 16, 1024, 2);
      int tile = 0;
      for (int i = 0; i < iters; i += 36, ++tile) {
        const uint32_t d = tmem + (mode >= 3 ? (tile & 1) * N : 0);
#pragma unroll
        for (int t = 0; t < 9; ++t)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(d, a0 + (((t / 3) * 34 + (t % 3)) * 128 + kk * 32) / 16, b0 + (t * N * 128 / 9 / 128 * 128 + kk * 32) / 16, idesc,
                      mode >= 4 ? ((t | kk) > 0) : ((i | t | kk) > 0));
        umma_commit(&bar2[tile & 1]);
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
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, N < 32 ? 64 : 2 * N); }
}

template <int N, int EVERY>
__global__ void __launch_bounds__(128, 1) mma_commit_loop(int iters, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, N < 32 ? 32 : N);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
    const uint64_t a0 = umma_smem_desc(smem_u32(smem), 16, 1024, 2);
    const uint64_t b0 = umma_smem_desc(smem_u32(smem + 32768), 16, 1024, 2);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += EVERY) {
#pragma unroll
      for (int j = 0; j < EVERY; ++j) umma_bf16(tmem, a0 + 2 * (j & 3), b0 + 2 * (j & 3), idesc, (i | j) > 0);
      umma_commit(&bar[(i / EVERY) & 1]);
    }
    umma_commit(&bar[0]);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, N < 32 ? 32 : N); }
}
// real halo pattern: A rows j0 + r*34 + s of a 30 KB stage (j0 varies per tile), B = 9 distinct
// resident tap tiles of N x 128 B (BMODE 1) or one shared tile (BMODE 0).
template <int N, int BMODE>
__global__ void __launch_bounds__(128, 1) mma_halo_loop(int tiles, long long* cycles, int fill) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  if (fill) {
    const int words = (4 * 30720 + 9 * N * 128) / 4;
    for (int i = threadIdx.x; i < words; i += blockDim.x) {
      uint32_t h = i * 2654435761u + blockIdx.x;
      h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
      // two bf16 in [-2, 2): sign, exponent 126..128, random mantissa
      const uint32_t lo = ((h & 1) << 15) | ((126 + (h >> 1) % 3) << 7) | ((h >> 3) & 0x7f);
      const uint32_t hi = (((h >> 10) & 1) << 15) | ((126 + (h >> 11) % 3) << 7) | ((h >> 13) & 0x7f);
      reinterpret_cast<uint32_t*>(smem)[i] = lo | (hi << 16);
    }
  }
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 2 * N);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
    const uint32_t bres = smem_u32(smem + 4 * 30720);
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const int st = t & 3;
      const int j0 = (t * 128) % 34;
      const uint64_t a0 = umma_smem_desc(smem_u32(smem + st * 30720) + j0 * 128, 16, 1024, 2);
      const uint64_t b0 = umma_smem_desc(bres, 16, 1024, 2);
      const uint32_t d = tmem + (t & 1) * N;
#pragma unroll
      for (int rr = 0; rr < 3; ++rr)
#pragma unroll
        for (int ss = 0; ss < 3; ++ss)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(d, a0 + ((rr * 34 + ss) * 128 + kk * 32) / 16,
                      b0 + (BMODE ? (rr * 3 + ss) * (N * 128) / 16 : 0) + kk * 2, idesc, (rr | ss | kk) > 0);
      umma_commit(&bar[t & 1]);
    }
    umma_commit(&bar[0]);
    mbar_wait(&bar[0], 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 2 * N); }
}
template <int N, int BMODE>
void runh(int fill) {
  long long* d; cudaMalloc(&d, 8);
  const int smem = 4 * 30720 + 9 * N * 128 + 2048;
  cudaFuncSetAttribute(mma_halo_loop<N, BMODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 128;
  for (int r = 0; r < 3; ++r) mma_halo_loop<N, BMODE><<<148, 128, smem>>>(tiles, d, fill);
  long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("halo N=%3d bmode=%d fill=%d: %.1f cycles/MMA (err=%s)\n", N, BMODE, fill, double(cyc) / (tiles * 36),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
template <int N, int EVERY>
void runc() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_commit_loop<N, EVERY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int iters = 4608;
  for (int r = 0; r < 2; ++r) mma_commit_loop<N, EVERY><<<148, 128, 80 * 1024>>>(iters, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_commit_loop<N, EVERY><<<148, 128, 80 * 1024>>>(iters, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 128 * N * 16 * iters * 148;
  printf("N=%3d commit every %2d MMAs: %.0f TFLOP/s -> %.1f ns/MMA (err=%s)\n", N, EVERY, flops / (ms * 1e-3) / 1e12,
         ms * 1e6 / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
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
  runh<64, 1>(0); runh<64, 1>(1); runh<32, 1>(0); runh<32, 1>(1);
  runc<128, 4608>(); runc<256, 4608>();
  return 0;
}
