// Microbenchmark: TMA tensor-load throughput per SM for the box shapes the conv kernels use.
// Each CTA streams `iters` boxes through a 4-deep ring (only TMA, no compute); boxes come from
// an L2-resident NHWC bf16 tensor (8 MB).  Reports per-SM GB/s with all 148 SMs loading.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2301_12443_b200/csrc/kernels/sm100.cuh"
#include "../../paper_2301_12443_b200/csrc/kernels/tmap.hpp"
using namespace pbdk;

struct Box { int dims; int c0max, c1max, c2max, c3max; };

template <int NBOX>
__global__ void __launch_bounds__(32, 1) tma_stream(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                                                    int box0_bytes, int box1_bytes, int rank0, int rank1, int iters, int lim1, int lim2, int lim3) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int stage = ((box0_bytes + (NBOX > 1 ? box1_bytes : 0)) + 1023) / 1024 * 1024;
  for (int i = 0; i < iters; ++i) {
    const int st = i & 3;
    if (i >= 4) mbar_wait(&bar[st], ((i >> 2) - 1) & 1);
    mbar_arrive_expect_tx(&bar[st], box0_bytes + (NBOX > 1 ? box1_bytes : 0));
    const int j = blockIdx.x * 131 + i * 7;
    if (rank0 == 4) tma_load_4d(smem + st * stage, &m0, &bar[st], 0, (j % lim1) - 1, ((j / lim1) % lim2) - 1, (j / 13) % lim3);
    else tma_load_2d(smem + st * stage, &m0, &bar[st], 64 * (j % 9), 0);
    if (NBOX > 1) tma_load_2d(smem + st * stage + box0_bytes, &m1, &bar[st], 64 * (j % 9), 256 * (j % 2));
  }
  for (int i = iters; i < iters + 4; ++i) mbar_wait(&bar[i & 3], ((i >> 2) - 1) & 1);
}

int main() {
  void* buf;
  cudaMalloc(&buf, 8 << 20);
  cudaMemset(buf, 0, 8 << 20);
  void* wbuf;
  cudaMalloc(&wbuf, 8 << 20);
  cudaMemset(wbuf, 0, 8 << 20);
  int sms = 148;
  struct Case { const char* name; int n, h, w, c, bw, bh, bn; int wrows; };
  // activation box (c=64 chunk, bw x bh x bn pixels = 128 rows) + optional weight box (64 x wrows)
  std::vector<Case> cases = {
      {"A 8x8 img box (8x8x2), no B", 64, 8, 8, 64, 8, 8, 2, 0},
      {"A 32x4 box (32x4x1), no B", 8, 32, 32, 64, 32, 4, 1, 0},
      {"A 4x4 box (4x4x8), no B", 256, 4, 4, 64, 4, 4, 8, 0},
      {"A 8x8 + B 256 rows", 64, 8, 8, 64, 8, 8, 2, 256},
      {"A 8x8 + B 128 rows", 64, 8, 8, 64, 8, 8, 2, 128},
      {"A 4x4 + B 256 rows", 256, 4, 4, 64, 4, 4, 8, 256},
      {"B only 256 rows (2D)", 0, 0, 0, 0, 0, 0, 0, 256},
      {"B only 128 rows (2D)", 0, 0, 0, 0, 0, 0, 0, 128},
  };
  for (auto& cs : cases) {
    CUtensorMap ma, mb;
    int abytes = 0, bbytes = 0, rank0 = 2;
    if (cs.n > 0) {
      const uint64_t dims[4] = {uint64_t(cs.c), uint64_t(cs.w), uint64_t(cs.h), uint64_t(cs.n)};
      const uint64_t strides[3] = {uint64_t(cs.c) * 2, uint64_t(cs.w) * cs.c * 2, uint64_t(cs.h) * cs.w * cs.c * 2};
      const uint32_t box[4] = {64, uint32_t(cs.bw), uint32_t(cs.bh), uint32_t(cs.bn)};
      const uint32_t es[4] = {1, 1, 1, 1};
      if (!encode_tmap_bf16(&ma, buf, 4, dims, strides, box, es, 128)) { printf("encode A failed\n"); return 1; }
      abytes = 128 * 128;
      rank0 = 4;
    }
    if (cs.wrows > 0) {
      const uint64_t dims[2] = {576, 512};
      const uint64_t strides[1] = {576 * 2};
      const uint32_t box[2] = {64, uint32_t(cs.wrows)};
      const uint32_t es[2] = {1, 1};
      if (!encode_tmap_bf16(&mb, wbuf, 2, dims, strides, box, es, 128)) { printf("encode B failed\n"); return 1; }
      bbytes = cs.wrows * 128;
    }
    const int iters = 2000;
    int total = abytes + bbytes;
    const int smem = 4 * ((total + 1023) / 1024 * 1024) + 1024;
    auto run = [&]() {
      if (cs.n > 0 && cs.wrows > 0) {
        cudaFuncSetAttribute(tma_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_stream<2><<<sms, 32, smem>>>(ma, mb, abytes, bbytes, 4, 2, iters, cs.w, cs.h, cs.n);
      } else if (cs.n > 0) {
        cudaFuncSetAttribute(tma_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_stream<1><<<sms, 32, smem>>>(ma, ma, abytes, 0, 4, 0, iters, cs.w, cs.h, cs.n);
      } else {
        cudaFuncSetAttribute(tma_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_stream<1><<<sms, 32, smem>>>(mb, mb, bbytes, 0, 2, 0, iters, 1, 1, 1);
      }
    };
    run();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(sms) * iters * total;
    printf("%-32s %6d B/iter: per-SM %6.1f GB/s, aggregate %5.2f TB/s (%s)\n", cs.name, total,
           bytes / sms / ms / 1e6, bytes / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
