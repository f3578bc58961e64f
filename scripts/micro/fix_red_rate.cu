// Microbenchmark: cost of the fixed-point reduction atomics of the student partial passes
// (fixacc.cuh fix_red: up to 3 RED.ADD.U64 per per-channel sum, every CTA of the grid adds its
// partials to the same nsum*3 words).  Grid = ctas x 256 threads; each CTA adds `nsum` values.
// mode 0: every CTA issues its own fix_red (the product pattern)
// mode 1: CTAs of a cluster of 8 first add their values into the leader CTA's shared memory
//         (DSMEM red.shared::cluster), the leader issues one fix_red per value
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2301_12443_b200/csrc/kernels \
//      scripts/micro/fix_red_rate.cu -o /tmp/fix_red_rate
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

#include "fixacc.cuh"

namespace cg = cooperative_groups;
using namespace pbdk;

__global__ void red_direct(unsigned long long* out, int nsum) {
  for (int i = threadIdx.x; i < nsum; i += blockDim.x) {
    const float v = 1.0f + 1e-3f * static_cast<float>(blockIdx.x) - 0.37f * static_cast<float>(i & 7);
    fix_red(out + static_cast<size_t>(i) * kFixWords, v);
  }
}

__global__ void __cluster_dims__(8, 1, 1) red_cluster(unsigned long long* out, int nsum) {
  extern __shared__ unsigned long long acc[];  // nsum * 2 words: fixed-point lo / hi of the cluster sum
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 2 * nsum; i += blockDim.x) acc[i] = 0ull;
  cl.sync();
  unsigned long long* lead = cl.map_shared_rank(acc, 0);
  for (int i = threadIdx.x; i < nsum; i += blockDim.x) {
    const float v = 1.0f + 1e-3f * static_cast<float>(blockIdx.x) - 0.37f * static_cast<float>(i & 7);
    const Fix128 f = fix_from(v);
    atomicAdd(lead + 2 * i, f.lo);
    atomicAdd(lead + 2 * i + 1, static_cast<unsigned long long>(f.hi));
  }
  cl.sync();
  if (cl.block_rank() != 0) return;
  for (int i = threadIdx.x; i < nsum; i += blockDim.x) {
    // the real version would carry lo into hi and red both words; here only the atomics' cost matters
    const double v = static_cast<double>(static_cast<long long>(acc[2 * i + 1])) * 1.8446744073709552e19 +
                     static_cast<double>(acc[2 * i]);
    fix_red(out + static_cast<size_t>(i) * kFixWords, static_cast<float>(v * 5.421010862427522e-20));
  }
}

int main() {
  unsigned long long* out;
  cudaMalloc(&out, 1 << 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nsums[] = {193, 385, 769, 1537, 3073};
  const int ctas[] = {64, 144, 296};
  for (int mode = 0; mode < 2; ++mode)
    for (int ns : nsums)
      for (int g : ctas) {
        const size_t smem = mode ? 2 * ns * sizeof(unsigned long long) : 0;
        if (mode) cudaFuncSetAttribute(red_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        for (int it = 0; it < 3; ++it) mode ? red_cluster<<<g, 256, smem>>>(out, ns) : red_direct<<<g, 256>>>(out, ns);
        cudaEventRecord(e0);
        const int reps = 50;
        for (int it = 0; it < reps; ++it)
          mode ? red_cluster<<<g, 256, smem>>>(out, ns) : red_direct<<<g, 256>>>(out, ns);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const cudaError_t err = cudaGetLastError();
        printf("mode %d nsum %5d ctas %4d : %7.2f us/launch  (%s)\n", mode, ns, g, 1e3f * ms / reps,
               cudaGetErrorString(err));
      }
  // empty-kernel launch floor
  cudaEventRecord(e0);
  for (int it = 0; it < 50; ++it) red_direct<<<144, 256>>>(out, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("empty launch: %.2f us\n", 1e3f * ms / 50);
  return 0;
}
