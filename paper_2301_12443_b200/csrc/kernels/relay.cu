// K11: peer relay of teacher activations between pipeline partitions (TR).
//
// The reference models this transfer as `ready = teacher_end(up) + max(C(b_up), C(b_down))`
// (simulate.cpp:203-214, cost_model.cpp:68-77).  On B200 the sender's SMs store the rows
// straight into the receiver's input buffer through NVLink peer memory (a CUDA IPC mapping
// when the receiver is another process), so no host thread and no NCCL call sit on the
// path and the whole per-rank step stays one CUDA graph.
//
// Protocol (single slot per receiver = its input buffer, monotone 64-bit sequence flags):
//   sender   relay_wait_kernel   : spin until every receiver's `consumed` flag >= seq-1
//            relay_copy_kernel   : 16-byte vector peer stores of every message; the last CTA
//                                  (atomic ticket) fences at system scope and publishes
//                                  ready[slot] = seq on every receiver, then seq_local = seq
//   receiver relay_wait_kernel   : spin until ready[slot] >= seq for every sender
//            ... teacher forward, student step read the input ...
//            relay_release_kernel: seq_local = seq; consumed[slot] = seq on every sender
// Every spin has a wall-clock bound (globaltimer): a peer that never arrives traps the
// kernel (a loud launch failure) instead of hanging the GPU.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "relay.hpp"

namespace pbdk {

namespace {

constexpr unsigned long long kSpinTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One warp: lane i waits on flags[i] >= *seq + bias (flags are written by peers).
__global__ void relay_wait_kernel(RelayWaitArgs a) {
  const int i = threadIdx.x;
  if (i >= a.count) return;
  const unsigned long long target = *a.seq + a.bias;
  const unsigned long long* f = a.flags[i];
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(f) < target) {
    __nanosleep(200);
    if (globaltimer() - t0 > kSpinTimeoutNs) {
      printf("pbd relay: timeout waiting on peer flag %d (want %llu, have %llu)\n", i, target, ld_acquire_sys(f));
      __trap();
    }
  }
}

// Grid-stride copy of every message (16-byte vectors; message sizes and offsets are multiples of
// 16 bytes because rows are NHWC bf16 with >= 16 channels), then the last CTA publishes.
__global__ void __launch_bounds__(256) relay_copy_kernel(RelayCopyArgs a) {
  __shared__ unsigned long long seq_s;
  if (threadIdx.x == 0) seq_s = *a.seq + 1;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (int m = 0; m < a.count; ++m) {
    const uint4* __restrict__ src = reinterpret_cast<const uint4*>(a.src[m]);
    uint4* dst = reinterpret_cast<uint4*>(a.dst[m]);
    const long long n = a.vec16[m];
    long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
      const uint4 v0 = src[i], v1 = src[i + stride], v2 = src[i + 2 * stride], v3 = src[i + 3 * stride];
      dst[i] = v0;
      dst[i + stride] = v1;
      dst[i + 2 * stride] = v2;
      dst[i + 3 * stride] = v3;
    }
    for (; i < n; i += stride) dst[i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int ticket = atomicAdd(a.ticket, 1u);
    if (ticket == gridDim.x - 1) {
      __threadfence_system();
      const unsigned long long seq = seq_s;
      for (int m = 0; m < a.count; ++m) st_release_sys(a.ready[m], seq);
      *a.seq = seq;
      *a.ticket = 0u;
    }
  }
}

// One thread: advance the local sequence and publish it to every peer flag.
__global__ void relay_release_kernel(RelayReleaseArgs a) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  const unsigned long long seq = *a.seq + (a.advance ? 1 : 0);
  *a.seq = seq;
  for (int i = 0; i < a.count; ++i) st_release_sys(a.flags[i], seq);
}

}  // namespace

int relay_wait(const RelayWaitArgs& a, cudaStream_t st) {
  if (a.count < 0 || a.count > kRelayMaxPeers || a.seq == nullptr) return 1;
  if (a.count == 0) return 0;
  relay_wait_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int relay_copy(const RelayCopyArgs& a, int ctas, cudaStream_t st) {
  if (a.count < 0 || a.count > kRelayMaxPeers || a.seq == nullptr || a.ticket == nullptr || ctas < 1) return 1;
  if (a.count == 0) return 0;
  relay_copy_kernel<<<ctas, 256, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int relay_release(const RelayReleaseArgs& a, cudaStream_t st) {
  if (a.count < 0 || a.count > kRelayMaxPeers || a.seq == nullptr) return 1;
  if (a.count == 0) return 0;
  relay_release_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace pbdk
