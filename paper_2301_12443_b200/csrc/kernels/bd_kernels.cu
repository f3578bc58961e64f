// HBM-bound kernels of the blockwise-distillation step (sm_100a):
//   K12 Philox synthetic input / host-image packing, weight init
//   K2/K3 training-mode BatchNorm statistics and apply+ReLU
//   K4  fused MSE distillation loss + ReLU backward + BN2/BNsc backward reductions
//   K5  BN backward apply (dy = gamma*rstd/M * (M g - sum g - xhat sum g xhat))
//   K10 fused SGD-momentum update + bf16 shadow refresh
// Layout: activations NHWC bf16 viewed as [M rows][C channels]; every thread
// owns 8 consecutive channels (one 16-byte vector) of a row.  Reductions are
// two-level and deterministic: per-CTA fp32 partials over a fixed row chunk,
// then a per-channel double-precision sum over the partials in chunk order.
// The arithmetic (operand order, explicit fmaf) is the contract shared with
// the CPU oracle (oracle/bd_oracle.c); see DESIGN.md §3.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "knobs.hpp"
#include "bd_kernels.hpp"
#include "pbdk.h"
#include "sm100.cuh"
#include "fixacc.cuh"

namespace pbdk {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void unpack8(const uint4 v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
}

__device__ __forceinline__ void philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
                                         uint32_t& o0) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c0;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  o0 = c0;
}

__device__ __forceinline__ float sym_unit(uint32_t u) {
  return 2.0f * (static_cast<float>(u >> 8) * (1.0f / 16777216.0f)) - 1.0f;
}

// ------------------------------------------------------------------ data / init

// x[n][32][32][16] bf16; channels 0..2 from Philox, 3..15 zero.
__global__ void philox_image_kernel(__nv_bfloat16* __restrict__ x, int n, int npix, long long first,
                                    const long long* counter, int global_batch, uint32_t seed) {
  const long long base = first + (counter != nullptr ? (*counter) * global_batch : 0);
  const long long total = static_cast<long long>(n) * npix;
  for (long long pix = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; pix < total;
       pix += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = pix / npix;
    const long long hw = pix - i * npix;
    float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const unsigned long long idx =
          static_cast<unsigned long long>(base + i) * (3ull * npix) + static_cast<unsigned long long>(hw * 3 + c);
      uint32_t o;
      philox10(static_cast<uint32_t>(idx), static_cast<uint32_t>(idx >> 32), 0u, 0u, seed, 0xDA7A0000u, o);
      v[c] = sym_unit(o);
    }
    uint4* dst = reinterpret_cast<uint4*>(x + static_cast<size_t>(pix) * 16);
    const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    dst[0] = pack8(v);
    dst[1] = pack8(z);
  }
}

__global__ void pack_image_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ x, long long total) {
  for (long long pix = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; pix < total;
       pix += static_cast<long long>(gridDim.x) * blockDim.x) {
    float v[8] = {src[pix * 3], src[pix * 3 + 1], src[pix * 3 + 2], 0, 0, 0, 0, 0};
    const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint4* dst = reinterpret_cast<uint4*>(x + static_cast<size_t>(pix) * 16);
    dst[0] = pack8(v);
    dst[1] = pack8(z);
  }
}

// double-buffered host input: the graph packs staging slot (*counter & 1) — the host copies the next
// step's images into the other slot while this step runs
__global__ void pack_image_parity_kernel(const float* __restrict__ s0, const float* __restrict__ s1,
                                         const long long* __restrict__ counter, __nv_bfloat16* __restrict__ x,
                                         long long total) {
  const float* __restrict__ src = (*counter & 1) ? s1 : s0;
  for (long long pix = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; pix < total;
       pix += static_cast<long long>(gridDim.x) * blockDim.x) {
    float v[8] = {src[pix * 3], src[pix * 3 + 1], src[pix * 3 + 2], 0, 0, 0, 0, 0};
    const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint4* dst = reinterpret_cast<uint4*>(x + static_cast<size_t>(pix) * 16);
    dst[0] = pack8(v);
    dst[1] = pack8(z);
  }
}

// fp32 workload image (conv_tf32.hpp split layout): x[pix][64] = [hi(32) | lo(32)], channels 0..2
// real, from Philox (mode 0), staging slot s0 (mode 1) or slot (*counter & 1) (mode 2).
constexpr int kF32ImageC = 32;
__global__ void image_split_kernel(float* __restrict__ x, int n, int npix, long long first,
                                   const long long* counter, int global_batch, uint32_t seed,
                                   const float* __restrict__ s0, const float* __restrict__ s1, int mode) {
  const long long base = first + (mode == 0 && counter != nullptr ? (*counter) * global_batch : 0);
  const float* __restrict__ src = mode == 2 && (*counter & 1) ? s1 : s0;
  const long long total = static_cast<long long>(n) * npix;
  for (long long pix = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; pix < total;
       pix += static_cast<long long>(gridDim.x) * blockDim.x) {
    float v[3];
    if (mode == 0) {
      const long long i = pix / npix;
      const long long hw = pix - i * npix;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const unsigned long long idx =
            static_cast<unsigned long long>(base + i) * (3ull * npix) + static_cast<unsigned long long>(hw * 3 + c);
        uint32_t o;
        philox10(static_cast<uint32_t>(idx), static_cast<uint32_t>(idx >> 32), 0u, 0u, seed, 0xDA7A0000u, o);
        v[c] = sym_unit(o);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) v[c] = src[pix * 3 + c];
    }
    float4* dst = reinterpret_cast<float4*>(x + static_cast<size_t>(pix) * 2 * kF32ImageC);
    const float h0 = tf32_hi(v[0]), h1 = tf32_hi(v[1]), h2 = tf32_hi(v[2]);
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    dst[0] = make_float4(h0, h1, h2, 0.f);
    for (int q = 1; q < kF32ImageC / 4; ++q) dst[q] = z;
    dst[kF32ImageC / 4] = make_float4(v[0] - h0, v[1] - h1, v[2] - h2, 0.f);
    for (int q = kF32ImageC / 4 + 1; q < kF32ImageC / 2; ++q) dst[q] = z;
  }
}

// dst[k][r][s][c_stored] = (k < k_true && c < c_true) ? U(-1,1)[counter=((k*r+..)*c_true+c, tensor)] * bound : 0
// (the counter is the flat index of the true [k_true][r][s][c_true] tensor)
__global__ void init_uniform_kernel(void* dst, int bf16_out, int k, int r, int s, int cs, int ct, uint32_t seed,
                                    uint32_t tensor, float bound, int kt) {
  const long long total = static_cast<long long>(k) * r * s * cs;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cs);
    const long long krs = i / cs;
    float v = 0.0f;
    if (c < ct && krs / (r * s) < kt) {
      const long long j = krs * ct + c;
      uint32_t o;
      philox10(static_cast<uint32_t>(j), tensor, 0u, 0u, seed, 0xB200B200u, o);
      v = sym_unit(o) * bound;
    }
    if (bf16_out == 1) {
      static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
    } else if (bf16_out == 2) {  // split fp32 [k][r][s][hi cs | lo cs]
      const float h = tf32_hi(v);
      static_cast<float*>(dst)[krs * 2 * cs + c] = h;
      static_cast<float*>(dst)[krs * 2 * cs + cs + c] = v - h;
    } else {
      static_cast<float*>(dst)[i] = v;
    }
  }
}

__global__ void fill_kernel(float* __restrict__ dst, size_t n, float v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = v;
}

// ------------------------------------------------------------------ row-wise kernels over [M][C]
// Thread (g, slot): g = tid % cg owns V consecutive channels for the whole kernel (its
// per-channel BN parameters are loaded once, into registers), slot = tid / cg picks rows.
// Partial reductions: CTA b covers the contiguous rows [b*rows_per_chunk, ...), fp32 sums
// per thread, fixed-order CTA combine into partial[chunk][NV][C]; finalize kernels add the
// chunk partials in a fixed strided order in fp64.  Deterministic for a given (M, C).

template <int V>
struct Vec;
template <>
struct Vec<8> {
  using T = uint4;
  __device__ static void load(const __nv_bfloat16* p, float (&f)[8]) { unpack8(*reinterpret_cast<const uint4*>(p), f); }
  __device__ static void store(__nv_bfloat16* p, const float (&f)[8]) { *reinterpret_cast<uint4*>(p) = pack8(f); }
};
template <>
struct Vec<4> {
  __device__ static void load(const __nv_bfloat16* p, float (&f)[4]) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    f[0] = __uint_as_float(v.x << 16);
    f[1] = __uint_as_float(v.x & 0xFFFF0000u);
    f[2] = __uint_as_float(v.y << 16);
    f[3] = __uint_as_float(v.y & 0xFFFF0000u);
  }
  __device__ static void store(__nv_bfloat16* p, const float (&f)[4]) {
    *reinterpret_cast<uint2*>(p) = make_uint2(pack2(f[0], f[1]), pack2(f[2], f[3]));
  }
};

// Row I/O policies of the [M][C] kernels: bf16 rows (the bf16 workloads), plain fp32 rows and split
// fp32 rows (the fp32 workload; conv_tf32.hpp: row r = [hi(C) | lo(C)] at r*2C, value = hi + lo,
// stored as hi = tf32(x), lo = x - hi).
struct IoBf16 {
  using T = __nv_bfloat16;
  template <int V>
  __device__ static void load(const T* p, size_t r, int C, int c0, float (&f)[V]) {
    Vec<V>::load(p + r * C + c0, f);
  }
  template <int V>
  __device__ static void store(T* p, size_t r, int C, int c0, const float (&f)[V]) {
    Vec<V>::store(p + r * C + c0, f);
  }
};
struct IoF32 {
  using T = float;
  template <int V>
  __device__ static void load(const T* p, size_t r, int C, int c0, float (&f)[V]) {
    const float4* q = reinterpret_cast<const float4*>(p + r * C + c0);
#pragma unroll
    for (int i = 0; i < V / 4; ++i) {
      const float4 v = q[i];
      f[4 * i] = v.x;
      f[4 * i + 1] = v.y;
      f[4 * i + 2] = v.z;
      f[4 * i + 3] = v.w;
    }
  }
  template <int V>
  __device__ static void store(T* p, size_t r, int C, int c0, const float (&f)[V]) {
    float4* q = reinterpret_cast<float4*>(p + r * C + c0);
#pragma unroll
    for (int i = 0; i < V / 4; ++i) q[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
  }
};
struct IoSplit {
  using T = float;
  template <int V>
  __device__ static void load(const T* p, size_t r, int C, int c0, float (&f)[V]) {
    const float4* h = reinterpret_cast<const float4*>(p + r * 2 * C + c0);
    const float4* l = reinterpret_cast<const float4*>(p + r * 2 * C + C + c0);
#pragma unroll
    for (int i = 0; i < V / 4; ++i) {
      const float4 a = h[i], b = l[i];
      f[4 * i] = a.x + b.x;
      f[4 * i + 1] = a.y + b.y;
      f[4 * i + 2] = a.z + b.z;
      f[4 * i + 3] = a.w + b.w;
    }
  }
  template <int V>
  __device__ static void store(T* p, size_t r, int C, int c0, const float (&f)[V]) {
    float4* h = reinterpret_cast<float4*>(p + r * 2 * C + c0);
    float4* l = reinterpret_cast<float4*>(p + r * 2 * C + C + c0);
#pragma unroll
    for (int i = 0; i < V / 4; ++i) {
      float hi[4], lo[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        hi[j] = tf32_hi(f[4 * i + j]);
        lo[j] = f[4 * i + j] - hi[j];
      }
      h[i] = make_float4(hi[0], hi[1], hi[2], hi[3]);
      l[i] = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
  }
};

struct RowTiling {
  int cg, rpp, chunks, rows_per_chunk;
};

int env_int(const char* name, int dflt) {
  const char* e = pbd::knob_env(name);
  return e != nullptr ? std::atoi(e) : dflt;
}
// Grid sizes of the reduction (partial) and elementwise (apply) passes (GridScope, bd_kernels.hpp).
// Measured, CUDA-graph ResNet step at b=256 (4 concurrent student streams): partials 296 -> 148 CTAs
// and applies 1184 -> 296 CTAs took the step from 0.997 to 0.932 ms although each kernel alone is
// slower — a one-CTA-per-SM wave leaves the other streams' convs their SMs.  The MBConv step (passes
// mostly alone) prefers 296 / 1184 (19.74 vs 20.17 ms).  PBDK_RED_TARGET / PBDK_APPLY_CTAS override.
thread_local int t_red = 0, t_apply = 0, t_fix_min = 0;
int red_target() {
  static const int e = env_int("PBDK_RED_TARGET", 0);
  return e > 0 ? e : (t_red > 0 ? t_red : 148 * 2);
}
int apply_cap() {
  static const int e = env_int("PBDK_APPLY_CTAS", 0);
  return e > 0 ? e : (t_apply > 0 ? t_apply : 148 * 8);
}

RowTiling tiling_for(int m, int c, int v, int target = -1) {
  if (target < 0) target = red_target();
  RowTiling t;
  t.cg = c / v;
  t.rpp = std::max(1, kThreads / t.cg);
  const int passes = (m + t.rpp - 1) / t.rpp;
  const int chunks = std::max(1, std::min(target, passes));
  t.rows_per_chunk = (passes + chunks - 1) / chunks * t.rpp;
  t.chunks = (m + t.rows_per_chunk - 1) / t.rows_per_chunk;
  return t;
}

int apply_grid(int m, int rpp) { return std::max(1, std::min((m + rpp - 1) / rpp, apply_cap())); }

// CTA-level fixed-order reduction of NV*V floats per thread into partial[chunk][NV][C].
template <int NV, int V>
__device__ void cta_reduce_store(float (&acc)[NV][V], int cg, int rpp, int C, float* __restrict__ partial) {
  __shared__ float sm[kThreads * NV * V];
  const int t = threadIdx.x;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int j = 0; j < V; ++j) sm[(v * V + j) * kThreads + t] = acc[v][j];
  __syncthreads();
  for (int o = t; o < NV * cg * V; o += kThreads) {
    const int v = o / (cg * V);
    const int rem = o - v * cg * V;
    const int g = rem / V;
    const int j = rem - g * V;
    float s = 0.0f;
    for (int r = 0; r < rpp; ++r) s += sm[(v * V + j) * kThreads + r * cg + g];
    partial[(static_cast<size_t>(blockIdx.x) * NV + v) * C + g * V + j] = s;
  }
}

constexpr int kFinWarps = 8;

// fp64 sum over chunks of partial[chunk][NV][C] for output o = v*C + c: one warp per output,
// lane l adds chunks l, l+32, ... (independent loads), then a fixed xor-shuffle tree.
// Deterministic for a given (chunks, C); every lane returns the total.
template <int NV>
__device__ __forceinline__ double warp_sum_chunks(const float* __restrict__ partial, int chunks, int C, int o) {
  const int lane = threadIdx.x & 31;
  const int v = o / C;
  const int c = o - v * C;
  const float* base = partial + static_cast<size_t>(v) * C + c;
  const size_t stride = static_cast<size_t>(NV) * C;
  double s = 0.0;
  for (int b = lane; b < chunks; b += 32) s += base[b * stride];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// fixed-order sum of n floats by one CTA of kFinWarps warps (strided per-thread sums,
// xor-shuffle tree per warp, warps added in order by thread 0).
__device__ __forceinline__ double cta_sum(const float* __restrict__ v, int n) {
  __shared__ double sm[kFinWarps];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sm[w];
  return t;
}

// -- BN statistics: per-channel (sum y, sum y^2) of one or two tensors of the same shape
template <int V, int NT, class IO = IoBf16>
__global__ void __launch_bounds__(kThreads) bn_stats_partial_kernel(const typename IO::T* __restrict__ y0,
                                                                    const typename IO::T* __restrict__ y1, int m,
                                                                    int C, int rows_per_chunk, int cg, int rpp,
                                                                    float* __restrict__ partial) {
  const int g = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float acc[2 * NT][V] = {};
  if (slot < rpp) {
    const int r0 = blockIdx.x * rows_per_chunk;
    const int r1 = min(m, r0 + rows_per_chunk);
#pragma unroll 4
    for (int r = r0 + slot; r < r1; r += rpp) {
      float f[NT][V];
      IO::template load<V>(y0, r, C, g * V, f[0]);
      if (NT == 2) IO::template load<V>(y1, r, C, g * V, f[NT - 1]);
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int j = 0; j < V; ++j) {
          acc[2 * t][j] += f[t][j];
          acc[2 * t + 1][j] += f[t][j] * f[t][j];
        }
    }
  }
  cta_reduce_store<2 * NT, V>(acc, cg, rpp, C, partial);
}

// grid: ceil(NT*C / 8) CTAs of 8 warps; warp = (tensor, channel).
template <int NT>
__global__ void bn_stats_finalize_kernel(const float* __restrict__ partial, int chunks, int C, int m,
                                         float* __restrict__ mr0, float* __restrict__ mr1) {
  const int o = blockIdx.x * kFinWarps + (threadIdx.x >> 5);
  if (o >= NT * C) return;
  const int t = o / C;
  const int c = o - t * C;
  const double s1 = warp_sum_chunks<2 * NT>(partial, chunks, C, 2 * t * C + c);
  const double s2 = warp_sum_chunks<2 * NT>(partial, chunks, C, (2 * t + 1) * C + c);
  if ((threadIdx.x & 31) == 0) {
    float* mr = t == 0 ? mr0 : mr1;
    const double mu = s1 / static_cast<double>(m);
    const double var = s2 / static_cast<double>(m) - mu * mu;
    mr[c] = static_cast<float>(mu);
    mr[C + c] = 1.0f / sqrtf(static_cast<float>(var) + 1e-5f);
  }
}

// -- BN apply + ReLU as a per-channel affine map: a = bf16(relu(fmaf(A, y, B))),
//    A = gamma*rstd, B = fmaf(-A, mean, beta)
template <int V, class IN = IoBf16, class OUT = IoBf16>
__global__ void __launch_bounds__(kThreads) bn_apply_relu_kernel(const typename IN::T* __restrict__ y,
                                                                 const float* __restrict__ mean_rstd,
                                                                 const float* __restrict__ gamma,
                                                                 const float* __restrict__ beta,
                                                                 typename OUT::T* __restrict__ a, int m, int C, int cg,
                                                                 int rpp) {
  const int g = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  if (slot >= rpp) return;
  const int c0 = g * V;
  float A[V], B[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    A[j] = gamma[c0 + j] * mean_rstd[C + c0 + j];
    B[j] = fmaf(-A[j], mean_rstd[c0 + j], beta[c0 + j]);
  }
  const int step = gridDim.x * rpp;
#pragma unroll 4
  for (int r = blockIdx.x * rpp + slot; r < m; r += step) {
    float f[V];
    IN::template load<V>(y, r, C, c0, f);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float z = fmaf(A[j], f[j], B[j]);
      f[j] = z > 0.0f ? z : 0.0f;
    }
    OUT::template store<V>(a, r, C, c0, f);
  }
}

// -- fused distillation loss.  z = A2*y2 + As*ysc + Bz (both BNs as affine maps), s = relu(z),
//    L += (s-t)^2, g = [z>0] (s-t)*gscale; partial sums of g, g*y2, g*ysc.
struct LossParams {
  const void* y2;  // IN rows
  const void* ys;  // IN rows
  const void* t;   // TG rows
  const float* st2;  // mean[C], rstd[C]
  const float* sts;
  const float* g2;
  const float* b2;
  const float* gs;
  const float* bs;
  int m, C;
  float gscale;
};

template <int V>
__device__ __forceinline__ void loss_affine(const LossParams& p, int c0, float (&A2)[V], float (&As)[V],
                                            float (&Bz)[V]) {
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int c = c0 + j;
    A2[j] = p.g2[c] * p.st2[p.C + c];
    As[j] = p.gs[c] * p.sts[p.C + c];
    Bz[j] = fmaf(-A2[j], p.st2[c], p.b2[c]) + fmaf(-As[j], p.sts[c], p.bs[c]);
  }
}

constexpr int kLossPartialV = 8;
const int kLossChunks = -1;  // = red_target(), as the BN partials
constexpr int kLossApplyV = 4;

template <class IN = IoBf16, class TG = IoBf16>
__global__ void __launch_bounds__(kThreads) loss_partial_kernel(const LossParams p, int rows_per_chunk, int cg, int rpp,
                                                                float* __restrict__ partial,
                                                                float* __restrict__ loss_partial) {
  constexpr int V = kLossPartialV;
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float acc[3][V] = {};
  float lsum = 0.0f;
  if (slot < rpp) {
    float A2[V], As[V], Bz[V];
    loss_affine<V>(p, gi * V, A2, As, Bz);
    const int r0 = blockIdx.x * rows_per_chunk;
    const int r1 = min(p.m, r0 + rows_per_chunk);
#pragma unroll 4
    for (int r = r0 + slot; r < r1; r += rpp) {
      float y2[V], ys[V], t[V];
      IN::template load<V>(static_cast<const typename IN::T*>(p.y2), r, p.C, gi * V, y2);
      IN::template load<V>(static_cast<const typename IN::T*>(p.ys), r, p.C, gi * V, ys);
      TG::template load<V>(static_cast<const typename TG::T*>(p.t), r, p.C, gi * V, t);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float z = fmaf(A2[j], y2[j], fmaf(As[j], ys[j], Bz[j]));
        const float d = (z > 0.0f ? z : 0.0f) - t[j];
        const float g = z > 0.0f ? d * p.gscale : 0.0f;
        lsum += d * d;
        acc[0][j] += g;
        acc[1][j] += g * y2[j];
        acc[2][j] += g * ys[j];
      }
    }
  }
  __shared__ float lred[kThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
  if ((threadIdx.x & 31) == 0) lred[threadIdx.x >> 5] = lsum;
  cta_reduce_store<3, V>(acc, cg, rpp, p.C, partial);
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.0f;
    for (int i = 0; i < kThreads / 32; ++i) s += lred[i];
    loss_partial[blockIdx.x] = s;
  }
}

// Finalize (fp64): sum g*xhat = rstd*(sum g*y - mean*sum g); gamma/beta grads; the coefficients
// of dy = A*g + Q*y + R: coef[0:C]=Q2, [C:2C]=R2, [2C:3C]=Qs, [3C:4C]=Rs.  Warp = channel; the
// last CTA sums the loss partials.
__global__ void loss_finalize_kernel(const LossParams p, const float* __restrict__ partial,
                                     const float* __restrict__ loss_partial, int chunks, double norm,
                                     float* __restrict__ coef, float* __restrict__ dg2, float* __restrict__ db2,
                                     float* __restrict__ dgs, float* __restrict__ dbs, double* __restrict__ loss_out) {
  const int C = p.C;
  if (blockIdx.x == gridDim.x - 1) {
    const double l = cta_sum(loss_partial, chunks);
    if (threadIdx.x == 0) *loss_out = l / norm;
    return;
  }
  const int c = blockIdx.x * kFinWarps + (threadIdx.x >> 5);
  if (c >= C) return;
  const double sg = warp_sum_chunks<3>(partial, chunks, C, c);
  const double sgy2 = warp_sum_chunks<3>(partial, chunks, C, C + c);
  const double sgys = warp_sum_chunks<3>(partial, chunks, C, 2 * C + c);
  if ((threadIdx.x & 31) == 0) {
    const float m2 = p.st2[c], r2 = p.st2[C + c], ms = p.sts[c], rs = p.sts[C + c];
    const float A2 = p.g2[c] * r2, As = p.gs[c] * rs;
    const double sgx2 = static_cast<double>(r2) * (sgy2 - static_cast<double>(m2) * sg);
    const double sgxs = static_cast<double>(rs) * (sgys - static_cast<double>(ms) * sg);
    db2[c] = static_cast<float>(sg);
    dbs[c] = static_cast<float>(sg);
    dg2[c] = static_cast<float>(sgx2);
    dgs[c] = static_cast<float>(sgxs);
    const double c2 = static_cast<double>(A2) / p.m, cs = static_cast<double>(As) / p.m;
    coef[c] = static_cast<float>(-c2 * sgx2 * r2);
    coef[C + c] = static_cast<float>(-c2 * (sg - sgx2 * r2 * m2));
    coef[2 * C + c] = static_cast<float>(-cs * sgxs * rs);
    coef[3 * C + c] = static_cast<float>(-cs * (sg - sgxs * rs * ms));
  }
}

template <class IN = IoBf16, class TG = IoBf16, class OUT = IoBf16>
__global__ void __launch_bounds__(kThreads) loss_bwd_apply_kernel(const LossParams p, const float* __restrict__ coef,
                                                                  int cg, int rpp, typename OUT::T* __restrict__ dy2,
                                                                  typename OUT::T* __restrict__ dys) {
  constexpr int V = kLossApplyV;
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  if (slot >= rpp) return;
  const int c0 = gi * V;
  float A2[V], As[V], Bz[V], Q2[V], R2[V], Qs[V], Rs[V];
  loss_affine<V>(p, c0, A2, As, Bz);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    Q2[j] = coef[c0 + j];
    R2[j] = coef[p.C + c0 + j];
    Qs[j] = coef[2 * p.C + c0 + j];
    Rs[j] = coef[3 * p.C + c0 + j];
  }
  const int step = gridDim.x * rpp;
#pragma unroll 4
  for (int r = blockIdx.x * rpp + slot; r < p.m; r += step) {
    float y2[V], ys[V], t[V], o2[V], os[V];
    IN::template load<V>(static_cast<const typename IN::T*>(p.y2), r, p.C, c0, y2);
    IN::template load<V>(static_cast<const typename IN::T*>(p.ys), r, p.C, c0, ys);
    TG::template load<V>(static_cast<const typename TG::T*>(p.t), r, p.C, c0, t);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float z = fmaf(A2[j], y2[j], fmaf(As[j], ys[j], Bz[j]));
      const float d = (z > 0.0f ? z : 0.0f) - t[j];
      const float g = z > 0.0f ? d * p.gscale : 0.0f;
      o2[j] = fmaf(A2[j], g, fmaf(Q2[j], y2[j], R2[j]));
      os[j] = fmaf(As[j], g, fmaf(Qs[j], ys[j], Rs[j]));
    }
    OUT::template store<V>(dy2, r, p.C, c0, o2);
    OUT::template store<V>(dys, r, p.C, c0, os);
  }
}

// -- BN backward (first BN of the unit): partial sums of g and g*y, finalize, apply
template <int V, class IN = IoBf16>
__global__ void __launch_bounds__(kThreads) bn_bwd_partial_kernel(const typename IN::T* __restrict__ gin,
                                                                  const typename IN::T* __restrict__ y, int m, int C,
                                                                  int rows_per_chunk, int cg, int rpp,
                                                                  float* __restrict__ partial) {
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float acc[2][V] = {};
  if (slot < rpp) {
    const int r0 = blockIdx.x * rows_per_chunk;
    const int r1 = min(m, r0 + rows_per_chunk);
#pragma unroll 4
    for (int r = r0 + slot; r < r1; r += rpp) {
      float fg[V], fy[V];
      IN::template load<V>(gin, r, C, gi * V, fg);
      IN::template load<V>(y, r, C, gi * V, fy);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        acc[0][j] += fg[j];
        acc[1][j] += fg[j] * fy[j];
      }
    }
  }
  cta_reduce_store<2, V>(acc, cg, rpp, C, partial);
}

// coef[0:C] = Q, coef[C:2C] = R of dy = A*g + Q*y + R
__global__ void bn_bwd_finalize_kernel(const float* __restrict__ partial, int chunks, int C, int m,
                                       const float* __restrict__ st, const float* __restrict__ gamma,
                                       float* __restrict__ coef, float* __restrict__ dgamma,
                                       float* __restrict__ dbeta) {
  const int c = blockIdx.x * kFinWarps + (threadIdx.x >> 5);
  if (c >= C) return;
  const double sg = warp_sum_chunks<2>(partial, chunks, C, c);
  const double sgy = warp_sum_chunks<2>(partial, chunks, C, C + c);
  if ((threadIdx.x & 31) == 0) {
    const float mu = st[c], rs = st[C + c];
    const float A = gamma[c] * rs;
    const double sgx = static_cast<double>(rs) * (sgy - static_cast<double>(mu) * sg);
    dbeta[c] = static_cast<float>(sg);
    dgamma[c] = static_cast<float>(sgx);
    const double k = static_cast<double>(A) / m;
    coef[c] = static_cast<float>(-k * sgx * rs);
    coef[C + c] = static_cast<float>(-k * (sg - sgx * rs * mu));
  }
}

template <int V, class IN = IoBf16, class OUT = IoBf16>
__global__ void __launch_bounds__(kThreads) bn_bwd_apply_kernel(const typename IN::T* __restrict__ gin,
                                                                const typename IN::T* __restrict__ y,
                                                                const float* __restrict__ st,
                                                                const float* __restrict__ gamma,
                                                                const float* __restrict__ coef, int m, int C, int cg,
                                                                int rpp, typename OUT::T* __restrict__ dy) {
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  if (slot >= rpp) return;
  const int c0 = gi * V;
  float A[V], Q[V], R[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    A[j] = gamma[c0 + j] * st[C + c0 + j];
    Q[j] = coef[c0 + j];
    R[j] = coef[C + c0 + j];
  }
  const int step = gridDim.x * rpp;
#pragma unroll 4
  for (int r = blockIdx.x * rpp + slot; r < m; r += step) {
    float fg[V], fy[V], o[V];
    IN::template load<V>(gin, r, C, c0, fg);
    IN::template load<V>(y, r, C, c0, fy);
#pragma unroll
    for (int j = 0; j < V; ++j) o[j] = fmaf(A[j], fg[j], fmaf(Q[j], fy[j], R[j]));
    OUT::template store<V>(dy, r, C, c0, o);
  }
}


// ------------------------------------------------------------------ self-finalizing partial passes
// The ResNet student step's reductions (BN statistics, loss sums, BN-backward sums) add each CTA's
// fp32 chunk partial EXACTLY into fixed-point accumulators (fixacc.cuh); the last CTA to finish
// (atomic ticket) turns the totals into the consumers' coefficients — the former finalize kernels'
// arithmetic — then zeroes the accumulators and its ticket for the next step.  One launch instead of
// two per reduction; integer adds commute, so the result does not depend on CTA completion order.

// CTA-level fixed-order reduction of NV*V floats per thread (as cta_reduce_store); the CTA's
// per-channel fp32 partial (v, c) is added exactly to the sum out[(v * C + c) * kFixWords ..].
template <int NV, int V>
__device__ void cta_reduce_fix(float (&acc)[NV][V], int cg, int rpp, int C, unsigned long long* __restrict__ out) {
  __shared__ float sm[kThreads * NV * V];
  const int t = threadIdx.x;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int j = 0; j < V; ++j) sm[(v * V + j) * kThreads + t] = acc[v][j];
  __syncthreads();
  for (int o = t; o < NV * cg * V; o += kThreads) {
    const int v = o / (cg * V);
    const int rem = o - v * cg * V;
    const int g = rem / V;
    const int j = rem - g * V;
    float s = 0.0f;
    for (int r = 0; r < rpp; ++r) s += sm[(v * V + j) * kThreads + r * cg + g];
    fix_red(out + (static_cast<size_t>(v) * C + g * V + j) * kFixWords, s);
  }
}

// true in the last CTA of the grid to pass (every thread's accumulator atomics are performed before
// its CTA takes a ticket); that CTA then sees every other CTA's adds.  Resets the ticket.
__device__ __forceinline__ bool last_cta(unsigned int* ticket) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(ticket, 1u);
    last = prev == gridDim.x - 1;
    if (last) *ticket = 0u;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__device__ __forceinline__ double fix_take(unsigned long long* p) {  // read a finished sum and zero it
  const unsigned long long v[kFixWords] = {__ldcg(p), __ldcg(p + 1), __ldcg(p + 2)};
  p[0] = 0ull;
  p[1] = 0ull;
  p[2] = 0ull;
  return fix_value(v);
}

// ------------------------------------------------------------------ TMA-staged row streams
// The student passes read [M][C] bf16 row ranges that are contiguous in HBM.  A CTA streams its range
// through a kPipeStages-deep shared-memory ring filled by 1D bulk copies (one per input tensor and
// tile of `tr` rows), so ~kPipeStages x kPipeStageBytes per SM are in flight instead of the handful of
// 16-byte loads per thread the register loops kept outstanding (those ran at 0.5-2 TB/s, latency-bound
// at one CTA per SM).  Thread (g, slot) visits rows r0 + slot + k*rpp in increasing order — the order
// of the register loops, so the fp32 partials are unchanged.
constexpr int kPipeStages = 4;
constexpr int kPipeStageBytes = 24 * 1024;  // all inputs of one stage

int pipe_tile_rows(int nin, int c, int rpp) {
  const int rows = kPipeStageBytes / (nin * c * 2);
  return std::max(rpp, rows / rpp * rpp);
}
size_t pipe_smem(int nin, int c, int tr) { return static_cast<size_t>(kPipeStages) * nin * tr * c * 2; }

template <int NIN>
struct PipeIn {
  const __nv_bfloat16* p[NIN];
};

// f(row, s) with s[k] = this thread's V-channel group of row `row` of input k in shared memory.
// pre() runs once per thread after the first tiles are requested: per-channel parameter loads placed
// there overlap the tiles' latency instead of delaying the requests.
template <int NIN, int V, class P, class F>
__device__ __forceinline__ void row_pipe(const PipeIn<NIN>& in, int C, int r0, int r1, int tr, int g, int slot,
                                         int rpp, P&& pre, F&& f) {
  extern __shared__ __align__(128) uint8_t pipe_smem_raw[];
  __shared__ uint64_t full[kPipeStages];
  const int tile_elems = tr * C;
  const int ntiles = r1 > r0 ? (r1 - r0 + tr - 1) / tr : 0;
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(pipe_smem_raw);
  auto issue = [&](int t) {
    const int st = t % kPipeStages;
    const int rows = min(tr, r1 - (r0 + t * tr));
    const uint32_t bytes = static_cast<uint32_t>(rows) * C * 2;
    mbar_arrive_expect_tx(&full[st], NIN * bytes);
#pragma unroll
    for (int k = 0; k < NIN; ++k)
      bulk_load(ring + (st * NIN + k) * tile_elems, in.p[k] + static_cast<size_t>(r0 + t * tr) * C, bytes, &full[st]);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPipeStages; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  grid_dep_wait();  // PDL (launch_pipe): every global access of the pass kernels comes after this point
  if (threadIdx.x == 0)
    for (int t = 0; t < min(ntiles, kPipeStages); ++t) issue(t);
  pre();
  for (int t = 0; t < ntiles; ++t) {
    const int st = t % kPipeStages;
    mbar_wait(&full[st], (t / kPipeStages) & 1);
    const int rows = min(tr, r1 - (r0 + t * tr));
    if (slot < rpp) {
      const __nv_bfloat16* s[NIN];
#pragma unroll
      for (int k = 0; k < NIN; ++k) s[k] = ring + (st * NIN + k) * tile_elems + g * V;
#pragma unroll 2
      for (int rr = slot; rr < rows; rr += rpp) {
        const __nv_bfloat16* sr[NIN];
#pragma unroll
        for (int k = 0; k < NIN; ++k) sr[k] = s[k] + rr * C;
        f(r0 + t * tr + rr, sr);
      }
    }
    __syncthreads();  // stage st fully read before it is refilled
    if (threadIdx.x == 0 && t + kPipeStages < ntiles) issue(t + kPipeStages);
  }
}

template <int NIN, int V, class F>
__device__ __forceinline__ void row_pipe(const PipeIn<NIN>& in, int C, int r0, int r1, int tr, int g, int slot,
                                         int rpp, F&& f) {
  row_pipe<NIN, V>(in, C, r0, r1, tr, g, slot, rpp, [] {}, f);
}

template <int V>
__device__ __forceinline__ void ld_smem(const __nv_bfloat16* p, float (&f)[V]) {
  Vec<V>::load(p, f);
}

// -- BN statistics of NT same-shape tensors -> mean / rstd (bn_stats_finalize_kernel's arithmetic)
template <int V, int NT>
__global__ void __launch_bounds__(kThreads) bn_stats_fix_kernel(const PipeIn<NT> in, int m, int C,
                                                                int rows_per_chunk, int cg, int rpp, int tr,
                                                                unsigned long long* __restrict__ acc,
                                                                unsigned int* ticket, float* __restrict__ mr0,
                                                                float* __restrict__ mr1) {
  const int g = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float a[2 * NT][V] = {};
  const int r0 = blockIdx.x * rows_per_chunk;
  row_pipe<NT, V>(in, C, r0, min(m, r0 + rows_per_chunk), tr, g, slot, rpp,
                  [&](int, const __nv_bfloat16* const* s) {
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                      float f[V];
                      ld_smem<V>(s[t], f);
#pragma unroll
                      for (int j = 0; j < V; ++j) {
                        a[2 * t][j] += f[j];
                        a[2 * t + 1][j] += f[j] * f[j];
                      }
                    }
                  });
  cta_reduce_fix<2 * NT, V>(a, cg, rpp, C, acc);  // acc[(2t + {0: sum, 1: sumsq}) * C + c]
  if (!last_cta(ticket)) return;
  for (int o = threadIdx.x; o < NT * C; o += blockDim.x) {
    const int t = o / C, c = o - t * C;
    const double s1 = fix_take(acc + (static_cast<size_t>(2 * t) * C + c) * kFixWords);
    const double s2 = fix_take(acc + (static_cast<size_t>(2 * t + 1) * C + c) * kFixWords);
    const double mu = s1 / static_cast<double>(m);
    const double var = s2 / static_cast<double>(m) - mu * mu;
    float* mr = t == 0 ? mr0 : mr1;
    mr[c] = static_cast<float>(mu);
    mr[C + c] = 1.0f / sqrtf(static_cast<float>(var) + 1e-5f);
  }
}

// -- BN apply + ReLU (bn_apply_relu_kernel's arithmetic), staged
template <int V>
__global__ void __launch_bounds__(kThreads) bn_apply_relu_pipe_kernel(const PipeIn<1> in,
                                                                      const float* __restrict__ mean_rstd,
                                                                      const float* __restrict__ gamma,
                                                                      const float* __restrict__ beta,
                                                                      __nv_bfloat16* __restrict__ out, int m, int C,
                                                                      int rows_per_chunk, int cg, int rpp, int tr) {
  const int g = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  const int c0 = g * V;
  float A[V], B[V];
  const int r0 = blockIdx.x * rows_per_chunk;
  row_pipe<1, V>(in, C, r0, min(m, r0 + rows_per_chunk), tr, g, slot, rpp, [&] {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      A[j] = gamma[c0 + j] * mean_rstd[C + c0 + j];
      B[j] = fmaf(-A[j], mean_rstd[c0 + j], beta[c0 + j]);
    }
  }, [&](int r, const __nv_bfloat16* const* s) {
    float f[V];
    ld_smem<V>(s[0], f);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float z = fmaf(A[j], f[j], B[j]);
      f[j] = z > 0.0f ? z : 0.0f;
    }
    Vec<V>::store(out + static_cast<size_t>(r) * C + c0, f);
  });
}

// -- loss partial sums (sum g, g*y2, g*ys per channel; sum (s-t)^2) -> coef / parameter gradients / loss
struct LossOut {
  double norm;
  unsigned long long* acc;  // sums [3][C] + [1] (loss), kFixWords each
  unsigned int* ticket;
  float* coef;  // [4C]: Q2, R2, Qs, Rs
  float *dg2, *db2, *dgs, *dbs;
  double* loss;
};

__global__ void __launch_bounds__(kThreads) loss_partial_fix_kernel(const LossParams p, const PipeIn<3> in,
                                                                    int rows_per_chunk, int cg, int rpp, int tr,
                                                                    const LossOut o) {
  constexpr int V = kLossPartialV;
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float acc[3][V] = {};
  float lsum = 0.0f;
  float A2[V], As[V], Bz[V];
  const int r0 = blockIdx.x * rows_per_chunk;
  row_pipe<3, V>(in, p.C, r0, min(p.m, r0 + rows_per_chunk), tr, gi, slot, rpp,
                 [&] { loss_affine<V>(p, gi * V, A2, As, Bz); },
                 [&](int, const __nv_bfloat16* const* s) {
                   float y2[V], ys[V], t[V];
                   ld_smem<V>(s[0], y2);
                   ld_smem<V>(s[1], ys);
                   ld_smem<V>(s[2], t);
#pragma unroll
                   for (int j = 0; j < V; ++j) {
                     const float z = fmaf(A2[j], y2[j], fmaf(As[j], ys[j], Bz[j]));
                     const float d = (z > 0.0f ? z : 0.0f) - t[j];
                     const float g = z > 0.0f ? d * p.gscale : 0.0f;
                     lsum += d * d;
                     acc[0][j] += g;
                     acc[1][j] += g * y2[j];
                     acc[2][j] += g * ys[j];
                   }
                 });
  __shared__ float lred[kThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
  if ((threadIdx.x & 31) == 0) lred[threadIdx.x >> 5] = lsum;
  cta_reduce_fix<3, V>(acc, cg, rpp, p.C, o.acc);
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.0f;
    for (int i = 0; i < kThreads / 32; ++i) s += lred[i];
    fix_red(o.acc + 3 * p.C * kFixWords, s);
  }
  if (!last_cta(o.ticket)) return;
  const int C = p.C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {  // loss_finalize_kernel's arithmetic
    const double sg = fix_take(o.acc + kFixWords * c);
    const double sgy2 = fix_take(o.acc + kFixWords * (C + c));
    const double sgys = fix_take(o.acc + kFixWords * (2 * C + c));
    const float m2 = p.st2[c], r2 = p.st2[C + c], ms = p.sts[c], rs = p.sts[C + c];
    const float A2c = p.g2[c] * r2, Asc = p.gs[c] * rs;
    const double sgx2 = static_cast<double>(r2) * (sgy2 - static_cast<double>(m2) * sg);
    const double sgxs = static_cast<double>(rs) * (sgys - static_cast<double>(ms) * sg);
    o.db2[c] = static_cast<float>(sg);
    o.dbs[c] = static_cast<float>(sg);
    o.dg2[c] = static_cast<float>(sgx2);
    o.dgs[c] = static_cast<float>(sgxs);
    const double c2 = static_cast<double>(A2c) / p.m, cs = static_cast<double>(Asc) / p.m;
    o.coef[c] = static_cast<float>(-c2 * sgx2 * r2);
    o.coef[C + c] = static_cast<float>(-c2 * (sg - sgx2 * r2 * m2));
    o.coef[2 * C + c] = static_cast<float>(-cs * sgxs * rs);
    o.coef[3 * C + c] = static_cast<float>(-cs * (sg - sgxs * rs * ms));
  }
  if (threadIdx.x == 0) *o.loss = fix_take(o.acc + kFixWords * 3 * C) / o.norm;
}

// -- dy2 / dys (loss_bwd_apply_kernel's arithmetic), staged
__global__ void __launch_bounds__(kThreads) loss_bwd_apply_pipe_kernel(const LossParams p, const PipeIn<3> in,
                                                                       const float* __restrict__ coef,
                                                                       int rows_per_chunk, int cg, int rpp, int tr,
                                                                       __nv_bfloat16* __restrict__ dy2,
                                                                       __nv_bfloat16* __restrict__ dys) {
  constexpr int V = kLossApplyV;
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  const int c0 = gi * V;
  float A2[V], As[V], Bz[V], Q2[V], R2[V], Qs[V], Rs[V];
  const int r0 = blockIdx.x * rows_per_chunk;
  row_pipe<3, V>(in, p.C, r0, min(p.m, r0 + rows_per_chunk), tr, gi, slot, rpp,
                 [&] {
                   loss_affine<V>(p, c0, A2, As, Bz);
#pragma unroll
                   for (int j = 0; j < V; ++j) {
                     Q2[j] = coef[c0 + j];
                     R2[j] = coef[p.C + c0 + j];
                     Qs[j] = coef[2 * p.C + c0 + j];
                     Rs[j] = coef[3 * p.C + c0 + j];
                   }
                 },
                 [&](int r, const __nv_bfloat16* const* s) {
                   float y2[V], ys[V], t[V], o2[V], os[V];
                   ld_smem<V>(s[0], y2);
                   ld_smem<V>(s[1], ys);
                   ld_smem<V>(s[2], t);
#pragma unroll
                   for (int j = 0; j < V; ++j) {
                     const float z = fmaf(A2[j], y2[j], fmaf(As[j], ys[j], Bz[j]));
                     const float d = (z > 0.0f ? z : 0.0f) - t[j];
                     const float g = z > 0.0f ? d * p.gscale : 0.0f;
                     o2[j] = fmaf(A2[j], g, fmaf(Q2[j], y2[j], R2[j]));
                     os[j] = fmaf(As[j], g, fmaf(Qs[j], ys[j], Rs[j]));
                   }
                   Vec<V>::store(dy2 + static_cast<size_t>(r) * p.C + c0, o2);
                   Vec<V>::store(dys + static_cast<size_t>(r) * p.C + c0, os);
                 });
}

// -- BN backward sums (sum g, sum g*y) -> coef [Q | R] and dgamma / dbeta (bn_bwd_finalize_kernel's arithmetic)
template <int V>
__global__ void __launch_bounds__(kThreads) bn_bwd_fix_partial_kernel(const PipeIn<2> in, int m, int C,
                                                                      int rows_per_chunk, int cg, int rpp, int tr,
                                                                      unsigned long long* __restrict__ acc,
                                                                      unsigned int* ticket, const float* __restrict__ st,
                                                                      const float* __restrict__ gamma,
                                                                      float* __restrict__ coef,
                                                                      float* __restrict__ dgamma,
                                                                      float* __restrict__ dbeta) {
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float a[2][V] = {};
  const int r0 = blockIdx.x * rows_per_chunk;
  row_pipe<2, V>(in, C, r0, min(m, r0 + rows_per_chunk), tr, gi, slot, rpp, [&](int, const __nv_bfloat16* const* s) {
    float fg[V], fy[V];
    ld_smem<V>(s[0], fg);
    ld_smem<V>(s[1], fy);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      a[0][j] += fg[j];
      a[1][j] += fg[j] * fy[j];
    }
  });
  cta_reduce_fix<2, V>(a, cg, rpp, C, acc);
  if (!last_cta(ticket)) return;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const double sg = fix_take(acc + kFixWords * c);
    const double sgy = fix_take(acc + kFixWords * (C + c));
    const float mu = st[c], rs = st[C + c];
    const float A = gamma[c] * rs;
    const double sgx = static_cast<double>(rs) * (sgy - static_cast<double>(mu) * sg);
    dbeta[c] = static_cast<float>(sg);
    dgamma[c] = static_cast<float>(sgx);
    const double k = static_cast<double>(A) / m;
    coef[c] = static_cast<float>(-k * sgx * rs);
    coef[C + c] = static_cast<float>(-k * (sg - sgx * rs * mu));
  }
}

// -- dy = A*g + Q*y + R (bn_bwd_apply_kernel's arithmetic), staged
template <int V>
__global__ void __launch_bounds__(kThreads) bn_bwd_apply_pipe_kernel(const PipeIn<2> in, const float* __restrict__ st,
                                                                     const float* __restrict__ gamma,
                                                                     const float* __restrict__ coef, int m, int C,
                                                                     int rows_per_chunk, int cg, int rpp, int tr,
                                                                     __nv_bfloat16* __restrict__ dy) {
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  const int c0 = gi * V;
  float A[V], Q[V], R[V];
  const int r0 = blockIdx.x * rows_per_chunk;
  row_pipe<2, V>(in, C, r0, min(m, r0 + rows_per_chunk), tr, gi, slot, rpp, [&] {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      A[j] = gamma[c0 + j] * st[C + c0 + j];
      Q[j] = coef[c0 + j];
      R[j] = coef[C + c0 + j];
    }
  }, [&](int r, const __nv_bfloat16* const* s) {
    float fg[V], fy[V], o[V];
    ld_smem<V>(s[0], fg);
    ld_smem<V>(s[1], fy);
#pragma unroll
    for (int j = 0; j < V; ++j) o[j] = fmaf(A[j], fg[j], fmaf(Q[j], fy[j], R[j]));
    Vec<V>::store(dy + static_cast<size_t>(r) * C + c0, o);
  });
}

// -- SGD with momentum + bf16 shadow:  v = fmaf(mu, v, g); w = fmaf(-lr, v, w); ws = bf16(w)
__global__ void sgd_kernel(float4* __restrict__ w, float4* __restrict__ v, const float4* __restrict__ g,
                           uint2* __restrict__ shadow, size_t n4, float lr, float mu, long long* counter) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float4 vv = v[i];
    const float4 gg = g[i];
    float4 ww = w[i];
    vv.x = fmaf(mu, vv.x, gg.x);
    vv.y = fmaf(mu, vv.y, gg.y);
    vv.z = fmaf(mu, vv.z, gg.z);
    vv.w = fmaf(mu, vv.w, gg.w);
    ww.x = fmaf(-lr, vv.x, ww.x);
    ww.y = fmaf(-lr, vv.y, ww.y);
    ww.z = fmaf(-lr, vv.z, ww.z);
    ww.w = fmaf(-lr, vv.w, ww.w);
    v[i] = vv;
    w[i] = ww;
    if (shadow != nullptr) shadow[i] = make_uint2(pack2(ww.x, ww.y), pack2(ww.z, ww.w));
  }
  if (counter != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *counter += 1;
}

// sgd_kernel + the flipped bf16 dgrad filters (FlipSet) written by the same launch: the flip launches
// that followed the update on the step's critical path are gone; values are bit-identical (same
// round-to-nearest bf16 of the same fp32 weight).  Regions whose k and c are multiples of 32 (and whose
// offset is float4-aligned) are updated by the trailing "tile" CTAs as 32x32 (k, c) tiles per tap —
// coalesced fp32 reads / writes along c, a shared-memory transpose, coalesced bf16 stores of the flipped
// copy along k — and skipped by the flat loop; any other region is scattered element by element.
struct FlipTiles {
  int count;                         // regions handled by tiles
  int region[FlipSet::kMax];         // FlipSet index of each tiled region
  int base[FlipSet::kMax + 1];       // first tile of each tiled region (prefix sums)
  // the flat loop's float4 index space: the gaps between the tiled regions, compacted
  int nseg;
  unsigned long long seg_lo[FlipSet::kMax + 1], seg_base[FlipSet::kMax + 2];
};

__device__ __forceinline__ void sgd1(float& w, float& v, float g, float lr, float mu) {
  v = fmaf(mu, v, g);
  w = fmaf(-lr, v, w);
}

__global__ void __launch_bounds__(kThreads) sgd_flip_kernel(float4* __restrict__ w, float4* __restrict__ v,
                                                           const float4* __restrict__ g, uint2* __restrict__ shadow,
                                                           float lr, float mu, long long* counter, const FlipSet fs,
                                                           const FlipTiles ft) {
  const int ntiles = ft.base[ft.count];
  if (static_cast<int>(blockIdx.x) < ntiles) {  // ---- tile part (first, so it starts early): one 32x32 (k, c) tile of one tap
    __shared__ __nv_bfloat16 tile[32][34];
    const int t = blockIdx.x;
    int q = 0;
    while (q + 1 < ft.count && t >= ft.base[q + 1]) ++q;
    const FlipRegion& R = fs.reg[ft.region[q]];
    const int taps = R.r * R.s;
    int rest = t - ft.base[q];
    const int tap = rest % taps;
    rest /= taps;
    const int cb = rest % (R.c / 32);
    const int kb = rest / (R.c / 32);
    const int rr = tap / R.s, ss = tap - rr * R.s;
    float* wf = reinterpret_cast<float*>(w);
    float* vf = reinterpret_cast<float*>(v);
    const float* gf = reinterpret_cast<const float*>(g);
    __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(shadow);
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    for (int kk = wp; kk < 32; kk += kThreads / 32) {  // row = output channel k, lanes along c
      const int k = kb * 32 + kk, c = cb * 32 + lane;
      const size_t e = R.off + (static_cast<size_t>(k) * taps + tap) * R.c + c;
      float ww = wf[e], vv = vf[e];
      sgd1(ww, vv, gf[e], lr, mu);
      wf[e] = ww;
      vf[e] = vv;
      const __nv_bfloat16 b = __float2bfloat16_rn(ww);
      sh[e] = b;
      tile[kk][lane] = b;
    }
    __syncthreads();
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(R.dst);
    const int ftap = (R.r - 1 - rr) * R.s + (R.s - 1 - ss);
    for (int cc = wp; cc < 32; cc += kThreads / 32) {  // row = input channel c, lanes along k
      const int c = cb * 32 + cc, k = kb * 32 + lane;
      dst[(static_cast<size_t>(c) * taps + ftap) * R.k + k] = tile[lane][cc];
    }
    return;
  }
  const unsigned long long total = ft.seg_base[ft.nseg];
  for (unsigned long long ci = (blockIdx.x - ntiles) * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
       ci < total; ci += static_cast<unsigned long long>(gridDim.x - ntiles) * blockDim.x) {
    int j = 0;
    while (j + 1 < ft.nseg && ci >= ft.seg_base[j + 1]) ++j;
    const size_t i = ft.seg_lo[j] + (ci - ft.seg_base[j]);
    float4 vv = v[i];
    const float4 gg = g[i];
    float4 ww = w[i];
    vv.x = fmaf(mu, vv.x, gg.x);
    vv.y = fmaf(mu, vv.y, gg.y);
    vv.z = fmaf(mu, vv.z, gg.z);
    vv.w = fmaf(mu, vv.w, gg.w);
    ww.x = fmaf(-lr, vv.x, ww.x);
    ww.y = fmaf(-lr, vv.y, ww.y);
    ww.z = fmaf(-lr, vv.z, ww.z);
    ww.w = fmaf(-lr, vv.w, ww.w);
    v[i] = vv;
    w[i] = ww;
    shadow[i] = make_uint2(pack2(ww.x, ww.y), pack2(ww.z, ww.w));
    const size_t e0 = 4 * i;
    for (int q = 0; q < fs.count; ++q) {
      const FlipRegion& R = fs.reg[q];
      const size_t len = static_cast<size_t>(R.k) * R.r * R.s * R.c;
      if (e0 + 4 <= R.off || e0 >= R.off + len) continue;
      const float f[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const size_t e = e0 + j;
        if (e < R.off || e >= R.off + len) continue;
        size_t t = e - R.off;  // [co][r][s][ci]
        const int ci = static_cast<int>(t % R.c);
        t /= R.c;
        const int ss = static_cast<int>(t % R.s);
        t /= R.s;
        const int rr = static_cast<int>(t % R.r);
        const int co = static_cast<int>(t / R.r);
        const size_t o = ((static_cast<size_t>(ci) * R.r + (R.r - 1 - rr)) * R.s + (R.s - 1 - ss)) * R.k + co;
        static_cast<__nv_bfloat16*>(R.dst)[o] = __float2bfloat16_rn(f[j]);
      }
    }
  }
  if (counter != nullptr && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *counter += 1;
}

// share_gradient + update_weight fused for a DP group: g = sum of the G members'
// gradient slabs read straight from their device memory (NVLink peer loads; CUDA IPC mappings across
// processes), added in member order on every member — so all members compute bit-identical weights
// without an NCCL allreduce — then the momentum SGD of sgd_kernel.
struct GradSources {
  const float4* g[8];
  int count;
};

__global__ void sgd_sum_kernel(float4* __restrict__ w, float4* __restrict__ v, const GradSources src,
                               uint2* __restrict__ shadow, size_t n4, float lr, float mu, long long* counter) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float4 gg = src.g[0][i];
    for (int r = 1; r < src.count; ++r) {
      const float4 o = src.g[r][i];
      gg.x = gg.x + o.x;
      gg.y = gg.y + o.y;
      gg.z = gg.z + o.z;
      gg.w = gg.w + o.w;
    }
    float4 vv = v[i];
    float4 ww = w[i];
    vv.x = fmaf(mu, vv.x, gg.x);
    vv.y = fmaf(mu, vv.y, gg.y);
    vv.z = fmaf(mu, vv.z, gg.z);
    vv.w = fmaf(mu, vv.w, gg.w);
    ww.x = fmaf(-lr, vv.x, ww.x);
    ww.y = fmaf(-lr, vv.y, ww.y);
    ww.z = fmaf(-lr, vv.z, ww.z);
    ww.w = fmaf(-lr, vv.w, ww.w);
    v[i] = vv;
    w[i] = ww;
    if (shadow != nullptr) shadow[i] = make_uint2(pack2(ww.x, ww.y), pack2(ww.z, ww.w));
  }
  if (counter != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *counter += 1;
}

// all-gather half of the DP exchange: float4 index i of a region belongs to member
// owner(i) = ((i+1)*G - 1) / n4 (slices [j*n4/G, (j+1)*n4/G)); copy every other member's updated slice
// of the master weights from its peer memory and refresh the bf16 shadow.
__global__ void dp_gather_kernel(float4* __restrict__ w, uint2* __restrict__ shadow, const GradSources peers, int me,
                                 size_t n4) {
  const unsigned long long G = static_cast<unsigned long long>(peers.count);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int owner = static_cast<int>(((i + 1) * G - 1) / n4);
    if (owner == me) continue;
    const float4 x = peers.g[owner][i];
    w[i] = x;
    if (shadow != nullptr) shadow[i] = make_uint2(pack2(x.x, x.y), pack2(x.z, x.w));
  }
}

int grid_for(long long work, int per_block = kThreads) {
  const long long b = (work + per_block - 1) / per_block;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(b, 148LL * 16)));
}

inline int ok(cudaError_t e) { return e == cudaSuccess ? PBDK_OK : PBDK_ECUDA; }

}  // namespace

GridScope::GridScope(int red_ctas, int apply_ctas, int fix_min_bytes)
    : saved_red(t_red), saved_apply(t_apply), saved_fix_min(t_fix_min) {
  t_red = red_ctas;
  t_apply = apply_ctas;
  t_fix_min = fix_min_bytes;
}
GridScope::~GridScope() {
  t_red = saved_red;
  t_apply = saved_apply;
  t_fix_min = saved_fix_min;
}

size_t reduce_workspace_floats(int m, int c, int nv) {
  int chunks = 1;
  for (int v : {4, 8}) chunks = std::max(chunks, tiling_for(m, c, v, 148 * 8).chunks);  // any target <= 8/SM
  return static_cast<size_t>(chunks) * std::max(nv, 4) * c + chunks;
}

int philox_image(void* x, int n, long long first, const long long* counter, int gb, uint32_t seed, cudaStream_t st,
                 int side, int prec) {
  const int npix = side * side;
  if (prec == 1) {
    image_split_kernel<<<grid_for(static_cast<long long>(n) * npix), kThreads, 0, st>>>(
        static_cast<float*>(x), n, npix, first, counter, gb, seed, nullptr, nullptr, 0);
    return ok(cudaGetLastError());
  }
  philox_image_kernel<<<grid_for(static_cast<long long>(n) * npix), kThreads, 0, st>>>(
      static_cast<__nv_bfloat16*>(x), n, npix, first, counter, gb, seed);
  return ok(cudaGetLastError());
}

int pack_image(const float* src, void* x, int n, cudaStream_t st, int side, int prec) {
  const long long total = static_cast<long long>(n) * side * side;
  if (prec == 1) {
    image_split_kernel<<<grid_for(total), kThreads, 0, st>>>(static_cast<float*>(x), n, side * side, 0, nullptr, 0, 0,
                                                             src, nullptr, 1);
    return ok(cudaGetLastError());
  }
  pack_image_kernel<<<grid_for(total), kThreads, 0, st>>>(src, static_cast<__nv_bfloat16*>(x), total);
  return ok(cudaGetLastError());
}

int pack_image_parity(const float* s0, const float* s1, const long long* counter, void* x, int n, cudaStream_t st,
                      int side, int prec) {
  const long long total = static_cast<long long>(n) * side * side;
  if (prec == 1) {
    image_split_kernel<<<grid_for(total), kThreads, 0, st>>>(static_cast<float*>(x), n, side * side, 0, counter, 0, 0,
                                                             s0, s1, 2);
    return ok(cudaGetLastError());
  }
  pack_image_parity_kernel<<<grid_for(total), kThreads, 0, st>>>(s0, s1, counter, static_cast<__nv_bfloat16*>(x),
                                                                 total);
  return ok(cudaGetLastError());
}

int init_uniform(void* dst, int bf16_out, int k, int r, int s, int cs, int ct, uint32_t seed, uint32_t tensor,
                 float bound, cudaStream_t st, int kt) {
  init_uniform_kernel<<<grid_for(static_cast<long long>(k) * r * s * cs), kThreads, 0, st>>>(dst, bf16_out, k, r, s,
                                                                                              cs, ct, seed, tensor,
                                                                                              bound, kt < 0 ? k : kt);
  return ok(cudaGetLastError());
}

int fill(float* dst, size_t n, float v, cudaStream_t st) {
  fill_kernel<<<grid_for(static_cast<long long>(n)), kThreads, 0, st>>>(dst, n, v);
  return ok(cudaGetLastError());
}

int bn_stats(const void* y, int m, int c, float* ws, float* mean_rstd, cudaStream_t st, int prec) {
  if (c % 8 != 0 || c / 8 > kThreads) return PBDK_EINVAL;
  const RowTiling t = tiling_for(m, c, 8);
  if (prec == 1)
    bn_stats_partial_kernel<8, 1, IoF32><<<t.chunks, kThreads, 0, st>>>(static_cast<const float*>(y), nullptr, m, c,
                                                                        t.rows_per_chunk, t.cg, t.rpp, ws);
  else
    bn_stats_partial_kernel<8, 1><<<t.chunks, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(y), nullptr, m, c,
                                                                 t.rows_per_chunk, t.cg, t.rpp, ws);
  bn_stats_finalize_kernel<1><<<(c + kFinWarps - 1) / kFinWarps, kFinWarps * 32, 0, st>>>(ws, t.chunks, c, m,
                                                                                          mean_rstd, nullptr);
  return ok(cudaGetLastError());
}

int bn_stats2(const void* y0, const void* y1, int m, int c, float* ws, float* mr0, float* mr1, cudaStream_t st,
              int prec) {
  if (c % 8 != 0 || c / 8 > kThreads) return PBDK_EINVAL;
  const RowTiling t = tiling_for(m, c, 8);
  if (prec == 1)
    bn_stats_partial_kernel<8, 2, IoF32><<<t.chunks, kThreads, 0, st>>>(
        static_cast<const float*>(y0), static_cast<const float*>(y1), m, c, t.rows_per_chunk, t.cg, t.rpp, ws);
  else
    bn_stats_partial_kernel<8, 2><<<t.chunks, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(y0),
                                                                 static_cast<const __nv_bfloat16*>(y1), m, c,
                                                                 t.rows_per_chunk, t.cg, t.rpp, ws);
  bn_stats_finalize_kernel<2><<<(2 * c + kFinWarps - 1) / kFinWarps, kFinWarps * 32, 0, st>>>(ws, t.chunks, c, m, mr0,
                                                                                              mr1);
  return ok(cudaGetLastError());
}

int bn_apply_relu(const void* y, const float* mean_rstd, const float* gamma, const float* beta, void* a, int m, int c,
                  cudaStream_t st, int prec) {
  if (c % 8 != 0 || c / 8 > kThreads) return PBDK_EINVAL;
  const RowTiling t = tiling_for(m, c, 8);
  if (prec == 1) {  // fp32 in, split fp32 out (the next convolution's operand)
    bn_apply_relu_kernel<8, IoF32, IoSplit><<<apply_grid(m, t.rpp), kThreads, 0, st>>>(
        static_cast<const float*>(y), mean_rstd, gamma, beta, static_cast<float*>(a), m, c, t.cg, t.rpp);
    return ok(cudaGetLastError());
  }
  bn_apply_relu_kernel<8><<<apply_grid(m, t.rpp), kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(y), mean_rstd,
                                                                     gamma, beta, static_cast<__nv_bfloat16*>(a), m, c,
                                                                     t.cg, t.rpp);
  return ok(cudaGetLastError());
}

int mse_bn_loss(const MseArgs& a, cudaStream_t st) {
  if (a.c % 8 != 0 || a.c / kLossApplyV > kThreads) return PBDK_EINVAL;
  LossParams p{a.y2, a.ysc, a.t, a.stats2, a.statssc, a.gamma2, a.beta2, a.gammasc, a.betasc,
               a.m, a.c, a.gscale};
  const RowTiling t = tiling_for(a.m, a.c, kLossPartialV, kLossChunks);
  float* partial = a.ws;
  float* loss_partial = a.ws + static_cast<size_t>(t.chunks) * 3 * a.c;
  if (a.prec == 1)  // y2 / ysc plain fp32, target split fp32
    loss_partial_kernel<IoF32, IoSplit><<<t.chunks, kThreads, 0, st>>>(p, t.rows_per_chunk, t.cg, t.rpp, partial,
                                                                       loss_partial);
  else
    loss_partial_kernel<<<t.chunks, kThreads, 0, st>>>(p, t.rows_per_chunk, t.cg, t.rpp, partial, loss_partial);
  loss_finalize_kernel<<<(a.c + kFinWarps - 1) / kFinWarps + 1, kFinWarps * 32, 0, st>>>(
      p, partial, loss_partial, t.chunks, a.norm, a.red, a.dgamma2, a.dbeta2, a.dgammasc, a.dbetasc, a.loss);
  const RowTiling ta = tiling_for(a.m, a.c, kLossApplyV);
  if (a.prec == 1)  // dy2 / dysc split fp32 (dgrad / wgrad operands)
    loss_bwd_apply_kernel<IoF32, IoSplit, IoSplit><<<apply_grid(a.m, ta.rpp), kThreads, 0, st>>>(
        p, a.red, ta.cg, ta.rpp, static_cast<float*>(a.dy2), static_cast<float*>(a.dysc));
  else
    loss_bwd_apply_kernel<<<apply_grid(a.m, ta.rpp), kThreads, 0, st>>>(p, a.red, ta.cg, ta.rpp,
                                                                        static_cast<__nv_bfloat16*>(a.dy2),
                                                                        static_cast<__nv_bfloat16*>(a.dysc));
  return ok(cudaGetLastError());
}

int bn_bwd(const void* g, const void* y, const float* mean_rstd, const float* gamma, int m, int c, float* ws,
           float* red, float* dgamma, float* dbeta, void* dy, cudaStream_t st, int prec) {
  if (c % 8 != 0 || c / 8 > kThreads) return PBDK_EINVAL;
  const RowTiling t = tiling_for(m, c, 8);
  if (prec == 1)
    bn_bwd_partial_kernel<8, IoF32><<<t.chunks, kThreads, 0, st>>>(static_cast<const float*>(g),
                                                                   static_cast<const float*>(y), m, c,
                                                                   t.rows_per_chunk, t.cg, t.rpp, ws);
  else
    bn_bwd_partial_kernel<8><<<t.chunks, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(g),
                                                            static_cast<const __nv_bfloat16*>(y), m, c,
                                                            t.rows_per_chunk, t.cg, t.rpp, ws);
  bn_bwd_finalize_kernel<<<(c + kFinWarps - 1) / kFinWarps, kFinWarps * 32, 0, st>>>(ws, t.chunks, c, m, mean_rstd,
                                                                                    gamma, red, dgamma, dbeta);
  if (prec == 1) {  // dy split fp32 (the wgrad operand)
    bn_bwd_apply_kernel<8, IoF32, IoSplit><<<apply_grid(m, t.rpp), kThreads, 0, st>>>(
        static_cast<const float*>(g), static_cast<const float*>(y), mean_rstd, gamma, red, m, c, t.cg, t.rpp,
        static_cast<float*>(dy));
    return ok(cudaGetLastError());
  }
  bn_bwd_apply_kernel<8><<<apply_grid(m, t.rpp), kThreads, 0, st>>>(
      static_cast<const __nv_bfloat16*>(g), static_cast<const __nv_bfloat16*>(y), mean_rstd, gamma, red, m, c, t.cg,
      t.rpp, static_cast<__nv_bfloat16*>(dy));
  return ok(cudaGetLastError());
}

// ---- self-finalizing reductions (bf16 rows)
size_t fix_acc_words(int c) { return (static_cast<size_t>(4) * c + 1) * kFixWords; }  // max over the four reductions

// grid of an elementwise staged pass: contiguous row chunks over apply_cap() CTAs (two per SM in the
// ResNet step's GridScope; each keeps up to 96 KB of loads in flight)
int apply_pipe_div() {  // PBDK_APPLY_PIPE_DIV: staged applies use apply_cap() / div CTAs (A/B runs)
  static const int d = env_int("PBDK_APPLY_PIPE_DIV", 2);
  return std::max(1, d);
}
bool apply_pipe() {  // PBDK_APPLY_PIPE=0: the register-loop apply kernels (A/B runs)
  static const bool on = env_int("PBDK_APPLY_PIPE", 1) != 0;
  return on;
}
// Staged passes over small [M][C] streams: a CTA that streams only a few tens of KB is latency bound
// (prologue, pipeline fill, reduction tail) while it holds an SM's shared memory against the other
// student streams' convs, so the grid is also capped at one CTA per `min_bytes` of input.  The
// cap is a function of the shape only, so a block's numerics stay independent of its placement.
int cap_chunks(int target, long long bytes, int min_bytes) {
  if (min_bytes <= 0) return target;
  const long long need = (bytes + min_bytes - 1) / min_bytes;
  return static_cast<int>(std::max(1LL, std::min<long long>(target, need)));
}
int fix_min_bytes() {  // PBDK_FIX_MIN_BYTES: reduction passes (CIFAR step 0.891 -> 0.873 ms at 256 KB; 128 KB-512 KB
                       // within 1 %, 1 MB 0.94 ms; r02_ab_minbytes.txt)
  static const int b = env_int("PBDK_FIX_MIN_BYTES", -1);  // experiments: 0 = no cap
  return b >= 0 ? b : (t_fix_min > 0 ? t_fix_min : 256 << 10);
}
int apply_min_bytes() {  // PBDK_APPLY_MIN_BYTES: elementwise passes (off: 256 KB measured neutral)
  static const int b = env_int("PBDK_APPLY_MIN_BYTES", 0);
  return b;
}
RowTiling fix_tiling(int m, int c, int v, int nin) {
  return tiling_for(m, c, v, cap_chunks(red_target(), 2LL * m * c * nin, fix_min_bytes()));
}
RowTiling apply_tiling(int m, int c, int v, int nin) {
  return tiling_for(m, c, v,
                    cap_chunks(std::max(1, apply_cap() / apply_pipe_div()), 2LL * m * c * nin, apply_min_bytes()));
}

bool pipe_pdl() {  // PBD_PDL=0 / PBDK_PIPE_PDL=0: plain launches (experiments build, A/B runs)
  static const bool on = pbd::pdl_enabled() && env_int("PBDK_PIPE_PDL", 1) != 0;
  return on;
}

template <class K, class... Args>
cudaError_t launch_pipe(K kernel, int grid, size_t smem, cudaStream_t st, Args... args) {
  constexpr size_t kMax = 2 * kPipeStages * kPipeStageBytes;  // tiles rounded up to rpp rows stay below
  if (smem > kMax) return cudaErrorInvalidValue;
  static bool attr_set = false;  // per instantiation: opt in to > 48 KB of dynamic shared memory once
  if (!attr_set) {
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(kMax));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  // programmatic dependent launch: the pass's CTAs are scheduled while the previous kernel of the stream
  // drains; row_pipe waits (griddepcontrol.wait) before its first global access
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pipe_pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

int bn_stats_fix(const void* y0, const void* y1, int m, int c, FixScratch fx, float* mr0, float* mr1,
                 cudaStream_t st) {
  if (c % 8 != 0 || c / 8 > kThreads) return PBDK_EINVAL;
  const int nin = y1 != nullptr ? 2 : 1;
  const RowTiling t = fix_tiling(m, c, 8, nin);
  const int tr = pipe_tile_rows(nin, c, t.rpp);
  const size_t smem = pipe_smem(nin, c, tr);
  if (y1 != nullptr)
    return ok(launch_pipe(bn_stats_fix_kernel<8, 2>, t.chunks, smem, st,
                          PipeIn<2>{{static_cast<const __nv_bfloat16*>(y0), static_cast<const __nv_bfloat16*>(y1)}}, m,
                          c, t.rows_per_chunk, t.cg, t.rpp, tr, fx.acc, fx.ticket, mr0, mr1));
  return ok(launch_pipe(bn_stats_fix_kernel<8, 1>, t.chunks, smem, st,
                        PipeIn<1>{{static_cast<const __nv_bfloat16*>(y0)}}, m, c, t.rows_per_chunk, t.cg, t.rpp, tr,
                        fx.acc, fx.ticket, mr0, static_cast<float*>(nullptr)));
}

int bn_apply_relu_fix(const void* y, const float* mean_rstd, const float* gamma, const float* beta, void* a, int m,
                      int c, cudaStream_t st) {
  if (c % 8 != 0 || c / 8 > kThreads) return PBDK_EINVAL;
  if (!apply_pipe()) return bn_apply_relu(y, mean_rstd, gamma, beta, a, m, c, st);
  const RowTiling t = apply_tiling(m, c, 8, 2);
  const int tr = pipe_tile_rows(1, c, t.rpp);
  return ok(launch_pipe(bn_apply_relu_pipe_kernel<8>, t.chunks, pipe_smem(1, c, tr), st,
                        PipeIn<1>{{static_cast<const __nv_bfloat16*>(y)}}, mean_rstd, gamma, beta,
                        static_cast<__nv_bfloat16*>(a), m, c, t.rows_per_chunk, t.cg, t.rpp, tr));
}

int mse_bn_loss_fix(const MseArgs& a, FixScratch fx, cudaStream_t st) {
  if (a.c % 8 != 0 || a.c / kLossApplyV > kThreads || a.prec != 0) return PBDK_EINVAL;
  LossParams p{a.y2, a.ysc, a.t, a.stats2, a.statssc, a.gamma2, a.beta2, a.gammasc, a.betasc, a.m, a.c, a.gscale};
  const PipeIn<3> in{{static_cast<const __nv_bfloat16*>(a.y2), static_cast<const __nv_bfloat16*>(a.ysc),
                      static_cast<const __nv_bfloat16*>(a.t)}};
  const RowTiling t = fix_tiling(a.m, a.c, kLossPartialV, 3);
  const int tr = pipe_tile_rows(3, a.c, t.rpp);
  const LossOut o{a.norm, fx.acc, fx.ticket, a.red, a.dgamma2, a.dbeta2, a.dgammasc, a.dbetasc, a.loss};
  cudaError_t e = launch_pipe(loss_partial_fix_kernel, t.chunks, pipe_smem(3, a.c, tr), st, p, in, t.rows_per_chunk,
                              t.cg, t.rpp, tr, o);
  if (e != cudaSuccess) return PBDK_ECUDA;
  if (!apply_pipe()) {
    const RowTiling ta = tiling_for(a.m, a.c, kLossApplyV);
    loss_bwd_apply_kernel<<<apply_grid(a.m, ta.rpp), kThreads, 0, st>>>(p, a.red, ta.cg, ta.rpp,
                                                                        static_cast<__nv_bfloat16*>(a.dy2),
                                                                        static_cast<__nv_bfloat16*>(a.dysc));
    return ok(cudaGetLastError());
  }
  const RowTiling ta = apply_tiling(a.m, a.c, kLossApplyV, 5);
  const int tra = pipe_tile_rows(3, a.c, ta.rpp);
  e = launch_pipe(loss_bwd_apply_pipe_kernel, ta.chunks, pipe_smem(3, a.c, tra), st, p, in,
                  static_cast<const float*>(a.red), ta.rows_per_chunk, ta.cg, ta.rpp, tra,
                  static_cast<__nv_bfloat16*>(a.dy2), static_cast<__nv_bfloat16*>(a.dysc));
  return ok(e);
}

int bn_bwd_fix(const void* g, const void* y, const float* mean_rstd, const float* gamma, int m, int c, FixScratch fx,
               float* red, float* dgamma, float* dbeta, void* dy, cudaStream_t st) {
  if (c % 8 != 0 || c / 8 > kThreads) return PBDK_EINVAL;
  const PipeIn<2> in{{static_cast<const __nv_bfloat16*>(g), static_cast<const __nv_bfloat16*>(y)}};
  const RowTiling t = fix_tiling(m, c, 8, 2);
  const int tr = pipe_tile_rows(2, c, t.rpp);
  cudaError_t e = launch_pipe(bn_bwd_fix_partial_kernel<8>, t.chunks, pipe_smem(2, c, tr), st, in, m, c,
                              t.rows_per_chunk, t.cg, t.rpp, tr, fx.acc, fx.ticket, mean_rstd, gamma, red, dgamma,
                              dbeta);
  if (e != cudaSuccess) return PBDK_ECUDA;
  if (!apply_pipe()) {
    bn_bwd_apply_kernel<8><<<apply_grid(m, t.rpp), kThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(g), static_cast<const __nv_bfloat16*>(y), mean_rstd, gamma, red, m, c, t.cg,
        t.rpp, static_cast<__nv_bfloat16*>(dy));
    return ok(cudaGetLastError());
  }
  const RowTiling ta = apply_tiling(m, c, 8, 3);
  const int tra = pipe_tile_rows(2, c, ta.rpp);
  e = launch_pipe(bn_bwd_apply_pipe_kernel<8>, ta.chunks, pipe_smem(2, c, tra), st, in, mean_rstd, gamma,
                  static_cast<const float*>(red), m, c, ta.rows_per_chunk, ta.cg, ta.rpp, tra,
                  static_cast<__nv_bfloat16*>(dy));
  return ok(e);
}

int sgd_momentum(float* w, float* v, const float* g, void* shadow, size_t n, float lr, float mu, long long* counter,
                 cudaStream_t st) {
  if (n % 4 != 0) return PBDK_EINVAL;
  sgd_kernel<<<grid_for(static_cast<long long>(n / 4)), kThreads, 0, st>>>(
      reinterpret_cast<float4*>(w), reinterpret_cast<float4*>(v), reinterpret_cast<const float4*>(g),
      static_cast<uint2*>(shadow), n / 4, lr, mu, counter);
  return ok(cudaGetLastError());
}

int sgd_momentum_flip(float* w, float* v, const float* g, void* shadow, size_t n, float lr, float mu,
                      long long* counter, const FlipSet& flips, cudaStream_t st) {
  if (n % 4 != 0 || shadow == nullptr || flips.count < 0 || flips.count > FlipSet::kMax) return PBDK_EINVAL;
  for (int q = 0; q < flips.count; ++q) {
    const FlipRegion& R = flips.reg[q];
    if (R.dst == nullptr || R.k < 1 || R.r < 1 || R.s < 1 || R.c < 1 ||
        R.off + static_cast<size_t>(R.k) * R.r * R.s * R.c > n)
      return PBDK_EINVAL;
  }
  // tiled regions (k, c multiples of 32, float4-aligned offset) first, then the scattered ones; the
  // flat loop skips the tiled regions' float4 ranges (their length is a multiple of 4)
  FlipTiles ft{};
  FlipSet packed;
  int tiles = 0;
  std::pair<size_t, size_t> cut[FlipSet::kMax];  // tiled float4 ranges
  for (int pass = 0; pass < 2; ++pass)
    for (int q = 0; q < flips.count; ++q) {
      const FlipRegion& R = flips.reg[q];
      const bool tiled = R.k % 32 == 0 && R.c % 32 == 0 && R.off % 4 == 0;
      if (tiled != (pass == 0)) continue;
      if (tiled) {
        const size_t len = static_cast<size_t>(R.k) * R.r * R.s * R.c;
        cut[ft.count] = {R.off / 4, (R.off + len) / 4};
        ft.region[ft.count] = packed.count;
        ft.base[ft.count] = tiles;
        tiles += R.r * R.s * (R.k / 32) * (R.c / 32);
        ++ft.count;
      }
      packed.reg[packed.count++] = R;
    }
  ft.base[ft.count] = tiles;
  for (int a = 1; a < ft.count; ++a)  // sort the (at most kMax) ranges by offset
    for (int b = a; b > 0 && cut[b].first < cut[b - 1].first; --b) std::swap(cut[b], cut[b - 1]);
  size_t at = 0, base = 0;
  for (int u = 0; u <= ft.count; ++u) {  // gaps [at, next cut) and the tail [at, n4)
    const size_t end = u < ft.count ? cut[u].first : n / 4;
    if (end < at) return PBDK_EINVAL;  // overlapping regions
    if (end > at) {
      ft.seg_lo[ft.nseg] = at;
      ft.seg_base[ft.nseg] = base;
      base += end - at;
      ++ft.nseg;
    }
    if (u < ft.count) at = cut[u].second;
  }
  if (ft.nseg == 0) ft.seg_lo[ft.nseg++] = 0;  // empty flat space: one empty segment
  ft.seg_base[ft.nseg] = base;
  const int flat = grid_for(static_cast<long long>(std::max<size_t>(base, 1)));
  sgd_flip_kernel<<<tiles + flat, kThreads, 0, st>>>(
      reinterpret_cast<float4*>(w), reinterpret_cast<float4*>(v), reinterpret_cast<const float4*>(g),
      static_cast<uint2*>(shadow), lr, mu, counter, packed, ft);
  return ok(cudaGetLastError());
}

int dp_gather(float* w, void* shadow, const float* const* peer_w, int count, int me, size_t n, cudaStream_t st) {
  if (n % 4 != 0 || count < 1 || count > 8 || me < 0 || me >= count) return PBDK_EINVAL;
  GradSources src{};
  for (int r = 0; r < count; ++r) src.g[r] = reinterpret_cast<const float4*>(peer_w[r]);
  src.count = count;
  dp_gather_kernel<<<grid_for(static_cast<long long>(n / 4)), kThreads, 0, st>>>(
      reinterpret_cast<float4*>(w), static_cast<uint2*>(shadow), src, me, n / 4);
  return ok(cudaGetLastError());
}

int sgd_momentum_sum(float* w, float* v, const float* const* g, int count, void* shadow, size_t n, float lr, float mu,
                     long long* counter, cudaStream_t st) {
  if (n % 4 != 0 || count < 1 || count > 8) return PBDK_EINVAL;
  GradSources src{};
  for (int r = 0; r < count; ++r) src.g[r] = reinterpret_cast<const float4*>(g[r]);
  src.count = count;
  sgd_sum_kernel<<<grid_for(static_cast<long long>(n / 4)), kThreads, 0, st>>>(
      reinterpret_cast<float4*>(w), reinterpret_cast<float4*>(v), src, static_cast<uint2*>(shadow), n / 4, lr, mu,
      counter);
  return ok(cudaGetLastError());
}

}  // namespace pbdk

// ------------------------------------------------------------------ C ABI
extern "C" {

int pbdk_philox_image(void* x, int n, long long first_sample, const long long* step_counter, int global_batch,
                      uint32_t seed, void* stream) {
  if (x == nullptr || n < 0) return PBDK_EINVAL;
  return pbdk::philox_image(x, n, first_sample, step_counter, global_batch, seed, static_cast<cudaStream_t>(stream));
}

int pbdk_pack_image(const float* src, void* x, int n, void* stream) {
  if (src == nullptr || x == nullptr || n < 0) return PBDK_EINVAL;
  return pbdk::pack_image(src, x, n, static_cast<cudaStream_t>(stream));
}

int pbdk_init_uniform(void* dst, int bf16_out, int k, int r, int s, int c_stored, int c_true, uint32_t seed,
                      uint32_t tensor_id, float bound, void* stream) {
  if (dst == nullptr || c_true > c_stored) return PBDK_EINVAL;
  return pbdk::init_uniform(dst, bf16_out, k, r, s, c_stored, c_true, seed, tensor_id, bound,
                            static_cast<cudaStream_t>(stream));
}

size_t pbdk_reduce_workspace_bytes(int m, int c) { return pbdk::reduce_workspace_floats(m, c, 3) * sizeof(float); }

int pbdk_bn_stats(const void* y, int m, int c, void* workspace, float* mean_rstd, void* stream) {
  return pbdk::bn_stats(y, m, c, static_cast<float*>(workspace), mean_rstd, static_cast<cudaStream_t>(stream));
}

int pbdk_bn_apply_relu(const void* y, const float* mean_rstd, const float* gamma, const float* beta, void* a, int m,
                       int c, void* stream) {
  return pbdk::bn_apply_relu(y, mean_rstd, gamma, beta, a, m, c, static_cast<cudaStream_t>(stream));
}

int pbdk_mse_bn_loss(const pbdk_mse_args* a, void* stream) {
  if (a == nullptr) return PBDK_EINVAL;
  pbdk::MseArgs m{a->y2, a->ysc, a->t, a->stats2, a->statssc, a->gamma2, a->beta2, a->gammasc, a->betasc,
                  a->m, a->c, a->gscale, a->norm, static_cast<float*>(a->workspace), a->red, a->dgamma2, a->dbeta2,
                  a->dgammasc, a->dbetasc, a->loss, a->dy2, a->dysc};
  return pbdk::mse_bn_loss(m, static_cast<cudaStream_t>(stream));
}

int pbdk_bn_bwd(const void* g, const void* y, const float* mean_rstd, const float* gamma, int m, int c,
                void* workspace, float* red, float* dgamma, float* dbeta, void* dy, void* stream) {
  return pbdk::bn_bwd(g, y, mean_rstd, gamma, m, c, static_cast<float*>(workspace), red, dgamma, dbeta, dy,
                      static_cast<cudaStream_t>(stream));
}

int pbdk_sgd_momentum(float* w, float* v, const float* g, void* w_bf16, size_t n, float lr, float momentum,
                      long long* step_counter, void* stream) {
  if (w == nullptr || v == nullptr || g == nullptr) return PBDK_EINVAL;
  return pbdk::sgd_momentum(w, v, g, w_bf16, n, lr, momentum, step_counter, static_cast<cudaStream_t>(stream));
}

int pbdk_sgd_momentum_flip(float* w, float* v, const float* g, void* w_bf16, size_t n, float lr, float momentum,
                           long long* step_counter, const pbdk_flip_region* regions, int count, void* stream) {
  if (w == nullptr || v == nullptr || g == nullptr || (count > 0 && regions == nullptr) || count < 0 ||
      count > pbdk::FlipSet::kMax)
    return PBDK_EINVAL;
  pbdk::FlipSet fs;
  for (int i = 0; i < count; ++i)
    fs.reg[fs.count++] = pbdk::FlipRegion{regions[i].off, regions[i].k, regions[i].r, regions[i].s, regions[i].c,
                                          regions[i].dst};
  return pbdk::sgd_momentum_flip(w, v, g, w_bf16, n, lr, momentum, step_counter, fs,
                                 static_cast<cudaStream_t>(stream));
}

}  // extern "C"
