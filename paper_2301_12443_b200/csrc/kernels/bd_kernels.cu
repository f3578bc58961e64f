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

#include "bd_kernels.hpp"
#include "pbdk.h"

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
__global__ void philox_image_kernel(__nv_bfloat16* __restrict__ x, int n, long long first, const long long* counter,
                                    int global_batch, uint32_t seed) {
  const long long base = first + (counter != nullptr ? (*counter) * global_batch : 0);
  const int total = n * 1024;
  for (int pix = blockIdx.x * blockDim.x + threadIdx.x; pix < total; pix += gridDim.x * blockDim.x) {
    const int i = pix / 1024;
    const int hw = pix - i * 1024;
    float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const unsigned long long idx =
          static_cast<unsigned long long>(base + i) * 3072ull + static_cast<unsigned long long>(hw * 3 + c);
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

__global__ void pack_image_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ x, int n) {
  const int total = n * 1024;
  for (int pix = blockIdx.x * blockDim.x + threadIdx.x; pix < total; pix += gridDim.x * blockDim.x) {
    float v[8] = {src[pix * 3], src[pix * 3 + 1], src[pix * 3 + 2], 0, 0, 0, 0, 0};
    const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint4* dst = reinterpret_cast<uint4*>(x + static_cast<size_t>(pix) * 16);
    dst[0] = pack8(v);
    dst[1] = pack8(z);
  }
}

// dst[k][r][s][c_stored] = c < c_true ? U(-1,1)[counter=((k*r+..)*c_true+c, tensor)] * bound : 0
__global__ void init_uniform_kernel(void* dst, int bf16_out, int k, int r, int s, int cs, int ct, uint32_t seed,
                                    uint32_t tensor, float bound) {
  const long long total = static_cast<long long>(k) * r * s * cs;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cs);
    const long long krs = i / cs;
    float v = 0.0f;
    if (c < ct) {
      const long long j = krs * ct + c;
      uint32_t o;
      philox10(static_cast<uint32_t>(j), tensor, 0u, 0u, seed, 0xB200B200u, o);
      v = sym_unit(o) * bound;
    }
    if (bf16_out)
      static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
    else
      static_cast<float*>(dst)[i] = v;
  }
}

__global__ void fill_kernel(float* __restrict__ dst, size_t n, float v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = v;
}

// ------------------------------------------------------------------ reductions
// Geometry of a row-chunked reduction over [M][C]: cg = C/8 channel groups per
// row, rpp = 256/cg rows per pass; CTA b covers rows [b*rows_per_chunk, ...).

struct RowTiling {
  int cg, rpp, chunks, rows_per_chunk;
};

RowTiling tiling_for(int m, int c) {
  RowTiling t;
  t.cg = c / 8;
  t.rpp = std::max(1, kThreads / t.cg);
  const int target = 148 * 4;
  int rpc = std::max(t.rpp, (m + target - 1) / target);
  rpc = (rpc + t.rpp - 1) / t.rpp * t.rpp;
  t.rows_per_chunk = rpc;
  t.chunks = (m + rpc - 1) / rpc;
  return t;
}

// CTA-level fixed-order reduction of NV*8 floats per thread into partial[chunk][NV][C].
template <int NV>
__device__ void cta_reduce_store(float (&acc)[NV][8], int cg, int rpp, int C, float* __restrict__ partial) {
  __shared__ float sm[kThreads * NV * 8];
  const int t = threadIdx.x;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int j = 0; j < 8; ++j) sm[(v * 8 + j) * kThreads + t] = acc[v][j];
  __syncthreads();
  // thread t < cg*8*NV reduces one (v, channel) over the rpp row slots in order
  for (int o = t; o < NV * cg * 8; o += kThreads) {
    const int v = o / (cg * 8);
    const int rem = o - v * cg * 8;
    const int g = rem / 8;
    const int j = rem - g * 8;
    float s = 0.0f;
    for (int r = 0; r < rpp; ++r) s += sm[(v * 8 + j) * kThreads + r * cg + g];
    partial[(static_cast<size_t>(blockIdx.x) * NV + v) * C + g * 8 + j] = s;
  }
}

// Fixed-order parallel sum of partial[chunk][NV][C] over chunks for 32 consecutive
// (v, c) outputs per CTA: warp w sums chunks [w*per, (w+1)*per) (lanes = 32
// consecutive outputs, coalesced), then the 8 warp partials are added in warp order.
// Deterministic for a given (chunks, C).  Returns the double sum in `out` for lane
// outputs o = blockIdx.x*32 + lane (valid when o < NV*C), visible to warp 0.
constexpr int kFinWarps = 8;

template <int NV>
__device__ __forceinline__ double sum_over_chunks(const float* __restrict__ partial, int chunks, int C, int o) {
  __shared__ double sm[kFinWarps][32];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double s = 0.0;
  if (o < NV * C) {
    const int v = o / C;
    const int c = o - v * C;
    const int per = (chunks + kFinWarps - 1) / kFinWarps;
    const int b0 = warp * per;
    const int b1 = min(chunks, b0 + per);
    for (int b = b0; b < b1; ++b) s += partial[(static_cast<size_t>(b) * NV + v) * C + c];
  }
  sm[warp][lane] = s;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
#pragma unroll
    for (int w = 0; w < kFinWarps; ++w) t += sm[w][lane];
  }
  return t;
}

// fixed-order sum of n floats by one CTA of kFinWarps*32 threads
__device__ __forceinline__ double cta_sum(const float* __restrict__ v, int n) {
  __shared__ double sm[kFinWarps * 32];
  double s = 0.0;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  const int b1 = min(n, b0 + per);
  for (int i = b0; i < b1; ++i) s += v[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < static_cast<int>(blockDim.x); ++i) t += sm[i];
  return t;
}

// -- BN statistics
__global__ void bn_stats_partial_kernel(const __nv_bfloat16* __restrict__ y, int m, int C, int rows_per_chunk, int cg,
                                        int rpp, float* __restrict__ partial) {
  const int g = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float acc[2][8] = {};
  if (slot < rpp) {
    const int r0 = blockIdx.x * rows_per_chunk;
    const int r1 = min(m, r0 + rows_per_chunk);
    for (int r = r0 + slot; r < r1; r += rpp) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(y + static_cast<size_t>(r) * C + g * 8), f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc[0][j] += f[j];
        acc[1][j] += f[j] * f[j];
      }
    }
  }
  cta_reduce_store<2>(acc, cg, rpp, C, partial);
}

// grid: ceil(C/32) CTAs of kFinWarps*32 threads; the (s1, s2) pair of channel c is
// summed by two independent fixed-order passes (v = 0 and v = 1).
__global__ void bn_stats_finalize_kernel(const float* __restrict__ partial, int chunks, int C, int m,
                                         float* __restrict__ mean_rstd) {
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const double s1 = sum_over_chunks<2>(partial, chunks, C, c);
  __syncthreads();
  const double s2 = sum_over_chunks<2>(partial, chunks, C, C + c);
  if ((threadIdx.x >> 5) == 0 && c < C) {
    const double mu = s1 / static_cast<double>(m);
    const double var = s2 / static_cast<double>(m) - mu * mu;
    mean_rstd[c] = static_cast<float>(mu);
    mean_rstd[C + c] = 1.0f / sqrtf(static_cast<float>(var) + 1e-5f);
  }
}

// -- BN apply + ReLU: a = bf16(relu(fmaf(gamma, (y-mu)*rstd, beta)))
__global__ void bn_apply_relu_kernel(const __nv_bfloat16* __restrict__ y, const float* __restrict__ mean_rstd,
                                     const float* __restrict__ gamma, const float* __restrict__ beta,
                                     __nv_bfloat16* __restrict__ a, int m, int C) {
  const int cg = C / 8;
  const long long total = static_cast<long long>(m) * cg;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c0 = static_cast<int>(i % cg) * 8;
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(y)[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float xh = (f[j] - mean_rstd[c0 + j]) * mean_rstd[C + c0 + j];
      const float z = fmaf(gamma[c0 + j], xh, beta[c0 + j]);
      f[j] = z > 0.0f ? z : 0.0f;
    }
    reinterpret_cast<uint4*>(a)[i] = pack8(f);
  }
}

// -- fused distillation loss: s = relu(BN2(y2) + BNsc(ysc)); L += (s-t)^2; g = [z>0] (s-t)*gscale
struct LossParams {
  const __nv_bfloat16* y2;
  const __nv_bfloat16* ys;
  const __nv_bfloat16* t;
  const float* st2;  // mean[C], rstd[C]
  const float* sts;
  const float* g2;
  const float* b2;
  const float* gs;
  const float* bs;
  int m, C;
  float gscale;
};

__device__ __forceinline__ void loss_point(const LossParams& p, size_t off, int c0, float (&g)[8], float (&xh2)[8],
                                           float (&xhs)[8], float (&d)[8]) {
  float fy2[8], fys[8], ft[8];
  unpack8(*reinterpret_cast<const uint4*>(p.y2 + off), fy2);
  unpack8(*reinterpret_cast<const uint4*>(p.ys + off), fys);
  unpack8(*reinterpret_cast<const uint4*>(p.t + off), ft);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = c0 + j;
    xh2[j] = (fy2[j] - p.st2[c]) * p.st2[p.C + c];
    xhs[j] = (fys[j] - p.sts[c]) * p.sts[p.C + c];
    const float z = fmaf(p.g2[c], xh2[j], p.b2[c]) + fmaf(p.gs[c], xhs[j], p.bs[c]);
    const float sv = z > 0.0f ? z : 0.0f;
    d[j] = sv - ft[j];
    g[j] = z > 0.0f ? d[j] * p.gscale : 0.0f;
  }
}

__global__ void loss_partial_kernel(const LossParams p, int rows_per_chunk, int cg, int rpp,
                                    float* __restrict__ partial, float* __restrict__ loss_partial) {
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float acc[3][8] = {};
  float lsum = 0.0f;
  if (slot < rpp) {
    const int r0 = blockIdx.x * rows_per_chunk;
    const int r1 = min(p.m, r0 + rows_per_chunk);
    for (int r = r0 + slot; r < r1; r += rpp) {
      float g[8], xh2[8], xhs[8], d[8];
      loss_point(p, static_cast<size_t>(r) * p.C + gi * 8, gi * 8, g, xh2, xhs, d);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        lsum += d[j] * d[j];
        acc[0][j] += g[j];
        acc[1][j] += g[j] * xh2[j];
        acc[2][j] += g[j] * xhs[j];
      }
    }
  }
  // loss: block reduction in fixed order
  __shared__ float lred[kThreads];
  lred[threadIdx.x] = lsum;
  cta_reduce_store<3>(acc, cg, rpp, p.C, partial);
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.0f;
    for (int i = 0; i < kThreads; ++i) s += lred[i];
    loss_partial[blockIdx.x] = s;
  }
}

// red (double [3C]) -> grads of gamma2/beta2/gammasc/betasc, float copies; the last
// CTA (blockIdx.x == gridDim.x-1, beyond the channel CTAs) sums the loss partials.
__global__ void loss_finalize_kernel(const float* __restrict__ partial, const float* __restrict__ loss_partial,
                                     int chunks, int C, double norm, float* __restrict__ red_f,
                                     float* __restrict__ dg2, float* __restrict__ db2, float* __restrict__ dgs,
                                     float* __restrict__ dbs, double* __restrict__ loss_out) {
  if (blockIdx.x == gridDim.x - 1) {
    const double l = cta_sum(loss_partial, chunks);
    if (threadIdx.x == 0) *loss_out = l / norm;
    return;
  }
  const int o = blockIdx.x * 32 + (threadIdx.x & 31);  // o in [0, 3C)
  const double sv = sum_over_chunks<3>(partial, chunks, C, o);
  if ((threadIdx.x >> 5) == 0 && o < 3 * C) {
    const int v = o / C;
    const int c = o - v * C;
    const float f = static_cast<float>(sv);
    red_f[o] = f;
    if (v == 0) {
      db2[c] = f;
      dbs[c] = f;
    } else if (v == 1) {
      dg2[c] = f;
    } else {
      dgs[c] = f;
    }
  }
}

__global__ void loss_bwd_apply_kernel(const LossParams p, const float* __restrict__ red_f,
                                      __nv_bfloat16* __restrict__ dy2, __nv_bfloat16* __restrict__ dys) {
  const int cg = p.C / 8;
  const long long total = static_cast<long long>(p.m) * cg;
  const float mf = static_cast<float>(p.m);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c0 = static_cast<int>(i % cg) * 8;
    float g[8], xh2[8], xhs[8], d[8], o2[8], os[8];
    loss_point(p, static_cast<size_t>(i) * 8, c0, g, xh2, xhs, d);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      const float sg = red_f[c];
      const float k2 = (p.g2[c] * p.st2[p.C + c]) / mf;
      const float ks = (p.gs[c] * p.sts[p.C + c]) / mf;
      const float base = fmaf(mf, g[j], -sg);
      o2[j] = k2 * fmaf(-xh2[j], red_f[p.C + c], base);
      os[j] = ks * fmaf(-xhs[j], red_f[2 * p.C + c], base);
    }
    reinterpret_cast<uint4*>(dy2)[i] = pack8(o2);
    reinterpret_cast<uint4*>(dys)[i] = pack8(os);
  }
}

// -- BN backward (first BN of the unit): reductions and apply
__global__ void bn_bwd_partial_kernel(const __nv_bfloat16* __restrict__ gin, const __nv_bfloat16* __restrict__ y,
                                      const float* __restrict__ st, int m, int C, int rows_per_chunk, int cg, int rpp,
                                      float* __restrict__ partial) {
  const int gi = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  float acc[2][8] = {};
  if (slot < rpp) {
    const int r0 = blockIdx.x * rows_per_chunk;
    const int r1 = min(m, r0 + rows_per_chunk);
    for (int r = r0 + slot; r < r1; r += rpp) {
      const size_t off = static_cast<size_t>(r) * C + gi * 8;
      float fg[8], fy[8];
      unpack8(*reinterpret_cast<const uint4*>(gin + off), fg);
      unpack8(*reinterpret_cast<const uint4*>(y + off), fy);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = gi * 8 + j;
        const float xh = (fy[j] - st[c]) * st[C + c];
        acc[0][j] += fg[j];
        acc[1][j] += fg[j] * xh;
      }
    }
  }
  cta_reduce_store<2>(acc, cg, rpp, C, partial);
}

__global__ void bn_bwd_finalize_kernel(const float* __restrict__ partial, int chunks, int C, float* __restrict__ red_f,
                                       float* __restrict__ dgamma, float* __restrict__ dbeta) {
  const int o = blockIdx.x * 32 + (threadIdx.x & 31);  // o in [0, 2C)
  const double sv = sum_over_chunks<2>(partial, chunks, C, o);
  if ((threadIdx.x >> 5) == 0 && o < 2 * C) {
    const int v = o / C;
    const int c = o - v * C;
    const float f = static_cast<float>(sv);
    red_f[o] = f;
    if (v == 0)
      dbeta[c] = f;
    else
      dgamma[c] = f;
  }
}

__global__ void bn_bwd_apply_kernel(const __nv_bfloat16* __restrict__ gin, const __nv_bfloat16* __restrict__ y,
                                    const float* __restrict__ st, const float* __restrict__ gamma,
                                    const float* __restrict__ red_f, int m, int C, __nv_bfloat16* __restrict__ dy) {
  const int cg = C / 8;
  const long long total = static_cast<long long>(m) * cg;
  const float mf = static_cast<float>(m);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c0 = static_cast<int>(i % cg) * 8;
    float fg[8], fy[8], o[8];
    unpack8(reinterpret_cast<const uint4*>(gin)[i], fg);
    unpack8(reinterpret_cast<const uint4*>(y)[i], fy);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      const float xh = (fy[j] - st[c]) * st[C + c];
      const float k1 = (gamma[c] * st[C + c]) / mf;
      o[j] = k1 * fmaf(-xh, red_f[C + c], fmaf(mf, fg[j], -red_f[c]));
    }
    reinterpret_cast<uint4*>(dy)[i] = pack8(o);
  }
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

int grid_for(long long work, int per_block = kThreads) {
  const long long b = (work + per_block - 1) / per_block;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(b, 148LL * 16)));
}

inline int ok(cudaError_t e) { return e == cudaSuccess ? PBDK_OK : PBDK_ECUDA; }

}  // namespace

size_t reduce_workspace_floats(int m, int c, int nv) {
  const RowTiling t = tiling_for(m, c);
  return static_cast<size_t>(t.chunks) * nv * c + t.chunks;
}

int philox_image(void* x, int n, long long first, const long long* counter, int gb, uint32_t seed, cudaStream_t st) {
  philox_image_kernel<<<grid_for(n * 1024LL), kThreads, 0, st>>>(static_cast<__nv_bfloat16*>(x), n, first, counter,
                                                                  gb, seed);
  return ok(cudaGetLastError());
}

int pack_image(const float* src, void* x, int n, cudaStream_t st) {
  pack_image_kernel<<<grid_for(n * 1024LL), kThreads, 0, st>>>(src, static_cast<__nv_bfloat16*>(x), n);
  return ok(cudaGetLastError());
}

int init_uniform(void* dst, int bf16_out, int k, int r, int s, int cs, int ct, uint32_t seed, uint32_t tensor,
                 float bound, cudaStream_t st) {
  init_uniform_kernel<<<grid_for(static_cast<long long>(k) * r * s * cs), kThreads, 0, st>>>(dst, bf16_out, k, r, s,
                                                                                              cs, ct, seed, tensor,
                                                                                              bound);
  return ok(cudaGetLastError());
}

int fill(float* dst, size_t n, float v, cudaStream_t st) {
  fill_kernel<<<grid_for(static_cast<long long>(n)), kThreads, 0, st>>>(dst, n, v);
  return ok(cudaGetLastError());
}

int bn_stats(const void* y, int m, int c, float* ws, float* mean_rstd, cudaStream_t st) {
  if (c % 8 != 0 || c > 8 * kThreads) return PBDK_EINVAL;
  const RowTiling t = tiling_for(m, c);
  bn_stats_partial_kernel<<<t.chunks, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(y), m, c,
                                                         t.rows_per_chunk, t.cg, t.rpp, ws);
  bn_stats_finalize_kernel<<<(c + 31) / 32, kFinWarps * 32, 0, st>>>(ws, t.chunks, c, m, mean_rstd);
  return ok(cudaGetLastError());
}

int bn_apply_relu(const void* y, const float* mean_rstd, const float* gamma, const float* beta, void* a, int m, int c,
                  cudaStream_t st) {
  bn_apply_relu_kernel<<<grid_for(static_cast<long long>(m) * c / 8), kThreads, 0, st>>>(
      static_cast<const __nv_bfloat16*>(y), mean_rstd, gamma, beta, static_cast<__nv_bfloat16*>(a), m, c);
  return ok(cudaGetLastError());
}

int mse_bn_loss(const MseArgs& a, cudaStream_t st) {
  if (a.c % 8 != 0) return PBDK_EINVAL;
  LossParams p{static_cast<const __nv_bfloat16*>(a.y2), static_cast<const __nv_bfloat16*>(a.ysc),
               static_cast<const __nv_bfloat16*>(a.t), a.stats2, a.statssc, a.gamma2, a.beta2, a.gammasc, a.betasc,
               a.m, a.c, a.gscale};
  const RowTiling t = tiling_for(a.m, a.c);
  float* partial = a.ws;
  float* loss_partial = a.ws + static_cast<size_t>(t.chunks) * 3 * a.c;
  loss_partial_kernel<<<t.chunks, kThreads, 0, st>>>(p, t.rows_per_chunk, t.cg, t.rpp, partial, loss_partial);
  loss_finalize_kernel<<<(3 * a.c + 31) / 32 + 1, kFinWarps * 32, 0, st>>>(partial, loss_partial, t.chunks, a.c, a.norm, a.red,
                                                          a.dgamma2, a.dbeta2, a.dgammasc, a.dbetasc, a.loss);
  loss_bwd_apply_kernel<<<grid_for(static_cast<long long>(a.m) * a.c / 8), kThreads, 0, st>>>(
      p, a.red, static_cast<__nv_bfloat16*>(a.dy2), static_cast<__nv_bfloat16*>(a.dysc));
  return ok(cudaGetLastError());
}

int bn_bwd(const void* g, const void* y, const float* mean_rstd, const float* gamma, int m, int c, float* ws,
           float* red, float* dgamma, float* dbeta, void* dy, cudaStream_t st) {
  if (c % 8 != 0) return PBDK_EINVAL;
  const RowTiling t = tiling_for(m, c);
  bn_bwd_partial_kernel<<<t.chunks, kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(g),
                                                       static_cast<const __nv_bfloat16*>(y), mean_rstd, m, c,
                                                       t.rows_per_chunk, t.cg, t.rpp, ws);
  bn_bwd_finalize_kernel<<<(2 * c + 31) / 32, kFinWarps * 32, 0, st>>>(ws, t.chunks, c, red, dgamma, dbeta);
  bn_bwd_apply_kernel<<<grid_for(static_cast<long long>(m) * c / 8), kThreads, 0, st>>>(
      static_cast<const __nv_bfloat16*>(g), static_cast<const __nv_bfloat16*>(y), mean_rstd, gamma, red, m, c,
      static_cast<__nv_bfloat16*>(dy));
  return ok(cudaGetLastError());
}

int sgd_momentum(float* w, float* v, const float* g, void* shadow, size_t n, float lr, float mu, long long* counter,
                 cudaStream_t st) {
  if (n % 4 != 0) return PBDK_EINVAL;
  sgd_kernel<<<grid_for(static_cast<long long>(n / 4)), kThreads, 0, st>>>(
      reinterpret_cast<float4*>(w), reinterpret_cast<float4*>(v), reinterpret_cast<const float4*>(g),
      static_cast<uint2*>(shadow), n / 4, lr, mu, counter);
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

}  // extern "C"
