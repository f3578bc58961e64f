// 3xTF32 convolutions on tcgen05 (kind::tf32) for the fp32 workload — see conv_tf32.hpp for the
// split-fp32 storage and the error argument.
//
//   fprop: D[m, k] = sum_{tap, c} X[pix(m, tap), c] * W[k, tap, c], 128-pixel M tiles (one 4D TMA
//          box per filter tap and channel chunk, OOB zero fill = padding, TMA element strides =
//          conv stride), N = BN output channels, K-major operands.  Every pipeline stage carries
//          the hi and lo halves of the A and B chunks (4 TMA boxes) and issues three MMAs per
//          K-step: lo*hi, hi*lo, hi*hi (small terms first).
//   wgrad: D[k, c] (per tap) = sum_m dY[m, k] * X[pix(m, tap), c], MN-major operands (pixels are the
//          reduction dim), 32 pixels per stage, split-K over pixel tiles with a fixed-order
//          reduction of the per-split slabs (deterministic for a given shape).
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (one thread), warps 2-5 epilogue
// (TMEM lane quarter = warp % 4); warp 2 owns the TMEM allocation.
#include "conv_tf32.hpp"

#include <algorithm>

#include "conv.hpp"
#include "knobs.hpp"
#include "sm100.cuh"
#include "tmap.hpp"

namespace pbdk {

namespace {
// programmatic dependent launch for the fp32 workload's tcgen05 convs and split sums (the kernels wait
// with griddepcontrol.wait before touching global memory); PBD_PDL=0 in the experiments build: plain
template <class... KArgs, class... Args>
cudaError_t f3_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pbd::pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
}  // namespace

namespace {

constexpr int kThreads = 192;
constexpr int kBudget = 200 * 1024;

__host__ __device__ constexpr int layout_of(int sw) { return sw == 128 ? 2 : (sw == 64 ? 4 : 6); }
__host__ __device__ constexpr int round_up(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ constexpr int tmem_cols(int n) { return n <= 32 ? 32 : (n <= 64 ? 64 : (n <= 128 ? 128 : 256)); }

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

template <int BN, int CK>
struct F3FpropCfg {
  static constexpr int SW = CK * 4;  // bytes per smem row == swizzle span (64 or 128)
  static constexpr int A = 128 * SW;
  static constexpr int B = BN * SW;
  static constexpr int STAGE = round_up(2 * (A + B), 1024);
  static constexpr int STAGES = (kBudget / STAGE) > 6 ? 6 : (kBudget / STAGE);
  static constexpr int TMEM_COLS = tmem_cols(BN);
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

template <int BN, int CK>
__global__ void __launch_bounds__(kThreads, 1)
    conv3x_fprop_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                        const F3FpropArgs a) {
  using C = F3FpropCfg<BN, CK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = warp_id();
  const int lane = lane_id();
  const int m_tile = blockIdx.x;
  const int k0 = blockIdx.y * BN;
  const int tq = m_tile % a.tiles_q;
  const int t2 = m_tile / a.tiles_q;
  const int ow0 = tq * a.bw, oh0 = (t2 % a.tiles_p) * a.bh, n0 = (t2 / a.tiles_p) * a.bn;
  const int num_kb = a.r * a.s * a.c_chunks;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmx);
    tma_prefetch(&tmw);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // PDL (f3_launch): the prologue above overlapped the previous kernel

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % C::STAGES;
        if (kb >= C::STAGES) mbar_wait(&empty[st], ((kb / C::STAGES) - 1) & 1);
        const int tap = kb / a.c_chunks;
        const int cc = (kb - tap * a.c_chunks) * CK;
        const int rr = tap / a.s;
        const int ss = tap - rr * a.s;
        const int iw = ow0 * a.stride + ss - a.pad, ih = oh0 * a.stride + rr - a.pad;
        uint8_t* sa = smem + st * C::STAGE;
        mbar_arrive_expect_tx(&full[st], 2 * (C::A + C::B));
        tma_load_4d(sa, &tmx, &full[st], cc, iw, ih, n0);                  // A hi
        tma_load_4d(sa + C::A, &tmx, &full[st], a.c + cc, iw, ih, n0);     // A lo
        const int wk = tap * 2 * a.c + cc;
        tma_load_2d(sa + 2 * C::A, &tmw, &full[st], wk, k0);               // B hi
        tma_load_2d(sa + 2 * C::A + C::B, &tmw, &full[st], wk + a.c, k0);  // B lo
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_tf32(128, BN, 0, 0);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % C::STAGES;
        mbar_wait(&full[st], (kb / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + st * C::STAGE);
        const uint64_t ahi = umma_smem_desc(sa, 16, 8 * C::SW, layout_of(C::SW));
        const uint64_t alo = umma_smem_desc(sa + C::A, 16, 8 * C::SW, layout_of(C::SW));
        const uint64_t bhi = umma_smem_desc(sa + 2 * C::A, 16, 8 * C::SW, layout_of(C::SW));
        const uint64_t blo = umma_smem_desc(sa + 2 * C::A + C::B, 16, 8 * C::SW, layout_of(C::SW));
#pragma unroll
        for (int kk = 0; kk < CK / 8; ++kk) {  // K = 8 tf32 = 32 B = +2 in descriptor units
          umma_tf32(tmem, alo + 2 * kk, bhi + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
          umma_tf32(tmem, ahi + 2 * kk, blo + 2 * kk, idesc, 1u);
          umma_tf32(tmem, ahi + 2 * kk, bhi + 2 * kk, idesc, 1u);
        }
        umma_commit(&empty[st]);
      }
      umma_commit(tfull);
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int iw = row % a.bw;
    const int ih = (row / a.bw) % a.bh;
    const int nn = n0 + row / (a.bw * a.bh);
    const bool valid = nn < a.n;
    const size_t m = (static_cast<size_t>(nn) * a.p + (oh0 + ih)) * a.q + (ow0 + iw);
    const bool bias = a.epi == PBDK_EPI_BIAS || a.epi == PBDK_EPI_BIAS_RELU || a.epi == PBDK_EPI_BIAS_RES_RELU;
    const bool res = a.epi == PBDK_EPI_BIAS_RES_RELU;
    const bool mask = a.epi == PBDK_EPI_RELU_MASK;
    const bool relu = a.epi == PBDK_EPI_BIAS_RELU || a.epi == PBDK_EPI_BIAS_RES_RELU;
    mbar_wait_backoff(tfull, 0, 64);
    tc_fence_after();
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      tmem_ld16(trow + c0, v);
      if (!valid) continue;
      const int col = k0 + c0;
      if (bias) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const float4 b = __ldg(reinterpret_cast<const float4*>(a.bias + col + j));
          v[j] += b.x;
          v[j + 1] += b.y;
          v[j + 2] += b.z;
          v[j + 3] += b.w;
        }
      }
      if (res || mask) {
        const float* hi = a.aux + m * 2 * a.k + col;
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const float4 h = __ldg(reinterpret_cast<const float4*>(hi + j));
          const float4 l = __ldg(reinterpret_cast<const float4*>(hi + a.k + j));
          const float r[4] = {h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) v[j + i] = res ? v[j + i] + r[i] : (r[i] > 0.f ? v[j + i] : 0.f);
        }
      }
      if (relu) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.f);
      }
      if (a.y_split) {
        float* dst = a.y + m * 2 * a.k + col;
        float hv[16], lv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          hv[j] = tf32_hi(v[j]);
          lv[j] = v[j] - hv[j];
        }
#pragma unroll
        for (int j = 0; j < 16; j += 8) {
          st_global_256(dst + j, make_uint4(__float_as_uint(hv[j]), __float_as_uint(hv[j + 1]),
                                            __float_as_uint(hv[j + 2]), __float_as_uint(hv[j + 3])),
                        make_uint4(__float_as_uint(hv[j + 4]), __float_as_uint(hv[j + 5]), __float_as_uint(hv[j + 6]),
                                   __float_as_uint(hv[j + 7])));
          st_global_256(dst + a.k + j, make_uint4(__float_as_uint(lv[j]), __float_as_uint(lv[j + 1]),
                                                  __float_as_uint(lv[j + 2]), __float_as_uint(lv[j + 3])),
                        make_uint4(__float_as_uint(lv[j + 4]), __float_as_uint(lv[j + 5]), __float_as_uint(lv[j + 6]),
                                   __float_as_uint(lv[j + 7])));
        }
      } else {
        float* dst = a.y + m * a.k + col;
#pragma unroll
        for (int j = 0; j < 16; j += 8)
          st_global_256(dst + j, make_uint4(__float_as_uint(v[j]), __float_as_uint(v[j + 1]),
                                            __float_as_uint(v[j + 2]), __float_as_uint(v[j + 3])),
                        make_uint4(__float_as_uint(v[j + 4]), __float_as_uint(v[j + 5]), __float_as_uint(v[j + 6]),
                                   __float_as_uint(v[j + 7])));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int BN, int CK>
cudaError_t launch_fprop(const F3FpropPlan& p, cudaStream_t st) {
  using C = F3FpropCfg<BN, CK>;
  if (st == reinterpret_cast<cudaStream_t>(-1))  // plan-time attribute setup
    return cudaFuncSetAttribute(conv3x_fprop_kernel<BN, CK>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  f3_launch(conv3x_fprop_kernel<BN, CK>, p.grid, dim3(kThreads), C::SMEM, st, p.tmx, p.tmw, p.args);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ wgrad
constexpr int kWgPix = 32;  // pixels per stage (the reduction K of one stage)

// MN-major 32-bit operands have one legal shared-memory layout: SWIZZLE_128B_BASE32B (layout type 1,
// TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) — 128-byte rows (32 channels), 32-byte chunks swizzled
// within 4-row atoms.  Descriptor: LBO = stride between 32-channel MN atoms, SBO = 4 rows (512 B);
// one K = 8 MMA covers 8 pixel rows = 1 KB.
constexpr int kLayout128Base32 = 1;

template <int BN>
struct F3WgradCfg {
  static constexpr int ATOM = kWgPix * 128;  // 32 channels (128 B) x 32 pixel rows
  static constexpr int A = 4 * ATOM;         // M = 128 k-channels
  static constexpr int B_ATOMS = BN / 32;
  static constexpr int B = B_ATOMS * ATOM;
  static constexpr int STAGE = round_up(2 * (A + B), 1024);
  static constexpr int STAGES = (kBudget / STAGE) > 6 ? 6 : (kBudget / STAGE);
  static constexpr int TMEM_COLS = tmem_cols(BN);
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    conv3x_wgrad_kernel(const __grid_constant__ CUtensorMap tmdy, const __grid_constant__ CUtensorMap tmx,
                        const F3WgradArgs a) {
  using C = F3WgradCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = warp_id();
  const int lane = lane_id();
  int t = blockIdx.x;
  const int ci0 = (t % a.ci_tiles) * BN;
  t /= a.ci_tiles;
  const int co0 = (t % a.co_tiles) * 128;
  const int tap = t / a.co_tiles;
  const int rr = tap / a.s;
  const int ss = tap - rr * a.s;
  const int split = blockIdx.y;
  const int mt0 = split * a.tiles_per_split;
  const int num_kb = max(0, min(a.m_tiles, mt0 + a.tiles_per_split) - mt0);
  const int a_atoms = min(4, (a.k - co0) / 32);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmdy);
    tma_prefetch(&tmx);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // PDL (f3_launch): the prologue above overlapped the previous kernel

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = static_cast<uint32_t>(2 * (a_atoms * C::ATOM + C::B));
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % C::STAGES;
        if (kb >= C::STAGES) mbar_wait(&empty[st], ((kb / C::STAGES) - 1) & 1);
        const int mt = mt0 + kb;
        const int tq = mt % a.tiles_q;
        const int t2 = mt / a.tiles_q;
        const int ow0 = tq * a.bw, oh0 = (t2 % a.tiles_p) * a.bh, n0 = (t2 / a.tiles_p) * a.bn;
        const int iw = ow0 * a.stride + ss - a.pad, ih = oh0 * a.stride + rr - a.pad;
        uint8_t* sa = smem + st * C::STAGE;
        uint8_t* sb = sa + 2 * C::A;
        mbar_arrive_expect_tx(&full[st], bytes);
        for (int i = 0; i < a_atoms; ++i) {
          tma_load_4d(sa + i * C::ATOM, &tmdy, &full[st], co0 + 32 * i, ow0, oh0, n0);
          tma_load_4d(sa + C::A + i * C::ATOM, &tmdy, &full[st], a.k + co0 + 32 * i, ow0, oh0, n0);
        }
#pragma unroll
        for (int i = 0; i < C::B_ATOMS; ++i) {
          tma_load_4d(sb + i * C::ATOM, &tmx, &full[st], ci0 + 32 * i, iw, ih, n0);
          tma_load_4d(sb + C::B + i * C::ATOM, &tmx, &full[st], a.c + ci0 + 32 * i, iw, ih, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_tf32(128, BN, 1, 1);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % C::STAGES;
        mbar_wait(&full[st], (kb / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + st * C::STAGE);
        const uint32_t sb = sa + 2 * C::A;
#pragma unroll
        for (int kk = 0; kk < kWgPix / 8; ++kk) {
          const uint32_t o = kk * 8 * 128;
          const uint64_t ahi = umma_smem_desc(sa + o, C::ATOM, 4 * 128, kLayout128Base32);
          const uint64_t alo = umma_smem_desc(sa + C::A + o, C::ATOM, 4 * 128, kLayout128Base32);
          const uint64_t bhi = umma_smem_desc(sb + o, C::ATOM, 4 * 128, kLayout128Base32);
          const uint64_t blo = umma_smem_desc(sb + C::B + o, C::ATOM, 4 * 128, kLayout128Base32);
          umma_tf32(tmem, alo, bhi, idesc, (kb | kk) != 0 ? 1u : 0u);
          umma_tf32(tmem, ahi, blo, idesc, 1u);
          umma_tf32(tmem, ahi, bhi, idesc, 1u);
        }
        umma_commit(&empty[st]);
      }
      if (num_kb > 0) umma_commit(tfull);
    }
  } else {
    const int quarter = warp & 3;
    const int co = co0 + quarter * 32 + lane;
    const int taps = a.r * a.s;
    float* dst = a.out + static_cast<size_t>(split) * a.k * taps * a.c + (static_cast<size_t>(co) * taps + tap) * a.c + ci0;
    if (num_kb > 0) {
      mbar_wait_backoff(tfull, 0, 64);
      tc_fence_after();
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(trow + c0, v);
        if (co < a.k) {
          float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
      }
    } else if (co < a.k) {
      for (int c0 = 0; c0 < BN; c0 += 4) *reinterpret_cast<float4*>(dst + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int BN>
cudaError_t launch_wgrad(const F3WgradPlan& p, cudaStream_t st) {
  using C = F3WgradCfg<BN>;
  if (st == reinterpret_cast<cudaStream_t>(-1))
    return cudaFuncSetAttribute(conv3x_wgrad_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  f3_launch(conv3x_wgrad_kernel<BN>, p.grid, dim3(kThreads), C::SMEM, st, p.tmdy, p.tmx, p.args);
  return cudaGetLastError();
}

// dw[i] = sum_s ws[s][i] in split order
__global__ void f3_split_sum_kernel(const float4* __restrict__ ws, float4* __restrict__ dw, size_t n4, int splits) {
  grid_dep_wait();  // PDL (f3_launch): the split slabs are complete after this
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float4 acc = ws[i];
    for (int s = 1; s < splits; ++s) {
      const float4 v = ws[s * n4 + i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    dw[i] = acc;
  }
}

__global__ void f3_split_kernel(const float* __restrict__ src, float* __restrict__ dst, size_t rows, int c) {
  const size_t total = rows * c;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / c;
    const int j = static_cast<int>(i - r * c);
    const float x = src[i];
    const float h = tf32_hi(x);
    dst[r * 2 * c + j] = h;
    dst[r * 2 * c + c + j] = x - h;
  }
}

// wt[ci][r'][s'][hi k | lo k] from w[co][R-1-r'][S-1-s'][ci]
__global__ void f3_flip_split_kernel(const float* __restrict__ w, float* __restrict__ wt, int k, int r, int s, int c) {
  const size_t total = static_cast<size_t>(k) * r * s * c;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int co = static_cast<int>(i % k);
    size_t t = i / k;  // (ci, r', s') row of wt
    const int sp = static_cast<int>(t % s);
    const int rp = static_cast<int>((t / s) % r);
    const int ci = static_cast<int>(t / (static_cast<size_t>(s) * r));
    const float x = w[((static_cast<size_t>(co) * r + (r - 1 - rp)) * s + (s - 1 - sp)) * c + ci];
    const float h = tf32_hi(x);
    wt[t * 2 * k + co] = h;
    wt[t * 2 * k + k + co] = x - h;
  }
}

int grid_for(size_t work) { return static_cast<int>(std::min<size_t>(std::max<size_t>(1, (work + 255) / 256), 148 * 8)); }

// fp32 NHWC tensor of 2c channels (the split layout) as a 4D map; box = chan x (bw x bh x bn pixels)
bool split_map(CUtensorMap* m, const float* base, int n, int h, int w, int c, int chan, int bw, int bh, int bn,
               int stride, int swizzle) {
  const uint64_t cc = 2ull * c;
  const uint64_t dims[4] = {cc, static_cast<uint64_t>(w), static_cast<uint64_t>(h), static_cast<uint64_t>(n)};
  const uint64_t strides[3] = {cc * 4, static_cast<uint64_t>(w) * cc * 4, static_cast<uint64_t>(h) * w * cc * 4};
  const uint32_t box[4] = {static_cast<uint32_t>(chan), static_cast<uint32_t>(bw * stride),
                           static_cast<uint32_t>(bh * stride), static_cast<uint32_t>(bn)};
  const uint32_t es[4] = {1, static_cast<uint32_t>(stride), static_cast<uint32_t>(stride), 1};
  return encode_tmap_f32(m, base, 4, dims, strides, box, es, swizzle);
}

bool chans_ok(int c) { return c == 16 || (c >= 32 && c % 32 == 0); }

// 32-pixel tiles of the wgrad reduction: (bn images) x (bh rows) x (bw cols) = 32
bool geom32(const pbdk_conv_desc& d, int* bw, int* bh, int* bn) {
  if (d.q > kWgPix || kWgPix % d.q != 0) return false;
  *bw = d.q;
  const int rows = kWgPix / d.q;
  *bh = std::min(d.p, rows);
  if (rows % *bh != 0 || d.p % *bh != 0) return false;
  *bn = rows / *bh;
  return *bw * d.stride <= 256 && *bh * d.stride <= 256;
}

int wgrad_splits(const pbdk_conv_desc& d, int m_tiles) {
  const int base = d.r * d.s * ((d.k + 127) / 128) * (d.c / std::min(d.c, 128));
  const int want = std::max(1, (2 * 148 + base - 1) / base);
  const int per = (m_tiles + std::min(want, m_tiles) - 1) / std::min(want, m_tiles);
  return (m_tiles + per - 1) / per;
}

}  // namespace

int f3_fprop_plan(const pbdk_conv_desc& d, const float* x, const float* w, float* y, int y_split, const float* bias,
                  const float* aux, int epi, F3FpropPlan* plan) {
  ConvGeom g;
  if (!make_geom(d, &g) || !chans_ok(d.c) || d.k % 16 != 0 || d.k < 16) return PBDK_EINVAL;
  const bool has_bias = epi == PBDK_EPI_BIAS || epi == PBDK_EPI_BIAS_RELU || epi == PBDK_EPI_BIAS_RES_RELU;
  const bool has_aux = epi == PBDK_EPI_BIAS_RES_RELU || epi == PBDK_EPI_RELU_MASK;
  if (epi != PBDK_EPI_STORE && !has_bias && !has_aux) return PBDK_EINVAL;
  if ((has_bias && bias == nullptr) || (has_aux && aux == nullptr) || x == nullptr || w == nullptr || y == nullptr)
    return PBDK_EINVAL;
  const int ck = d.c == 16 ? 16 : 32;
  const int bn = d.k >= 128 ? 128 : d.k;  // 16, 32, 64 or 128 (k multiple of 16 below 128)
  if (d.k % bn != 0 || (bn != 16 && bn != 32 && bn != 64 && bn != 128)) return PBDK_EINVAL;
  if (!split_map(&plan->tmx, x, d.n, d.h, d.w, d.c, ck, g.bw, g.bh, g.bn, d.stride, ck * 4)) return PBDK_ECUDA;
  {
    const uint64_t ktot = static_cast<uint64_t>(d.r) * d.s * 2 * d.c;
    const uint64_t dims[2] = {ktot, static_cast<uint64_t>(d.k)};
    const uint64_t strides[1] = {ktot * 4};
    const uint32_t box[2] = {static_cast<uint32_t>(ck), static_cast<uint32_t>(bn)};
    const uint32_t es[2] = {1, 1};
    if (!encode_tmap_f32(&plan->tmw, w, 2, dims, strides, box, es, ck * 4)) return PBDK_ECUDA;
  }
  F3FpropArgs& a = plan->args;
  a = F3FpropArgs{d.n, d.p, d.q, d.k, d.c, d.stride, d.pad, d.r, d.s, g.bw, g.bh, g.bn, g.tiles_q, g.tiles_p,
                  d.c / ck, epi, y_split ? 1 : 0, y, bias, aux};
  plan->grid = dim3(static_cast<unsigned>(g.m_tiles), static_cast<unsigned>(d.k / bn), 1);
  using L = cudaError_t (*)(const F3FpropPlan&, cudaStream_t);
  L l = nullptr;
  if (ck == 16) {
    l = bn == 16 ? launch_fprop<16, 16> : bn == 32 ? launch_fprop<32, 16> : bn == 64 ? launch_fprop<64, 16>
                                                                                   : launch_fprop<128, 16>;
  } else {
    l = bn == 16 ? launch_fprop<16, 32> : bn == 32 ? launch_fprop<32, 32> : bn == 64 ? launch_fprop<64, 32>
                                                                                   : launch_fprop<128, 32>;
  }
  plan->launch = l;
  return l(*plan, reinterpret_cast<cudaStream_t>(-1)) == cudaSuccess ? PBDK_OK : PBDK_ECUDA;
}

int f3_fprop_run(const F3FpropPlan& plan, cudaStream_t st) {
  if (plan.launch == nullptr) return PBDK_EINVAL;
  return plan.launch(plan, st) == cudaSuccess ? PBDK_OK : PBDK_ECUDA;
}

// MN-major tf32 operands come in 32-channel atoms (SWIZZLE_128B_BASE32B)
bool wgrad_ok(const pbdk_conv_desc& d) { return d.c % 32 == 0 && d.k % 32 == 0; }

size_t f3_wgrad_workspace_bytes(const pbdk_conv_desc& d) {
  int bw, bh, bn;
  if (!geom32(d, &bw, &bh, &bn) || !wgrad_ok(d)) return 0;
  const int m_tiles = (d.q / bw) * (d.p / bh) * ((d.n + bn - 1) / bn);
  const int splits = wgrad_splits(d, m_tiles);
  return splits > 1 ? static_cast<size_t>(splits) * d.k * d.r * d.s * d.c * sizeof(float) : 0;
}

int f3_wgrad_plan(const pbdk_conv_desc& d, const float* x, const float* dy, float* dw, void* ws, size_t ws_bytes,
                  F3WgradPlan* plan) {
  int bw, bh, bn;
  if (!geom32(d, &bw, &bh, &bn) || !wgrad_ok(d) || x == nullptr || dy == nullptr || dw == nullptr) return PBDK_EINVAL;
  const int bnt = std::min(d.c, 128);
  F3WgradArgs& a = plan->args;
  a.n = d.n;
  a.p = d.p;
  a.q = d.q;
  a.k = d.k;
  a.c = d.c;
  a.stride = d.stride;
  a.pad = d.pad;
  a.r = d.r;
  a.s = d.s;
  a.bw = bw;
  a.bh = bh;
  a.bn = bn;
  a.tiles_q = d.q / bw;
  a.tiles_p = d.p / bh;
  a.m_tiles = a.tiles_q * a.tiles_p * ((d.n + bn - 1) / bn);
  a.co_tiles = (d.k + 127) / 128;
  a.ci_tiles = d.c / bnt;
  const int splits = wgrad_splits(d, a.m_tiles);
  a.tiles_per_split = (a.m_tiles + splits - 1) / splits;
  plan->splits = splits;
  plan->dw = dw;
  plan->slab = static_cast<size_t>(d.k) * d.r * d.s * d.c;
  if (splits > 1) {
    if (ws == nullptr || ws_bytes < plan->slab * splits * sizeof(float)) return PBDK_EINVAL;
    a.out = static_cast<float*>(ws);
  } else {
    a.out = dw;
  }
  if (!split_map(&plan->tmdy, dy, d.n, d.p, d.q, d.k, 32, bw, bh, bn, 1, kSwizzle128Atom32)) return PBDK_ECUDA;
  if (!split_map(&plan->tmx, x, d.n, d.h, d.w, d.c, 32, bw, bh, bn, d.stride, kSwizzle128Atom32)) return PBDK_ECUDA;
  plan->grid = dim3(static_cast<unsigned>(d.r * d.s * a.co_tiles * a.ci_tiles), static_cast<unsigned>(splits), 1);
  using L = cudaError_t (*)(const F3WgradPlan&, cudaStream_t);
  L l = launch_wgrad<128>;
  if (bnt == 32) l = launch_wgrad<32>;
  if (bnt == 64) l = launch_wgrad<64>;
  plan->launch = l;
  return l(*plan, reinterpret_cast<cudaStream_t>(-1)) == cudaSuccess ? PBDK_OK : PBDK_ECUDA;
}

int f3_wgrad_run(const F3WgradPlan& plan, cudaStream_t st) {
  if (plan.launch == nullptr) return PBDK_EINVAL;
  if (plan.launch(plan, st) != cudaSuccess) return PBDK_ECUDA;
  if (plan.splits > 1) {
    const size_t n4 = plan.slab / 4;
    if (f3_launch(f3_split_sum_kernel, dim3(grid_for(n4)), dim3(256), 0, st,
                  reinterpret_cast<const float4*>(plan.args.out), reinterpret_cast<float4*>(plan.dw), n4,
                  plan.splits) != cudaSuccess)
      return PBDK_ECUDA;
  }
  return PBDK_OK;
}

int f3_split(const float* src, float* dst, size_t rows, int c, cudaStream_t st) {
  if (src == nullptr || dst == nullptr || c < 1) return PBDK_EINVAL;
  f3_split_kernel<<<grid_for(rows * c), 256, 0, st>>>(src, dst, rows, c);
  return cudaGetLastError() == cudaSuccess ? PBDK_OK : PBDK_ECUDA;
}

int f3_flip_split(const float* w, float* wt, int k, int r, int s, int c, cudaStream_t st) {
  if (w == nullptr || wt == nullptr || k < 1 || r < 1 || s < 1 || c < 1) return PBDK_EINVAL;
  f3_flip_split_kernel<<<grid_for(static_cast<size_t>(k) * r * s * c), 256, 0, st>>>(w, wt, k, r, s, c);
  return cudaGetLastError() == cudaSuccess ? PBDK_OK : PBDK_ECUDA;
}

}  // namespace pbdk

// ------------------------------------------------------------------ C ABI (include/pbdk.h)
extern "C" {

int pbdk_conv3x_fprop(const pbdk_conv_desc* d, const float* x, const float* w, float* y, int y_split,
                      const float* bias, const float* aux, int epilogue, void* stream) {
  if (d == nullptr) return PBDK_EINVAL;
  pbdk::F3FpropPlan plan;
  const int rc = pbdk::f3_fprop_plan(*d, x, w, y, y_split, bias, aux, epilogue, &plan);
  return rc != PBDK_OK ? rc : pbdk::f3_fprop_run(plan, static_cast<cudaStream_t>(stream));
}

size_t pbdk_conv3x_wgrad_workspace_bytes(const pbdk_conv_desc* d) {
  return d == nullptr ? 0 : pbdk::f3_wgrad_workspace_bytes(*d);
}

int pbdk_conv3x_wgrad(const pbdk_conv_desc* d, const float* x, const float* dy, float* dw, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (d == nullptr) return PBDK_EINVAL;
  pbdk::F3WgradPlan plan;
  const int rc = pbdk::f3_wgrad_plan(*d, x, dy, dw, workspace, workspace_bytes, &plan);
  return rc != PBDK_OK ? rc : pbdk::f3_wgrad_run(plan, static_cast<cudaStream_t>(stream));
}

int pbdk_split_tf32(const float* src, float* dst, size_t rows, int c, void* stream) {
  return pbdk::f3_split(src, dst, rows, c, static_cast<cudaStream_t>(stream));
}

int pbdk_weight_flip_split(const float* w, float* wt, int k, int r, int s, int c, void* stream) {
  return pbdk::f3_flip_split(w, wt, k, r, s, c, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
