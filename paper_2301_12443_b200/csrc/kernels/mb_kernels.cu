// CUDA-core kernels of the MobileNetV2 -> ProxylessNAS workload (sm_100a), DESIGN.md §10:
//   depthwise k x k conv (k = 3/5/7, stride 1/2): forward (+bias+ReLU6 for the teacher),
//     data gradient with the ReLU6 mask of the stored activation, weight gradient (two-level,
//     fixed-order reduction);
//   stem 3x3/s2 conv on the 16-channel padded image: forward and weight gradient;
//   BN apply as a per-channel affine map with {none, ReLU6} and an optional residual add;
//   MSE distillation loss + its gradient on z = BN(y) [+ residual] (no activation).
// The 1x1 expand / project convolutions run on the tcgen05 implicit-GEMM engine (conv.cu).
// Layout: NHWC bf16, every thread owns 8 consecutive channels (one 16-byte vector).
// Depthwise weights are stored flipped and tap-major, wt[r'][s'][c] = w[c][K-1-r'][K-1-s']
// (pbdk_weight_flip with c = 1), so one array serves the forward and the data gradient.
// Accumulation order (fmaf over taps, r then s ascending) is the contract with the oracle
// (oracle/mb_oracle.c), which makes these kernels bit-exact against it on identical inputs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "knobs.hpp"
#include "mb_kernels.hpp"
#include "pbdk.h"
#include "sm100.cuh"
#include "tmap.hpp"

namespace pbdk {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint32_t pk2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&f)[8]) {
  *reinterpret_cast<uint4*>(p) = make_uint4(pk2(f[0], f[1]), pk2(f[2], f[3]), pk2(f[4], f[5]), pk2(f[6], f[7]));
}

// acc[j] = fmaf(x[j], w[j], acc[j]) for j < 8 as four packed FFMA2 (fma.rn.f32x2: per-lane IEEE fma,
// bit-identical to the scalar chain, half the fma-pipe issue slots)
__device__ __forceinline__ void fma8(float (&acc)[8], const float (&x)[8], const float (&w)[8]) {
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    unsigned long long a = (static_cast<unsigned long long>(__float_as_uint(acc[j + 1])) << 32) | __float_as_uint(acc[j]);
    const unsigned long long xx =
        (static_cast<unsigned long long>(__float_as_uint(x[j + 1])) << 32) | __float_as_uint(x[j]);
    const unsigned long long ww =
        (static_cast<unsigned long long>(__float_as_uint(w[j + 1])) << 32) | __float_as_uint(w[j]);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(xx), "l"(ww));
    acc[j] = __uint_as_float(static_cast<uint32_t>(a));
    acc[j + 1] = __uint_as_float(static_cast<uint32_t>(a >> 32));
  }
}

__device__ __forceinline__ float relu6f(float z) { return fminf(fmaxf(z, 0.0f), 6.0f); }
// EfficientNet's swish / sigmoid in fast math (ex2.approx + approximate division, a few ulp of fp32):
// the libm expf + IEEE division made the swish epilogues compute-bound (the 3x3/s2 depthwise of the
// EfficientNet teacher ran at 1.0 TB/s vs 3.1 TB/s with ReLU6).  Far below one bf16 rounding step; the
// oracle keeps expf and '/', parity is within the bf16 teacher tolerance (tests/test_gpu_mb.py).
__device__ __forceinline__ float swishf(float z) { return __fdividef(z, 1.0f + __expf(-z)); }
__device__ __forceinline__ float sigmoidf(float z) { return __fdividef(1.0f, 1.0f + __expf(-z)); }
// activation codes (mb_kernels.hpp): 0 none, 1 ReLU6, 2 swish
__device__ __forceinline__ float act_fn(int act, float v) {
  return act == 1 ? relu6f(v) : act == 2 ? swishf(v) : v;
}

int grid_for(long long work) {
  const long long b = (work + kT - 1) / kT;
  static const long long cap = [] {
    const char* e = pbd::knob_env("PBDK_MB_CTAS");
    return e != nullptr ? std::max(1LL, std::atoll(e)) : 148LL * 16;
  }();
  return static_cast<int>(std::max<long long>(1, std::min<long long>(b, cap)));
}

// Programmatic dependent launch for the MBConv kernels (every kernel calls grid_dep_wait() first): a
// kernel's CTAs are scheduled while its predecessor in the stream drains.  PBD_PDL=0 / PBDK_MB_PDL=0
// (experiments build): plain launches.
template <class... KArgs, class... Args>
cudaError_t mb_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  static const bool pdl = [] {
    const char* e = pbd::knob_env("PBDK_MB_PDL");
    return pbd::pdl_enabled() && (e == nullptr || e[0] != '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

inline int ok(cudaError_t e) { return e == cudaSuccess ? PBDK_OK : PBDK_ECUDA; }

// ------------------------------------------------------------------ depthwise forward
// Work item = (output row n,p ; strip of QT output columns ; 8-channel group).  For every filter
// row r the thread walks the strip's input window once (each input vector loaded once per r) and
// scatters it into the QT accumulators; per output the fmaf order is (r, s) ascending, exactly the
// oracle's.  Consecutive threads take consecutive channel groups (coalesced 16-byte loads).
constexpr int kQT = 4;

template <int K, int ST>
__global__ void __launch_bounds__(kT) dw_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                    const __nv_bfloat16* __restrict__ wt,
                                                    const float* __restrict__ bias, __nv_bfloat16* __restrict__ y,
                                                    int N, int H, int W, int C, int P, int Q, int relu6) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  constexpr int PAD = K / 2;
  constexpr int WIN = (kQT - 1) * ST + K;
  const int G = C / 8;
  const int QS = (Q + kQT - 1) / kQT;
  const int total = N * P * QS * G;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % G;
    const int t = i / G;
    const int q0 = (t % QS) * kQT;
    const int row = t / QS;  // n * P + p
    const int p = row % P;
    const int n = row / P;
    const int c0 = g * 8;
    float acc[kQT][8];
#pragma unroll
    for (int u = 0; u < kQT; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[u][j] = 0.0f;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int h = p * ST + r - PAD;
      if (h < 0 || h >= H) continue;
      float wr[K][8];  // filter row r of this channel group (w[c][r][s] = wt[K-1-r][K-1-s][c])
#pragma unroll
      for (int sidx = 0; sidx < K; ++sidx)
        ld8(wt + static_cast<size_t>((K - 1 - r) * K + (K - 1 - sidx)) * C + c0, wr[sidx]);
      const __nv_bfloat16* xrow = x + (static_cast<size_t>(n) * H + h) * W * C + c0;
#pragma unroll
      for (int j = 0; j < WIN; ++j) {
        const int w = q0 * ST - PAD + j;
        if (w < 0 || w >= W) continue;
        float xv[8];
        ld8(xrow + static_cast<size_t>(w) * C, xv);
#pragma unroll
        for (int u = 0; u < kQT; ++u) {
          const int sidx = j - u * ST;
          if (sidx < 0 || sidx >= K) continue;
          fma8(acc[u], xv, wr[sidx]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kQT; ++u) {
      if (q0 + u >= Q) break;
      float o[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        float v = acc[u][jj];
        if (bias != nullptr) v = v + bias[c0 + jj];
        o[jj] = act_fn(relu6, v);
      }
      st8(y + ((static_cast<size_t>(row) * Q) + q0 + u) * C + c0, o);
    }
  }
}

// ------------------------------------------------------------------ depthwise forward, shared-memory tiles
// Tile = (image n, TP output rows, all Q columns, CT channels).  ONE 4D TMA box per tile stages the
// input window — (TP-1)*ST + K rows x (Q-1)*ST + K columns x CT channels, the padding zero-filled by
// the TMA out-of-bounds handling — plus a 2D box of the filter slice [K*K][CT], double-buffered across
// the CTA's tiles on mbarriers; every input vector leaves HBM/L2 once per tile instead of once per
// (filter row, output strip) as in dw_fwd_kernel, which was memory-latency bound (ncu: 1.7 TB/s,
// long-scoreboard stalls at 33 % occupancy).  Thread item = (output row, strip of kQTT = 7 columns —
// the MBConv maps are 7 * 2^i wide — , 8-channel group); TP is chosen so a tile holds a whole number
// of 256-item rounds where the shared-memory budget allows.  Per output the fmaf order is (r, s)
// ascending — bit-identical to dw_fwd_kernel and the oracle (padding taps add +-0 products to an
// accumulator that is never -0).
constexpr int kQTT = 7;
// output columns per thread item: 7 for 3x3 filters; 4 for 5x5 / 7x7, whose filter rows and input
// windows would otherwise push the kernel to one CTA per SM (ncu: 154-158 registers at kQTT = 7)
__host__ __device__ constexpr int dw_qt(int k) { return k == 3 ? kQTT : 4; }
constexpr int kDwStages = 2;
constexpr int kDwTileBytes = 64 * 1024;  // one stage (input window + filter)

// DG: the stride-1 depthwise DATA gradient on the same tiles — dx = the correlation of dy with the
// spatially flipped filter, taps visited in descending window order so every output's fmaf chain is
// dw_dgrad_kernel's (r, s) ascending; epilogue = the ReLU6 mask of the stored activation `amask`.
template <int K, int ST, int CT, bool DG = false>
__global__ void __launch_bounds__(kT) dw_fwd_tiled_kernel(const __grid_constant__ CUtensorMap tmx,
                                                          const __grid_constant__ CUtensorMap tmw,
                                                          const float* __restrict__ bias,
                                                          __nv_bfloat16* __restrict__ y, int N, int C, int P, int Q,
                                                          int act, int TP,
                                                          const __nv_bfloat16* __restrict__ amask = nullptr) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  constexpr int PAD = K / 2;
  constexpr int G = CT / 8;
  constexpr int QT = dw_qt(K);
  constexpr int WIN = (QT - 1) * ST + K;
  extern __shared__ __align__(128) uint8_t dsm_base[];
  uint8_t* dsm_raw = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_base) + 127) & ~uintptr_t(127));
  __shared__ uint64_t full[kDwStages];
  const int cols_in = (Q - 1) * ST + K;
  const int rows_in = (TP - 1) * ST + K;
  const uint32_t x_bytes = static_cast<uint32_t>(rows_in) * cols_in * CT * 2;
  const uint32_t x_off = (x_bytes + 127) / 128 * 128;  // the filter box starts 128-B aligned
  const uint32_t w_bytes = K * K * CT * 2;
  const uint32_t stage_bytes = (x_off + w_bytes + 127) / 128 * 128;
  const int pblocks = (P + TP - 1) / TP;
  const int cblocks = C / CT;
  const int ntiles = N * pblocks * cblocks;
  const int strips = (Q + QT - 1) / QT;

  auto tile_of = [&](int t, int& n, int& p0, int& c0) {
    const int cb = t % cblocks;
    const int rest = t / cblocks;
    p0 = (rest % pblocks) * TP;
    n = rest / pblocks;
    c0 = cb * CT;
  };
  auto issue = [&](int t, int slot) {
    int n, p0, c0;
    tile_of(t, n, p0, c0);
    uint8_t* buf = dsm_raw + slot * stage_bytes;
    mbar_arrive_expect_tx(&full[slot], x_bytes + w_bytes);
    tma_load_4d(buf, &tmx, &full[slot], c0, -PAD, p0 * ST - PAD, n);
    tma_load_2d(buf + x_off, &tmw, &full[slot], c0, 0);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < kDwStages; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < kDwStages; ++s)
      if (blockIdx.x + s * gridDim.x < ntiles) issue(blockIdx.x + s * gridDim.x, s);
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int slot = it % kDwStages;
    mbar_wait(&full[slot], (it / kDwStages) & 1);
    const uint4* cur = reinterpret_cast<const uint4*>(dsm_raw + slot * stage_bytes);
    const uint4* wsm = reinterpret_cast<const uint4*>(dsm_raw + slot * stage_bytes + x_off);
    int n, p0, c0;
    tile_of(t, n, p0, c0);
    const int rows = min(TP, P - p0);
    const int items = rows * strips * G;
    for (int i = threadIdx.x; i < items; i += blockDim.x) {
      const int g = i % G;
      const int rest = i / G;
      const int q0 = (rest % strips) * QT;
      const int pr = rest / strips;
      float acc[QT][8];
#pragma unroll
      for (int u = 0; u < QT; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[u][j] = 0.0f;
      const size_t orow = (static_cast<size_t>(n) * P + p0 + pr) * Q;
      // data gradient: the ReLU6 mask rows requested before the taps (latency hidden); not for 5x5, whose
      // 128 registers (two CTAs per SM) the prefetch would exceed
      constexpr bool PF = DG && K != 5;
      uint4 am[PF ? QT : 1];
      if constexpr (PF) {
#pragma unroll
        for (int u = 0; u < QT; ++u)
          if (amask != nullptr && q0 + u < Q)
            am[u] = __ldg(reinterpret_cast<const uint4*>(amask + (orow + q0 + u) * C + c0 + 8 * g));
      }
#pragma unroll
      for (int ri = 0; ri < K; ++ri) {
        const int r = DG ? K - 1 - ri : ri;  // window row
        float wr[K][8];  // forward: w[c][r][s] = wt[K-1-r][K-1-s][c]; data gradient: w[c][K-1-r][K-1-s] = wt[r][s][c]
#pragma unroll
        for (int sidx = 0; sidx < K; ++sidx)
          ld8(reinterpret_cast<const __nv_bfloat16*>(
                  wsm + (DG ? r * K + sidx : (K - 1 - r) * K + (K - 1 - sidx)) * G + g),
              wr[sidx]);
        const uint4* xrow = cur + ((pr * ST + r) * cols_in + q0 * ST) * G + g;
#pragma unroll
        for (int jj = 0; jj < WIN; ++jj) {
          const int j = DG ? WIN - 1 - jj : jj;
          if (q0 * ST + j >= cols_in) continue;
          float xv[8];
          ld8(reinterpret_cast<const __nv_bfloat16*>(xrow + j * G), xv);
#pragma unroll
          for (int u = 0; u < QT; ++u) {
            const int sidx = j - u * ST;
            if (sidx < 0 || sidx >= K) continue;
            fma8(acc[u], xv, wr[sidx]);
          }
        }
      }
      float bv[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) bv[jj] = bias != nullptr ? bias[c0 + 8 * g + jj] : 0.0f;
#pragma unroll
      for (int u = 0; u < QT; ++u) {
        if (q0 + u >= Q) break;
        float o[8];
        if constexpr (DG) {
          if (amask != nullptr) {
            float av[8];
            if constexpr (PF) {
              const uint32_t w4[4] = {am[u].x, am[u].y, am[u].z, am[u].w};
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                av[2 * jj] = __uint_as_float(w4[jj] << 16);
                av[2 * jj + 1] = __uint_as_float(w4[jj] & 0xFFFF0000u);
              }
            } else {
              ld8(amask + (orow + q0 + u) * C + c0 + 8 * g, av);
            }
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) o[jj] = (av[jj] > 0.0f && av[jj] < 6.0f) ? acc[u][jj] : 0.0f;
          } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) o[jj] = acc[u][jj];
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            float v = acc[u][jj];
            if (bias != nullptr) v = v + bv[jj];
            o[jj] = act_fn(act, v);
          }
        }
        st8(y + (orow + q0 + u) * C + c0 + 8 * g, o);
      }
    }
    __syncthreads();  // slot fully read: refill it with the tile kDwStages ahead
    if (threadIdx.x == 0 && t + kDwStages * gridDim.x < ntiles) issue(t + kDwStages * gridDim.x, slot);
  }
}

// ------------------------------------------------------------------ depthwise data gradient
// dx[n,h,w,c] = fmaf chain over (r, s) ascending of dy[n,(h+PAD-r)/ST,(w+PAD-s)/ST,c] w[c][r][s],
// then the ReLU6 mask of the stored activation `act` (0 < a < 6) when given.
// Stride 2 with even H, W (`par`): pixels are walked parity class by parity class ((h&1, w&1) major,
// then h/2, w/2), so the lanes of a warp share one set of valid taps and the tap branches no longer
// diverge; the per-pixel tap order is unchanged.
template <int K, int ST>
__global__ void __launch_bounds__(kT) dw_dgrad_kernel(const __nv_bfloat16* __restrict__ dy,
                                                      const __nv_bfloat16* __restrict__ wt,
                                                      const __nv_bfloat16* __restrict__ act,
                                                      __nv_bfloat16* __restrict__ dx, int N, int H, int W, int C, int P,
                                                      int Q, bool par) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  constexpr int PAD = K / 2;
  const int G = C / 8;
  const int total = N * H * W * G;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % G;
    int pix, w, h, n;
    if (ST == 2 && par) {
      const int t = i / G;
      const int W2 = W / 2, H2 = H / 2;
      const int ww = t % W2;
      const int hh = (t / W2) % H2;
      const int cls = (t / (W2 * H2)) & 3;
      n = t / (W2 * H2 * 4);
      h = 2 * hh + (cls >> 1);
      w = 2 * ww + (cls & 1);
      pix = (n * H + h) * W + w;
    } else {
      pix = i / G;
      w = pix % W;
      h = (pix / W) % H;
      n = pix / (H * W);
    }
    const int c0 = g * 8;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint4 am = make_uint4(0u, 0u, 0u, 0u);  // the ReLU6 mask row, requested before the taps
    if (act != nullptr) am = __ldg(reinterpret_cast<const uint4*>(act + static_cast<size_t>(pix) * C + c0));
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const int pn = h + PAD - r;
      if (pn < 0 || pn % ST != 0 || pn / ST >= P) continue;
      const __nv_bfloat16* grow = dy + (static_cast<size_t>(n) * P + pn / ST) * Q * C + c0;
      const __nv_bfloat16* wrow = wt + static_cast<size_t>(K - 1 - r) * K * C + c0;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const int qn = w + PAD - s;
        if (qn < 0 || qn % ST != 0 || qn / ST >= Q) continue;
        float gv[8], wv[8];
        ld8(grow + static_cast<size_t>(qn / ST) * C, gv);
        ld8(wrow + static_cast<size_t>(K - 1 - s) * C, wv);
        fma8(acc, gv, wv);
      }
    }
    if (act != nullptr) {
      const uint32_t w4[4] = {am.x, am.y, am.z, am.w};
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const float a0 = __uint_as_float(w4[jj] << 16), a1 = __uint_as_float(w4[jj] & 0xFFFF0000u);
        acc[2 * jj] = (a0 > 0.0f && a0 < 6.0f) ? acc[2 * jj] : 0.0f;
        acc[2 * jj + 1] = (a1 > 0.0f && a1 < 6.0f) ? acc[2 * jj + 1] : 0.0f;
      }
    }
    st8(dx + static_cast<size_t>(pix) * C + c0, acc);
  }
}

// ------------------------------------------------------------------ depthwise weight gradient
// Pass 1, grid (chunks, channel windows, K): CTA = lanes_c channel groups x lanes_p pixel lanes,
// filter row r = blockIdx.z; every thread accumulates K x 8 fp32 sums over its pixels, then the
// CTA adds the pixel lanes in lane order -> partial[chunk][c][r][s].
template <int K, int ST>
__global__ void __launch_bounds__(kT, K >= 7 ? 2 : 1) dw_wgrad_partial_kernel(const __nv_bfloat16* __restrict__ a,
                                                              const __nv_bfloat16* __restrict__ dy,
                                                              float* __restrict__ partial, int N, int H, int W, int C,
                                                              int P, int Q, int lanes_c, int rows_per_chunk) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  // Thread = (channel group, row lane): walks whole output rows (n, p) of its chunk, q ascending, with the
  // K input vectors of filter row r the current q touches held in a register window that slides by ST
  // per q — one dy load and ST activation loads per pixel instead of 1 + K.
  constexpr int PAD = K / 2;
  __shared__ float red[kT * 8];
  const int G = C / 8;
  const int cl = threadIdx.x % lanes_c;
  const int pl = threadIdx.x / lanes_c;
  const int lanes_p = kT / lanes_c;
  const int g = blockIdx.y * lanes_c + cl;
  const int r = blockIdx.z;
  const int rows = N * P;
  const int r0 = blockIdx.x * rows_per_chunk;
  const int r1 = min(rows, r0 + rows_per_chunk);
  float acc[K][8];
#pragma unroll
  for (int s = 0; s < K; ++s)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[s][j] = 0.0f;
  if (g < G && pl < lanes_p) {
    const int c0 = g * 8;
    for (int row = r0 + pl; row < r1; row += lanes_p) {
      const int p = row % P;
      const int n = row / P;
      const int h = p * ST + r - PAD;
      if (h < 0 || h >= H) continue;
      const __nv_bfloat16* arow = a + (static_cast<size_t>(n) * H + h) * W * C + c0;
      const __nv_bfloat16* grow = dy + static_cast<size_t>(row) * Q * C + c0;
      float win[K][8];  // win[s] = a[h][q*ST + s - PAD] (zero outside the image)
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const int w = s - PAD;
        if (w >= 0 && w < W) {
          ld8(arow + static_cast<size_t>(w) * C, win[s]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) win[s][j] = 0.0f;
        }
      }
      // K q-steps per trip with the window rotated at compile time: tap s of step u lives in slot
      // (ST*u + s) % K, and the ST vectors loaded after step u replace the slots of taps 0..ST-1 —
      // no register moves; the fmaf order per sum (q ascending) is unchanged.
      constexpr int U = K >= 5 ? K : 1;  // K = 3: the plain shift (2 x 8 moves) measured faster
      // K = 3, stride 1: four q-steps unrolled so the next steps' loads are issued ahead of this step's fmas
#pragma unroll(K >= 5 || ST != 1 ? 1 : 4)
      for (int q0 = 0; q0 < Q; q0 += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = q0 + u;
          if (q >= Q) break;
          float gv[8];
          ld8(grow + static_cast<size_t>(q) * C, gv);
#pragma unroll
          for (int s = 0; s < K; ++s)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[s][j] = fmaf(gv[j], win[(ST * u + s) % K][j], acc[s][j]);
          if constexpr (U == 1) {  // slide by ST: the next q needs a[(q+1)*ST + s - PAD]
#pragma unroll
            for (int s = 0; s < K - ST; ++s)
#pragma unroll
              for (int j = 0; j < 8; ++j) win[s][j] = win[s + ST][j];
          }
#pragma unroll
          for (int t = 0; t < ST; ++t) {
            const int w = (q + 1) * ST + (K - ST + t) - PAD;
            const int slot = U == 1 ? K - ST + t : (ST * u + t) % K;
            if (w >= 0 && w < W) {
              ld8(arow + static_cast<size_t>(w) * C, win[slot]);
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j) win[slot][j] = 0.0f;
            }
          }
        }
      }
    }
  }
  const size_t cKK = static_cast<size_t>(C) * K * K;
#pragma unroll
  for (int s = 0; s < K; ++s) {
#pragma unroll
    for (int j = 0; j < 8; ++j) red[(pl * lanes_c + cl) * 8 + j] = acc[s][j];
    __syncthreads();
    for (int o = threadIdx.x; o < lanes_c * 8; o += kT) {
      const int l = o / 8, j = o % 8;
      const int gg = blockIdx.y * lanes_c + l;
      if (gg < G) {
        float t = 0.0f;
        for (int pp = 0; pp < lanes_p; ++pp) t += red[(pp * lanes_c + l) * 8 + j];
        partial[blockIdx.x * cKK + (static_cast<size_t>(gg * 8 + j) * K + r) * K + s] = t;
      }
    }
    __syncthreads();
  }
}

// Pass 2: dw[o] = sum over chunks (chunk order, fp64) of partial[chunk][o].
// out[o] = sum over chunks of partial[chunk][o] in fp64, fixed order: CTA = 32 consecutive outputs
// (threadIdx.x, coalesced) x 32 chunk lanes (threadIdx.y sums chunks y, y + 32, ...), the 32 lane sums
// added in lane order.  (A thread walking all chunks serially was latency bound: 25 us per launch.)
constexpr int kSumLanes = 32;
__global__ void __launch_bounds__(32 * kSumLanes) chunk_sum_kernel(const float* __restrict__ partial, int chunks,
                                                                   size_t n, float* __restrict__ out) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  __shared__ double part[kSumLanes][33];
  const size_t o = blockIdx.x * static_cast<size_t>(32) + threadIdx.x;
  double acc = 0.0;
  if (o < n) {
    int c = threadIdx.y;
    for (; c + 3 * kSumLanes < chunks; c += 4 * kSumLanes) {  // four independent loads in flight
      const float a0 = partial[static_cast<size_t>(c) * n + o];
      const float a1 = partial[static_cast<size_t>(c + kSumLanes) * n + o];
      const float a2 = partial[static_cast<size_t>(c + 2 * kSumLanes) * n + o];
      const float a3 = partial[static_cast<size_t>(c + 3 * kSumLanes) * n + o];
      acc += a0;
      acc += a1;
      acc += a2;
      acc += a3;
    }
    for (; c < chunks; c += kSumLanes) acc += partial[static_cast<size_t>(c) * n + o];
  }
  part[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && o < n) {
    double s = 0.0;
    for (int l = 0; l < kSumLanes; ++l) s += part[l][threadIdx.x];
    out[o] = static_cast<float>(s);
  }
}

// ------------------------------------------------------------------ stem weight gradient, staged rows
// dw[k][r][s][c] = sum_{n,p,q} dy[n,p,q,k] x[n, 2p+r-1, 2q+s-1, c] (c < 3).  A CTA walks its chunk of
// output rows one at a time: the dy row (Q x 32, bf16 -> fp32) and the three input rows (3 real
// channels, fp32, zero outside the image) are staged in shared memory, then thread (4-channel group of
// k, tap) sweeps the row's q with 12 fp32 fmas per 2 shared loads.  (The register kernel re-read 9
// broadcast 8-byte x vectors per q from L1/L2 and was latency bound: 588 GB/s.)  Per-thread fp32
// partials over the chunk's rows, CTA partial -> fixed-order chunk sum (as before).
constexpr int kStemLanes = 3;  // q-lanes per CTA: 72 (k4, tap) threads each

__global__ void __launch_bounds__(kT) stem_wgrad_staged_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ dy,
                                                               float* __restrict__ partial, int N, int S,
                                                               int rows_per_chunk) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  extern __shared__ float4 ssm[];
  const int P = S / 2;
  float4* xs = ssm;                             // [3][S + 2] pixels (c0, c1, c2, 0), column -1 .. S
  float4* gs = ssm + 3 * (S + 2);               // [P][8] = 32 k as 8 float4
  __shared__ float red[kStemLanes][72][4];
  const int t = threadIdx.x;
  const int lane_q = t / 72;                    // q-lane
  const int pair = t - lane_q * 72;             // (k4, tap)
  const int k4 = pair / 9, tap = pair - k4 * 9;
  const int r = tap / 3, sc = tap - r * 3;
  float acc[4][3] = {};
  const int r0 = blockIdx.x * rows_per_chunk;
  const int r1 = min(N * P, r0 + rows_per_chunk);
  for (int row = r0; row < r1; ++row) {
    const int p = row % P, n = row / P;
    __syncthreads();  // previous row's compute done
    for (int i = t; i < 3 * (S + 2); i += blockDim.x) {
      const int rr = i / (S + 2), w = i - rr * (S + 2) - 1;
      const int h = 2 * p + rr - 1;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (h >= 0 && h < S && w >= 0 && w < S) {
        const uint2 u = *reinterpret_cast<const uint2*>(x + ((static_cast<size_t>(n) * S + h) * S + w) * 16);
        v = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                        0.f);
      }
      xs[i] = v;
    }
    const __nv_bfloat16* grow = dy + static_cast<size_t>(row) * P * 32;
    for (int i = t; i < P * 8; i += blockDim.x) {
      const uint2 u = *reinterpret_cast<const uint2*>(grow + 4 * static_cast<size_t>(i));
      gs[i] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                          __uint_as_float(u.y & 0xFFFF0000u));
    }
    __syncthreads();
    if (lane_q < kStemLanes) {
      const float4* xr = xs + r * (S + 2) + sc;  // column 2q + sc - 1 -> index 2q + sc
      for (int q = lane_q; q < P; q += kStemLanes) {
        const float4 g = gs[q * 8 + k4];
        const float4 xv = xr[2 * q];
        const float gg[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[j][0] = fmaf(gg[j], xv.x, acc[j][0]);
          acc[j][1] = fmaf(gg[j], xv.y, acc[j][1]);
          acc[j][2] = fmaf(gg[j], xv.z, acc[j][2]);
        }
      }
    }
  }
  // CTA partial: lanes added in lane order; layout = the weight layout [32][3][3][16] (pad channels 0)
  float* out = partial + static_cast<size_t>(blockIdx.x) * (32 * 9 * 16);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    __syncthreads();
    if (lane_q < kStemLanes)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[lane_q][pair][j] = acc[j][c];
    __syncthreads();
    for (int o = t; o < 72 * 4; o += blockDim.x) {
      const int pr = o / 4, j = o - pr * 4;
      float v = 0.f;
#pragma unroll
      for (int l = 0; l < kStemLanes; ++l) v += red[l][pr][j];
      const int kk = (pr / 9) * 4 + j, tp = pr % 9;
      out[(kk * 9 + tp) * 16 + c] = v;
    }
  }
  for (int o = t; o < 32 * 9 * 13; o += blockDim.x) {
    const int k = o / (9 * 13), rem = o % (9 * 13);
    out[(k * 9 + rem / 13) * 16 + 3 + rem % 13] = 0.0f;
  }
}

// ------------------------------------------------------------------ stem 3x3 / stride 2 (3 -> 32)
// x: [N][S][S][16] bf16 (channels 3..15 zero), w: [32][3][3][16] bf16 (the product layout);
// y[n,p,q,k] = fmaf chain over (r, s, c < 3).  Thread = (output pixel, 16 output channels); the
// channel half is warp-uniform (32 consecutive pixels per warp), so every filter read is a
// broadcast float4 from shared memory.  Measured per launch (MobileNetV2 b=256, 224²): 8 channels
// per thread 419 µs, 16 channels 315 µs, all 32 channels 407 µs (181 registers, one CTA per SM).
__global__ void __launch_bounds__(kT) stem_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const __nv_bfloat16* __restrict__ w,
                                                      const float* __restrict__ bias, __nv_bfloat16* __restrict__ y,
                                                      int N, int S, int relu6) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  __shared__ __align__(16) float ws[27][32];  // [r*9 + s*3 + c][k]
  for (int i = threadIdx.x; i < 27 * 32; i += blockDim.x) {
    const int k = i % 32, t = i / 32;
    ws[t][k] = __bfloat162float(w[(k * 9 + t / 3) * 16 + t % 3]);
  }
  __syncthreads();
  const int P = S / 2;
  const int npix = N * P * P;
  const int total = (npix + 31) / 32 * 64;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = (i >> 5) & 1;
    const int pix = ((i >> 6) << 5) | (i & 31);
    if (pix >= npix) continue;
    const int q = pix % P;
    const int p = (pix / P) % P;
    const int n = pix / (P * P);
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0f;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int h = 2 * p + r - 1;
      if (h < 0 || h >= S) continue;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int ww = 2 * q + s - 1;
        if (ww < 0 || ww >= S) continue;
        const uint2 v = *reinterpret_cast<const uint2*>(x + ((static_cast<size_t>(n) * S + h) * S + ww) * 16);
        const float xc[3] = {__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xFFFF0000u),
                             __uint_as_float(v.y << 16)};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float4* wr = reinterpret_cast<const float4*>(&ws[r * 9 + s * 3 + c][g * 16]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 wv = wr[u];
            acc[4 * u + 0] = fmaf(xc[c], wv.x, acc[4 * u + 0]);
            acc[4 * u + 1] = fmaf(xc[c], wv.y, acc[4 * u + 1]);
            acc[4 * u + 2] = fmaf(xc[c], wv.z, acc[4 * u + 2]);
            acc[4 * u + 3] = fmaf(xc[c], wv.w, acc[4 * u + 3]);
          }
        }
      }
    }
#pragma unroll
    for (int h8 = 0; h8 < 2; ++h8) {
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float v = acc[8 * h8 + j];
        if (bias != nullptr) v = v + bias[g * 16 + 8 * h8 + j];
        o[j] = act_fn(relu6, v);
      }
      st8(y + static_cast<size_t>(pix) * 32 + g * 16 + 8 * h8, o);
    }
  }
}

// dw[k][r][s][c] (c < 3; pad channels stay 0) = sum_pix dy[pix][k] x[...][c].  Pass 1: warp lane =
// output channel k, 8 warps split the chunk's pixels, 27 fp32 sums per lane; warps added in order.
__global__ void __launch_bounds__(kT) stem_wgrad_partial_kernel(const __nv_bfloat16* __restrict__ x,
                                                                const __nv_bfloat16* __restrict__ dy,
                                                                float* __restrict__ partial, int N, int S,
                                                                int rows_per_chunk) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  __shared__ float red[8][27][32];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int P = S / 2;
  const int r0 = blockIdx.x * rows_per_chunk;
  const int r1 = min(N * P, r0 + rows_per_chunk);
  float acc[27];
#pragma unroll
  for (int t = 0; t < 27; ++t) acc[t] = 0.0f;
  for (int row = r0 + wp; row < r1; row += 8) {  // output row (n, p)
    const int p = row % P;
    const int n = row / P;
    const __nv_bfloat16* grow = dy + static_cast<size_t>(row) * P * 32 + lane;
    // the three input rows of this output row, clamped; out-of-image taps contribute 0 * x (branch-free)
    float hv[3];
    const __nv_bfloat16* xr[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int h = 2 * p + r - 1;
      hv[r] = (h >= 0 && h < S) ? 1.0f : 0.0f;
      xr[r] = x + (static_cast<size_t>(n) * S + min(max(h, 0), S - 1)) * S * 16;
    }
#pragma unroll 2
    for (int q = 0; q < P; ++q) {
      const float g = __bfloat162float(grow[static_cast<size_t>(q) * 32]);
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int ww = 2 * q + s - 1;
        const float wv = (ww >= 0 && ww < S) ? 1.0f : 0.0f;
        const int wc = min(max(ww, 0), S - 1);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const uint2 v = *reinterpret_cast<const uint2*>(xr[r] + static_cast<size_t>(wc) * 16);
          const float gm = g * (hv[r] * wv);
          acc[r * 9 + s * 3 + 0] = fmaf(gm, __uint_as_float(v.x << 16), acc[r * 9 + s * 3 + 0]);
          acc[r * 9 + s * 3 + 1] = fmaf(gm, __uint_as_float(v.x & 0xFFFF0000u), acc[r * 9 + s * 3 + 1]);
          acc[r * 9 + s * 3 + 2] = fmaf(gm, __uint_as_float(v.y << 16), acc[r * 9 + s * 3 + 2]);
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 27; ++t) red[wp][t][lane] = acc[t];
  __syncthreads();
  for (int o = threadIdx.x; o < 27 * 32; o += kT) {
    const int t = o / 32, k = o % 32;
    float s = 0.0f;
    for (int i = 0; i < 8; ++i) s += red[i][t][k];
    // partial layout = the weight layout [32][3][3][16] (pad channels written as 0 here)
    partial[blockIdx.x * (32 * 9 * 16) + (k * 9 + t / 3) * 16 + t % 3] = s;
  }
  for (int o = threadIdx.x; o < 32 * 9 * 13; o += kT) {
    const int k = o / (9 * 13), rem = o % (9 * 13);
    partial[blockIdx.x * (32 * 9 * 16) + (k * 9 + rem / 13) * 16 + 3 + rem % 13] = 0.0f;
  }
}

// ------------------------------------------------------------------ BN apply (affine) + act [+ residual]
// Thread = one 8-channel group for rows slot, slot + rpp, ... (cg = C/8 groups, rpp = 256/cg rows
// per CTA pass), so A, B live in registers for the whole kernel.
template <int ACT, bool RES>
__global__ void __launch_bounds__(kT) bn_apply_act_kernel(const __nv_bfloat16* __restrict__ y,
                                                          const float* __restrict__ mean_rstd,
                                                          const float* __restrict__ gamma,
                                                          const float* __restrict__ beta,
                                                          const __nv_bfloat16* __restrict__ res,
                                                          __nv_bfloat16* __restrict__ out, int m, int C) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  const int cg = C / 8;
  const int rpp = kT / cg;
  const int g = threadIdx.x % cg;
  const int slot = threadIdx.x / cg;
  if (slot >= rpp) return;
  const int c0 = g * 8;
  float A[8], B[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    A[j] = gamma[c0 + j] * mean_rstd[C + c0 + j];
    B[j] = fmaf(-A[j], mean_rstd[c0 + j], beta[c0 + j]);
  }
  for (int r = blockIdx.x * rpp + slot; r < m; r += gridDim.x * rpp) {
    const size_t off = static_cast<size_t>(r) * C + c0;
    float f[8], rv[8];
    ld8(y + off, f);
    if (RES) ld8(res + off, rv);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float z = fmaf(A[j], f[j], B[j]);
      if (ACT == 6) z = relu6f(z);
      if (RES) z = z + rv[j];
      f[j] = z;
    }
    st8(out + off, f);
  }
}

// ------------------------------------------------------------------ MSE loss on z = BN(y) [+ res]
// g = bf16((z - t) * gscale); per-CTA loss partial (fp64 per thread, fixed-order CTA tree),
// then one CTA sums the partials in chunk order.
__global__ void __launch_bounds__(kT) mse_affine_partial_kernel(const __nv_bfloat16* __restrict__ y,
                                                                const float* __restrict__ mean_rstd,
                                                                const float* __restrict__ gamma,
                                                                const float* __restrict__ beta,
                                                                const __nv_bfloat16* __restrict__ res,
                                                                const __nv_bfloat16* __restrict__ t, long long m,
                                                                int C, float gscale, __nv_bfloat16* __restrict__ g,
                                                                double* __restrict__ loss_partial) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  __shared__ double sm[kT / 32];
  const int G = C / 8;
  const long long total = m * G;
  double ls = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c0 = static_cast<int>(i % G) * 8;
    const size_t off = static_cast<size_t>(i / G) * C + c0;
    float f[8], tv[8], rv[8];
    ld8(y + off, f);
    ld8(t + off, tv);
    if (res != nullptr) ld8(res + off, rv);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      const float A = gamma[c] * mean_rstd[C + c];
      const float B = fmaf(-A, mean_rstd[c], beta[c]);
      float z = fmaf(A, f[j], B);
      if (res != nullptr) z = z + rv[j];
      const float d = z - tv[j];
      ls += static_cast<double>(d) * d;
      f[j] = d * gscale;
    }
    st8(g + off, f);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = ls;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kT / 32; ++w) s += sm[w];
    loss_partial[blockIdx.x] = s;
  }
}

// one CTA: strided per-thread sums, xor-shuffle tree per warp, warps added in order (deterministic)
__global__ void loss_sum_kernel(const double* __restrict__ part, int n, double norm, double* __restrict__ loss) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  __shared__ double sm[kT / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kT / 32; ++w) t += sm[w];
    *loss = t / norm;
  }
}

// ------------------------------------------------------------------ squeeze-excite (EfficientNet teacher)
// pooled[n][c] = (sum_q y[n][q][c]) / hw: CTA per (n, 8-channel group window of 32 groups); threads
// stride over q in double, fixed-order tree over the CTA.
// pooled[n][c] = mean over the hw pixels of y[n][.][c].  CTA = (sample, 32 channel groups):
// a warp reads 32 consecutive 16-byte channel vectors of one pixel (coalesced), 8 pixel slots per CTA.
// (One CTA per 8-channel group strided the pixels at E*2 bytes: 32 sectors per warp load, 1.9 TB/s.)
constexpr int kPoolSlots = kT / 32;
__global__ void __launch_bounds__(kT) se_pool_kernel(const __nv_bfloat16* __restrict__ y, int hw, int E,
                                                     float* __restrict__ pooled) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  __shared__ double red[kPoolSlots][32][8];
  const int n = blockIdx.x;
  const int gl = threadIdx.x & 31, slot = threadIdx.x >> 5;
  const int g = blockIdx.y * 32 + gl;  // 8-channel group
  const bool live = g < E / 8;
  // per-thread fp32 sums over its pixel slot (the fp64 adds were the limit), fp64 across slots
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (live) {
    const __nv_bfloat16* base = y + static_cast<size_t>(n) * hw * E + g * 8;
#pragma unroll 4
    for (int q = slot; q < hw; q += kPoolSlots) {
      float f[8];
      ld8(base + static_cast<size_t>(q) * E, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += f[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[slot][gl][j] = acc[j];
  __syncthreads();
  for (int o = threadIdx.x; o < 32 * 8; o += kT) {
    const int gg = o / 8, j = o % 8;
    const int go = blockIdx.y * 32 + gg;
    if (go >= E / 8) continue;
    double t = 0.0;
    for (int sl = 0; sl < kPoolSlots; ++sl) t += red[sl][gg][j];
    pooled[static_cast<size_t>(n) * E + go * 8 + j] = static_cast<float>(t / hw);
  }
}

// gate[n][c] = sigmoid(b2[c] + W2[c] . swish(b1 + W1 pooled[n])): one CTA per sample, fmaf order of
// the oracle (c ascending for W1, j ascending for W2); bf16 weights, fp32 math.
__global__ void __launch_bounds__(kT) se_fc_kernel(const float* __restrict__ pooled, const __nv_bfloat16* __restrict__ w1,
                                                   const float* __restrict__ b1, const __nv_bfloat16* __restrict__ w2,
                                                   const float* __restrict__ b2, int E, int cs,
                                                   float* __restrict__ gate) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  extern __shared__ float sm[];  // pooled[E], h[cs]
  float* pl = sm;
  float* h = sm + E;
  const int n = blockIdx.x;
  for (int c = threadIdx.x; c < E; c += kT) pl[c] = pooled[static_cast<size_t>(n) * E + c];
  __syncthreads();
  // FC1: one warp per hidden unit, lanes stride the E inputs (coalesced weight rows), fixed xor tree
  // (a thread walking E serially left the SM idle: 47 us per launch)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < cs; j += kT / 32) {
    const __nv_bfloat16* wr = w1 + static_cast<size_t>(j) * E;
    float acc = 0.0f;
    for (int c = lane; c < E; c += 32) acc = fmaf(__bfloat162float(wr[c]), pl[c], acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) h[j] = swishf(acc + b1[j]);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < E; c += kT) {
    float acc = b2[c];
    const __nv_bfloat16* wr = w2 + static_cast<size_t>(c) * cs;
    for (int j = 0; j < cs; ++j) acc = fmaf(__bfloat162float(wr[j]), h[j], acc);
    gate[static_cast<size_t>(n) * E + c] = sigmoidf(acc);
  }
}

// y[n][q][c] = bf16(y * gate[n][c]) in place
__global__ void __launch_bounds__(kT) se_scale_kernel(__nv_bfloat16* __restrict__ y, const float* __restrict__ gate,
                                                      int hw, int E, int total) {
  grid_dep_wait();  // PDL (mb_launch): every global access comes after this
  const int G = E / 8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % G;
    const int pix = i / G;
    const int n = pix / hw;
    float f[8];
    __nv_bfloat16* p = y + static_cast<size_t>(pix) * E + g * 8;
    ld8(p, f);
    const float* gt = gate + static_cast<size_t>(n) * E + g * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] * gt[j];
    st8(p, f);
  }
}

template <int K>
cudaError_t launch_dw_fwd(int st, const DwArgs& d, const void* x, const void* wt, const float* bias, void* y,
                          int relu6, cudaStream_t s) {
  const int g = grid_for(static_cast<long long>(d.n) * d.p * ((d.q + kQT - 1) / kQT) * (d.c / 8));
  if (st == 1)
    mb_launch(dw_fwd_kernel<K, 1>, dim3(g), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(x),
                                         static_cast<const __nv_bfloat16*>(wt), bias,
                                         static_cast<__nv_bfloat16*>(y), d.n, d.h, d.w, d.c, d.p, d.q, relu6);
  else
    mb_launch(dw_fwd_kernel<K, 2>, dim3(g), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(x),
                                         static_cast<const __nv_bfloat16*>(wt), bias,
                                         static_cast<__nv_bfloat16*>(y), d.n, d.h, d.w, d.c, d.p, d.q, relu6);
  return cudaGetLastError();
}

template <int K>
cudaError_t launch_dw_dgrad(int st, const DwArgs& d, const void* dy, const void* wt, const void* act, void* dx,
                            cudaStream_t s) {
  const int g = grid_for(static_cast<long long>(d.n) * d.h * d.w * (d.c / 8));
  auto* a = static_cast<const __nv_bfloat16*>(act);
  if (st == 1)
    mb_launch(dw_dgrad_kernel<K, 1>, dim3(g), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(dy),
                                           static_cast<const __nv_bfloat16*>(wt), a,
                                           static_cast<__nv_bfloat16*>(dx), d.n, d.h, d.w, d.c, d.p, d.q, false);
  else
    mb_launch(dw_dgrad_kernel<K, 2>, dim3(g), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(dy),
                                           static_cast<const __nv_bfloat16*>(wt), a,
                                           static_cast<__nv_bfloat16*>(dx), d.n, d.h, d.w, d.c, d.p, d.q,
                                           d.h % 2 == 0 && d.w % 2 == 0);
  return cudaGetLastError();
}

struct WgradTiling {
  int lanes_c, cwin, chunks, per_chunk;  // per_chunk = output rows (n, p) per chunk
};

WgradTiling dw_wgrad_tiling(const DwArgs& d) {
  WgradTiling t;
  const int G = d.c / 8;
  t.lanes_c = std::min(G, 32);
  t.cwin = (G + t.lanes_c - 1) / t.lanes_c;
  const int rows = d.n * d.p;
  const int lanes_p = 256 / t.lanes_c;
  const int target = 148 * 4;
  // every row lane of a chunk walks >= 2 whole output rows
  t.chunks = std::max(1, std::min(rows / (2 * lanes_p) + 1, target / (t.cwin * d.k) + 1));
  t.per_chunk = (rows + t.chunks - 1) / t.chunks;
  t.chunks = (rows + t.per_chunk - 1) / t.per_chunk;
  return t;
}

template <int K>
cudaError_t launch_dw_wgrad(int st, const DwArgs& d, const void* a, const void* dy, float* partial, float* dw,
                            cudaStream_t s) {
  const WgradTiling t = dw_wgrad_tiling(d);
  const dim3 grid(t.chunks, t.cwin, K);
  if (st == 1)
    mb_launch(dw_wgrad_partial_kernel<K, 1>, dim3(grid), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(a),
                                                      static_cast<const __nv_bfloat16*>(dy), partial, d.n, d.h, d.w,
                                                      d.c, d.p, d.q, t.lanes_c, t.per_chunk);
  else
    mb_launch(dw_wgrad_partial_kernel<K, 2>, dim3(grid), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(a),
                                                      static_cast<const __nv_bfloat16*>(dy), partial, d.n, d.h, d.w,
                                                      d.c, d.p, d.q, t.lanes_c, t.per_chunk);
  const size_t n = static_cast<size_t>(d.c) * K * K;
  mb_launch(chunk_sum_kernel, dim3(static_cast<int>((n + 31) / 32)), dim3(dim3(32, kSumLanes)), 0, s, partial, t.chunks, n, dw);
  return cudaGetLastError();
}

bool dw_ok(const DwArgs& d) {
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.c % 8 != 0 || d.c < 8) return false;
  if (d.k != 3 && d.k != 5 && d.k != 7) return false;
  if (d.stride != 1 && d.stride != 2) return false;
  const int pad = d.k / 2;
  if (static_cast<long long>(d.n) * d.h * d.w * d.c >= (1LL << 31)) return false;  // 32-bit work indices
  return d.p == (d.h + 2 * pad - d.k) / d.stride + 1 && d.q == (d.w + 2 * pad - d.k) / d.stride + 1;
}

int stem_chunk_rows(int n, int S) {  // output rows (n, p) per chunk: ~2 waves of CTAs
  const int rows = n * (S / 2);
  const int chunks = std::max(1, std::min(148 * 8, rows / 8 + 1));
  return (rows + chunks - 1) / chunks;
}

}  // namespace

size_t dw_wgrad_workspace_floats(const DwArgs& d) {
  if (!dw_ok(d)) return 0;
  return static_cast<size_t>(dw_wgrad_tiling(d).chunks) * d.c * d.k * d.k;
}

// staged-tile plan of dw_fwd_tiled_kernel: CT channels per tile (64 / 128 for narrow maps), TP output rows
// = the largest that fits kDwTileBytes, rounded down to a whole number of 256-item rounds when possible
struct DwTilePlan {
  int ct = 0, tp = 0;
  size_t smem = 0;
};
DwTilePlan dw_tile_plan(const DwArgs& d) {
  DwTilePlan t;
  if (pbd::knob_env("PBDK_DW_TILED") != nullptr && std::atoi(pbd::knob_env("PBDK_DW_TILED")) == 0) return t;
  int ct = d.q <= 7 && d.c % 128 == 0 ? 128 : d.q <= 14 && d.c % 64 == 0 ? 64 : d.c % 32 == 0 ? 32 : 0;
  if (ct == 0) return t;
  const int cols_in = (d.q - 1) * d.stride + d.k;
  if (cols_in > 256) return t;  // TMA box extent
  const size_t row_bytes = static_cast<size_t>(cols_in) * ct * 2;
  const size_t w_bytes = static_cast<size_t>(d.k) * d.k * ct * 2;
  const int rows_max = static_cast<int>((kDwTileBytes - w_bytes) / row_bytes);
  if (rows_max < d.k) return t;
  const int tp_max = std::min({d.p, (rows_max - d.k) / d.stride + 1, (256 - d.k) / d.stride + 1});
  const int per_row = ((d.q + dw_qt(d.k) - 1) / dw_qt(d.k)) * (ct / 8);
  int tp = tp_max;
  for (int c = tp_max; c >= 1; --c)  // prefer whole 256-item rounds (no idle half-round at the barrier)
    if ((c * per_row) % kT == 0) {
      tp = c;
      break;
    }
  if (tp < tp_max / 2) tp = tp_max;
  t.ct = ct;
  t.tp = tp;
  const size_t rows_in = static_cast<size_t>(tp - 1) * d.stride + d.k;
  t.smem = kDwStages * ((((rows_in * row_bytes + 127) / 128 * 128) + w_bytes + 127) / 128 * 128) + 128;
  return t;
}

template <int K, int ST, int CT, bool DG = false>
cudaError_t launch_dw_fwd_tiled(const DwArgs& d, const DwTilePlan& t, const void* x, const void* wt,
                                const float* bias, void* y, int act, cudaStream_t s, const void* amask = nullptr) {
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(dw_fwd_tiled_kernel<K, ST, CT, DG>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               kDwStages * (kDwTileBytes + 256) + 128);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tmx, tmw;
  {
    const int cols_in = (d.q - 1) * d.stride + d.k, rows_in = (t.tp - 1) * d.stride + d.k;
    const uint64_t dims[4] = {static_cast<uint64_t>(d.c), static_cast<uint64_t>(d.w), static_cast<uint64_t>(d.h),
                              static_cast<uint64_t>(d.n)};
    const uint64_t strides[3] = {static_cast<uint64_t>(d.c) * 2, static_cast<uint64_t>(d.w) * d.c * 2,
                                 static_cast<uint64_t>(d.h) * d.w * d.c * 2};
    const uint32_t box[4] = {static_cast<uint32_t>(CT), static_cast<uint32_t>(cols_in),
                             static_cast<uint32_t>(rows_in), 1};
    const uint32_t es[4] = {1, 1, 1, 1};
    if (!encode_tmap_bf16(&tmx, x, 4, dims, strides, box, es, 0)) return cudaErrorInvalidValue;
    const uint64_t wd[2] = {static_cast<uint64_t>(d.c), static_cast<uint64_t>(K * K)};
    const uint64_t ws[1] = {static_cast<uint64_t>(d.c) * 2};
    const uint32_t wb[2] = {static_cast<uint32_t>(CT), static_cast<uint32_t>(K * K)};
    const uint32_t we[2] = {1, 1};
    if (!encode_tmap_bf16(&tmw, wt, 2, wd, ws, wb, we, 0)) return cudaErrorInvalidValue;
  }
  const long long tiles = static_cast<long long>(d.n) * ((d.p + t.tp - 1) / t.tp) * (d.c / CT);
  const int per_sm = t.smem * 2 <= 200 * 1024 ? 2 : 1;
  const int grid = static_cast<int>(std::min<long long>(tiles, 148LL * per_sm));
  mb_launch(dw_fwd_tiled_kernel<K, ST, CT, DG>, dim3(grid), dim3(kT), t.smem, s, tmx, tmw, bias, static_cast<__nv_bfloat16*>(y), d.n,
                                                             d.c, d.p, d.q, act, t.tp,
                                                             static_cast<const __nv_bfloat16*>(amask));
  return cudaGetLastError();
}

template <int K>
cudaError_t dw_fwd_tiled(const DwArgs& d, const DwTilePlan& t, const void* x, const void* wt, const float* bias,
                         void* y, int act, cudaStream_t s) {
  if (d.stride == 1)
    return t.ct == 128 ? launch_dw_fwd_tiled<K, 1, 128>(d, t, x, wt, bias, y, act, s)
           : t.ct == 64 ? launch_dw_fwd_tiled<K, 1, 64>(d, t, x, wt, bias, y, act, s)
                        : launch_dw_fwd_tiled<K, 1, 32>(d, t, x, wt, bias, y, act, s);
  return t.ct == 128 ? launch_dw_fwd_tiled<K, 2, 128>(d, t, x, wt, bias, y, act, s)
         : t.ct == 64 ? launch_dw_fwd_tiled<K, 2, 64>(d, t, x, wt, bias, y, act, s)
                      : launch_dw_fwd_tiled<K, 2, 32>(d, t, x, wt, bias, y, act, s);
}

int dw_fwd(const DwArgs& d, const void* x, const void* wt, const float* bias, void* y, int relu6, cudaStream_t s,
           int variant) {
  if (!dw_ok(d)) return PBDK_EINVAL;
  const DwTilePlan t = dw_tile_plan(d);
  if (variant == 1 && t.ct == 0) return PBDK_EINVAL;
  if (variant != 0 && t.ct != 0) {
    switch (d.k) {
      case 3: return ok(dw_fwd_tiled<3>(d, t, x, wt, bias, y, relu6, s));
      case 5: return ok(dw_fwd_tiled<5>(d, t, x, wt, bias, y, relu6, s));
      default: return ok(dw_fwd_tiled<7>(d, t, x, wt, bias, y, relu6, s));
    }
  }
  switch (d.k) {
    case 3: return ok(launch_dw_fwd<3>(d.stride, d, x, wt, bias, y, relu6, s));
    case 5: return ok(launch_dw_fwd<5>(d.stride, d, x, wt, bias, y, relu6, s));
    default: return ok(launch_dw_fwd<7>(d.stride, d, x, wt, bias, y, relu6, s));
  }
}

// stride-1 data gradient on the staged tiles: the tile geometry of the forward over dy (H = P, W = Q)
template <int K>
cudaError_t dw_dgrad_tiled(const DwArgs& d, const DwTilePlan& t, const void* dy, const void* wt, const void* act,
                           void* dx, cudaStream_t s) {
  const DwArgs g{d.n, d.p, d.q, d.c, d.k, 1, d.h, d.w};
  return t.ct == 128 ? launch_dw_fwd_tiled<K, 1, 128, true>(g, t, dy, wt, nullptr, dx, 0, s, act)
         : t.ct == 64 ? launch_dw_fwd_tiled<K, 1, 64, true>(g, t, dy, wt, nullptr, dx, 0, s, act)
                      : launch_dw_fwd_tiled<K, 1, 32, true>(g, t, dy, wt, nullptr, dx, 0, s, act);
}

int dw_dgrad(const DwArgs& d, const void* dy, const void* wt, const void* act, void* dx, cudaStream_t s,
             int variant) {
  if (!dw_ok(d)) return PBDK_EINVAL;
  if (variant != 0 && d.stride == 1) {
    const DwTilePlan t = dw_tile_plan(d);  // stride 1: the same geometry as the forward
    if (t.ct != 0) {
      switch (d.k) {
        case 3: return ok(dw_dgrad_tiled<3>(d, t, dy, wt, act, dx, s));
        case 5: return ok(dw_dgrad_tiled<5>(d, t, dy, wt, act, dx, s));
        default: return ok(dw_dgrad_tiled<7>(d, t, dy, wt, act, dx, s));
      }
    }
  }
  if (variant == 1) return PBDK_EINVAL;
  switch (d.k) {
    case 3: return ok(launch_dw_dgrad<3>(d.stride, d, dy, wt, act, dx, s));
    case 5: return ok(launch_dw_dgrad<5>(d.stride, d, dy, wt, act, dx, s));
    default: return ok(launch_dw_dgrad<7>(d.stride, d, dy, wt, act, dx, s));
  }
}

int dw_wgrad(const DwArgs& d, const void* a, const void* dy, float* ws, size_t ws_floats, float* dw, cudaStream_t s) {
  if (!dw_ok(d) || ws == nullptr || ws_floats < dw_wgrad_workspace_floats(d)) return PBDK_EINVAL;
  switch (d.k) {
    case 3: return ok(launch_dw_wgrad<3>(d.stride, d, a, dy, ws, dw, s));
    case 5: return ok(launch_dw_wgrad<5>(d.stride, d, a, dy, ws, dw, s));
    default: return ok(launch_dw_wgrad<7>(d.stride, d, a, dy, ws, dw, s));
  }
}

int stem_fwd(const void* x, const void* w, const float* bias, void* y, int n, int S, int relu6, cudaStream_t s) {
  if (n < 1 || S < 2 || S % 2 != 0 || static_cast<long long>(n) * S * S >= (1LL << 29)) return PBDK_EINVAL;
  mb_launch(stem_fwd_kernel, dim3(grid_for((static_cast<long long>(n) * (S / 2) * (S / 2) + 31) / 32 * 64)), dim3(kT), 0, s, 
      static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w), bias,
      static_cast<__nv_bfloat16*>(y), n, S, relu6);
  return ok(cudaGetLastError());
}

size_t stem_wgrad_workspace_floats(int n, int S) {
  const int rows = n * (S / 2);
  const int per = stem_chunk_rows(n, S);
  return static_cast<size_t>((rows + per - 1) / per) * 32 * 9 * 16;
}

int stem_wgrad(const void* x, const void* dy, int n, int S, float* ws, size_t ws_floats, float* dw, cudaStream_t s) {
  if (n < 1 || S < 2 || S % 2 != 0 || ws == nullptr || ws_floats < stem_wgrad_workspace_floats(n, S))
    return PBDK_EINVAL;
  const int rows = n * (S / 2);
  const int per = stem_chunk_rows(n, S);
  const int chunks = (rows + per - 1) / per;
  const size_t smem = (3 * static_cast<size_t>(S + 2) + static_cast<size_t>(S / 2) * 8) * sizeof(float4);
  static const bool staged = [] {  // PBDK_STEM_STAGED=0: the register kernel (A/B runs)
    const char* e = pbd::knob_env("PBDK_STEM_STAGED");
    return e == nullptr || e[0] != '0';
  }();
  if (staged && smem <= 48 * 1024) {
    mb_launch(stem_wgrad_staged_kernel, dim3(chunks), dim3(kT), smem, s, static_cast<const __nv_bfloat16*>(x),
                                                      static_cast<const __nv_bfloat16*>(dy), ws, n, S, per);
  } else {
    mb_launch(stem_wgrad_partial_kernel, dim3(chunks), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(x),
                                                    static_cast<const __nv_bfloat16*>(dy), ws, n, S, per);
  }
  mb_launch(chunk_sum_kernel, dim3((32 * 9 * 16 + 31) / 32), dim3(dim3(32, kSumLanes)), 0, s, ws, chunks, 32 * 9 * 16, dw);
  return ok(cudaGetLastError());
}

int bn_apply_act(const void* y, const float* mean_rstd, const float* gamma, const float* beta, const void* res,
                 void* out, long long m, int c, int relu6, cudaStream_t s) {
  if (c % 8 != 0 || c / 8 > kT || m < 1 || m >= (1LL << 31)) return PBDK_EINVAL;
  const int rpp = kT / (c / 8);
  const int g = static_cast<int>(std::max<long long>(1, std::min<long long>((m + rpp - 1) / rpp, 148LL * 8)));
  auto* yy = static_cast<const __nv_bfloat16*>(y);
  auto* rr = static_cast<const __nv_bfloat16*>(res);
  auto* oo = static_cast<__nv_bfloat16*>(out);
  if (relu6 && res == nullptr)
    mb_launch(bn_apply_act_kernel<6, false>, dim3(g), dim3(kT), 0, s, yy, mean_rstd, gamma, beta, rr, oo, static_cast<int>(m), c);
  else if (!relu6 && res == nullptr)
    mb_launch(bn_apply_act_kernel<0, false>, dim3(g), dim3(kT), 0, s, yy, mean_rstd, gamma, beta, rr, oo, static_cast<int>(m), c);
  else if (!relu6)
    mb_launch(bn_apply_act_kernel<0, true>, dim3(g), dim3(kT), 0, s, yy, mean_rstd, gamma, beta, rr, oo, static_cast<int>(m), c);
  else
    return PBDK_EINVAL;
  return ok(cudaGetLastError());
}

int se_apply(void* y, int n, int hw, int E, int cs, const void* w1, const float* b1, const void* w2,
             const float* b2, float* pooled, float* gate, cudaStream_t s) {
  if (E % 8 != 0 || cs < 1 || n < 1 || static_cast<long long>(n) * hw * E >= (1LL << 31)) return PBDK_EINVAL;
  mb_launch(se_pool_kernel, dim3(dim3(n, (E / 8 + 31) / 32)), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(y), hw, E, pooled);
  mb_launch(se_fc_kernel, dim3(n), dim3(kT), (E + cs) * sizeof(float), s, pooled, static_cast<const __nv_bfloat16*>(w1), b1,
                                                        static_cast<const __nv_bfloat16*>(w2), b2, E, cs, gate);
  const int total = n * hw * (E / 8);
  mb_launch(se_scale_kernel, dim3(grid_for(total)), dim3(kT), 0, s, static_cast<__nv_bfloat16*>(y), gate, hw, E, total);
  return ok(cudaGetLastError());
}

size_t mse_affine_workspace_doubles(long long m, int c) { return static_cast<size_t>(grid_for(m * (c / 8))); }

int mse_affine(const void* y, const float* mean_rstd, const float* gamma, const float* beta, const void* res,
               const void* t, long long m, int c, float gscale, double norm, void* g, double* ws, double* loss,
               cudaStream_t s) {
  if (c % 8 != 0 || m < 1) return PBDK_EINVAL;
  const int grid = grid_for(m * (c / 8));
  mb_launch(mse_affine_partial_kernel, dim3(grid), dim3(kT), 0, s, static_cast<const __nv_bfloat16*>(y), mean_rstd, gamma, beta,
                                                static_cast<const __nv_bfloat16*>(res),
                                                static_cast<const __nv_bfloat16*>(t), m, c, gscale,
                                                static_cast<__nv_bfloat16*>(g), ws);
  mb_launch(loss_sum_kernel, dim3(1), dim3(kT), 0, s, ws, grid, norm, loss);
  return ok(cudaGetLastError());
}

}  // namespace pbdk

// ------------------------------------------------------------------ C ABI
extern "C" int pbdk_dw_dgrad(const pbdk_dw_desc* d, const void* dy, const void* wt, const void* act, void* dx,
                             int variant, void* stream) {
  if (d == nullptr || dy == nullptr || wt == nullptr || dx == nullptr || variant < -1 || variant > 1)
    return PBDK_EINVAL;
  const pbdk::DwArgs a{d->n, d->h, d->w, d->c, d->k, d->stride, d->p, d->q};
  return pbdk::dw_dgrad(a, dy, wt, act, dx, static_cast<cudaStream_t>(stream), variant);
}

extern "C" int pbdk_dw_fwd(const pbdk_dw_desc* d, const void* x, const void* wt, const float* bias, void* y, int act,
                           int variant, void* stream) {
  if (d == nullptr || x == nullptr || wt == nullptr || y == nullptr || act < 0 || act > 2 || variant < -1 ||
      variant > 1)
    return PBDK_EINVAL;
  const pbdk::DwArgs a{d->n, d->h, d->w, d->c, d->k, d->stride, d->p, d->q};
  return pbdk::dw_fwd(a, x, wt, bias, y, act, static_cast<cudaStream_t>(stream), variant);
}
