// tcgen05 implicit-GEMM convolutions for sm_100a.
//
//   fprop: D[m, k] = sum_{tap, c} X[pix(m, tap), c] * W[k, tap, c]
//          A = X tile (128 output pixels x BKC channels, K-major) via one 4D TMA box per
//          (tap, channel chunk); out-of-image taps are zero-filled by TMA OOB handling,
//          stride-2 convs use TMA element strides. B = W tile (BN x BKC, K-major).
//          Accumulator in TMEM (128 lanes x BN fp32 columns); fused epilogue.
//   wgrad: D[k, c] (per tap) = sum_m dY[m, k] * X[pix(m, tap), c]
//          A = dY tile, B = X tile, both MN-major (pixels are the reduction dim),
//          split-K over output-pixel tiles, deterministic fixed-order reduction.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (one thread),
// warps 2-5 epilogue (TMEM lane quarter = warp % 4); warp 2 owns TMEM alloc.
#include "knobs.hpp"
#include "conv.hpp"
#include "sm100.cuh"
#include "tmap.hpp"

#include <algorithm>
#include <cstdlib>

// timing-experiment modes of FpropArgs::debug: compiled out of the product build (knobs.hpp)
#define DBG_IS(args, v) (pbd::kExperiments && (args).debug == (v))
#define DBG_GE(args, v) (pbd::kExperiments && (args).debug >= (v))

namespace pbdk {

namespace {

constexpr int kThreads = 192;
constexpr int kSmemBudget = 200 * 1024;      // wgrad pipeline
constexpr int kFpropBudget = 220 * 1024;     // fprop ring + resident filter

__host__ __device__ constexpr int layout_for_sw(int sw) { return sw == 128 ? 2 : (sw == 64 ? 4 : 6); }
__host__ __device__ constexpr int round_up(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ constexpr int tmem_cols_for(int n) {
  return n <= 32 ? 32 : (n <= 64 ? 64 : (n <= 128 ? 128 : (n <= 256 ? 256 : 512)));
}

// Persistent fprop: grid = min(tiles, #SMs); each CTA walks tiles t = blockIdx.x + i*gridDim.x
// (N tile fastest, so CTAs working on one M tile at the same time share its A boxes in L2).
// Two TMEM accumulators (2*BN columns): the epilogue of tile i overlaps the MMAs of tile i+1.
// BRES: the whole filter (all K blocks of the single N tile) is loaded into shared memory once
// per CTA and stays resident; the ring then carries only the activation boxes.
template <int BN, int BKC, bool BRES>
struct FpropCfg {
  static constexpr int SW = BKC * 2;  // bytes per smem row == swizzle span
  static constexpr int LAYOUT = layout_for_sw(SW);
  static constexpr int A_BYTES = 128 * SW;
  static constexpr int B_BYTES = BN * SW;
  static constexpr int B_RES_MAX = 96 * 1024;  // resident filter budget
  static constexpr int STAGE = round_up(A_BYTES + (BRES ? 0 : B_BYTES), 1024);
  static constexpr int RING = (BRES ? kFpropBudget - B_RES_MAX : kFpropBudget);
  // small stages (16 / 32-channel inputs: 32 / 64-byte box rows) need more of them in flight
  static constexpr int MAX_STAGES = STAGE <= 4096 ? 24 : STAGE <= 8192 ? 16 : 8;
  static constexpr int STAGES = (RING / STAGE) > MAX_STAGES ? MAX_STAGES : (RING / STAGE);
  static constexpr int ACC_COLS = BN < 32 ? 32 : BN;
  // TMEM accumulators in rotation (conv_fprop_kernel): four for N <= 128 tiles (up to all 512 columns:
  // every TMEM-using kernel needs > 114 KB of shared memory, so no two of their CTAs share an SM), two above
  static constexpr int NACC = ACC_COLS <= 128 ? 4 : 2;
  static constexpr int TMEM_COLS = tmem_cols_for(NACC * ACC_COLS);
  static constexpr int BAR_BYTES = round_up(2 * STAGES * 8 + (2 * NACC + 1) * 8 + 4, 256);
  static constexpr int SMEM = STAGES * STAGE + (BRES ? B_RES_MAX : 0) + 1024 + BAR_BYTES;
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Launch with optional thread-block clusters and programmatic dependent launch (PDL: the kernel may
// start — prologue: barriers, TMEM, tensor-map prefetch — while the previous kernel in the stream
// drains; it calls grid_dep_wait() before touching global memory).
template <class... KArgs, class... Args>
cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, bool pdl,
                      unsigned cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Epilogue semantics (pbdk.h PBDK_EPI_*): y = act(aux_op(acc + bias, aux)), fp32, one bf16 rounding.
struct EpiFlags {
  bool bias, aux, add, mask0, mask6, relu, relu6, swish;
};
__host__ __device__ constexpr EpiFlags epi_flags(int e) {
  return EpiFlags{e == PBDK_EPI_BIAS || e == PBDK_EPI_BIAS_RELU || e == PBDK_EPI_BIAS_RES_RELU ||
                      e == PBDK_EPI_BIAS_RELU6 || e == PBDK_EPI_BIAS_RES || e == PBDK_EPI_BIAS_SWISH,
                  e == PBDK_EPI_BIAS_RES_RELU || e == PBDK_EPI_RELU_MASK || e == PBDK_EPI_BIAS_RES ||
                      e == PBDK_EPI_RELU6_MASK || e == PBDK_EPI_ADD,
                  e == PBDK_EPI_BIAS_RES_RELU || e == PBDK_EPI_BIAS_RES || e == PBDK_EPI_ADD,
                  e == PBDK_EPI_RELU_MASK,
                  e == PBDK_EPI_RELU6_MASK,
                  e == PBDK_EPI_BIAS_RELU || e == PBDK_EPI_BIAS_RES_RELU,
                  e == PBDK_EPI_BIAS_RELU6,
                  e == PBDK_EPI_BIAS_SWISH};
}
__device__ __forceinline__ float epi_aux(const EpiFlags& f, float v, float r) {
  if (f.add) return v + r;
  if (f.mask0) return r > 0.f ? v : 0.f;
  return (r > 0.f && r < 6.f) ? v : 0.f;  // mask6: ReLU6 backward from the stored activation
}
__device__ __forceinline__ float epi_act(const EpiFlags& f, float v) {
  if (f.relu) return fmaxf(v, 0.f);
  if (f.relu6) return fminf(fmaxf(v, 0.f), 6.f);
  if (f.swish) return __fdividef(v, 1.0f + __expf(-v));  // fast-math swish (mb_kernels.cu swishf)
  return v;
}

// Epilogue: thread = accumulator row (TMEM lane).  tcgen05.ld 16 columns at a time, fused
// bias / residual / ReLU / ReLU-mask in fp32, one bf16 rounding, 2 x 16 B stores straight
// from registers.  No shared-memory staging on purpose: for N <= 128 the tensor core is
// bound by its shared-memory read port (SS operands), so the epilogue must not compete
// for it.  RowMap(r) -> (valid, output pixel index) of tile row r.
// `wait` blocks until the tile's accumulator is complete (tfull barrier); the first column group's
// aux / bias vectors are requested BEFORE it, so their latency hides behind the tile's last MMAs.
struct NoWait {
  __device__ __forceinline__ void operator()() const {}
};

template <int BN, class RowMap, class Wait = NoWait>
__device__ __forceinline__ void fprop_epilogue(const FpropArgs& a, uint32_t trow, int row, int k0,
                                               const RowMap& rowmap, const Wait& wait = Wait()) {
  bool valid;
  size_t m;
  rowmap(row, valid, m);
  const EpiFlags f = epi_flags(a.epi);
  const bool has_bias = f.bias;
  if (DBG_IS(a, 3) || DBG_IS(a, 9) || DBG_IS(a, 7)) {
    wait();
    return;
  }
  // Columns in groups of up to 64: the group's aux (residual / mask) vectors are requested up front,
  // so one global-load latency is paid per 64 columns instead of one per 16 (the epilogue of a
  // N = 64 tile was latency-bound on them and fell behind the MMAs: 64->64 conv + residual
  // 50 -> see DESIGN.md §6).
  constexpr int GC = BN < 64 ? BN : 64;
  const bool live = valid && !DBG_IS(a, 1);
#pragma unroll 1
  for (int g0 = 0; g0 < BN; g0 += GC) {
    uint4 ra[GC / 8];
    float4 rb[GC / 4];
    if (f.aux && live) {
      const uint4* r4 = reinterpret_cast<const uint4*>(a.aux + m * a.k + k0 + g0);
#pragma unroll
      for (int i = 0; i < GC / 8; ++i) ra[i] = __ldg(r4 + i);
    }
    if (has_bias && live) {  // warp-uniform addresses: one broadcast wavefront per load
      const float4* b4 = reinterpret_cast<const float4*>(a.bias + k0 + g0);
#pragma unroll
      for (int i = 0; i < GC / 4; ++i) rb[i] = __ldg(b4 + i);
    }
    if (g0 == 0) wait();
#pragma unroll
    for (int c = 0; c < GC; c += 16) {
      float v[16];
      tmem_ld16(trow + g0 + c, v);
      if (!live) continue;
      const int col = k0 + g0 + c;
      if (has_bias) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 b = rb[c / 4 + j];
          v[4 * j + 0] += b.x;
          v[4 * j + 1] += b.y;
          v[4 * j + 2] += b.z;
          v[4 * j + 3] += b.w;
        }
      }
      if (f.aux) {
        const uint4 r0 = ra[c / 8], r1 = ra[c / 8 + 1];
        const uint32_t rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[2 * j] = epi_aux(f, v[2 * j], bf16_lo(rw[j]));
          v[2 * j + 1] = epi_aux(f, v[2 * j + 1], bf16_hi(rw[j]));
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = epi_act(f, v[j]);
      uint4 o0, o1;
      o0.x = pack_bf16x2(v[0], v[1]);
      o0.y = pack_bf16x2(v[2], v[3]);
      o0.z = pack_bf16x2(v[4], v[5]);
      o0.w = pack_bf16x2(v[6], v[7]);
      o1.x = pack_bf16x2(v[8], v[9]);
      o1.y = pack_bf16x2(v[10], v[11]);
      o1.z = pack_bf16x2(v[12], v[13]);
      o1.w = pack_bf16x2(v[14], v[15]);
      st_global_256(a.y + m * a.k + col, o0, o1);
    }
  }
}

struct TileRows {  // regular tiles: a (bn images) x (bh rows) x (bw cols) box of output pixels
  const FpropArgs* a;
  int n0, oh0, ow0;
  __device__ __forceinline__ void operator()(int row, bool& valid, size_t& m) const {
    const int iw = row % a->bw;
    const int ih = (row / a->bw) % a->bh;
    const int in = row / (a->bw * a->bh);
    const int nn = n0 + in;
    valid = nn < a->n;
    m = (static_cast<size_t>(nn) * a->p + (oh0 + ih)) * a->q + (ow0 + iw);
  }
};

struct HaloRows {  // halo tiles: 128 consecutive positions of a (W+2)-wide padded image
  const FpropArgs* a;
  int img, p0, wp;
  __device__ __forceinline__ void operator()(int row, bool& valid, size_t& m) const {
    const int p = p0 + row;
    const int h = p / wp;
    const int w = p - h * wp;
    valid = h < a->p && w < a->q;
    m = (static_cast<size_t>(img) * a->p + h) * a->q + w;
  }
};

// EPW epilogue warps per TMEM lane quarter (each takes BN/EPW columns): 2 for convs whose short K
// leaves the tile's epilogue, not its MMAs, on the critical path.
constexpr int epi_threads(int epw) { return 64 + 128 * epw; }

template <int BN, int BKC, bool BRES, int EPW = 1>
__global__ void __launch_bounds__(epi_threads(EPW), 1)
    conv_fprop_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                      const FpropArgs a) {
  using C = FpropCfg<BN, BKC, BRES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* bres = smem + C::STAGES * C::STAGE;  // resident filter (BRES)
  uint64_t* full = reinterpret_cast<uint64_t*>(bres + (BRES ? C::B_RES_MAX : 0));
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;  // [NACC]
  uint64_t* tempty = tfull + C::NACC;   // [NACC]
  uint64_t* bfull = tempty + C::NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = warp_id();
  const int lane = lane_id();
  const int num_kb = a.r * a.s * a.c_chunks;
  const int total = a.m_tiles * a.n_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmx);
    tma_prefetch(&tmw);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < C::NACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4 * EPW);
    }
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel; its outputs are visible now

  if (warp == 0) {
    if (lane == 0) {
      const int cin_stored = a.c_chunks * BKC;
      if (BRES) {
        mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(num_kb * C::B_BYTES));
        for (int kb = 0; kb < num_kb; ++kb) {
          const int tap = kb / a.c_chunks;
          const int cc = kb - tap * a.c_chunks;
          tma_load_2d(bres + kb * C::B_BYTES, &tmw, bfull, tap * cin_stored + cc * BKC, 0);
        }
      }
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int m_tile = t / a.n_tiles;
        const int k0 = (t - m_tile * a.n_tiles) * BN;
        const int tq = m_tile % a.tiles_q;
        const int t2 = m_tile / a.tiles_q;
        const int tp = t2 % a.tiles_p;
        const int tn = t2 / a.tiles_p;
        const int ow0 = tq * a.bw, oh0 = tp * a.bh, n0 = tn * a.bn;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int st = it % C::STAGES;
          if (it >= C::STAGES) mbar_wait(&empty[st], ((it / C::STAGES) - 1) & 1);
          const int tap = kb / a.c_chunks;
          const int cc = kb - tap * a.c_chunks;
          const int rr = tap / a.s;
          const int ss = tap - rr * a.s;
          uint8_t* sa = smem + st * C::STAGE;
          mbar_arrive_expect_tx(&full[st], C::A_BYTES + (BRES ? 0 : C::B_BYTES));
          tma_load_4d(sa, &tmx, &full[st], cc * BKC, ow0 * a.stride + ss - a.pad, oh0 * a.stride + rr - a.pad, n0);
          if (!BRES) tma_load_2d(sa + C::A_BYTES, &tmw, &full[st], tap * cin_stored + cc * BKC, k0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN, 0, 0);
      if (BRES) mbar_wait(bfull, 0);
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
        const int acc = lt % C::NACC;
        if (lt >= C::NACC) mbar_wait(&tempty[acc], ((lt / C::NACC) - 1) & 1);
        tc_fence_after();
        const uint32_t dacc = tmem + static_cast<uint32_t>(acc * C::ACC_COLS);
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int st = it % C::STAGES;
          mbar_wait(&full[st], (it / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * C::STAGE);
          const uint32_t sb = BRES ? smem_u32(bres + kb * C::B_BYTES) : sa + C::A_BYTES;
          const uint64_t a0 = umma_smem_desc(sa, 16, 8 * C::SW, C::LAYOUT);
          const uint64_t b0 = umma_smem_desc(sb, 16, 8 * C::SW, C::LAYOUT);
#pragma unroll
          for (int kk = 0; kk < BKC / 16; ++kk) {
            if (!DBG_IS(a, 2)) umma_bf16(dacc, a0 + 2 * kk, b0 + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[st]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // epilogue: warps 2.., TMEM lane quarter = warp % 4, column slice (warp - 2) / 4
    const int quarter = warp & 3;
    constexpr int CW = BN / EPW;
    const int c_lo = ((warp - 2) >> 2) * CW;
    int lt = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
      const int acc = lt % C::NACC;
      const int m_tile = t / a.n_tiles;
      const int k0 = (t - m_tile * a.n_tiles) * BN;
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * C::ACC_COLS);
      const int tq = m_tile % a.tiles_q;
      const int t2 = m_tile / a.tiles_q;
      const TileRows rows{&a, (t2 / a.tiles_p) * a.bn, (t2 % a.tiles_p) * a.bh, tq * a.bw};
      fprop_epilogue<CW>(a, trow + c_lo, quarter * 32 + lane, k0 + c_lo, rows, [&] {
        mbar_wait(&tfull[acc], (lt / C::NACC) & 1);
        tc_fence_after();
      });
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ split-K fprop (clusters + DSMEM)
// For convs with too few output tiles to fill the GPU (4x4 / 8x8 maps at 256-512 channels) a
// cluster of S CTAs shares one 128 x BN output tile: CTA s accumulates the K blocks
// [s*kb/S, (s+1)*kb/S) in its TMEM and stages the fp32 partial in its (by then idle) pipeline
// shared memory; after a cluster barrier CTA s reduces rows [s*128/S, (s+1)*128/S) over DSMEM,
// adding the S partials in split order (deterministic), applies the fused epilogue and stores
// bf16.  No global workspace and no second kernel.
template <int BN, int BKC>
struct SplitCfg {
  using F = FpropCfg<BN, BKC, false>;
  static constexpr int PITCH = BN + 4;  // floats per staged row; the 16 B pad makes row stores conflict-free
  static constexpr int TMEM_COLS = tmem_cols_for(BN < 32 ? 32 : BN);
  static_assert(128 * PITCH * 4 <= F::STAGES * F::STAGE, "partial tile does not fit the ring");
};

__device__ __forceinline__ void epi_store4(const FpropArgs& a, size_t m, int col, float4 v) {
  float x[4] = {v.x, v.y, v.z, v.w};
  const EpiFlags f = epi_flags(a.epi);
  if (f.bias) {
    const float4 b = __ldg(reinterpret_cast<const float4*>(a.bias + col));
    x[0] += b.x;
    x[1] += b.y;
    x[2] += b.z;
    x[3] += b.w;
  }
  if (f.aux) {
    const uint2 r = __ldg(reinterpret_cast<const uint2*>(a.aux + m * a.k + col));
    const float rv[4] = {bf16_lo(r.x), bf16_hi(r.x), bf16_lo(r.y), bf16_hi(r.y)};
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = epi_aux(f, x[j], rv[j]);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = epi_act(f, x[j]);
  uint2 o;
  o.x = pack_bf16x2(x[0], x[1]);
  o.y = pack_bf16x2(x[2], x[3]);
  *reinterpret_cast<uint2*>(a.y + m * a.k + col) = o;
}

template <int BN, int BKC>
__global__ void __launch_bounds__(kThreads, 1)
    conv_fprop_splitk_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                             const FpropArgs a) {
  using F = FpropCfg<BN, BKC, false>;
  using C = SplitCfg<BN, BKC>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + F::STAGES * F::STAGE);
  uint64_t* empty = full + F::STAGES;
  uint64_t* tfull = empty + F::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* part = reinterpret_cast<float*>(smem);  // staged partial, reuses the ring

  const int warp = warp_id();
  const int lane = lane_id();
  const int splits = static_cast<int>(gridDim.x);
  const int rank = static_cast<int>(cluster_rank());
  const int t = blockIdx.y;
  const int m_tile = t / a.n_tiles;
  const int k0 = (t - m_tile * a.n_tiles) * BN;
  const int tq = m_tile % a.tiles_q;
  const int t2 = m_tile / a.tiles_q;
  const int tp = t2 % a.tiles_p;
  const int tn = t2 / a.tiles_p;
  const int num_kb = a.r * a.s * a.c_chunks;
  const int kb_lo = rank * num_kb / splits;
  const int kb_hi = (rank + 1) * num_kb / splits;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmx);
    tma_prefetch(&tmw);
    for (int i = 0; i < F::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  __syncwarp();  // warp 0 reconverges after the lane-0 barrier init (aligned barrier below)
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();  // (a cluster-wide barrier also covers the CTA: the split CTAs start in step)
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel; its outputs are visible now

  if (warp == 0) {
    if (lane == 0) {
      const int cin_stored = a.c_chunks * BKC;
      const int ow0 = tq * a.bw, oh0 = tp * a.bh, n0 = tn * a.bn;
      int st = 0;
      uint32_t ph = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb) {
        if (kb - kb_lo >= F::STAGES) mbar_wait(&empty[st], ph ^ 1);
        const int tap = kb / a.c_chunks;
        const int cc = kb - tap * a.c_chunks;
        const int rr = tap / a.s;
        const int ss = tap - rr * a.s;
        uint8_t* sa = smem + st * F::STAGE;
        mbar_arrive_expect_tx(&full[st], F::A_BYTES + F::B_BYTES);
        tma_load_4d(sa, &tmx, &full[st], cc * BKC, ow0 * a.stride + ss - a.pad, oh0 * a.stride + rr - a.pad, n0);
        tma_load_2d(sa + F::A_BYTES, &tmw, &full[st], tap * cin_stored + cc * BKC, k0);
        if (++st == F::STAGES) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN, 0, 0);
      const uint64_t adesc0 = umma_smem_desc(smem_u32(smem), 16, 8 * F::SW, F::LAYOUT);
      int st = 0;
      uint32_t ph = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        const uint64_t a0 = adesc0 + static_cast<uint32_t>((st * F::STAGE) >> 4);
        const uint64_t b0 = a0 + static_cast<uint32_t>(F::A_BYTES >> 4);
#pragma unroll
        for (int kk = 0; kk < BKC / 16; ++kk)
          umma_bf16(tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, (kb != kb_lo || kk != 0) ? 1u : 0u);
        umma_commit(&empty[st]);
        if (++st == F::STAGES) {
          st = 0;
          ph ^= 1;
        }
      }
      umma_commit(tfull);
    }
  } else {
    // stage this CTA's fp32 partial: thread = accumulator row
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    mbar_wait(tfull, 0);
    tc_fence_after();
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    float4* dst = reinterpret_cast<float4*>(part + row * C::PITCH);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      tmem_ld16(trow + c0, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[c0 / 4 + j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
    tc_fence_before();
  }
  __syncwarp();
  cluster_sync();

  // reduce rows [rank*128/S, (rank+1)*128/S) across the cluster, fixed split order
  {
    const int rows_per = 128 / splits;
    const TileRows rows{&a, tn * a.bn, tp * a.bh, tq * a.bw};
    const uint32_t part_u32 = smem_u32(part);
    for (int r = rank * rows_per + warp; r < (rank + 1) * rows_per; r += kThreads / 32) {
      bool valid;
      size_t m;
      rows(r, valid, m);
      if (!valid) continue;
#pragma unroll
      for (int c4 = lane; c4 < BN / 4; c4 += 32) {
        const uint32_t off = part_u32 + static_cast<uint32_t>((r * C::PITCH + 4 * c4) * 4);
        float4 v[8];
#pragma unroll
        for (int sp = 0; sp < 8; ++sp)
          if (sp < splits) v[sp] = dsmem_ld4(dsmem_addr(off, static_cast<uint32_t>(sp)));
        float4 acc = v[0];
#pragma unroll
        for (int sp = 1; sp < 8; ++sp) {
          if (sp < splits) {
            acc.x += v[sp].x;
            acc.y += v[sp].y;
            acc.z += v[sp].z;
            acc.w += v[sp].w;
          }
        }
        epi_store4(a, m, k0 + 4 * c4, acc);
      }
    }
  }
  __syncwarp();    // the lane-strided column loop may leave a warp diverged: reconverge before the
  cluster_sync();  // .aligned cluster barrier; every CTA's partial stays alive until all reads are done
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int BN, int BKC>
cudaError_t launch_fprop_splitk(const FpropPlan& p, cudaStream_t stream) {
  using F = FpropCfg<BN, BKC, false>;
  if (stream == reinterpret_cast<cudaStream_t>(-1)) {
    return cudaFuncSetAttribute(conv_fprop_splitk_kernel<BN, BKC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                F::SMEM);
  }
  return launch_ex(conv_fprop_splitk_kernel<BN, BKC>, p.grid, dim3(kThreads, 1, 1), F::SMEM, stream, p.pdl, p.grid.x,
                   p.tmx, p.tmw, p.args);
}

// ------------------------------------------------------------------ 2-CTA fprop (cta_group::2)
// Each SM ingests at most ~100 B/clk from L2, and a 128 x BN tile with BKC = 64 needs
// (16 KB A + BN*128 B of B) per K block: 94 B/clk at the MMA rate for BN = 256, 125 for
// BN = 128, so one-CTA tiles are load-bound.  A CTA pair computes a 256 x BN tile (two
// consecutive M tiles) with 256 x BN x 16 MMAs issued by the even CTA: each CTA loads its own
// A box and HALF of the filter tile, so per-SM traffic drops to 16 KB + BN*64 B per K block.
// Persistent over pair tiles, double-buffered TMEM accumulators, fused register epilogue.
template <int BN, int BKC>
struct PairCfg {
  static constexpr int SW = BKC * 2;
  static constexpr int LAYOUT = layout_for_sw(SW);
  static constexpr int A_BYTES = 128 * SW;
  static constexpr int B_BYTES = (BN / 2) * SW;  // this CTA's half of the filter tile
  static constexpr int STAGE = round_up(A_BYTES + B_BYTES, 1024);
  static constexpr int STAGES = (kFpropBudget / STAGE) > 8 ? 8 : (kFpropBudget / STAGE);
  static constexpr int TMEM_COLS = tmem_cols_for(2 * BN);
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

template <int BN, int BKC>
__global__ void __launch_bounds__(kThreads, 1)
    conv_fprop_pair_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                           const FpropArgs a) {
  using C = PairCfg<BN, BKC>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);  // leader's are used
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2], leader's: 4 epilogue warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int rank = static_cast<int>(cluster_rank());
  const int pair = blockIdx.x >> 1;
  const int pairs = gridDim.x >> 1;
  const int num_kb = a.r * a.s * a.c_chunks;
  const int total = (a.m_tiles >> 1) * a.n_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmx);
    tma_prefetch(&tmw);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel; its outputs are visible now

  if (warp == 0) {
    if (lane == 0) {
      const int cin_stored = a.c_chunks * BKC;
      int it = 0, st = 0;
      uint32_t ph = 0;
      for (int t = pair; t < total; t += pairs) {
        const int mp = t / a.n_tiles;
        const int k0 = (t - mp * a.n_tiles) * BN;
        const int m_tile = 2 * mp + rank;
        const int tq = m_tile % a.tiles_q;
        const int t2 = m_tile / a.tiles_q;
        const int tp = t2 % a.tiles_p;
        const int tn = t2 / a.tiles_p;
        const int ow0 = tq * a.bw, oh0 = tp * a.bh, n0 = tn * a.bn;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          if (it >= C::STAGES) mbar_wait(&empty[st], ph ^ 1);
          const uint32_t fb = dsmem_addr(smem_u32(&full[st]), 0);  // leader's full barrier
          if (rank == 0) mbar_arrive_expect_tx(&full[st], 2 * (C::A_BYTES + C::B_BYTES));
          const int tap = kb / a.c_chunks;
          const int cc = kb - tap * a.c_chunks;
          const int rr = tap / a.s;
          const int ss = tap - rr * a.s;
          uint8_t* sa = smem + st * C::STAGE;
          tma_load_4d_pair(sa, &tmx, fb, cc * BKC, ow0 * a.stride + ss - a.pad, oh0 * a.stride + rr - a.pad, n0);
          tma_load_2d_pair(sa + C::A_BYTES, &tmw, fb, tap * cin_stored + cc * BKC, k0 + rank * (BN / 2));
          if (++st == C::STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, BN, 0, 0);
      const uint64_t adesc0 = umma_smem_desc(smem_u32(smem), 16, 8 * C::SW, C::LAYOUT);
      int st = 0, lt = 0;
      uint32_t ph = 0;
      for (int t = pair; t < total; t += pairs, ++lt) {
        const int acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dacc = tmem + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint64_t a0 = adesc0 + static_cast<uint32_t>((st * C::STAGE) >> 4);
          const uint64_t b0 = a0 + static_cast<uint32_t>(C::A_BYTES >> 4);
#pragma unroll
          for (int kk = 0; kk < BKC / 16; ++kk)
            umma_bf16_pair(dacc, a0 + 2 * kk, b0 + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
          umma_commit_pair(&empty[st]);
          if (++st == C::STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else {
    const int quarter = warp & 3;
    int lt = 0;
    for (int t = pair; t < total; t += pairs, ++lt) {
      const int acc = lt & 1;
      const int mp = t / a.n_tiles;
      const int k0 = (t - mp * a.n_tiles) * BN;
      const int m_tile = 2 * mp + rank;
      const int tq = m_tile % a.tiles_q;
      const int t2 = m_tile / a.tiles_q;
      const TileRows rows{&a, (t2 / a.tiles_p) * a.bn, (t2 % a.tiles_p) * a.bh, tq * a.bw};
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * BN);
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      fprop_epilogue<BN>(a, trow, quarter * 32 + lane, k0, rows);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(dsmem_addr(smem_u32(&tempty[acc]), 0));
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, C::TMEM_COLS);
  }
}

template <int BN, int BKC>
cudaError_t launch_fprop_pair(const FpropPlan& p, cudaStream_t stream) {
  using C = PairCfg<BN, BKC>;
  if (stream == reinterpret_cast<cudaStream_t>(-1)) {
    return cudaFuncSetAttribute(conv_fprop_pair_kernel<BN, BKC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM);
  }
  return launch_ex(conv_fprop_pair_kernel<BN, BKC>, p.grid, dim3(kThreads, 1, 1), C::SMEM, stream, p.pdl, 2u, p.tmx,
                   p.tmw, p.args);
}

// ------------------------------------------------------------------ halo fprop (3x3, stride 1, pad 1)
// For wide images (W = 32) the per-tap boxes re-read every input pixel 9 times through L2.
// Here the GEMM rows index a zero-padded image: output position p = h*(W+2) + w' (w' in
// [0, W+2), w' >= W are discarded), and the input tile is ONE TMA box of padded rows
// (columns -1..W, rows from p0/(W+2)-1, OOB zero = padding).  Tap (r, s) is then the same
// smem tile read from row offset (p0 % (W+2)) + r*(W+2) + s: all 9 taps come from a single
// load, so activation traffic drops ~5x for a ~6% row overhead (32x32: 9 tiles of 128 rows
// cover the 1088 padded positions of an image).  Filters stay resident in shared memory.
//
// The MMA issuer is instruction-latency bound unless every descriptor offset is a compile-time
// constant (measured: 74 cycles/MMA with runtime row/tap strides vs the 48-cycle SS-operand
// rate at N = 64), so the padded width WP is a template parameter and the resident filter is
// laid out [channel chunk][tap]: per tile only the stage base and j0 = p0 % WP are runtime.
template <int BN, int BKC, int WP>
struct HaloCfg {
  static constexpr int SW = BKC * 2;
  static constexpr int LAYOUT = layout_for_sw(SW);
  static constexpr int B_BYTES = BN * SW;
  static constexpr int B_RES_MAX = 96 * 1024;
  static constexpr int ACC_COLS = BN < 32 ? 32 : BN;
  // TMEM accumulators in rotation: the MMA warp may run up to NACC-1 tiles ahead of the epilogue
  static constexpr int NACC = ACC_COLS <= 128 ? 4 : 2;
  static constexpr int TMEM_COLS = tmem_cols_for(NACC * ACC_COLS);
  static constexpr int ROWS = 3 + (129 + WP - 1) / WP;  // padded rows one 128-row tile touches
  static constexpr int BOX_BYTES = ROWS * WP * SW;
  static constexpr int STAGE = round_up(BOX_BYTES, 1024);
  static constexpr int STAGES = ((kFpropBudget - B_RES_MAX) / STAGE) > 8 ? 8 : ((kFpropBudget - B_RES_MAX) / STAGE);
  static constexpr int SMEM = STAGES * STAGE + B_RES_MAX + 1024 + 256;
  static_assert(STAGES >= 2, "halo stage does not fit");
};

template <int BN, int BKC, int WP, int EPW = 1>
__global__ void __launch_bounds__(epi_threads(EPW), 1)
    conv_fprop_halo_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                           const FpropArgs a) {
  using C = HaloCfg<BN, BKC, WP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* bres = smem + C::STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(bres + C::B_RES_MAX);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + C::NACC;
  uint64_t* bfull = tempty + C::NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = warp_id();
  const int lane = lane_id();
  const int total = a.m_tiles;  // single N tile
  const int chunks = a.c_chunks;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmx);
    tma_prefetch(&tmw);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < C::NACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4 * EPW);
    }
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel; its outputs are visible now

  if (warp == 0) {
    if (lane == 0) {
      const int cin_stored = chunks * BKC;
      mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(9 * chunks * C::B_BYTES));
      for (int cc = 0; cc < chunks; ++cc)
        for (int tap = 0; tap < 9; ++tap)
          tma_load_2d(bres + (cc * 9 + tap) * C::B_BYTES, &tmw, bfull, tap * cin_stored + cc * BKC, 0);
      int it = 0, st = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < (DBG_IS(a, 8) ? 0 : total); t += gridDim.x) {
        const int img = t / a.tiles_img;
        const int p0 = (t - img * a.tiles_img) * 128;
        for (int cc = 0; cc < chunks; ++cc, ++it) {
          if (it >= C::STAGES) mbar_wait(&empty[st], ph ^ 1);
          if (DBG_GE(a, 6)) {  // timing only: no activation loads (MMA + epilogue pipeline alone)
            mbar_arrive(&full[st]);
          } else {
            mbar_arrive_expect_tx(&full[st], C::BOX_BYTES);
            tma_load_4d(smem + st * C::STAGE, &tmx, &full[st], cc * BKC, -1, p0 / WP - 1, img);
          }
          if (++st == C::STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN, 0, 0);
      // Descriptors advance by adding (byte offset >> 4) to the start-address field (smem
      // addresses < 256 KB never carry out of the 14-bit field).
      const uint64_t adesc0 = umma_smem_desc(smem_u32(smem), 16, 8 * C::SW, C::LAYOUT);
      const uint64_t bdesc0 = umma_smem_desc(smem_u32(bres), 16, 8 * C::SW, C::LAYOUT);
      mbar_wait(bfull, 0);
      int lt = 0, st = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
        const int acc = lt % C::NACC;
        if (lt >= C::NACC && !DBG_IS(a, 8)) mbar_wait(&tempty[acc], ((lt / C::NACC) - 1) & 1);
        tc_fence_after();
        const uint32_t dacc = tmem + static_cast<uint32_t>(acc * C::ACC_COLS);
        const int j0 = (t % a.tiles_img) * 128 % WP;
        for (int cc = 0; cc < chunks; ++cc) {
          if (!DBG_IS(a, 8)) mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint64_t a0 = adesc0 + static_cast<uint32_t>((st * C::STAGE + j0 * C::SW) >> 4);
          const uint64_t b0 = bdesc0 + static_cast<uint32_t>((cc * 9 * C::B_BYTES) >> 4);
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
#pragma unroll
            for (int kk = 0; kk < BKC / 16; ++kk) {
              const uint32_t aoff = static_cast<uint32_t>((((tap / 3) * WP + tap % 3) * C::SW + kk * 32) >> 4);
              const uint32_t boff = static_cast<uint32_t>((tap * C::B_BYTES + kk * 32) >> 4);
              if (!DBG_IS(a, 2)) umma_bf16(dacc, a0 + aoff, b0 + boff, idesc, (cc | tap | kk) != 0 ? 1u : 0u);
            }
          }
          umma_commit(&empty[st]);
          if (++st == C::STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    const int quarter = warp & 3;
    constexpr int CW = BN / EPW;
    const int c_lo = ((warp - 2) >> 2) * CW;
    int lt = 0;
    for (int t = blockIdx.x; t < (DBG_IS(a, 8) ? 0 : total); t += gridDim.x, ++lt) {
      const int acc = lt % C::NACC;
      const int img = t / a.tiles_img;
      const HaloRows rows{&a, img, (t - img * a.tiles_img) * 128, WP};
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * C::ACC_COLS);
      fprop_epilogue<CW>(a, trow + c_lo, quarter * 32 + lane, c_lo, rows, [&] {
        mbar_wait(&tfull[acc], (lt / C::NACC) & 1);
        tc_fence_after();
      });
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ fprop, two M tiles per filter load
// Non-resident filters (128..512-channel 3x3 convs) make the implicit GEMM L2-throughput bound: the
// chip-wide TMA/L2 ingest (~6300 B/clk, B300_MICROARCH.md "TMA chip-throughput") is reached long
// before the tensor pipe, and half of the bytes are the filter tile re-streamed for every M tile.
// Here each work item is a PAIR of M tiles with the same N tile: every stage carries A0, A1 and one
// B box, the MMA issuer runs both 128 x BN x 16 MMAs off the same B descriptor into two TMEM
// accumulators, so B bytes per FLOP halve.  Four accumulators (2 tiles x double buffer) = 4 x BN
// TMEM columns, hence BN <= 128.
template <int BN, int BKC>
struct FpropM2Cfg {
  static constexpr int SW = BKC * 2;
  static constexpr int LAYOUT = layout_for_sw(SW);
  static constexpr int A_BYTES = 128 * SW;
  static constexpr int B_BYTES = BN * SW;
  static constexpr int STAGE = round_up(2 * A_BYTES + B_BYTES, 1024);
  static constexpr int STAGES = (kFpropBudget / STAGE) > 8 ? 8 : (kFpropBudget / STAGE);
  static constexpr int ACC_COLS = BN < 32 ? 32 : BN;
  // accumulator pairs in rotation: four for BN = 64 (all 512 columns), two for BN = 128
  static constexpr int NBUF = 2 * 4 * ACC_COLS <= 512 ? 4 : 2;
  static constexpr int TMEM_COLS = tmem_cols_for(2 * NBUF * ACC_COLS);
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static_assert(2 * NBUF * ACC_COLS <= 512, "the accumulator pairs must fit TMEM");
};

template <int BN, int BKC>
__global__ void __launch_bounds__(kThreads, 1)
    conv_fprop_m2_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                         const FpropArgs a) {
  using C = FpropM2Cfg<BN, BKC>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;  // [NBUF]
  uint64_t* tempty = tfull + C::NBUF;   // [NBUF]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::NBUF);

  const int warp = warp_id();
  const int lane = lane_id();
  const int num_kb = a.r * a.s * a.c_chunks;
  const int m_pairs = (a.m_tiles + 1) / 2;
  const int total = m_pairs * a.n_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmx);
    tma_prefetch(&tmw);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < C::NBUF; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel; its outputs are visible now

  if (warp == 0) {
    if (lane == 0) {
      const int cin_stored = a.c_chunks * BKC;
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int mp = t / a.n_tiles;
        const int k0 = (t - mp * a.n_tiles) * BN;
        const int nval = (2 * mp + 1 < a.m_tiles) ? 2 : 1;
        int ow0[2], oh0[2], n0[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int m_tile = 2 * mp + u;
          const int tq = m_tile % a.tiles_q;
          const int t2 = m_tile / a.tiles_q;
          ow0[u] = tq * a.bw;
          oh0[u] = (t2 % a.tiles_p) * a.bh;
          n0[u] = (t2 / a.tiles_p) * a.bn;
        }
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int st = it % C::STAGES;
          if (it >= C::STAGES) mbar_wait(&empty[st], ((it / C::STAGES) - 1) & 1);
          const int tap = kb / a.c_chunks;
          const int cc = kb - tap * a.c_chunks;
          const int rr = tap / a.s;
          const int ss = tap - rr * a.s;
          uint8_t* sa = smem + st * C::STAGE;
          mbar_arrive_expect_tx(&full[st], nval * C::A_BYTES + C::B_BYTES);
          for (int u = 0; u < nval; ++u)
            tma_load_4d(sa + u * C::A_BYTES, &tmx, &full[st], cc * BKC, ow0[u] * a.stride + ss - a.pad,
                        oh0[u] * a.stride + rr - a.pad, n0[u]);
          tma_load_2d(sa + 2 * C::A_BYTES, &tmw, &full[st], tap * cin_stored + cc * BKC, k0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN, 0, 0);
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
        const int mp = t / a.n_tiles;
        const int nval = (2 * mp + 1 < a.m_tiles) ? 2 : 1;
        const int acc = lt % C::NBUF;
        if (lt >= C::NBUF) mbar_wait(&tempty[acc], ((lt / C::NBUF) - 1) & 1);
        tc_fence_after();
        const uint32_t d0 = tmem + static_cast<uint32_t>(acc * 2 * C::ACC_COLS);
        const uint32_t d1 = d0 + static_cast<uint32_t>(C::ACC_COLS);
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int st = it % C::STAGES;
          mbar_wait(&full[st], (it / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * C::STAGE);
          const uint64_t a0 = umma_smem_desc(sa, 16, 8 * C::SW, C::LAYOUT);
          const uint64_t a1 = umma_smem_desc(sa + C::A_BYTES, 16, 8 * C::SW, C::LAYOUT);
          const uint64_t b0 = umma_smem_desc(sa + 2 * C::A_BYTES, 16, 8 * C::SW, C::LAYOUT);
#pragma unroll
          for (int kk = 0; kk < BKC / 16; ++kk) {
            const uint32_t accum = (kb | kk) != 0 ? 1u : 0u;
            umma_bf16(d0, a0 + 2 * kk, b0 + 2 * kk, idesc, accum);
            if (nval == 2) umma_bf16(d1, a1 + 2 * kk, b0 + 2 * kk, idesc, accum);
          }
          umma_commit(&empty[st]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    const int quarter = warp & 3;
    int lt = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++lt) {
      const int acc = lt % C::NBUF;
      const int mp = t / a.n_tiles;
      const int k0 = (t - mp * a.n_tiles) * BN;
      const int nval = (2 * mp + 1 < a.m_tiles) ? 2 : 1;
      for (int u = 0; u < nval; ++u) {
        const int m_tile = 2 * mp + u;
        const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16) +
                              static_cast<uint32_t>((acc * 2 + u) * C::ACC_COLS);
        const int tq = m_tile % a.tiles_q;
        const int t2 = m_tile / a.tiles_q;
        const TileRows rows{&a, (t2 / a.tiles_p) * a.bn, (t2 % a.tiles_p) * a.bh, tq * a.bw};
        if (u == 0) {
          fprop_epilogue<BN>(a, trow, quarter * 32 + lane, k0, rows, [&] {
            mbar_wait(&tfull[acc], (lt / C::NBUF) & 1);
            tc_fence_after();
          });
        } else {
          fprop_epilogue<BN>(a, trow, quarter * 32 + lane, k0, rows);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int BN, int BKC>
cudaError_t launch_fprop_m2(const FpropPlan& p, cudaStream_t stream) {
  using C = FpropM2Cfg<BN, BKC>;
  if (stream == reinterpret_cast<cudaStream_t>(-1)) {
    return cudaFuncSetAttribute(conv_fprop_m2_kernel<BN, BKC>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  }
  return launch_ex(conv_fprop_m2_kernel<BN, BKC>, p.grid, dim3(kThreads, 1, 1), C::SMEM, stream, p.pdl, 1u, p.tmx,
                   p.tmw, p.args);
}

template <int BN, int BKC, int WP, int EPW = 1>
cudaError_t launch_fprop_halo(const FpropPlan& p, cudaStream_t stream) {
  using C = HaloCfg<BN, BKC, WP>;
  if (stream == reinterpret_cast<cudaStream_t>(-1)) {
    return cudaFuncSetAttribute(conv_fprop_halo_kernel<BN, BKC, WP, EPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM);
  }
  return launch_ex(conv_fprop_halo_kernel<BN, BKC, WP, EPW>, p.grid, dim3(epi_threads(EPW), 1, 1), C::SMEM, stream,
                   p.pdl, 1u, p.tmx, p.tmw, p.args);
}

template <int BN, int BKC, bool BRES, int EPW = 1>
cudaError_t launch_fprop(const FpropPlan& p, cudaStream_t stream) {
  using C = FpropCfg<BN, BKC, BRES>;
  if (stream == reinterpret_cast<cudaStream_t>(-1)) {  // prepare: set the smem attribute outside any capture
    return cudaFuncSetAttribute(conv_fprop_kernel<BN, BKC, BRES, EPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM);
  }
  return launch_ex(conv_fprop_kernel<BN, BKC, BRES, EPW>, p.grid, dim3(epi_threads(EPW), 1, 1), C::SMEM, stream,
                   p.pdl, 1u, p.tmx, p.tmw, p.args);
}

// ------------------------------------------------------------------ wgrad

template <int BN, int SWA, int SWB>
struct WgradCfg {
  static constexpr int KT = 128;                       // pixels per stage
  static constexpr int A_ATOM = KT * SWA;              // one MN atom of A (SWA/2 channels of k)
  static constexpr int A_BYTES = 128 * KT * 2;         // full M=128 region
  static constexpr int B_ATOM = KT * SWB;
  static constexpr int B_ATOMS = BN / (SWB / 2);
  static constexpr int B_BYTES = B_ATOMS * B_ATOM;
  static constexpr int STAGE = round_up(A_BYTES + B_BYTES, 1024);
  static constexpr int STAGES = (kSmemBudget / STAGE) > 6 ? 6 : (kSmemBudget / STAGE);
  static constexpr int TMEM_COLS = tmem_cols_for(BN);
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

template <int BN, int SWA, int SWB>
__global__ void __launch_bounds__(kThreads, 1)
    conv_wgrad_kernel(const __grid_constant__ CUtensorMap tmdy, const __grid_constant__ CUtensorMap tmx,
                      const WgradArgs a) {
  using C = WgradCfg<BN, SWA, SWB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = warp_id();
  const int lane = lane_id();
  int t = blockIdx.x;
  const int ci_t = t % a.ci_tiles;
  t /= a.ci_tiles;
  const int co_t = t % a.co_tiles;
  const int tap = t / a.co_tiles;
  const int rr = tap / a.s;
  const int ss = tap - rr * a.s;
  const int co0 = co_t * 128;
  const int ci0 = ci_t * BN;
  const int split = blockIdx.y;
  const int mt0 = split * a.tiles_per_split;
  const int mt1 = min(a.m_tiles, mt0 + a.tiles_per_split);
  const int num_kb = max(0, mt1 - mt0);

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
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel; its outputs are visible now

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = static_cast<uint32_t>(a.a_atoms * C::A_ATOM + C::B_BYTES);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % C::STAGES;
        if (kb >= C::STAGES) mbar_wait(&empty[st], ((kb / C::STAGES) - 1) & 1);
        const int mt = mt0 + kb;
        const int tq = mt % a.tiles_q;
        const int t2 = mt / a.tiles_q;
        const int tp = t2 % a.tiles_p;
        const int tn = t2 / a.tiles_p;
        const int ow0 = tq * a.bw, oh0 = tp * a.bh, n0 = tn * a.bn;
        uint8_t* sa = smem + st * C::STAGE;
        uint8_t* sb = sa + C::A_BYTES;
        mbar_arrive_expect_tx(&full[st], bytes);
        for (int i = 0; i < a.a_atoms; ++i)
          tma_load_4d(sa + i * C::A_ATOM, &tmdy, &full[st], co0 + i * (SWA / 2), ow0, oh0, n0);
#pragma unroll
        for (int i = 0; i < C::B_ATOMS; ++i)
          tma_load_4d(sb + i * C::B_ATOM, &tmx, &full[st], ci0 + i * (SWB / 2), ow0 * a.stride + ss - a.pad,
                      oh0 * a.stride + rr - a.pad, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN, 1, 1);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % C::STAGES;
        mbar_wait(&full[st], (kb / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + st * C::STAGE);
        const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < C::KT / 16; ++kk) {
          // MN-major canonical layout: LBO = stride between MN atoms, SBO = 8 K-rows.
          const uint64_t ad = umma_smem_desc(sa + kk * 16 * SWA, C::A_ATOM, 8 * SWA, layout_for_sw(SWA));
          const uint64_t bd = umma_smem_desc(sb + kk * 16 * SWB, C::B_ATOM, 8 * SWB, layout_for_sw(SWB));
          umma_bf16(tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[st]);
      }
      if (num_kb > 0) umma_commit(tfull);
    }
  } else {
    const int quarter = warp & 3;
    const int co = co0 + quarter * 32 + lane;
    const int taps = a.r * a.s;
    float* dst_row = a.out + static_cast<size_t>(split) * a.k * taps * a.c +
                     (static_cast<size_t>(co) * taps + tap) * a.c + ci0;
    if (num_kb > 0) {
      mbar_wait(tfull, 0);
      tc_fence_after();
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(trow + c0, v);
        if (co < a.k) {
          float4* d4 = reinterpret_cast<float4*>(dst_row + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
      }
    } else if (co < a.k) {
      for (int c0 = 0; c0 < BN; c0 += 4)
        *reinterpret_cast<float4*>(dst_row + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// Multi-tap wgrad for narrow inputs (c = CB in {16, 32}, k <= 128): ONE CTA computes every tap of
// the filter for its pixel range.  Per 128-pixel stage it loads the dy box once (A, MN-major) and
// the TAPS shifted x boxes side by side as the N atoms of B, so one MMA covers up to 256/CB taps:
// D[k][tap*CB + c] = dW[k][tap][c] is exactly the row-major filter-gradient layout.  Versus the
// per-tap kernel (one CTA per tap) this reads dy once instead of TAPS times and replaces TAPS
// narrow MMAs (each re-reading the whole 128-row A from shared memory) with one or two wide ones.
// A's rows beyond k (M = 128) are never loaded: their atoms alias the B region (read, discarded).
template <int CB, int SWA, int AAT, int TAPS>
struct WgradMtCfg {
  static constexpr int KT = 128;
  static constexpr int SWB = 2 * CB;  // CB <= 64: one swizzle atom of B per tap
  static constexpr int A_ATOM = KT * SWA;
  static constexpr int B_ATOM = KT * SWB;
  static constexpr int G0 = TAPS < 256 / CB ? TAPS : 256 / CB;  // taps in MMA group 0
  static constexpr int G1 = TAPS - G0;
  static constexpr int N0 = G0 * CB, N1 = G1 * CB;
  static constexpr int STAGE = round_up(AAT * A_ATOM + TAPS * B_ATOM, 1024);
  static constexpr int STAGES = (kSmemBudget / STAGE) > 6 ? 6 : (kSmemBudget / STAGE);
  static constexpr int TMEM_COLS = tmem_cols_for(N0 + N1);
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static_assert(N1 <= 256 && N0 + N1 <= 512, "taps x channels must fit two MMAs / TMEM");
  static_assert(STAGE >= 128 * KT * 2, "aliased A atoms must stay inside the stage");
};

template <int CB, int SWA, int AAT, int TAPS>
__global__ void __launch_bounds__(kThreads, 1)
    conv_wgrad_mt_kernel(const __grid_constant__ CUtensorMap tmdy, const __grid_constant__ CUtensorMap tmx,
                         const WgradArgs a) {
  using C = WgradMtCfg<CB, SWA, AAT, TAPS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = warp_id();
  const int lane = lane_id();
  const int split = blockIdx.x;
  // blockIdx.y = (tap group, co tile, ci tile), ci fastest
  int grp = blockIdx.y;
  const int ci0 = (grp % a.ci_tiles) * CB;
  grp /= a.ci_tiles;
  const int co0 = (grp % a.co_tiles) * 128;
  const int tap0 = (grp / a.co_tiles) * TAPS;
  const int mt0 = split * a.tiles_per_split;
  const int mt1 = min(a.m_tiles, mt0 + a.tiles_per_split);
  const int num_kb = max(0, mt1 - mt0);

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
  grid_dep_wait();  // PDL: the prologue above overlapped the previous kernel; its outputs are visible now

  if (warp == 0) {
    if (lane == 0) {
      constexpr uint32_t bytes = static_cast<uint32_t>(AAT * C::A_ATOM + TAPS * C::B_ATOM);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % C::STAGES;
        if (kb >= C::STAGES) mbar_wait(&empty[st], ((kb / C::STAGES) - 1) & 1);
        const int mt = mt0 + kb;
        const int tq = mt % a.tiles_q;
        const int t2 = mt / a.tiles_q;
        const int tp = t2 % a.tiles_p;
        const int tn = t2 / a.tiles_p;
        const int ow0 = tq * a.bw, oh0 = tp * a.bh, n0 = tn * a.bn;
        uint8_t* sa = smem + st * C::STAGE;
        uint8_t* sb = sa + AAT * C::A_ATOM;
        mbar_arrive_expect_tx(&full[st], bytes);
#pragma unroll
        for (int i = 0; i < AAT; ++i)
          tma_load_4d(sa + i * C::A_ATOM, &tmdy, &full[st], co0 + i * (SWA / 2), ow0, oh0, n0);
#pragma unroll
        for (int t = 0; t < TAPS; ++t) {
          const int rr = (tap0 + t) / a.s, ss = (tap0 + t) - rr * a.s;
          tma_load_4d(sb + t * C::B_ATOM, &tmx, &full[st], ci0, ow0 * a.stride + ss - a.pad,
                      oh0 * a.stride + rr - a.pad, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc0 = umma_idesc_bf16(128, C::N0, 1, 1);
      constexpr uint32_t idesc1 = umma_idesc_bf16(128, C::N1 > 0 ? C::N1 : 16, 1, 1);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % C::STAGES;
        mbar_wait(&full[st], (kb / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + st * C::STAGE);
        const uint32_t sb = sa + AAT * C::A_ATOM;
#pragma unroll
        for (int kk = 0; kk < C::KT / 16; ++kk) {
          const uint32_t acc = (kb | kk) != 0 ? 1u : 0u;
          const uint64_t ad = umma_smem_desc(sa + kk * 16 * SWA, C::A_ATOM, 8 * SWA, layout_for_sw(SWA));
          const uint64_t b0 = umma_smem_desc(sb + kk * 16 * C::SWB, C::B_ATOM, 8 * C::SWB, layout_for_sw(C::SWB));
          umma_bf16(tmem, ad, b0, idesc0, acc);
          if constexpr (C::N1 > 0) {
            const uint64_t b1 = umma_smem_desc(sb + C::G0 * C::B_ATOM + kk * 16 * C::SWB, C::B_ATOM, 8 * C::SWB,
                                               layout_for_sw(C::SWB));
            umma_bf16(tmem + C::N0, ad, b1, idesc1, acc);
          }
        }
        umma_commit(&empty[st]);
      }
      if (num_kb > 0) umma_commit(tfull);
    }
  } else {
    const int quarter = warp & 3;
    const int co = co0 + quarter * 32 + lane;
    const int taps = a.r * a.s;
    // D column t*CB + c = dW[co][tap0 + t][ci0 + c]
    float* dst_row = a.out + static_cast<size_t>(split) * a.k * taps * a.c + (static_cast<size_t>(co) * taps + tap0) * a.c + ci0;
    if (num_kb > 0) {
      mbar_wait(tfull, 0);
      tc_fence_after();
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < TAPS * CB; c0 += 16) {
        float v[16];
        tmem_ld16(trow + c0, v);
        if (co < a.k) {
          float4* d4 = reinterpret_cast<float4*>(dst_row + (c0 / CB) * a.c + c0 % CB);
#pragma unroll
          for (int j = 0; j < 4; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
      }
    } else if (co < a.k) {
      for (int c0 = 0; c0 < TAPS * CB; c0 += 4)
        *reinterpret_cast<float4*>(dst_row + (c0 / CB) * a.c + c0 % CB) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int CB, int SWA, int AAT, int TAPS>
cudaError_t launch_wgrad_mt(const WgradPlan& p, cudaStream_t stream) {
  using C = WgradMtCfg<CB, SWA, AAT, TAPS>;
  if (stream == reinterpret_cast<cudaStream_t>(-1)) {
    return cudaFuncSetAttribute(conv_wgrad_mt_kernel<CB, SWA, AAT, TAPS>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  }
  return launch_ex(conv_wgrad_mt_kernel<CB, SWA, AAT, TAPS>, p.grid, dim3(kThreads, 1, 1), C::SMEM, stream, p.pdl, 1u,
                   p.tmdy, p.tmx, p.args);
}

template <int BN, int SWA, int SWB>
cudaError_t launch_wgrad(const WgradPlan& p, cudaStream_t stream) {
  using C = WgradCfg<BN, SWA, SWB>;
  if (stream == reinterpret_cast<cudaStream_t>(-1)) {
    return cudaFuncSetAttribute(conv_wgrad_kernel<BN, SWA, SWB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM);
  }
  return launch_ex(conv_wgrad_kernel<BN, SWA, SWB>, p.grid, dim3(kThreads, 1, 1), C::SMEM, stream, p.pdl, 1u, p.tmdy,
                   p.tmx, p.args);
}

// Fixed-order split reduction: dw[i] = sum_s ws[s][i]  (deterministic).  CTA = 32 float4 lanes x 8
// split lanes: split lane l adds splits l, l+8, ... in order, then the 8 partial sums are added in
// lane order through shared memory — every split slab is read by 8x more threads in flight than a
// serial walk, which matters for the small slabs of the early blocks (up to 148 splits).
constexpr int kRedLanes = 32, kRedSplitLanes = 8;
__global__ void __launch_bounds__(kRedLanes * kRedSplitLanes)
    split_reduce_kernel(const float4* __restrict__ ws, float4* __restrict__ dw, size_t n4, int splits) {
  __shared__ float4 part[kRedSplitLanes][kRedLanes];
  const int e = threadIdx.x % kRedLanes;
  const int sl = threadIdx.x / kRedLanes;
  grid_dep_wait();  // PDL (launched with the wgrad plan's pdl flag): the split slabs are complete after this
  for (size_t base = static_cast<size_t>(blockIdx.x) * kRedLanes; base < n4;
       base += static_cast<size_t>(gridDim.x) * kRedLanes) {
    const size_t i = base + e;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < n4) {
      int s = sl;
      for (; s + 3 * kRedSplitLanes < splits; s += 4 * kRedSplitLanes) {  // 4 loads in flight, in order
        const float4 v0 = ws[s * n4 + i];
        const float4 v1 = ws[(s + kRedSplitLanes) * n4 + i];
        const float4 v2 = ws[(s + 2 * kRedSplitLanes) * n4 + i];
        const float4 v3 = ws[(s + 3 * kRedSplitLanes) * n4 + i];
        acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w;
        acc.x += v1.x; acc.y += v1.y; acc.z += v1.z; acc.w += v1.w;
        acc.x += v2.x; acc.y += v2.y; acc.z += v2.z; acc.w += v2.w;
        acc.x += v3.x; acc.y += v3.y; acc.z += v3.z; acc.w += v3.w;
      }
      for (; s < splits; s += kRedSplitLanes) {
        const float4 v = ws[s * n4 + i];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    part[sl][e] = acc;
    __syncthreads();
    if (sl == 0 && i < n4) {
      float4 t = part[0][e];
      for (int l = 1; l < kRedSplitLanes; ++l) {
        const float4 v = part[l][e];
        t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
      }
      dw[i] = t;
    }
    __syncthreads();
  }
}

__global__ void weight_flip_kernel(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ wt, int k, int r,
                                   int s, int c) {
  const size_t total = static_cast<size_t>(k) * r * s * c;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    // i indexes wt[ci][r'][s'][co]
    const int co = static_cast<int>(i % k);
    size_t t = i / k;
    const int sp = static_cast<int>(t % s);
    t /= s;
    const int rp = static_cast<int>(t % r);
    const int ci = static_cast<int>(t / r);
    wt[i] = w[((static_cast<size_t>(co) * r + (r - 1 - rp)) * s + (s - 1 - sp)) * c + ci];
  }
}

bool chan_ok(int c) { return c == 16 || c == 32 || (c >= 64 && c % 64 == 0); }
int chan_block(int c) { return c >= 64 ? 64 : c; }

}  // namespace

bool make_geom(const pbdk_conv_desc& d, ConvGeom* g) {
  if (d.n < 1 || d.h < 1 || d.w < 1 || d.r < 1 || d.s < 1 || d.stride < 1 || d.pad < 0) return false;
  if (d.p != (d.h + 2 * d.pad - d.r) / d.stride + 1) return false;
  if (d.q != (d.w + 2 * d.pad - d.s) / d.stride + 1) return false;
  if (d.q > 128 || 128 % d.q != 0) return false;
  g->d = d;
  g->bw = d.q;
  const int rows = 128 / d.q;
  g->bh = std::min(d.p, rows);
  if (rows % g->bh != 0 || d.p % g->bh != 0) return false;
  g->bn = rows / g->bh;
  if (g->bw * d.stride > 256 || g->bh * d.stride > 256 || g->bn > 256) return false;
  g->tiles_q = d.q / g->bw;
  g->tiles_p = d.p / g->bh;
  g->tiles_n = (d.n + g->bn - 1) / g->bn;
  g->m_tiles = g->tiles_q * g->tiles_p * g->tiles_n;
  return true;
}

namespace {

// 4D map over an NHWC bf16 activation, box = one 128-pixel tile of `chan` channels.
bool act_map(CUtensorMap* m, const void* base, int n, int h, int w, int c, int chan, int bw, int bh, int bn,
             int stride) {
  const uint64_t dims[4] = {static_cast<uint64_t>(c), static_cast<uint64_t>(w), static_cast<uint64_t>(h),
                            static_cast<uint64_t>(n)};
  const uint64_t strides[3] = {static_cast<uint64_t>(c) * 2, static_cast<uint64_t>(w) * c * 2,
                               static_cast<uint64_t>(h) * w * c * 2};
  const uint32_t box[4] = {static_cast<uint32_t>(chan), static_cast<uint32_t>(bw * stride),
                           static_cast<uint32_t>(bh * stride), static_cast<uint32_t>(bn)};
  const uint32_t es[4] = {1, static_cast<uint32_t>(stride), static_cast<uint32_t>(stride), 1};
  return encode_tmap_bf16(m, base, 4, dims, strides, box, es, chan * 2);
}

using FpropLauncher = cudaError_t (*)(const FpropPlan&, cudaStream_t);

template <int BKC, bool BRES>
FpropLauncher pick_fprop(int bn, int epw = 1) {
  if (epw == 2) {
    switch (bn) {
      case 32: return launch_fprop<32, BKC, BRES, 2>;
      case 64: return launch_fprop<64, BKC, BRES, 2>;
      case 128: return launch_fprop<128, BKC, BRES, 2>;
      default: break;
    }
  }
  switch (bn) {
    case 16: return launch_fprop<16, BKC, BRES>;
    case 32: return launch_fprop<32, BKC, BRES>;
    case 64: return launch_fprop<64, BKC, BRES>;
    case 128: return launch_fprop<128, BKC, BRES>;
    case 256: return launch_fprop<256, BKC, BRES>;
    default: return nullptr;
  }
}

constexpr int kHaloWP = 34;  // halo kernel instantiated for 32-wide images (W + 2 padded columns)

template <int BKC>
FpropLauncher pick_halo(int bn, int epw = 1) {
  if (epw == 2) {
    switch (bn) {
      case 32: return launch_fprop_halo<32, BKC, kHaloWP, 2>;
      case 64: return launch_fprop_halo<64, BKC, kHaloWP, 2>;
      default: break;
    }
  }
  switch (bn) {
    case 16: return launch_fprop_halo<16, BKC, kHaloWP>;
    case 32: return launch_fprop_halo<32, BKC, kHaloWP>;
    case 64: return launch_fprop_halo<64, BKC, kHaloWP>;
    case 128: return launch_fprop_halo<128, BKC, kHaloWP>;
    default: return nullptr;
  }
}

bool halo_enabled() {
  static const bool on = [] {
    const char* e = pbd::knob_env("PBDK_NO_HALO");
    return e == nullptr || e[0] == '0';
  }();
  return on;
}

thread_local int t_grid_sms = 0;  // ConvGridScope
thread_local int t_epw = 0;       // ConvGridScope: preferred epilogue warps per lane quarter (0 = by shape)
// SMs a plan may spread over (persistent grids, one-wave split counts)
int grid_sms();

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

int grid_sms() { return t_grid_sms > 0 ? std::min(t_grid_sms, num_sms()) : num_sms(); }



using WgradLauncher = cudaError_t (*)(const WgradPlan&, cudaStream_t);

template <int SWA>
WgradLauncher pick_wgrad_b(int bn, int swb) {
  if (swb == 32 && bn == 16) return launch_wgrad<16, SWA, 32>;
  if (swb == 64 && bn == 32) return launch_wgrad<32, SWA, 64>;
  if (swb == 128 && bn == 64) return launch_wgrad<64, SWA, 128>;
  if (swb == 128 && bn == 128) return launch_wgrad<128, SWA, 128>;
  return nullptr;
}

WgradLauncher pick_wgrad(int bn, int swa, int swb) {
  switch (swa) {
    case 32: return pick_wgrad_b<32>(bn, swb);
    case 64: return pick_wgrad_b<64>(bn, swb);
    case 128: return pick_wgrad_b<128>(bn, swb);
    default: return nullptr;
  }
}

int wgrad_bn(int c) { return c % 128 == 0 ? 128 : c >= 64 ? 64 : c; }  // c in {16, 32} or a multiple of 64

// multi-tap wgrad (conv_wgrad_mt_kernel) for 3x3 filters: c in {16, 32} with all 9 taps per CTA (k <= 128),
// or c = 64 with one filter row (3 taps, N = 192) per CTA (any k: 128-row co tiles)
template <int CB>
WgradLauncher pick_wgrad_mt_c(int swa, int aat) {
  if (swa == 32 && aat == 1) return launch_wgrad_mt<CB, 32, 1, 9>;
  if (swa == 64 && aat == 1) return launch_wgrad_mt<CB, 64, 1, 9>;
  if (swa == 128 && aat == 1) return launch_wgrad_mt<CB, 128, 1, 9>;
  if constexpr (CB == 16)
    if (swa == 128 && aat == 2) return launch_wgrad_mt<CB, 128, 2, 9>;
  return nullptr;
}

int wgrad_mt_taps(const pbdk_conv_desc& d) { return d.c >= 64 ? 3 : 9; }

WgradLauncher pick_wgrad_mt(const pbdk_conv_desc& d) {
  static const int mode = [] {
    const char* e = pbd::knob_env("PBDK_WGRAD_MT");  // 0 off, 1 narrow inputs only, 2 (default) + 64-ch tiles
    return e != nullptr ? std::atoi(e) : 2;
  }();
  if (mode == 0 || d.r * d.s != 9) return nullptr;
  const int swa = chan_block(d.k) * 2;
  const int aat = (std::min(128, d.k) + swa / 2 - 1) / (swa / 2);
  if (d.c >= 64) {  // measured (scripts/time_wgrad.py): a win at c = 64 (s2 19.4 -> 14.6 us), a loss at c >= 128
    if (mode < 2 || swa != 128 || d.c != 64) return nullptr;
    return aat == 1 ? launch_wgrad_mt<64, 128, 1, 3> : launch_wgrad_mt<64, 128, 2, 3>;
  }
  if (d.k > 128 || (d.c != 16 && d.c != 32)) return nullptr;
  return d.c == 16 ? pick_wgrad_mt_c<16>(swa, aat) : pick_wgrad_mt_c<32>(swa, aat);
}

template <int BKC>
FpropLauncher pick_splitk(int bn) {
  switch (bn) {
    case 128: return launch_fprop_splitk<128, BKC>;
    case 256: return launch_fprop_splitk<256, BKC>;
    default: return nullptr;
  }
}

bool fprop_bres(const pbdk_conv_desc& d, int bn, int bkc) {
  return d.k == bn && d.r * d.s * (d.c / bkc) * bn * bkc * 2 <= 96 * 1024;
}

// Tile width and split count from a throughput model measured on B200:
// 128 x N x 16 MMA = 46/48/64/128 cycles for N = 32/64/128/256, and each SM ingests at most
// ~100 B/clk from L2 with ~192 KB of TMA loads in flight (latency ~1 us under load;
// scripts/micro/tma_rate.cu, l2_ingress.cu), so a K block costs
// max(MMA cycles, bytes loaded / kIngress).  Persistent (S = 1) kernels pay ceil(tiles / SMs) tiles per
// CTA; split-K (S in 2..8, one wave, K blocks divided S ways) pays a DSMEM reduction.
struct FpropChoice {
  int bn;
  int splits;
  bool pair;  // 2-CTA (cta_group::2) tiles of 256 x bn
  bool m2 = false;  // two M tiles per filter load (conv_fprop_m2_kernel)
};

constexpr double kIngress = 100.0;  // L2 -> smem bytes per SM clock with ~192 KB of loads in flight

FpropChoice choose_fprop(const pbdk_conv_desc& d, const ConvGeom& g, int bkc) {
  const int num_kb = d.r * d.s * (d.c / bkc);
  const int sms = num_sms();
  static const int forced = [] {
    const char* e = pbd::knob_env("PBDK_FPROP_SPLITS");  // 1: never split (A/B runs)
    return e != nullptr ? std::atoi(e) : 0;
  }();
  // 2-CTA tiles measured no faster than one-CTA tiles on the step's shapes (the K loop is
  // not load-bound once enough bytes are in flight); opt-in for experiments.
  static const int no_pair = [] {
    const char* e = pbd::knob_env("PBDK_PAIR");
    return e == nullptr || e[0] == '0';
  }();
  FpropChoice best{0, 1, false};
  double best_cost = 1e300;
  for (int bn : {256, 128, 64, 32, 16}) {
    if (d.k % bn != 0) continue;
    const bool bres = fprop_bres(d, bn, bkc);
    const double mma = (bkc / 16) * (bn <= 32 ? 46.0 : bn == 64 ? 48.0 : bn == 128 ? 64.0 : 128.0);
    const double bytes = 128.0 * bkc * 2 + (bres ? 0.0 : static_cast<double>(bn) * bkc * 2);
    const double kb_cost = std::max(mma, bytes / kIngress);
    const int tiles = g.m_tiles * (d.k / bn);
    for (int sp : {1, 2, 4, 8}) {
      if (sp > 1) {
        if (bkc != 64 || (bn != 128 && bn != 256) || tiles * sp > sms || num_kb < 4 * sp) continue;
      }
      if (forced == 1 && sp > 1) continue;
      double cost;
      if (sp == 1) {
        const int per_cta = (tiles + std::min(tiles, sms) - 1) / std::min(tiles, sms);
        cost = per_cta * num_kb * kb_cost + 4.0 * bn;
      } else {
        cost = ((num_kb + sp - 1) / sp) * kb_cost + 8.0 * bn + 6500.0;  // measured reduction + sync cost
      }
      if (cost < best_cost) {
        best_cost = cost;
        best = {bn, sp, false};
      }
    }
    // 2-CTA: per SM a K block loads 16 KB of A and half the filter tile
    if (!no_pair && bkc == 64 && (bn == 128 || bn == 256) && !bres && g.m_tiles % 2 == 0) {
      const double pbytes = 128.0 * bkc * 2 + static_cast<double>(bn / 2) * bkc * 2;
      const double pkb = std::max(mma, pbytes / kIngress);
      const int ptiles = tiles / 2;
      const int pairs = std::min(ptiles, sms / 2);
      const double cost = ((ptiles + pairs - 1) / pairs) * num_kb * pkb + 4.0 * bn + 500.0;
      if (cost < best_cost) {
        best_cost = cost;
        best = {bn, 1, true};
      }
    }
  }
  return best;
}

// Pairing halves the re-streamed filter bytes but leaves half as many work items to spread over the
// SMs; take it when the chip-wide L2 ingest (not the wave count) bounds the persistent kernel:
// compare max(items/SMs rounds x MMA, bytes / chip ingest) of both variants.
constexpr double kChipIngest = 6300.0;  // B/clk, whole chip (B300_MICROARCH.md TMA chip-throughput)

bool m2_auto(const pbdk_conv_desc& d, const ConvGeom& g, int bn) {
  const int bkc = 64;
  const int num_kb = d.r * d.s * (d.c / bkc);
  const int sms = num_sms();
  const double mma = (bkc / 16) * (bn == 64 ? 48.0 : 64.0);
  const double a_b = 128.0 * bkc * 2, b_b = static_cast<double>(bn) * bkc * 2;
  const int n_tiles = d.k / bn;
  const int tiles = g.m_tiles * n_tiles;
  const int items = (g.m_tiles + 1) / 2 * n_tiles;
  const double t1 = std::max(((tiles + sms - 1) / sms) * num_kb * mma, tiles * num_kb * (a_b + b_b) / kChipIngest);
  const double t2 = std::max(((items + sms - 1) / sms) * num_kb * 2 * mma,
                             items * num_kb * (2 * a_b + b_b) / kChipIngest);
  return t2 < 0.95 * t1;
}

}  // namespace

ConvGridScope::ConvGridScope(int sms, int epw) : saved(t_grid_sms), saved_epw(t_epw) {
  t_grid_sms = sms;
  t_epw = epw;
}
ConvGridScope::~ConvGridScope() {
  t_grid_sms = saved;
  t_epw = saved_epw;
}

int fprop_plan(const pbdk_conv_desc& d, const void* x, const void* w, void* y, const float* bias, const void* aux,
               int epi, FpropPlan* plan) {
  ConvGeom g;
  if (!make_geom(d, &g) || !chan_ok(d.c) || d.k % 16 != 0 || d.k < 16) return PBDK_EINVAL;
  if (epi < PBDK_EPI_STORE || epi > PBDK_EPI_BIAS_SWISH) return PBDK_EINVAL;
  if (epi_flags(epi).bias && bias == nullptr) return PBDK_EINVAL;
  if (epi_flags(epi).aux && aux == nullptr) return PBDK_EINVAL;
  const int bkc = chan_block(d.c);
  FpropChoice ch = choose_fprop(d, g, bkc);
  {
    static const int m2_mode = [] {
      const char* e = pbd::knob_env("PBDK_M2");  // 0 off, 1 auto (default), 2 force where legal
      return e != nullptr ? std::atoi(e) : 1;
    }();
    const bool legal = ch.splits == 1 && !ch.pair && (ch.bn == 64 || ch.bn == 128) && bkc == 64 &&
                       g.m_tiles >= 2 && !fprop_bres(d, ch.bn, bkc) && d.r * d.s > 1;
    // measured (scripts/time_conv.py): a win when the pairs still fill every SM (128->128 @16x16:
    // 24.4 -> 21.9 us), a loss on the small-M strided / 4x4 convs
    const int items = (g.m_tiles + 1) / 2 * (d.k / ch.bn);
    if (legal && m2_mode == 2) ch.m2 = true;
    if (legal && m2_mode == 1) ch.m2 = items >= num_sms() && m2_auto(d, g, ch.bn);
  }
  const int bn = ch.bn;
  const int splits = ch.splits;
  const bool pair = ch.pair;
  const bool bres = !pair && !ch.m2 && fprop_bres(d, bn, bkc);
  const bool halo = splits == 1 && !pair && halo_enabled() && bres && bn <= 128 && d.r == 3 && d.s == 3 && d.stride == 1 && d.pad == 1 &&
                    d.q + 2 == kHaloWP && d.w == d.q;
  // short-K convs (3x3 over <= 32 channels, 1x1 over <= 64): the epilogue bounds the tile, so two
  // epilogue warps per TMEM lane quarter (PBDK_EPW=1/2 forces)
  static const int epw_env = [] {
    const char* e = pbd::knob_env("PBDK_EPW");
    return e != nullptr ? std::atoi(e) : 0;
  }();
  const bool short_k = (d.r * d.s == 9 && d.c <= 32) || (d.r * d.s == 1 && d.c <= 64);
  const int epw = bn >= 32 && bn <= 128 && (epw_env == 2 || (epw_env == 0 && (short_k || t_epw == 2))) ? 2 : 1;
  FpropLauncher l = nullptr;
  switch (bkc) {
    case 16: l = bres ? pick_fprop<16, true>(bn, epw) : pick_fprop<16, false>(bn, epw); break;
    case 32: l = bres ? pick_fprop<32, true>(bn, epw) : pick_fprop<32, false>(bn, epw); break;
    case 64: l = bres ? pick_fprop<64, true>(bn, epw) : pick_fprop<64, false>(bn, epw); break;
    default: break;
  }
  if (splits > 1) l = bkc == 64 ? pick_splitk<64>(bn) : nullptr;
  if (pair) l = bkc != 64 ? nullptr : bn == 256 ? launch_fprop_pair<256, 64> : bn == 128 ? launch_fprop_pair<128, 64> : nullptr;
  if (halo) {
    switch (bkc) {
      case 16: l = pick_halo<16>(bn, epw); break;
      case 32: l = pick_halo<32>(bn, epw); break;
      case 64: l = pick_halo<64>(bn, epw); break;
      default: l = nullptr; break;
    }
  }
  if (ch.m2) l = bn == 128 ? launch_fprop_m2<128, 64> : bn == 64 ? launch_fprop_m2<64, 64> : nullptr;
  if (l == nullptr) return PBDK_EINVAL;
  FpropArgs& a0 = plan->args;
  if (halo) {
    const int wp = kHaloWP;
    const int halo_rows = 3 + (129 + wp - 1) / wp;
    a0.tiles_img = (d.p * wp + 127) / 128;
    const uint64_t dims[4] = {static_cast<uint64_t>(d.c), static_cast<uint64_t>(d.w), static_cast<uint64_t>(d.h),
                              static_cast<uint64_t>(d.n)};
    const uint64_t strides[3] = {static_cast<uint64_t>(d.c) * 2, static_cast<uint64_t>(d.w) * d.c * 2,
                                 static_cast<uint64_t>(d.h) * d.w * d.c * 2};
    const uint32_t box[4] = {static_cast<uint32_t>(bkc), static_cast<uint32_t>(wp),
                             static_cast<uint32_t>(halo_rows), 1};
    const uint32_t es[4] = {1, 1, 1, 1};
    if (!encode_tmap_bf16(&plan->tmx, x, 4, dims, strides, box, es, bkc * 2)) return PBDK_ECUDA;
  } else if (!act_map(&plan->tmx, x, d.n, d.h, d.w, d.c, bkc, g.bw, g.bh, g.bn, d.stride)) {
    return PBDK_ECUDA;
  }
  {
    const uint64_t ktot = static_cast<uint64_t>(d.r) * d.s * d.c;
    const uint64_t dims[2] = {ktot, static_cast<uint64_t>(d.k)};
    const uint64_t strides[1] = {ktot * 2};
    const uint32_t box[2] = {static_cast<uint32_t>(bkc), static_cast<uint32_t>(pair ? bn / 2 : bn)};
    const uint32_t es[2] = {1, 1};
    if (!encode_tmap_bf16(&plan->tmw, w, 2, dims, strides, box, es, bkc * 2)) return PBDK_ECUDA;
  }
  FpropArgs& a = plan->args;
  a.n = d.n;
  a.p = d.p;
  a.q = d.q;
  a.k = d.k;
  a.stride = d.stride;
  a.pad = d.pad;
  a.r = d.r;
  a.s = d.s;
  a.bw = g.bw;
  a.bh = g.bh;
  a.bn = g.bn;
  a.tiles_q = g.tiles_q;
  a.tiles_p = g.tiles_p;
  a.c_chunks = d.c / bkc;
  a.epi = epi;
  {
    const char* dbg = pbd::knob_env("PBDK_CONV_DEBUG");
    a.debug = dbg != nullptr ? std::atoi(dbg) : 0;
    a.dbg_buf = (DBG_GE(a, 4) && aux != nullptr) ? static_cast<long long*>(const_cast<void*>(aux)) : nullptr;
  }
  a.y = static_cast<__nv_bfloat16*>(y);
  a.bias = bias;
  a.aux = static_cast<const __nv_bfloat16*>(aux);
  a.n_tiles = d.k / bn;
  a.m_tiles = halo ? d.n * a.tiles_img : g.m_tiles;
  const int tiles = a.n_tiles * a.m_tiles;
  if (ch.m2) {
    const int items = (a.m_tiles + 1) / 2 * a.n_tiles;
    plan->grid = dim3(static_cast<unsigned>(std::min(items, grid_sms())), 1, 1);
  } else if (pair) {
    plan->grid = dim3(static_cast<unsigned>(2 * std::min(tiles / 2, grid_sms() / 2)), 1, 1);
  } else if (splits > 1) {
    plan->grid = dim3(static_cast<unsigned>(splits), static_cast<unsigned>(tiles), 1);
  } else {
    plan->grid = dim3(static_cast<unsigned>(std::min(tiles, grid_sms())), 1, 1);
  }
  plan->bn_tile = bn;
  plan->bkc = bkc;
  plan->smem_bytes = 0;
  plan->launch = l;
  if (l(*plan, reinterpret_cast<cudaStream_t>(-1)) != cudaSuccess) return PBDK_ECUDA;
  return PBDK_OK;
}

int fprop_run(const FpropPlan& plan, cudaStream_t stream) {
  if (plan.launch == nullptr) return PBDK_EINVAL;
  return plan.launch(plan, stream) == cudaSuccess ? PBDK_OK : PBDK_ECUDA;
}

// the multi-tap kernel wants >= 4 pixel tiles per CTA in one wave (else the per-tap grid, whose
// CTAs split the taps, fills the GPU with far fewer partial slabs)
int wgrad_mt_groups(const pbdk_conv_desc& d) {
  return d.c >= 64 ? ((d.k + 127) / 128) * (d.c / 64) * (9 / wgrad_mt_taps(d)) : 1;
}

bool use_wgrad_mt(const ConvGeom& g) {
  if (pick_wgrad_mt(g.d) == nullptr) return false;
  const int groups = wgrad_mt_groups(g.d);
  return g.m_tiles * groups >= 4 * 148;  // >= 4 pixel tiles per CTA in one wave
}

// CTAs of one wgrad split grid.  A constant, not a function of the partition that plans it: the split
// count fixes the summation order, so a block's gradients must not depend on its placement.  The
// wgrads run beside the other student streams; measured on the 4-block step at b=256: a 148-CTA wave
// 0.928 ms, 96 / 64 / 48 CTAs 0.907 / 0.908 / 0.902 ms (fewer splits also shrink the reduction).
// PBDK_WGRAD_WAVE overrides.
int wgrad_wave() {
  static const int w = [] {
    const char* e = pbd::knob_env("PBDK_WGRAD_WAVE");
    return e != nullptr ? std::max(1, std::atoi(e)) : 64;
  }();
  return w;
}

int wgrad_splits(const ConvGeom& g) {
  if (use_wgrad_mt(g)) {  // one wave: groups x splits ~ #SMs
    const int groups = wgrad_mt_groups(g.d);
    const int want = std::max(1, wgrad_wave() / groups);
    const int tps = (g.m_tiles + want - 1) / want;
    return (g.m_tiles + tps - 1) / tps;
  }
  const int co_tiles = (g.d.k + 127) / 128;
  const int ci_tiles = g.d.c / wgrad_bn(g.d.c);
  const int tiles = co_tiles * ci_tiles * g.d.r * g.d.s;
  // one wave of CTAs: the student streams run concurrently, so the wgrads need not fill the
  // GPU alone, and every split costs a partial slab in the fixed-order reduction.
  const int target = wgrad_wave();
  int splits = std::max(1, target / tiles);
  splits = std::min(splits, std::max(1, g.m_tiles / 8));  // >= 8 pixel tiles per split
  return splits;
}

size_t wgrad_workspace_bytes(const pbdk_conv_desc& d) {
  ConvGeom g;
  if (!make_geom(d, &g)) return 0;
  const int splits = wgrad_splits(g);
  if (splits <= 1) return 0;
  return static_cast<size_t>(splits) * d.k * d.r * d.s * d.c * sizeof(float);
}

int wgrad_plan(const pbdk_conv_desc& d, const void* x, const void* dy, float* dw, void* ws, size_t ws_bytes,
               WgradPlan* plan) {
  ConvGeom g;
  if (!make_geom(d, &g) || !chan_ok(d.c) || !chan_ok(d.k)) return PBDK_EINVAL;
  const int swa = chan_block(d.k) * 2;
  const int swb = chan_block(d.c) * 2;
  const WgradLauncher mt = use_wgrad_mt(g) ? pick_wgrad_mt(d) : nullptr;
  const int bn = mt != nullptr ? std::min(d.c, 64) : wgrad_bn(d.c);
  WgradLauncher l = mt != nullptr ? mt : pick_wgrad(bn, swa, swb);
  if (l == nullptr) return PBDK_EINVAL;
  const int splits = wgrad_splits(g);
  const size_t slab = static_cast<size_t>(d.k) * d.r * d.s * d.c;
  if (splits > 1 && (ws == nullptr || ws_bytes < splits * slab * sizeof(float))) return PBDK_EINVAL;
  if (!act_map(&plan->tmdy, dy, d.n, d.p, d.q, d.k, swa / 2, g.bw, g.bh, g.bn, 1)) return PBDK_ECUDA;
  if (!act_map(&plan->tmx, x, d.n, d.h, d.w, d.c, swb / 2, g.bw, g.bh, g.bn, d.stride)) return PBDK_ECUDA;
  WgradArgs& a = plan->args;
  a.n = d.n;
  a.p = d.p;
  a.q = d.q;
  a.k = d.k;
  a.c = d.c;
  a.stride = d.stride;
  a.pad = d.pad;
  a.r = d.r;
  a.s = d.s;
  a.bw = g.bw;
  a.bh = g.bh;
  a.bn = g.bn;
  a.tiles_q = g.tiles_q;
  a.tiles_p = g.tiles_p;
  a.m_tiles = g.m_tiles;
  a.co_tiles = (d.k + 127) / 128;
  a.ci_tiles = d.c / bn;
  a.tiles_per_split = (g.m_tiles + splits - 1) / splits;
  a.a_atoms = (std::min(128, d.k) + swa / 2 - 1) / (swa / 2);
  a.out = splits > 1 ? static_cast<float*>(ws) : dw;
  plan->grid = mt != nullptr ? dim3(static_cast<unsigned>(splits), static_cast<unsigned>(wgrad_mt_groups(d)), 1)
                              : dim3(static_cast<unsigned>(a.co_tiles * a.ci_tiles * d.r * d.s),
                                     static_cast<unsigned>(splits), 1);
  plan->splits = splits;
  plan->bn_tile = bn;
  plan->dw = dw;
  plan->slab = slab;
  plan->launch = l;
  if (l(*plan, reinterpret_cast<cudaStream_t>(-1)) != cudaSuccess) return PBDK_ECUDA;
  return PBDK_OK;
}

int split_reduce_cap() {
  static const int cap = [] {
    const char* e = pbd::knob_env("PBDK_SPLITRED_CTAS");
    return e != nullptr ? std::max(1, std::atoi(e)) : 148 * 8;
  }();
  return cap;
}

int wgrad_run(const WgradPlan& plan, cudaStream_t stream) {
  if (plan.launch == nullptr) return PBDK_EINVAL;
  if (plan.launch(plan, stream) != cudaSuccess) return PBDK_ECUDA;
  if (plan.splits > 1) {
    const size_t n4 = plan.slab / 4;
    const int blocks =
        static_cast<int>(std::max<size_t>(1, std::min<size_t>((n4 + kRedLanes - 1) / kRedLanes, split_reduce_cap())));
    if (launch_ex(split_reduce_kernel, dim3(blocks, 1, 1), dim3(kRedLanes * kRedSplitLanes, 1, 1), 0, stream, plan.pdl,
                  1u, reinterpret_cast<const float4*>(plan.args.out), reinterpret_cast<float4*>(plan.dw), n4,
                  plan.splits) != cudaSuccess)
      return PBDK_ECUDA;
  }
  return PBDK_OK;
}

}  // namespace pbdk

// ------------------------------------------------------------------ C ABI
extern "C" {

const char* pbdk_build_info(void) { return "pbdk sm_100a tcgen05"; }

void pbdk_conv_scope(int sms, int epw) {
  pbdk::t_grid_sms = sms > 0 ? sms : 0;
  pbdk::t_epw = epw == 2 ? 2 : 0;
}

int pbdk_conv_fprop(const pbdk_conv_desc* d, const void* x, const void* w, void* y, const float* bias,
                    const void* aux, int epilogue, void* stream) {
  if (d == nullptr) return PBDK_EINVAL;
  pbdk::FpropPlan plan;
  const int rc = pbdk::fprop_plan(*d, x, w, y, bias, aux, epilogue, &plan);
  if (rc != PBDK_OK) return rc;
  return pbdk::fprop_run(plan, static_cast<cudaStream_t>(stream));
}

size_t pbdk_conv_wgrad_workspace_bytes(const pbdk_conv_desc* d) {
  return d == nullptr ? 0 : pbdk::wgrad_workspace_bytes(*d);
}

int pbdk_conv_wgrad(const pbdk_conv_desc* d, const void* x, const void* dy, float* dw, void* workspace,
                    size_t workspace_bytes, void* stream) {
  if (d == nullptr) return PBDK_EINVAL;
  pbdk::WgradPlan plan;
  const int rc = pbdk::wgrad_plan(*d, x, dy, dw, workspace, workspace_bytes, &plan);
  if (rc != PBDK_OK) return rc;
  return pbdk::wgrad_run(plan, static_cast<cudaStream_t>(stream));
}

int pbdk_weight_flip(const void* w, void* wt, int k, int r, int s, int c, void* stream) {
  if (w == nullptr || wt == nullptr || k < 1 || r < 1 || s < 1 || c < 1) return PBDK_EINVAL;
  const size_t total = static_cast<size_t>(k) * r * s * c;
  const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16));
  pbdk::weight_flip_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(wt), k, r, s, c);
  return cudaGetLastError() == cudaSuccess ? PBDK_OK : PBDK_ECUDA;
}

}  // extern "C"
