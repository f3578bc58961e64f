// Internal C++ interface of the tcgen05 implicit-GEMM convolution engine.
// The executor builds plans once per layer (tensor maps baked in) and replays
// them every step; the C-ABI entry points in pbdk.h build a plan per call.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>

#include "pbdk.h"

namespace pbdk {

// Output-pixel tiling shared by fprop and wgrad: a 128-row GEMM tile is a
// (bn images) x (bh rows) x (bw cols) box of output pixels, which is exactly
// what one 4D TMA box of the input delivers for one filter tap.
struct ConvGeom {
  pbdk_conv_desc d;
  int bw, bh, bn;
  int tiles_q, tiles_p, tiles_n;
  int m_tiles;
};

bool make_geom(const pbdk_conv_desc& d, ConvGeom* g);

struct FpropArgs {
  int n, p, q, k;
  int stride, pad, r, s;
  int bw, bh, bn, tiles_q, tiles_p;
  int c_chunks;
  int n_tiles, m_tiles;
  int tiles_img;  // halo variant only
  int epi;
  int debug;  // timing experiments (PBDK_CONV_DEBUG): 0 normal; 1 skip epilogue stores; 2 skip MMAs;
              // 3 skip epilogue; 4 cycle counters; halo kernel: 6 no activation loads, 7 = 6 + 3,
              // 8 MMA warp alone (no producer / epilogue, no barrier waits)
  long long* dbg_buf;  // debug 4: per CTA {total, wait_tempty, wait_full, issue, epi_wait, epi_work}
  __nv_bfloat16* y;
  const float* bias;
  const __nv_bfloat16* aux;
};

struct FpropPlan {
  CUtensorMap tmx;
  CUtensorMap tmw;
  FpropArgs args;
  dim3 grid;
  int bn_tile = 0;
  int bkc = 0;
  int smem_bytes = 0;
  bool pdl = false;  // launch with programmatic dependent launch (the kernels call griddepcontrol.wait)
  cudaError_t (*launch)(const FpropPlan&, cudaStream_t) = nullptr;
};

int fprop_plan(const pbdk_conv_desc& d, const void* x, const void* w, void* y, const float* bias, const void* aux,
               int epi, FpropPlan* plan);
int fprop_run(const FpropPlan& plan, cudaStream_t stream);

struct WgradArgs {
  int n, p, q, k, c;
  int stride, pad, r, s;
  int bw, bh, bn, tiles_q, tiles_p;
  int m_tiles;
  int co_tiles, ci_tiles;
  int tiles_per_split;
  int a_atoms;  // A (dy) atoms actually loaded per stage
  float* out;   // dw (splits == 1) or workspace
};

// While alive, fprop plans built by this thread spread their persistent grid over at most `sms` SMs
// (0 = all).  Results do not depend on it (tiles are independent); wgrad split counts, which fix a
// summation order, ignore it.
// `epw` = 2 asks for two epilogue warps per TMEM lane quarter on every eligible conv (0 = by shape).
struct ConvGridScope {
  explicit ConvGridScope(int sms, int epw = 0);
  ~ConvGridScope();
  int saved, saved_epw;
};

struct WgradPlan {
  CUtensorMap tmdy;
  CUtensorMap tmx;
  WgradArgs args;
  dim3 grid;
  int splits = 1;
  int bn_tile = 0;
  int smem_bytes = 0;
  float* dw = nullptr;
  size_t slab = 0;  // elements of dw
  bool pdl = false;  // as FpropPlan::pdl (the split reduction after it is a plain launch)
  cudaError_t (*launch)(const WgradPlan&, cudaStream_t) = nullptr;
};

int wgrad_splits(const ConvGeom& g);
size_t wgrad_workspace_bytes(const pbdk_conv_desc& d);
int wgrad_plan(const pbdk_conv_desc& d, const void* x, const void* dy, float* dw, void* ws, size_t ws_bytes,
               WgradPlan* plan);
int wgrad_run(const WgradPlan& plan, cudaStream_t stream);

}  // namespace pbdk
