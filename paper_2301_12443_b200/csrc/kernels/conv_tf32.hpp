// fp32 convolutions on the tensor cores (3xTF32, tcgen05 kind::tf32) for the fp32 workload
// (BASELINE configs[0]: the reference's smallest case, batch 64, fp32).
//
// Storage ("split fp32"): a tensor that feeds a convolution as an operand is kept as
// [rows][2c] fp32 with row = [hi(c) | lo(c)], hi = tf32(x) (round to nearest), lo = x - hi (exact).
// hi + lo == x bit-exactly, so consumers that need the value (residual adds, the distillation
// target, ReLU masks) read it losslessly; a convolution computes sum a*b as
// a_hi*b_hi + a_hi*b_lo + a_lo*b_hi on the tensor cores with fp32 accumulation in TMEM (the
// dropped a_lo*b_lo term and the tf32 reading of the lo parts leave ~2^-21 relative error per
// product, fp32-class accuracy).  Tensors that only feed elementwise kernels stay plain fp32.
//
// Descriptors use pbdk_conv_desc with c / k = channels per half (true fp32 channel counts,
// multiples of 16; the 3-channel image is stored as 16).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>

#include "pbdk.h"

namespace pbdk {

struct F3FpropArgs {
  int n, p, q, k, c;
  int stride, pad, r, s;
  int bw, bh, bn, tiles_q, tiles_p;
  int c_chunks;
  int epi;
  int y_split;  // 1: y is split fp32 [m][2k]; 0: plain fp32 [m][k]
  float* y;
  const float* bias;
  const float* aux;  // split fp32 [m][2k] (residual / ReLU mask)
};

struct F3FpropPlan {
  CUtensorMap tmx, tmw;
  F3FpropArgs args;
  dim3 grid;
  cudaError_t (*launch)(const F3FpropPlan&, cudaStream_t) = nullptr;
};

// x: split [n][h][w][2c]; w: split [k][r][s][2c]; y / aux per F3FpropArgs.
int f3_fprop_plan(const pbdk_conv_desc& d, const float* x, const float* w, float* y, int y_split, const float* bias,
                  const float* aux, int epi, F3FpropPlan* plan);
int f3_fprop_run(const F3FpropPlan& plan, cudaStream_t st);

struct F3WgradArgs {
  int n, p, q, k, c;
  int stride, pad, r, s;
  int bw, bh, bn, tiles_q, tiles_p;
  int m_tiles, co_tiles, ci_tiles, tiles_per_split;
  float* out;  // dw [k][r][s][c] (1 split) or the split slabs
};

struct F3WgradPlan {
  CUtensorMap tmdy, tmx;
  F3WgradArgs args;
  dim3 grid;
  int splits = 1;
  float* dw = nullptr;
  size_t slab = 0;
  cudaError_t (*launch)(const F3WgradPlan&, cudaStream_t) = nullptr;
};

size_t f3_wgrad_workspace_bytes(const pbdk_conv_desc& d);
// x: split [n][h][w][2c]; dy: split [n][p][q][2k]; dw: plain fp32 [k][r][s][c].
int f3_wgrad_plan(const pbdk_conv_desc& d, const float* x, const float* dy, float* dw, void* ws, size_t ws_bytes,
                  F3WgradPlan* plan);
int f3_wgrad_run(const F3WgradPlan& plan, cudaStream_t st);

// plain [rows][c] -> split [rows][2c]
int f3_split(const float* src, float* dst, size_t rows, int c, cudaStream_t st);
// master [k][r][s][c] -> split flipped [c][r][s][2k] (weights of the dgrad convolution)
int f3_flip_split(const float* w, float* wt, int k, int r, int s, int c, cudaStream_t st);

}  // namespace pbdk
