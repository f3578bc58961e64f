// Internal interface of the MobileNetV2 -> ProxylessNAS CUDA-core kernels (mb_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace pbdk {

// depthwise k x k conv, NHWC bf16, pad = k / 2
struct DwArgs {
  int n, h, w, c;  // input
  int k, stride;
  int p, q;  // output
};

// activation codes of dw_fwd / stem_fwd: 0 none, 1 ReLU6, 2 swish
// y = act(dw(x) [+ bias]); wt = flipped tap-major weights wt[r'][s'][c]
// variant: -1 product choice (staged tiles where they fit), 0 per-strip kernel, 1 staged tiles (bit-identical)
int dw_fwd(const DwArgs& d, const void* x, const void* wt, const float* bias, void* y, int relu6, cudaStream_t s,
           int variant = -1);
// dx = dw^T(dy) [masked by 0 < act < 6]
// variant as dw_fwd (the staged tiles serve stride 1)
int dw_dgrad(const DwArgs& d, const void* dy, const void* wt, const void* act, void* dx, cudaStream_t s,
             int variant = -1);
// dw[c][r][s] (fp32, the parameter layout) = sum dy * shifted a
size_t dw_wgrad_workspace_floats(const DwArgs& d);
int dw_wgrad(const DwArgs& d, const void* a, const void* dy, float* ws, size_t ws_floats, float* dw, cudaStream_t s);

// stem 3x3 / stride 2, 3 (stored 16) -> 32 channels on an S x S image
int stem_fwd(const void* x, const void* w, const float* bias, void* y, int n, int S, int relu6, cudaStream_t s);
size_t stem_wgrad_workspace_floats(int n, int S);
int stem_wgrad(const void* x, const void* dy, int n, int S, float* ws, size_t ws_floats, float* dw, cudaStream_t s);

// squeeze-excite (EfficientNet teacher) in place on y [n][hw][E]: gate = sigmoid(W2 swish(W1 mean_hw(y) + b1)
// + b2), y *= gate.  w1 [cs][E], w2 [E][cs] bf16; pooled, gate: n*E floats of workspace each.
int se_apply(void* y, int n, int hw, int E, int cs, const void* w1, const float* b1, const void* w2,
             const float* b2, float* pooled, float* gate, cudaStream_t s);

// out = bf16(act(fmaf(A, y, B)) [+ res]), A = gamma*rstd, B = fmaf(-A, mean, beta)
int bn_apply_act(const void* y, const float* mean_rstd, const float* gamma, const float* beta, const void* res,
                 void* out, long long m, int c, int relu6, cudaStream_t s);

// z = fmaf(A, y, B) [+ res]; g = bf16((z - t) * gscale); *loss = sum (z - t)^2 / norm
size_t mse_affine_workspace_doubles(long long m, int c);
int mse_affine(const void* y, const float* mean_rstd, const float* gamma, const float* beta, const void* res,
               const void* t, long long m, int c, float gscale, double norm, void* g, double* ws, double* loss,
               cudaStream_t s);

}  // namespace pbdk
