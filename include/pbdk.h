/*
 * pbdk.h — C-ABI of the B200 (sm_100a) blockwise-distillation kernels.
 *
 * The reference (Pipe-BD, /root/reference) has no device code: it models each
 * of these operations as a cost term of Algorithm 1.  The
 * entry points below are the device implementation of those terms:
 *
 *   pbdk_conv_fprop   teacher T_i.forward / student S_i.forward convolutions,
 *                     and the student dgrad (conv with flipped weights)
 *                     — "teacher_fwd" / "student_fwd_bwd", simulate.cpp:217-235
 *   pbdk_conv_wgrad   student weight gradient — inside S_k (cost_model.cpp:38-66)
 *   pbdk_bn_*         training-mode BatchNorm of the student (forward/backward)
 *   pbdk_mse_*        fused distillation loss L(s,t) + dL/ds
 *   pbdk_sgd_momentum S_i.update_weight() (simulate.cpp:243-261)
 *   pbdk_philox_*     load_data() for the first partition
 *
 * Conventions: POD descriptors, caller-owned device memory,
 * no allocation inside the calls, explicit stream (a cudaStream_t passed as
 * void*), int status.  Activations are NHWC bf16; channel counts are the
 * STORED (padded) counts — the image's 3 channels are stored as 16.
 * Weights are [K][R][S][C] bf16 (K-major for the implicit GEMM).
 */
#ifndef PBDK_H_
#define PBDK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define PBDK_OK 0
#define PBDK_EINVAL 1  /* unsupported / inconsistent shape: maps to pbd::ValidationError */
#define PBDK_ECUDA 2   /* CUDA launch or driver error: maps to pbd::DeviceError */

/* convolution epilogues (fprop) */
#define PBDK_EPI_STORE 0          /* y = acc                                   */
#define PBDK_EPI_BIAS 1           /* y = acc + bias[k]                         */
#define PBDK_EPI_BIAS_RELU 2      /* y = relu(acc + bias[k])                   */
#define PBDK_EPI_BIAS_RES_RELU 3  /* y = relu(acc + bias[k] + aux[m][k])       */
#define PBDK_EPI_RELU_MASK 4      /* y = aux[m][k] > 0 ? acc : 0   (relu bwd)  */
#define PBDK_EPI_BIAS_RELU6 5     /* y = min(max(acc + bias[k], 0), 6)          */
#define PBDK_EPI_BIAS_RES 6       /* y = acc + bias[k] + aux[m][k]              */
#define PBDK_EPI_RELU6_MASK 7     /* y = 0 < aux[m][k] < 6 ? acc : 0 (relu6 bwd) */
#define PBDK_EPI_ADD 8            /* y = acc + aux[m][k]                        */
#define PBDK_EPI_BIAS_SWISH 9     /* y = z * sigmoid(z), z = acc + bias[k]      */

typedef struct pbdk_conv_desc {
  int n, h, w, c;  /* input NHWC, c = stored channels (multiple of 16) */
  int k;           /* output channels (multiple of 16)                */
  int r, s;        /* filter height / width                           */
  int stride, pad; /* symmetric                                       */
  int p, q;        /* output height / width                           */
} pbdk_conv_desc;

/* Library identity: returns "sm_100a" build tag; used by loaders to fail loudly. */
const char* pbdk_build_info(void);

/* y[n,p,q,k] = epi( sum_{r,s,c} x[n, p*st+r-pad, q*st+s-pad, c] * w[k,r,s,c] )
 * tcgen05 implicit GEMM: M = n*p*q pixels (128 per tile), N = k, K = r*s*c. */
/* Plans built by later pbdk_conv_fprop calls on this thread use at most `sms` SMs (0 = all) and, with
 * epw = 2, two epilogue warps per TMEM lane quarter — the settings the ResNet executor builds its
 * plans with (ConvGridScope); pbdk_conv_scope(0, 0) restores the shape defaults. */
void pbdk_conv_scope(int sms, int epw);
int pbdk_conv_fprop(const pbdk_conv_desc* d, const void* x, const void* w, void* y, const float* bias,
                    const void* aux, int epilogue, void* stream);

/* dw[k,r,s,c] = sum_{n,p,q} dy[n,p,q,k] * x[n, p*st+r-pad, q*st+s-pad, c]   (fp32 out)
 * tcgen05 GEMM with MN-major operands, split-K over pixels; `workspace` must hold
 * pbdk_conv_wgrad_workspace_bytes(d) bytes (may be 0 => no workspace needed). */
size_t pbdk_conv_wgrad_workspace_bytes(const pbdk_conv_desc* d);
int pbdk_conv_wgrad(const pbdk_conv_desc* d, const void* x, const void* dy, float* dw, void* workspace,
                    size_t workspace_bytes, void* stream);

/* wt[c,r',s',k] = w[k,R-1-r',S-1-s',c]  (bf16 -> bf16): weights of the dgrad conv. */
int pbdk_weight_flip(const void* w, void* wt, int k, int r, int s, int c, void* stream);


/* ------------------------------------------------------------------ fp32 convolutions (3xTF32, configs[0]) */
/* Split-fp32 storage: an operand tensor [rows][2c] holds hi = tf32(x) (round to nearest) in channels
 * [0, c) and lo = x - hi (exact) in [c, 2c); hi + lo == x.  The tensor cores compute every product as
 * a_hi*b_hi + a_hi*b_lo + a_lo*b_hi (tcgen05 kind::tf32, fp32 accumulation).  d->c / d->k are the
 * channels per half (multiples of 16; 16 or a multiple of 32 for inputs).
 * x: split [n][h][w][2c]; w: split [k][r][s][2c]; y: split [m][2k] (y_split = 1) or plain [m][k];
 * aux (residual for PBDK_EPI_BIAS_RES_RELU, mask source for PBDK_EPI_RELU_MASK): split [m][2k].
 * Epilogues: STORE, BIAS, BIAS_RELU, BIAS_RES_RELU, RELU_MASK. */
int pbdk_conv3x_fprop(const pbdk_conv_desc* d, const float* x, const float* w, float* y, int y_split,
                      const float* bias, const float* aux, int epilogue, void* stream);
/* dw[k,r,s,c] (plain fp32) from split x [n][h][w][2c] and split dy [n][p][q][2k] (k multiple of 32) */
size_t pbdk_conv3x_wgrad_workspace_bytes(const pbdk_conv_desc* d);
int pbdk_conv3x_wgrad(const pbdk_conv_desc* d, const float* x, const float* dy, float* dw, void* workspace,
                      size_t workspace_bytes, void* stream);
/* plain [rows][c] -> split [rows][2c] */
int pbdk_split_tf32(const float* src, float* dst, size_t rows, int c, void* stream);
/* master w [k][r][s][c] -> split flipped wt [c][r][s][2k] (dgrad weights) */
int pbdk_weight_flip_split(const float* w, float* wt, int k, int r, int s, int c, void* stream);

/* ------------------------------------------------------------------ K12: synthetic input (load_data) */
/* x[n][32][32][16] bf16 (3 Philox channels + 13 zero pad channels) for global samples
 * first_sample + (*step_counter)*global_batch + i  (step_counter may be NULL). */
int pbdk_philox_image(void* x, int n, long long first_sample, const long long* step_counter, int global_batch,
                      uint32_t seed, void* stream);
/* device fp32 NHWC [n][32][32][3] -> padded bf16 [n][32][32][16] */
int pbdk_pack_image(const float* src, void* x, int n, void* stream);
/* weights: dst[k][r][s][c_stored] = c < c_true ? U(-1,1)*bound : 0 (Philox counter = (flat unpadded idx, tensor_id)) */
int pbdk_init_uniform(void* dst, int bf16_out, int k, int r, int s, int c_stored, int c_true, uint32_t seed,
                      uint32_t tensor_id, float bound, void* stream);

/* ------------------------------------------------------------------ K2/K3/K5: training-mode BatchNorm */
/* workspace bytes for any of the [m][c] reductions below */
size_t pbdk_reduce_workspace_bytes(int m, int c);
/* mean_rstd[0:c] = batch mean, mean_rstd[c:2c] = 1/sqrt(biased var + 1e-5) */
int pbdk_bn_stats(const void* y, int m, int c, void* workspace, float* mean_rstd, void* stream);
/* a = bf16(relu(gamma*(y-mean)*rstd + beta)) */
int pbdk_bn_apply_relu(const void* y, const float* mean_rstd, const float* gamma, const float* beta, void* a, int m,
                       int c, void* stream);
/* BN backward given dL/d(bn out) g: dbeta = sum g, dgamma = sum g*xhat (= rstd*(sum g*y - mean*sum g)),
 * dy = gamma*rstd/m * (m*g - sum g - xhat*sum g*xhat) evaluated as dy = A*g + Q*y + R (A = gamma*rstd);
 * red receives {Q[c], R[c]} (2c floats). */
int pbdk_bn_bwd(const void* g, const void* y, const float* mean_rstd, const float* gamma, int m, int c,
                void* workspace, float* red, float* dgamma, float* dbeta, void* dy, void* stream);

/* ------------------------------------------------------------------ K4: fused distillation loss + backward */
/* s = relu(BN2(y2) + BNsc(ysc)); loss = sum (s-t)^2 / norm; g = [s>0] (s-t)*gscale (gscale = 2/norm);
 * writes dgamma/dbeta of both BNs, red[4c] = {Q2, R2, Qsc, Rsc} (the coefficients of dy = A*g + Q*y + R)
 * and dy2 / dysc (bf16). */
typedef struct pbdk_mse_args {
  const void* y2;
  const void* ysc;
  const void* t;
  const float* stats2;
  const float* statssc;
  const float* gamma2;
  const float* beta2;
  const float* gammasc;
  const float* betasc;
  int m, c;
  float gscale;
  double norm;
  void* workspace;
  float* red;
  float* dgamma2;
  float* dbeta2;
  float* dgammasc;
  float* dbetasc;
  double* loss;
  void* dy2;
  void* dysc;
} pbdk_mse_args;
int pbdk_mse_bn_loss(const pbdk_mse_args* a, void* stream);

/* ------------------------------------------------------------------ K8: depthwise convolution */
/* y[n,p,q,c] = act(sum_{r,s} x[n, p*stride+r-k/2, q*stride+s-k/2, c] * w[c][r][s] (+ bias[c])), NHWC bf16,
 * fmaf over (r, s) ascending; wt = the flipped tap-major filter [k][k][c] (pbdk_weight_flip with c = 1).
 * act: 0 none, 1 ReLU6, 2 swish.  variant: 0 per-strip register kernel, 1 shared-memory staged tiles,
 * -1 the product's choice — both variants are bit-identical. */
typedef struct pbdk_dw_desc {
  int n, h, w, c, k, stride, p, q;
} pbdk_dw_desc;
int pbdk_dw_fwd(const pbdk_dw_desc* d, const void* x, const void* wt, const float* bias, void* y, int act,
                int variant, void* stream);
/* dx[n,h,w,c] = fmaf chain over (r, s) ascending of dy[n,(h+k/2-r)/stride,(w+k/2-s)/stride,c] * w[c][r][s],
 * then the ReLU6 mask of `act` (0 < a < 6; NULL: none).  variant as pbdk_dw_fwd (staged tiles: stride 1). */
int pbdk_dw_dgrad(const pbdk_dw_desc* d, const void* dy, const void* wt, const void* act, void* dx, int variant,
                  void* stream);

/* ------------------------------------------------------------------ K10: SGD-momentum update */
/* v = mu*v + g; w = w - lr*v (fmaf); w_bf16 (may be NULL) = bf16(w); ++*step_counter (may be NULL).
 * n must be a multiple of 4. */
int pbdk_sgd_momentum(float* w, float* v, const float* g, void* w_bf16, size_t n, float lr, float momentum,
                      long long* step_counter, void* stream);
/* The same update, also storing the flipped bf16 dgrad operand of up to 4 filters inside w: region i
 * covers w[off, off + k*r*s*c) laid out [k][r][s][c]; dst[c'][r-1-r'][s-1-s'][k'] = w_bf16 of that
 * element (bit-identical to pbdk_weight_flip of the updated w_bf16, without its launch).  w_bf16 must be
 * non-NULL. */
typedef struct {
  size_t off;
  int k, r, s, c;
  void* dst;
} pbdk_flip_region;
int pbdk_sgd_momentum_flip(float* w, float* v, const float* g, void* w_bf16, size_t n, float lr, float momentum,
                           long long* step_counter, const pbdk_flip_region* regions, int count, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PBDK_H_ */
