// Internal C++ interface of the HBM-bound blockwise-distillation kernels (bd_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pbdk {

struct MseArgs {
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
  float* ws;
  float* red;
  float* dgamma2;
  float* dbeta2;
  float* dgammasc;
  float* dbetasc;
  double* loss;
  void* dy2;
  void* dysc;
  int prec = 0;  // 0: bf16 rows; 1: y2/ysc fp32, t / dy2 / dysc split fp32 (the fp32 workload)
};

size_t reduce_workspace_floats(int m, int c, int nv);

// Grid sizes of the reduction (partial) and elementwise (apply) passes launched by this thread while
// the scope is alive.  Default (no scope): 2 partial CTAs and 8 apply CTAs per SM, best when the
// passes run mostly alone (MBConv step).  The ResNet step runs them beside the conv kernels of the
// other student streams and uses GridScope(148, 296) (see bd_kernels.cu).
struct GridScope {
  GridScope(int red_ctas, int apply_ctas, int fix_min_bytes = 0);  // 0: the default
  ~GridScope();
  int saved_red, saved_apply, saved_fix_min;
};
// synthetic / host images of side x side pixels, stored [n][side][side][16] bf16
// prec 1: split fp32 [n][side][side][2*32] (conv_tf32.hpp) instead
int philox_image(void* x, int n, long long first, const long long* counter, int gb, uint32_t seed, cudaStream_t st,
                 int side = 32, int prec = 0);
int pack_image(const float* src, void* x, int n, cudaStream_t st, int side = 32, int prec = 0);
int pack_image_parity(const float* s0, const float* s1, const long long* counter, void* x, int n, cudaStream_t st,
                      int side = 32, int prec = 0);
// bf16_out: 0 fp32, 1 bf16, 2 split fp32 [k][r][s][2cs]
int init_uniform(void* dst, int bf16_out, int k, int r, int s, int cs, int ct, uint32_t seed, uint32_t tensor,
                 float bound, cudaStream_t st, int kt = -1);  // kt: true output channels (rows >= kt zero)
int fill(float* dst, size_t n, float v, cudaStream_t st);
// prec 1 (fp32 workload): fp32 inputs; outputs that feed convolutions are split fp32
int bn_stats(const void* y, int m, int c, float* ws, float* mean_rstd, cudaStream_t st, int prec = 0);
// statistics of two same-shape tensors in one pass (the student's y2 and shortcut y)
int bn_stats2(const void* y0, const void* y1, int m, int c, float* ws, float* mr0, float* mr1, cudaStream_t st,
              int prec = 0);
int bn_apply_relu(const void* y, const float* mean_rstd, const float* gamma, const float* beta, void* a, int m, int c,
                  cudaStream_t st, int prec = 0);
int mse_bn_loss(const MseArgs& a, cudaStream_t st);
int bn_bwd(const void* g, const void* y, const float* mean_rstd, const float* gamma, int m, int c, float* ws,
           float* red, float* dgamma, float* dbeta, void* dy, cudaStream_t st, int prec = 0);
int sgd_momentum(float* w, float* v, const float* g, void* shadow, size_t n, float lr, float mu, long long* counter,
                 cudaStream_t st);
// Flipped dgrad copies written by the update itself: region i covers elements [off, off + k*r*s*c) of
// the updated vector (a [k][r][s][c] filter); its bf16 value (the shadow's rounding) is also stored at
// dst[c'][r-1-r'][s-1-s'][k'] — what pbdk_weight_flip would produce from the shadow, without the launch.
struct FlipRegion {
  size_t off;
  int k, r, s, c;
  void* dst;
};
struct FlipSet {
  static constexpr int kMax = 4;
  int count = 0;
  FlipRegion reg[kMax];
};
int sgd_momentum_flip(float* w, float* v, const float* g, void* shadow, size_t n, float lr, float mu,
                      long long* counter, const FlipSet& flips, cudaStream_t st);

// ---- self-finalizing variants of bn_stats / bn_stats2 / mse_bn_loss / bn_bwd (bf16 rows): one partial
// launch per reduction instead of partial + finalize; every pass streams its rows through a TMA-staged
// shared-memory ring (bd_kernels.cu row_pipe).  Each CTA adds its chunk partial exactly into
// fixed-point accumulators (fixacc.cuh); the last CTA to finish writes the same outputs the finalize
// kernels wrote (mean/rstd, coefficients, parameter gradients, loss) and re-zeroes its scratch.
// FixScratch: fix_acc_words(c) zero-initialised words + one zeroed ticket, per concurrent reduction.
struct FixScratch {
  unsigned long long* acc;
  unsigned int* ticket;
};
size_t fix_acc_words(int c);
int bn_stats_fix(const void* y0, const void* y1, int m, int c, FixScratch fx, float* mr0, float* mr1,
                 cudaStream_t st);
int bn_apply_relu_fix(const void* y, const float* mean_rstd, const float* gamma, const float* beta, void* a, int m,
                      int c, cudaStream_t st);  // the same arithmetic as bn_apply_relu, TMA-staged rows
int mse_bn_loss_fix(const MseArgs& a, FixScratch fx, cudaStream_t st);
int bn_bwd_fix(const void* g, const void* y, const float* mean_rstd, const float* gamma, int m, int c, FixScratch fx,
               float* red, float* dgamma, float* dbeta, void* dy, cudaStream_t st);
// the same update on g = g[0] + g[1] + ... (member order), the DP group's gradient slabs in peer memory
int sgd_momentum_sum(float* w, float* v, const float* const* g, int count, void* shadow, size_t n, float lr, float mu,
                     long long* counter, cudaStream_t st);
// DP all-gather: w[slice j] = peer_w[j][slice j] for every member j != me (slices: float4 index i belongs to
// ((i+1)*G-1)/(n/4)), bf16 shadow refreshed when non-null.  peer_w[me] is ignored.
int dp_gather(float* w, void* shadow, const float* const* peer_w, int count, int me, size_t n, cudaStream_t st);

// element range [lo, hi) of member j's slice of an n-element region (n multiple of 4) in a G-member group
inline void dp_slice(size_t n, int G, int j, size_t* lo, size_t* hi) {
  const size_t n4 = n / 4;
  *lo = 4 * (static_cast<size_t>(j) * n4 / static_cast<size_t>(G));
  *hi = 4 * ((static_cast<size_t>(j) + 1) * n4 / static_cast<size_t>(G));
}

}  // namespace pbdk
