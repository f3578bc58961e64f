/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement (oracle) of one Pipe-BD
 * blockwise-distillation step.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, as the checker.
 *
 * What it restates (there is no executable reference for the numeric path:
 * SPEC.md:15 puts training out of scope):
 *   Algorithm 1 body  PAPER.md:345-374   load_data / T_i.forward / S_i.forward /
 *                                         S_i.backward(L(s,t)) / update_weight
 *   blockwise loss    PAPER.md:192-194    (S_i(T_{i-1} out), T_i out) pairs
 *   batch share       schedule.cpp:63 + SPEC.md:231 (ceil share, first b%g take one extra)
 *   SGD               PAPER.md:428-429   (lr 0.1; momentum 0.9 as torch.optim.SGD)
 * Model and numerics contract: DESIGN.md §3 (ResNet-18-CIFAR teacher, slim
 * residual student, training-mode BN, MSE, SGD-momentum; Philox4x32-10 inputs
 * and weights).  With bf16 != 0 every tensor the GPU path stores in bf16 is
 * rounded to bf16 (round-to-nearest-even) at the same point, so GPU results
 * differ only by fp32 accumulation order.  Parity of this oracle is pinned by
 * tests/golden/ (torch fp32, independent implementation) and Philox KATs.
 */
#ifndef BD_ORACLE_H_
#define BD_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BDO_BLOCKS 4

/* geometry of the CIFAR ResNet-18 teacher / slim student */
int bdo_in_channels(int block);   /* 3, 64, 128, 256 */
int bdo_out_channels(int block);  /* 64, 128, 256, 512 */
int bdo_in_hw(int block);         /* 32, 32, 16, 8 */
int bdo_out_hw(int block);        /* 32, 16, 8, 4 */
size_t bdo_student_param_count(int block);
size_t bdo_teacher_param_count(int block);

/* Philox4x32-10: 4 output words for (counter c[4], key k[2]). */
void bdo_philox(const uint32_t c[4], const uint32_t k[2], uint32_t out[4]);

/* Synthetic input: n samples starting at global sample index `first`,
 * NHWC [n,32,32,3] floats in [-1,1). */
void bdo_input(int n, int64_t first, uint32_t seed, float* out, int bf16);

/* Teacher parameters of block k (flat: per conv W[K][R][S][C] then bias[K],
 * convs in program order) and student parameters (W1, W2, Wsc, g1, b1, g2, b2, gsc, bsc). */
void bdo_teacher_init(int block, uint32_t seed, float* params, int bf16);
void bdo_student_init(int block, uint32_t seed, float* params);

/* Teacher forward of block k on n samples: in NHWC [n, Hin, Hin, Cin] -> out [n, Hout, Hout, Cout]. */
int bdo_teacher_fwd(int block, const float* tparams, int n, const float* in, float* out, int bf16);

/* Student forward + backward of block k on an n-sample shard.
 * `norm` = global_batch * Cout * Hout * Hout (the MSE denominator of the whole step);
 * writes the gradient of sum_shard (s-t)^2 / norm into grads (layout of params)
 * and that partial loss into *loss. */
int bdo_student_fwd_bwd(int block, const float* sparams, int n, const float* in, const float* t_out, double norm,
                        int bf16, float* grads, double* loss);

/* SGD with momentum (torch.optim.SGD semantics, dampening 0, no weight decay):
 * v = mu*v + g ; w = w - lr*v. */
void bdo_sgd(size_t count, float* w, float* v, const float* g, float lr, float mu);

/* bf16 round-to-nearest-even of x (returned as float). */
float bdo_bf16(float x);

/* threads used by the OpenMP loops (for the cpu_baseline record). */
int bdo_threads(void);

#ifdef __cplusplus
}
#endif

#endif /* BD_ORACLE_H_ */
