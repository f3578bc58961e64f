/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement (oracle) of the blockwise-distillation step for the
 * ImageNet-shaped workload of BASELINE.json configs[2]: a MobileNetV2-style
 * teacher (BN folded, frozen) split into 6 blocks at stage boundaries, distilled block by block into
 * a ProxylessNAS-style single-path supernet student (every searchable MBConv layer holds the
 * candidates {k3, k5, k7} x {e3, e6}; one candidate per layer is active per step).  Only tests/,
 * __graft_entry__.smoke() and bench.py's baseline legs may load it.
 *
 * There is no executable reference for this path (SPEC.md:15 excludes training):
 * it restates Algorithm 1 with the block pairs of PAPER.md:192-194, the
 * ProxylessNAS supernet + MobileNetV2 teacher of PAPER.md:409-414 (Table 2 row, :533-534), SGD as PAPER.md:428-429.  The
 * tensor shapes are ours (the reference defines none): MobileNetV2-1.0 / EfficientNet-B0
 * with their true channel widths, stored rounded up to the tensor-tile granularity with the extra
 * channels identically zero (zero weights, zero gradients).  Numerics contract =
 * the GPU path and this oracle round to bf16 at the same points; depthwise and stem
 * convolutions accumulate in the same fmaf order on both sides, 1x1 convolutions (tensor cores)
 * differ only in fp32 accumulation order.  Deterministic for any OpenMP thread count.
 */
#ifndef MB_ORACLE_H_
#define MB_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MBO_BLOCKS 6
#define MBO_CANDIDATES 6 /* candidate c: kernel {3,5,7}[c % 3], expansion {3,6}[c / 3] */

/* teacher family (process-wide, test infrastructure): 0 = MobileNetV2 (ReLU6; configs[2]),
 * 1 = EfficientNet-B0 (swish, squeeze-excite, k5 stages; configs[3]).  The student supernet is the
 * same ProxylessNAS space over the family's block / layer structure. */
void mbo_set_family(int family);
int mbo_family(void);

/* geometry (image side S, e.g. 224): boundary b in 0..6 (0 = the image, stored as 16 channels) */
int mbo_channels(int boundary);                 /* stored: 3, 32, 32, 64, 128, 192, 320 */
int mbo_true_channels(int boundary);            /* the architecture's: 3, 24, 32, 64, 96, 160, 320 (MBv2) */
int mbo_hw(int boundary, int S);                /* S, S/4, S/8, S/16, S/16, S/32, S/32 */
int mbo_student_layers(int block);              /* incl. block 0's stem and fixed MBConv1 */
int mbo_layer_candidates(int block, int layer); /* 1 (fixed) or MBO_CANDIDATES */
size_t mbo_teacher_param_count(int block);
size_t mbo_student_param_count(int block); /* the whole supernet of the block */
/* element offset and count of candidate c of layer l inside the block's flat student params */
size_t mbo_candidate_offset(int block, int layer, int cand, size_t* count);

/* synthetic image, NHWC [n, S, S, 3] in [-1, 1) (same Philox stream as the CIFAR workload) */
void mbo_input(int n, int64_t first, int S, uint32_t seed, float* out, int bf16);
void mbo_teacher_init(int block, uint32_t seed, float* params, int bf16);
void mbo_student_init(int block, uint32_t seed, float* params);
/* seeded single-path sampler: path[l] for the block's layers at sampling index `draw` */
void mbo_sample_path(int block, uint32_t seed, int64_t draw, int* path);

/* in: NHWC at boundary `block` ([n,S,S,3] for block 0), out: NHWC at boundary block+1 */
int mbo_teacher_fwd(int block, const float* tparams, int n, int S, const float* in, float* out, int bf16);
/* student fwd + bwd of the active path on an n-sample shard; grads in the params layout (inactive
 * candidates stay 0), loss = sum_shard (s - t)^2 / norm */
int mbo_student_fwd_bwd(int block, const float* sparams, const int* path, int n, int S, const float* in,
                        const float* t_out, double norm, int bf16, float* grads, double* loss);
/* SGD-momentum over the active path only (inactive candidates: no gradient, untouched — torch
 * semantics for parameters whose .grad is None) */
void mbo_sgd_path(int block, const int* path, float* w, float* v, const float* g, float lr, float mu);

#ifdef __cplusplus
}
#endif

#endif /* MB_ORACLE_H_ */
