/*
 * pbdx.h — C-ABI of the per-GPU partition executor (libpbd.so).
 *
 * One executor = one device's share of a Pipe-BD schedule: the contiguous
 * block range [block_lo, block_hi] of a PartitionSpec (schedule.hpp:28-38)
 * at a shard of `n` samples of each global batch.  It runs the per-device body
 * of Algorithm 1 as three phases so the host driver can
 * put the relay and the gradient allreduce between them:
 *
 *   pbdx_teacher_forward   load_data() (block 0) + T_i.forward          (lines 8,10)
 *                          -> the boundary activation is ready to send   (line 11)
 *   pbdx_student_step      S_i.forward, L(s,t), S_i.backward            (lines 12-13)
 *                          -> gradients ready for share_gradient()       (line 14)
 *   pbdx_apply_update      S_i.update_weight() (fused SGD-momentum)      (line 15)
 *
 * Its simulated counterpart is the step loop of simulate.cpp:193-262; the
 * executor reports the same per-block teacher / student times (CUDA events)
 * that profile.hpp:30-42 BlockProfile holds, so the partitioner can run on
 * device-measured T_k(b), S_k(b).
 *
 * All device memory is owned by the executor (cudaMalloc).  Buffers that the
 * driver moves with NCCL are exposed as raw device pointers (pbdx_buffer).
 * Return codes are pbdk.h's (0 ok, 1 invalid, 2 CUDA error).
 */
#ifndef PBDX_H_
#define PBDX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* workloads */
#define PBDX_MODEL_RESNET_CIFAR 0    /* configs[0..1]: ResNet-18-CIFAR teacher -> slim residual student, 4 blocks */
#define PBDX_MODEL_MBV2_PROXYLESS 1  /* configs[2]: MobileNetV2 teacher -> ProxylessNAS supernet student, 6 blocks */
#define PBDX_MODEL_EFFB0_PROXYLESS 2 /* configs[3]: EfficientNet-B0 teacher (swish, squeeze-excite) -> same space */
#define PBDX_MODEL_RESNET_CIFAR_FP32 3 /* configs[0]: the CIFAR workload in fp32 (3xTF32 tensor-core convolutions;
                                          activations stored split fp32, see pbdk_conv3x_fprop) */

typedef struct pbdx_desc {
  int block_lo, block_hi; /* inclusive block range of the model's chain        */
  int n_max;              /* largest shard this executor will run               */
  int global_batch;       /* b: MSE normalisation + synthetic sample indexing   */
  uint32_t seed_data, seed_teacher, seed_student;
  float lr, momentum;
  int model;              /* PBDX_MODEL_*                                        */
  int image;              /* input side S (CIFAR: 32; MBV2: e.g. 224)           */
} pbdx_desc;

/* buffers for pbdx_buffer */
#define PBDX_BUF_INPUT 0        /* input activation of block_lo (bf16 NHWC; block 0: padded image [n,32,32,16]) */
#define PBDX_BUF_TEACHER_OUT 1  /* teacher output of block_hi (bf16 NHWC) — the relayed activation */
#define PBDX_BUF_GRADS 2        /* fp32 flat student gradients of the partition (allreduce target) */
#define PBDX_BUF_PARAMS 3       /* fp32 flat student master weights */
#define PBDX_BUF_MOMENTUM 4     /* fp32 flat momentum */
#define PBDX_BUF_LOSSES 5       /* double[num_blocks]: per-block partial loss of the last step */
#define PBDX_BUF_STEP 6         /* int64 step counter (advanced by apply_update) */
#define PBDX_BUF_TEACHER_PARAMS 7 /* bf16 teacher conv weights of block_lo..hi (flat, program order) */
#define PBDX_BUF_MAILBOX 8      /* 80 uint64 flags written by peers (own allocation, IPC-exportable):
                                   [0,16) relay ready (per sender slot), [16,32) relay consumed (per
                                   receiver slot), [32,48) DP ready, [48,64) DP consumed, [64,80) DP
                                   slice updated (per member) */

int pbdx_create(const pbdx_desc* d, void** handle);
void pbdx_destroy(void* handle);

/* Deterministic Philox initialisation of teacher and student parameters. */
int pbdx_init_params(void* handle, void* stream);

/* Current shard: n samples starting at offset `first` inside the global batch. */
int pbdx_set_shard(void* handle, int n, int first);

/* 0: block 0 input generated on device by Philox (synthetic data);
 * 1: block 0 input comes from pbdx_upload_images (host data, e2e path);
 * 2: block 0 input staged by pbdx_stage_images into two slots (overlapped host input). */
int pbdx_set_input_mode(void* handle, int external);
/* host fp32 NHWC [n][32][32][3] (pinned for async) -> device padded bf16 input */
int pbdx_upload_images(void* handle, const float* host, int n, void* stream);
/* input mode 2 (double-buffered host input): copy the images of a step into staging slot 0/1 on any
 * stream (a copy stream, overlapping the previous step); the step itself packs slot (step counter & 1),
 * so one captured graph serves every step.  CIFAR model. */
int pbdx_stage_images(void* handle, const float* host, int n, int slot, void* stream);

int pbdx_teacher_forward(void* handle, void* stream);
int pbdx_student_step(void* handle, void* stream);
int pbdx_apply_update(void* handle, void* stream);
/* teacher_forward + student_step + apply_update */
int pbdx_step(void* handle, void* stream);

/* Capture teacher_forward + student_step + apply_update as one CUDA graph (single-GPU path) and replay it. */
int pbdx_capture(void* handle, void* stream);
int pbdx_replay(void* handle, void* stream);
/* Capture the three phases as separate graphs (0 teacher_forward, 1 student_step, 2 apply_update)
 * so a multi-GPU driver can put the NCCL relay / allreduce between replays.  fuse_ts != 0: phase 0
 * holds teacher_forward + student_step (overlapped per block) and phase 1 is empty — for ranks
 * that relay nothing downstream. */
int pbdx_capture_phases(void* handle, int fuse_ts, void* stream);
int pbdx_replay_phase(void* handle, int phase, void* stream);

int pbdx_buffer(void* handle, int which, void** ptr, size_t* bytes);
int pbdx_num_blocks(void* handle);
/* teacher output t_k (bf16 NHWC [n_max][H][W][C]) of block k inside the partition */
int pbdx_teacher_act(void* handle, int block, void** ptr, size_t* bytes);

/* Re-derive the bf16 GEMM shadows (and flipped dgrad weights) from the fp32 master weights after
 * the driver overwrote PBDX_BUF_PARAMS / PBDX_BUF_MOMENTUM (state migration on reconfiguration).
 * Requires PBDX_BUF_GRADS to be zero (momentum is kept unchanged). */
int pbdx_refresh_shadows(void* handle, void* stream);

/* Per-block CUDA-event timing of the last step (ms): teacher[k], student[k] for k in the range. */
int pbdx_set_timing(void* handle, int enabled);
int pbdx_block_times(void* handle, float* teacher_ms, float* student_ms);
/* Student blocks that train (bit i = block block_lo + i; default all).  The paper's DP baseline
 * trains blocks one after another, each step recomputing the teacher prefix:
 * partition [0, k] with mask 1 << k.  Untrained blocks run only their teacher part. */
int pbdx_set_train_mask(void* handle, unsigned int mask);

/* Measured timelines (the reference's SimReport, simulate.hpp:27-86, built from real runs): record a
 * reference event on `stream`, then after a timed step read every block's teacher / student
 * [start, end] relative to it (ms, per block in the range). */
int pbdx_trace_mark(void* handle, void* stream);
int pbdx_block_trace(void* handle, float* teacher_start, float* teacher_end, float* student_start,
                     float* student_end);

/* Supernet layout of the MBConv models (host-only queries, no device needed): student layers of a
 * block, candidates of a layer, a candidate's (offset, count) inside the block's flat parameters,
 * and the block's parameter count.  -1 on bad arguments. */
int pbdx_mb_layers(int model, int block);
int pbdx_mb_candidates(int model, int block, int layer);
long pbdx_mb_candidate_offset(int model, int block, int layer, int cand, long* count);
long pbdx_mb_block_params(int model, int block);

/* Search space (PBDX_MODEL_MBV2_PROXYLESS / _EFFB0_PROXYLESS): active candidate of every student layer of `block`
 * (path[l] in [0, candidates); fixed layers 0).  Only the active path runs forward/backward and is
 * updated (inactive candidates keep weights and momentum: torch semantics for params without
 * .grad).  Invalidates captured graphs.  Layout of the supernet parameters: DESIGN.md §10. */
int pbdx_set_path(void* handle, int block, const int* path, int n);

/* Flat student-parameter layout of one block (element offsets, padded storage):
 * out[9] = {w1, w2, wsc, g1, b1, g2, b2, gsc, bsc}; returns the block's element count
 * (negative on error).  Block 0 stores its 3 input channels padded to 16. */
long pbdx_student_layout(int block, long* offsets);
/* The same for PBDX_MODEL_RESNET_CIFAR_FP32 (block 0 stores its 3 input channels padded to 32). */
long pbdx_student_layout_fp32(int block, long* offsets);

/* ------------------------------------------------------------------ K11 peer relay (TR)
 * The reference models the hand-over of t_hi as ready = teacher_end + max(C(b_up), C(b_down))
 * (simulate.cpp:203-214).  Here the SENDER's SMs store its rows directly into the receiver's
 * PBDX_BUF_INPUT through peer memory (NVLink; a CUDA IPC mapping across processes) on a side
 * stream right after T.forward, then publish a sequence number into the receiver's mailbox.
 * The receiver's teacher_forward first waits for every sender's flag; its student_step ends by
 * publishing "consumed" into each sender's mailbox, which gates the next overwrite (one slot).
 * All of it is device-side, so a rank's whole step (and its CUDA graph) needs no host handshake.
 *
 * Receiver: remote_consumed_flags[i] = &mailbox_of_sender_i[16 + (my slot in sender i's list)];
 *           sender i writes my mailbox[i].
 * Sender:   msgs[j] = rows [src_row, src_row+rows) of my PBDX_BUF_TEACHER_OUT -> dst (peer pointer into
 *           receiver j's input, already offset), remote_flag = &mailbox_of_receiver_j[my slot there];
 *           receiver j writes my mailbox[16 + j]. */
typedef struct pbdx_relay_msg {
  long long src_row, rows;
  void* dst;
  void* remote_flag;
} pbdx_relay_msg;
int pbdx_relay_set_recv(void* handle, int nsenders, void* const* remote_consumed_flags);
/* bytes per sample of the relayed activation (teacher output of block_hi) */
size_t pbdx_relay_row_bytes(void* handle);
int pbdx_relay_set_send(void* handle, int nmsgs, const pbdx_relay_msg* msgs);
/* DP group over peer memory (share_gradient; AHD partitions with |G| > 1): instead of an
 * NCCL allreduce, every member announces its gradients after S_i.backward (device-side flag into each
 * peer's mailbox), waits for all members, and the update kernel reads the group's gradient slabs straight
 * from the peers' PBDX_BUF_GRADS (NVLink loads), adds them in member order and applies SGD-momentum —
 * bit-identical weights on every member, no host round trip, and the whole step stays one CUDA graph.
 * peer_grads[j] / peer_mailbox[j]: member j's buffers as seen from this process (j == me ignored). */
int pbdx_dp_set_group(void* handle, int size, int me, void* const* peer_grads, void* const* peer_mailbox);
/* The exchange itself is a reduce-scatter + all-gather over peer memory: member `me` sums and updates
 * slice `me` of every parameter region (its peers' gradient slices, member order), publishes a
 * device-side "updated" flag (mailbox slots [64, 80)), then copies every other member's updated slice
 * of the master weights — 2(G-1)/G * 4P bytes of NVLink reads per member, the ring-allreduce volume of
 * cost_model.cpp:79-86.  peer_params[j]: member j's PBDX_BUF_PARAMS (the allocation also holds its
 * momentum).  Required when size > 1. */
int pbdx_dp_set_params(void* handle, int size, void* const* peer_params);
/* Momentum is sharded by the exchange (only a slice's owner keeps it current): pull every other
 * member's slices of weights and momentum before the host reads block state (checkpoint, migration). */
int pbdx_dp_sync_state(void* handle, void* stream);
/* Host-only: peer bytes read per member and step by the exchange for an n-float region (n % 4 == 0). */
long long pbdx_dp_peer_bytes(long long n, int size, int me);

/* CUDA IPC of an executor buffer (the allocation base: PBDX_BUF_INPUT / PBDX_BUF_MAILBOX) for ranks in
 * other processes; handle = 64 bytes (cudaIpcMemHandle_t). */
int pbdx_ipc_export(void* dev_ptr, void* handle);
int pbdx_ipc_open(const void* handle, void** dev_ptr);
int pbdx_ipc_close(void* dev_ptr);

/* Kernel launches issued per step by this executor (for the bench's gpu_launches claim). */
int pbdx_launches_per_step(void* handle);

#ifdef __cplusplus
}
#endif

#endif /* PBDX_H_ */
