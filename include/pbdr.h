/*
 * pbdr.h — C-ABI of the single-process multi-GPU driver (libpbd.so).
 *
 * Runs a whole Pipe-BD schedule (the AHD partitioner's document, schedule.hpp:28-74 /
 * pbd_capi.h) inside ONE host process: one pbdx executor per schedule device (include/pbdx.h), the
 * K11 peer relay between consecutive partitions and the DP gradient exchange inside every partition
 * with |G| > 1 wired over CUDA peer memory (cudaDeviceEnablePeerAccess; NVLink on B200 nodes).
 * Because both exchanges are device-side (sequence flags in the executors' mailboxes), a step is
 * one CUDA graph per device enqueued back to back from the calling thread — the C++ counterpart of
 * the per-device loop the reference simulates (simulate.cpp:193-264) and of the torch.distributed
 * driver paper_2301_12443_b200/runtime.py (one process per GPU).  Return codes are pbdk.h's.
 */
#ifndef PBDR_H_
#define PBDR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pbdr_desc {
  int global_batch;                     /* b */
  int model;                            /* PBDX_MODEL_* */
  int image;                            /* input side (0: the model's default) */
  uint32_t seed_data, seed_teacher, seed_student;
  float lr, momentum;
  int graphs;                           /* 1: each device's step is replayed as one CUDA graph */
} pbdr_desc;

/* schedule_json: the schedule document (save_schedule format; devices are ranks 0..R-1).
 * device_of_rank[r]: the CUDA device that runs schedule device r (several ranks may share one GPU). */
int pbdr_create(const char* schedule_json, const pbdr_desc* d, const int* device_of_rank, int nranks,
                void** handle);
void pbdr_destroy(void* handle);
int pbdr_step(void* handle);                 /* enqueue one step of Algorithm 1 on every rank */
int pbdr_sync(void* handle);                 /* wait for every rank */
int pbdr_num_blocks(void* handle);
/* per-block loss of the last step (summed over the block's DP group); synchronizes */
int pbdr_block_losses(void* handle, double* out);
/* the executor of rank r (pbdx.h handle, for buffers / block state) and its CUDA device */
int pbdr_rank(void* handle, int rank, void** pbdx_handle, int* device);

/* CUDA devices visible to the library (0 without a GPU) */
int pbdr_device_count(void);

/* Host-only wiring (CPU-testable): the relay messages across partition boundary `boundary`
 * (partition boundary-1 -> boundary) as (sender rank, receiver rank, sender row, receiver row, rows)
 * quintuples — the overlapping row ranges of the two groups' DP shards.
 * Returns the message count (> max_msgs: only the first max_msgs written), < 0 on error. */
int pbdr_relay_plan(const char* schedule_json, int global_batch, int boundary, long long* out, int max_msgs);

#ifdef __cplusplus
}
#endif

#endif /* PBDR_H_ */
