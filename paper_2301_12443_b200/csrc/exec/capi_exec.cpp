// C-ABI of the per-GPU partition executor (include/pbdx.h): model dispatch + exception -> status.
#include <cuda_runtime.h>

#include <cstring>
#include <new>

#include "partition_base.hpp"
#include "pbdk.h"
#include "pbdx.h"

// ------------------------------------------------------------------ C ABI
namespace {

using pbd::exec::PartitionBase;

template <class F>
int guard(F&& f) {
  try {
    f();
    return PBDK_OK;
  } catch (const pbd::exec::BadArg&) {
    return PBDK_EINVAL;
  } catch (const std::bad_alloc&) {
    return PBDK_ECUDA;
  } catch (const std::exception&) {
    return PBDK_ECUDA;
  }
}

PartitionBase* P(void* h) { return static_cast<PartitionBase*>(h); }
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int pbdx_create(const pbdx_desc* d, void** handle) {
  if (d == nullptr || handle == nullptr) return PBDK_EINVAL;
  return guard([&] {
    switch (d->model) {
      case PBDX_MODEL_RESNET_CIFAR: *handle = pbd::exec::make_resnet_partition(*d); break;
      case PBDX_MODEL_RESNET_CIFAR_FP32: *handle = pbd::exec::make_resnet_f32_partition(*d); break;
      case PBDX_MODEL_MBV2_PROXYLESS:
      case PBDX_MODEL_EFFB0_PROXYLESS: *handle = pbd::exec::make_mb_partition(*d); break;
      default: throw pbd::exec::BadArg("unknown model");
    }
  });
}

void pbdx_destroy(void* handle) { delete P(handle); }

size_t pbdx_relay_row_bytes(void* h) { return h == nullptr ? 0 : P(h)->relay_row_bytes(); }

int pbdx_init_params(void* h, void* st) { return guard([&] { P(h)->init_params(S(st)); }); }
int pbdx_set_shard(void* h, int n, int first) { return guard([&] { P(h)->set_shard(n, first); }); }
int pbdx_set_input_mode(void* h, int external) { return guard([&] { P(h)->set_external_input(external); }); }
int pbdx_stage_images(void* h, const float* host, int n, int slot, void* st) {
  return guard([&] { P(h)->stage_images(host, n, slot, S(st)); });
}
int pbdx_upload_images(void* h, const float* host, int n, void* st) {
  return guard([&] { P(h)->upload_images(host, n, S(st)); });
}
int pbdx_teacher_forward(void* h, void* st) { return guard([&] { P(h)->teacher_forward(S(st)); }); }
int pbdx_student_step(void* h, void* st) { return guard([&] { P(h)->student_step(S(st)); }); }
int pbdx_apply_update(void* h, void* st) { return guard([&] { P(h)->apply_update(S(st)); }); }
int pbdx_step(void* h, void* st) { return guard([&] { P(h)->step(S(st)); }); }
int pbdx_capture(void* h, void* st) { return guard([&] { P(h)->capture(S(st)); }); }
int pbdx_replay(void* h, void* st) { return guard([&] { P(h)->replay(S(st)); }); }
int pbdx_capture_phases(void* h, int fuse_ts, void* st) {
  return guard([&] { P(h)->capture_phases(S(st), fuse_ts != 0); });
}
int pbdx_replay_phase(void* h, int phase, void* st) { return guard([&] { P(h)->replay_phase(phase, S(st)); }); }
int pbdx_buffer(void* h, int which, void** ptr, size_t* bytes) {
  return guard([&] { P(h)->buffer(which, ptr, bytes); });
}
int pbdx_num_blocks(void* h) { return P(h)->nblocks(); }
int pbdx_teacher_act(void* h, int block, void** ptr, size_t* bytes) {
  return guard([&] { P(h)->teacher_act(block, ptr, bytes); });
}
int pbdx_refresh_shadows(void* h, void* st) { return guard([&] { P(h)->refresh_shadows(S(st)); }); }
int pbdx_set_timing(void* h, int enabled) { return guard([&] { P(h)->set_timing(enabled != 0); }); }
int pbdx_block_times(void* h, float* t, float* s) { return guard([&] { P(h)->block_times(t, s); }); }
int pbdx_dp_set_group(void* h, int size, int me, void* const* peer_grads, void* const* peer_mailbox) {
  if (size > 1 && (peer_grads == nullptr || peer_mailbox == nullptr)) return PBDK_EINVAL;
  return guard([&] { P(h)->dp_set_group(size, me, peer_grads, peer_mailbox); });
}
int pbdx_dp_set_params(void* h, int size, void* const* peer_params) {
  if (size > 1 && peer_params == nullptr) return PBDK_EINVAL;
  return guard([&] { P(h)->dp_set_params(size, peer_params); });
}
int pbdx_dp_sync_state(void* h, void* st) { return guard([&] { P(h)->dp_sync_state(S(st)); }); }
long long pbdx_dp_peer_bytes(long long n, int size, int me) {
  if (n < 0 || n % 4 != 0 || size < 1 || me < 0 || me >= size) return -1;
  long long bytes = 0;
  for (int j = 0; j < size; ++j) {  // reduce-scatter: my slice from each peer; all-gather: each peer's slice
    size_t lo = 0, hi = 0;
    pbdk::dp_slice(static_cast<size_t>(n), size, j, &lo, &hi);
    const long long mine_lo = static_cast<long long>(lo), mine_hi = static_cast<long long>(hi);
    if (j == me) {
      bytes += (size - 1) * (mine_hi - mine_lo) * 4;
    } else {
      bytes += (mine_hi - mine_lo) * 4;
    }
  }
  return bytes;
}
int pbdx_set_train_mask(void* h, unsigned int mask) { return guard([&] { P(h)->set_train_mask(mask); }); }
int pbdx_trace_mark(void* h, void* st) { return guard([&] { P(h)->trace_mark(S(st)); }); }
int pbdx_block_trace(void* h, float* t0, float* t1, float* s0, float* s1) {
  return guard([&] { P(h)->block_trace(t0, t1, s0, s1); });
}
int pbdx_launches_per_step(void* h) { return P(h)->launches_per_step(); }
int pbdx_relay_set_recv(void* h, int nsenders, void* const* remote_consumed_flags) {
  if (nsenders > 0 && remote_consumed_flags == nullptr) return PBDK_EINVAL;
  return guard([&] { P(h)->relay_set_recv(nsenders, remote_consumed_flags); });
}
int pbdx_relay_set_send(void* h, int nmsgs, const pbdx_relay_msg* msgs) {
  if (nmsgs > 0 && msgs == nullptr) return PBDK_EINVAL;
  return guard([&] { P(h)->relay_set_send(nmsgs, msgs); });
}
int pbdx_ipc_export(void* dev_ptr, void* handle) {
  if (dev_ptr == nullptr || handle == nullptr) return PBDK_EINVAL;
  cudaIpcMemHandle_t hd;
  if (cudaIpcGetMemHandle(&hd, dev_ptr) != cudaSuccess) return PBDK_ECUDA;
  std::memcpy(handle, &hd, sizeof(hd));
  return PBDK_OK;
}
int pbdx_ipc_open(const void* handle, void** dev_ptr) {
  if (dev_ptr == nullptr || handle == nullptr) return PBDK_EINVAL;
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, sizeof(hd));
  return cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? PBDK_OK : PBDK_ECUDA;
}
int pbdx_ipc_close(void* dev_ptr) { return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? PBDK_OK : PBDK_ECUDA; }

int pbdx_set_path(void* h, int block, const int* path, int n) {
  if (path == nullptr || n < 1) return PBDK_EINVAL;
  return guard([&] { P(h)->set_path(block, path, n); });
}

}  // extern "C"
