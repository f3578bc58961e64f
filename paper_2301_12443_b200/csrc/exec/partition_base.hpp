// Model-independent half of the per-GPU partition executor (include/pbdx.h): the phases of
// Algorithm 1 around the model's own teacher / student / update bodies,
// the K11 peer relay hooks (relay.cu), CUDA-graph capture of a whole step or of its phases,
// and the device arena.  Models: ResNetPartition (CIFAR ResNet-18 -> slim residual student,
// partition.cpp) and MbPartition (MobileNetV2 -> ProxylessNAS supernet, mb_partition.cpp).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "knobs.hpp"
#include "bd_kernels.hpp"
#include "pbdk.h"
#include "pbdx.h"
#include "relay.hpp"

namespace pbd::exec {

struct CudaFail : std::runtime_error {
  explicit CudaFail(const std::string& m) : std::runtime_error(m) {}
};
struct BadArg : std::runtime_error {
  explicit BadArg(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int rc, const char* what) {
  if (rc == PBDK_EINVAL) throw BadArg(what);
  if (rc != PBDK_OK) throw CudaFail(std::string(what) + ": " + cudaGetErrorString(cudaGetLastError()));
}
inline void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail(std::string(what) + ": " + cudaGetErrorString(e));
}

class Arena {
 public:
  ~Arena() {
    for (void* p : ptrs_) cudaFree(p);
  }
  template <class T = void>
  T* get(size_t bytes) {
    void* p = nullptr;
    bytes = (bytes + 255) / 256 * 256;
    if (bytes == 0) bytes = 256;
    cuda(cudaMalloc(&p, bytes), "cudaMalloc");
    cuda(cudaMemset(p, 0, bytes), "cudaMemset");
    ptrs_.push_back(p);
    bytes_ += bytes;
    return static_cast<T*>(p);
  }
  size_t bytes() const { return bytes_; }

 private:
  std::vector<void*> ptrs_;
  size_t bytes_ = 0;
};

class PartitionBase {
 public:
  explicit PartitionBase(const pbdx_desc& d) : d_(d), n_(d.n_max) {
    if (d.n_max < 1 || d.global_batch < 1) throw BadArg("bad batch");
  }
  virtual ~PartitionBase() {
    if (graph_exec_ != nullptr) cudaGraphExecDestroy(graph_exec_);
    for (auto g : phase_exec_)
      if (g != nullptr) cudaGraphExecDestroy(g);
    if (cap_stream_ != nullptr) cudaStreamDestroy(cap_stream_);
    if (relay_stream_ != nullptr) cudaStreamDestroy(relay_stream_);
    if (relay_fork_ != nullptr) cudaEventDestroy(relay_fork_);
    if (relay_done_ != nullptr) cudaEventDestroy(relay_done_);
    for (auto e : ev_t_) cudaEventDestroy(e);
    for (auto e : ev_s_) cudaEventDestroy(e);
    if (trace_ref_ != nullptr) cudaEventDestroy(trace_ref_);
  }

  // ---- model hooks
  virtual int nblocks() const = 0;
  virtual void init_params(cudaStream_t st) = 0;
  virtual void rebuild_for_shard() = 0;  // n_ changed
  virtual void upload_images(const float* host, int n, cudaStream_t st) = 0;
  // input mode 2: host images copied into staging slot 0/1 (any stream); the step packs slot (step & 1)
  virtual void stage_images(const float*, int, int, cudaStream_t) { throw BadArg("model has no staged input"); }
  virtual void teacher_body(cudaStream_t st) = 0;
  // student blocks; fork: start from the caller's stream (standalone phase) instead of the
  // per-block teacher events.  Must join every side stream back into `caller`.
  virtual void student_body(cudaStream_t caller, bool fork) = 0;
  virtual void update_body(cudaStream_t st) = 0;
  virtual void refresh_shadows(cudaStream_t st) = 0;
  virtual void buffer(int which, void** ptr, size_t* bytes) = 0;
  virtual void teacher_act(int k, void** ptr, size_t* bytes) = 0;
  // Per-block CUDA-event timing (teacher block on the caller's stream, student block on its own).
  void set_timing(bool on) {
    timing_ = on;
    if (on && ev_t_.empty()) {
      ev_t_.resize(2 * static_cast<size_t>(nblocks()));
      ev_s_.resize(2 * static_cast<size_t>(nblocks()));
      for (auto& e : ev_t_) cuda(cudaEventCreate(&e), "event create");
      for (auto& e : ev_s_) cuda(cudaEventCreate(&e), "event create");
    }
  }
  void block_times(float* tms, float* sms) {
    if (ev_t_.empty()) throw BadArg("timing not enabled");
    for (int i = 0; i < nblocks(); ++i) {
      cuda(cudaEventSynchronize(ev_t_[2 * i + 1]), "event sync");
      cuda(cudaEventElapsedTime(&tms[i], ev_t_[2 * i], ev_t_[2 * i + 1]), "elapsed");
      cuda(cudaEventSynchronize(ev_s_[2 * i + 1]), "event sync");
      cuda(cudaEventElapsedTime(&sms[i], ev_s_[2 * i], ev_s_[2 * i + 1]), "elapsed");
    }
  }
  // Measured timelines (SimReport of real runs, §8f): a reference event on the caller's stream, and
  // every block's [start, end] of the last step relative to it (ms).
  void trace_mark(cudaStream_t st) {
    if (trace_ref_ == nullptr) cuda(cudaEventCreate(&trace_ref_), "event create");
    cuda(cudaEventRecord(trace_ref_, st), "event");
  }
  void block_trace(float* t0, float* t1, float* s0, float* s1) {
    if (ev_t_.empty() || trace_ref_ == nullptr) throw BadArg("timing / trace mark not enabled");
    for (int i = 0; i < nblocks(); ++i) {
      cuda(cudaEventSynchronize(ev_s_[2 * i + 1]), "event sync");
      cuda(cudaEventSynchronize(ev_t_[2 * i + 1]), "event sync");
      cuda(cudaEventElapsedTime(&t0[i], trace_ref_, ev_t_[2 * i]), "elapsed");
      cuda(cudaEventElapsedTime(&t1[i], trace_ref_, ev_t_[2 * i + 1]), "elapsed");
      cuda(cudaEventElapsedTime(&s0[i], trace_ref_, ev_s_[2 * i]), "elapsed");
      cuda(cudaEventElapsedTime(&s1[i], trace_ref_, ev_s_[2 * i + 1]), "elapsed");
    }
  }
  virtual int body_launches_per_step() const = 0;
  virtual void set_path(int /*block*/, const int* /*path*/, int /*n*/) { throw BadArg("model has no search space"); }
  // relayed activation (teacher output of block_hi) and its bytes per sample
  virtual const void* relay_source() const = 0;
  virtual size_t relay_row_bytes() const = 0;

  // ---- Algorithm 1 phases
  void set_shard(int n, int first) {
    if (n < 1 || n > d_.n_max || first < 0 || first + n > d_.global_batch) throw BadArg("bad shard");
    first_ = first;
    if (n != n_) {
      n_ = n;
      rebuild_for_shard();
      invalidate_graphs();
    }
  }

  void set_external_input(int mode) {
    if (mode < 0 || mode > 2) throw BadArg("input mode 0/1/2");
    external_ = mode;
    invalidate_graphs();
  }

  void teacher_forward(cudaStream_t st) {
    dp_wait_consumed(st);  // the previous step's DP peers finished reading my gradients
    relay_wait_input(st);
    teacher_body(st);
    relay_send_output(st);
  }
  void student_step(cudaStream_t caller) { student_step_impl(caller, true); }
  void student_step_impl(cudaStream_t caller, bool fork) {
    student_body(caller, fork);
    relay_finish(caller);
    dp_exchange(caller);  // share_gradient: announce mine, wait for every member's
  }
  void apply_update(cudaStream_t st) {
    update_body(st);
    dp_release(st);
  }
  void step(cudaStream_t st) {
    teacher_forward(st);
    student_step_impl(st, false);
    apply_update(st);
  }

  int launches_per_step() const {
    int n = body_launches_per_step();
    if (!recv_consumed_.empty()) n += 2;  // relay wait + release
    if (!send_.empty()) n += 2;           // relay wait + copy
    if (dp_active()) n += 6;              // dp wait consumed, ready, wait ready, updated, wait updated, consumed
    return n;
  }

  // ---- CUDA graphs
  // Three graphs (teacher_forward / student_step / apply_update) for the multi-GPU driver, which
  // interleaves NCCL collectives between them.  fuse_ts: phase 0 = teacher_forward + student_step
  // with the per-block teacher->student overlap of step(), phase 1 empty.
  void capture_phases(cudaStream_t caller, bool fuse_ts) {
    ensure_cap_stream();
    cuda(cudaStreamSynchronize(caller), "sync");
    const bool was_timing = timing_;
    timing_ = false;
    for (int ph = 0; ph < 3; ++ph) {
      if (phase_exec_[ph] != nullptr) {
        cudaGraphExecDestroy(phase_exec_[ph]);
        phase_exec_[ph] = nullptr;
      }
      cudaGraph_t g = nullptr;
      cuda(cudaStreamBeginCapture(cap_stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        if (ph == 0) {
          teacher_forward(cap_stream_);
          if (fuse_ts) student_step_impl(cap_stream_, false);
        }
        if (ph == 1 && !fuse_ts) student_step_impl(cap_stream_, true);
        if (ph == 2) apply_update(cap_stream_);
      } catch (...) {
        cudaStreamEndCapture(cap_stream_, &g);
        if (g) cudaGraphDestroy(g);
        timing_ = was_timing;
        throw;
      }
      cuda(cudaStreamEndCapture(cap_stream_, &g), "end capture");
      size_t nodes = 0;
      cuda(cudaGraphGetNodes(g, nullptr, &nodes), "graph nodes");
      if (nodes > 0) cuda(cudaGraphInstantiate(&phase_exec_[ph], g, graph_flags()), "instantiate");
      cudaGraphDestroy(g);
    }
    timing_ = was_timing;
    phases_valid_ = true;
  }

  void replay_phase(int ph, cudaStream_t st) {
    if (ph < 0 || ph > 2 || !phases_valid_) throw BadArg("no captured phase graph");
    if (phase_exec_[ph] != nullptr) cuda(cudaGraphLaunch(phase_exec_[ph], st), "graph launch");
  }

  // Captures on a private non-blocking stream (the legacy default stream cannot be captured);
  // the instantiated graph is replayed on the caller's stream.
  void capture(cudaStream_t caller) {
    if (graph_exec_ != nullptr) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
    ensure_cap_stream();
    cuda(cudaStreamSynchronize(caller), "sync");
    cudaGraph_t g = nullptr;
    cuda(cudaStreamBeginCapture(cap_stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
    const bool was_timing = timing_;
    timing_ = false;
    try {
      step(cap_stream_);
    } catch (...) {
      cudaStreamEndCapture(cap_stream_, &g);
      if (g) cudaGraphDestroy(g);
      timing_ = was_timing;
      throw;
    }
    timing_ = was_timing;
    cuda(cudaStreamEndCapture(cap_stream_, &g), "end capture");
    cuda(cudaGraphInstantiate(&graph_exec_, g, graph_flags()), "instantiate");
    cudaGraphDestroy(g);
    graph_valid_ = true;
  }

  void replay(cudaStream_t st) {
    if (!graph_valid_ || graph_exec_ == nullptr) throw BadArg("no captured graph for the current shard");
    cuda(cudaGraphLaunch(graph_exec_, st), "graph launch");
  }

  // ---- K11 peer relay (relay.cu): the receiver's input buffer is written by its senders
  void relay_set_recv(int n, void* const* remote_consumed) {
    if (n < 0 || n > pbdk::kRelayMaxPeers) throw BadArg("relay: too many senders");
    if (n > 0 && d_.block_lo == 0) throw BadArg("relay: partition 0 loads data, it receives nothing");
    recv_consumed_.assign(remote_consumed, remote_consumed + n);
    invalidate_graphs();
  }

  void relay_set_send(int n, const pbdx_relay_msg* msgs) {
    if (n < 0 || n > pbdk::kRelayMaxPeers) throw BadArg("relay: too many receivers");
    const size_t row = relay_row_bytes();
    send_.clear();
    for (int i = 0; i < n; ++i) {
      const pbdx_relay_msg& m = msgs[i];
      if (m.src_row < 0 || m.rows < 0 || m.src_row + m.rows > n_ || m.dst == nullptr || m.remote_flag == nullptr)
        throw BadArg("relay: bad message");
      if ((row * m.rows) % 16 != 0 || reinterpret_cast<uintptr_t>(m.dst) % 16 != 0) throw BadArg("relay: alignment");
      send_.push_back(m);
    }
    if (!send_.empty() && relay_stream_ == nullptr) {
      cuda(cudaStreamCreateWithFlags(&relay_stream_, cudaStreamNonBlocking), "stream");
      cuda(cudaEventCreateWithFlags(&relay_fork_, cudaEventDisableTiming), "event");
      cuda(cudaEventCreateWithFlags(&relay_done_, cudaEventDisableTiming), "event");
    }
    invalidate_graphs();
  }

  const pbdx_desc& desc() const { return d_; }

  // ---- DP group over peer memory (share_gradient fused into the update, bd_kernels.cu sgd_sum_kernel)
  // peer_grads[j] / peer_mailbox[j]: member j's PBDX_BUF_GRADS and PBDX_BUF_MAILBOX (device pointers
  // valid here; j == me is ignored).  Slots: member j writes my mailbox[32 + j] (ready) and
  // mailbox[48 + j] (consumed).
  void dp_set_group(int size, int me, void* const* peer_grads, void* const* peer_mailbox) {
    if (size < 1 || size > pbdk::kDpMaxGroup || me < 0 || me >= size) throw BadArg("dp group: bad size / index");
    dp_size_ = size;
    dp_me_ = me;
    dp_grads_.assign(static_cast<size_t>(size), nullptr);
    dp_mail_.assign(static_cast<size_t>(size), nullptr);
    for (int j = 0; j < size; ++j) {
      if (j == me) continue;
      if (peer_grads[j] == nullptr || peer_mailbox[j] == nullptr) throw BadArg("dp group: null peer pointer");
      dp_grads_[static_cast<size_t>(j)] = static_cast<const float*>(peer_grads[j]);
      dp_mail_[static_cast<size_t>(j)] = static_cast<unsigned long long*>(peer_mailbox[j]);
    }
    invalidate_graphs();
  }
  bool dp_active() const { return dp_size_ > 1; }

  // members' master-weight buffers (PBDX_BUF_PARAMS) as seen from this process, member order
  void dp_set_params(int size, void* const* peer_params) {
    if (size != dp_size_) throw BadArg("dp params: size differs from the group");
    dp_params_.assign(static_cast<size_t>(size), nullptr);
    for (int j = 0; j < size; ++j) {
      if (j == dp_me_) continue;
      if (peer_params[j] == nullptr) throw BadArg("dp params: null peer pointer");
      dp_params_[static_cast<size_t>(j)] = static_cast<const float*>(peer_params[j]);
    }
    invalidate_graphs();
  }

  // Complete the sharded momentum (and weights) of every parameter region from the slice owners'
  // peer memory: before a checkpoint / migration reads block_state (only the owner's slice is current).
  void dp_sync_state(cudaStream_t st) {
    if (!dp_active()) return;
    float *w = nullptr, *v = nullptr;
    size_t bytes = 0;
    buffer(PBDX_BUF_PARAMS, reinterpret_cast<void**>(&w), &bytes);
    buffer(PBDX_BUF_MOMENTUM, reinterpret_cast<void**>(&v), &bytes);
    require_dp_params();
    // momentum lives in the params allocation at +total (every model allocates them together), so a
    // peer's momentum is its params pointer + the same offset
    const ptrdiff_t dv = v - w;
    if (dv != static_cast<ptrdiff_t>(bytes / sizeof(float))) throw BadArg("dp sync: momentum not adjacent to params");
    for (const DpRegion& r : dp_all_regions()) {
      std::vector<const float*> pw(static_cast<size_t>(dp_size_)), pv(static_cast<size_t>(dp_size_));
      for (int j = 0; j < dp_size_; ++j) {
        const float* base = j == dp_me_ ? w : dp_params_[static_cast<size_t>(j)];
        pw[static_cast<size_t>(j)] = base + r.off;
        pv[static_cast<size_t>(j)] = base + dv + r.off;
      }
      check(pbdk::dp_gather(w + r.off, nullptr, pw.data(), dp_size_, dp_me_, r.n, st), "dp sync w");
      check(pbdk::dp_gather(v + r.off, nullptr, pv.data(), dp_size_, dp_me_, r.n, st), "dp sync v");
    }
  }

  // Which student blocks of the range train (bit i = block block_lo + i).  All by default; the DP
  // baseline of the paper (blocks trained one after another, every step
  // recomputing the teacher prefix) runs partition [0, k] with only block k training.
  void set_train_mask(uint32_t mask) {
    const uint32_t full = nblocks() >= 32 ? 0xFFFFFFFFu : ((1u << nblocks()) - 1u);
    if ((mask & full) == 0) throw BadArg("train mask selects no block");
    train_mask_ = mask & full;
    invalidate_graphs();
  }

 protected:
  void invalidate_graphs() { graph_valid_ = phases_valid_ = false; }

  // Scheduling priorities: the teacher chain (caller / capture stream) is the step's critical path
  // (every student block waits for its teacher block; the last student block starts only after the
  // whole chain), so its kernels get the highest priority, the last student block next, the
  // earlier student blocks (which have the whole remaining chain to hide behind) the lowest.
  // Graphs keep the captured per-node priorities (cudaGraphInstantiateFlagUseNodePriority).
  static int priority_high() {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    return pbd::knob_env("PBD_NO_PRIORITY") != nullptr ? 0 : hi;
  }
  static int priority_low() {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    return pbd::knob_env("PBD_NO_PRIORITY") != nullptr ? 0 : lo;
  }
  static unsigned long long graph_flags() {
    return pbd::knob_env("PBD_NO_PRIORITY") != nullptr
               ? 0ull
               : static_cast<unsigned long long>(cudaGraphInstantiateFlagUseNodePriority);
  }

  void ensure_cap_stream() {
    if (cap_stream_ == nullptr)
      cuda(cudaStreamCreateWithPriority(&cap_stream_, cudaStreamNonBlocking, priority_high()), "stream");
  }

  // relay / DP flag storage (call from the model's allocate())
  void allocate_relay() {
    mailbox_ = arena_.get<unsigned long long>(kMailboxSlots * sizeof(unsigned long long));
    relay_seq_ = arena_.get<unsigned long long>(3 * sizeof(unsigned long long));
    relay_ticket_ = arena_.get<unsigned int>(sizeof(unsigned int));
  }

  // gradient sources of a DP-group update: member order, `mine` at my index, peers' slabs at the same
  // element offset
  std::vector<const float*> dp_sources(const float* mine, size_t offset) const {
    std::vector<const float*> v(static_cast<size_t>(dp_size_));
    for (int j = 0; j < dp_size_; ++j) v[static_cast<size_t>(j)] = (j == dp_me_ ? mine : dp_grads_[static_cast<size_t>(j)]) + offset;
    return v;
  }

  void dp_exchange(cudaStream_t st) {
    if (!dp_active()) return;
    pbdk::RelayReleaseArgs r{};  // ready(seq+1) into every peer's mailbox[32 + me]
    pbdk::RelayWaitArgs w{};     // then every peer's ready in my mailbox[32 + j]
    int n = 0;
    for (int j = 0; j < dp_size_; ++j) {
      if (j == dp_me_) continue;
      r.flags[n] = dp_mail_[static_cast<size_t>(j)] + 32 + dp_me_;
      w.flags[n] = mailbox_ + 32 + j;
      ++n;
    }
    r.count = w.count = n;
    r.seq = relay_seq_ + 2;
    w.seq = relay_seq_ + 2;
    r.advance = 1;
    w.bias = 0;
    check(pbdk::relay_release(r, st), "dp ready");
    check(pbdk::relay_wait(w, st), "dp wait ready");
  }

  void dp_release(cudaStream_t st) {  // I have read every peer's gradients of this step
    if (!dp_active()) return;
    pbdk::RelayReleaseArgs r{};
    int n = 0;
    for (int j = 0; j < dp_size_; ++j)
      if (j != dp_me_) r.flags[n++] = dp_mail_[static_cast<size_t>(j)] + 48 + dp_me_;
    r.count = n;
    r.seq = relay_seq_ + 2;
    r.advance = 0;
    check(pbdk::relay_release(r, st), "dp consumed");
  }

  void dp_wait_consumed(cudaStream_t st) {  // before this step's wgrads overwrite my gradients
    if (!dp_active()) return;
    pbdk::RelayWaitArgs w{};
    int n = 0;
    for (int j = 0; j < dp_size_; ++j)
      if (j != dp_me_) w.flags[n++] = mailbox_ + 48 + j;
    w.count = n;
    w.seq = relay_seq_ + 2;
    w.bias = 0;
    check(pbdk::relay_wait(w, st), "dp wait consumed");
  }

  // share_gradient + update_weight of a DP group as reduce-scatter + all-gather over peer memory
  // (DESIGN.md §8).  Every parameter region [off, off+n) of the step is cut into G slices
  // (pbdk::dp_slice); member `me`:
  //   1. sums slice `me` of the group's gradient slabs in member order (peer loads) and applies the
  //      momentum SGD to that slice of w / v (+ bf16 shadow);
  //   2. publishes "updated" to every member and waits for theirs (device-side flags, mailbox 64+j);
  //   3. copies every other member's updated slice of w from its peer memory (+ bf16 shadow).
  // Per member and step that is (G-1)/G * P fp32 read in 1 and again in 3: 2(G-1)/G * 4P bytes over
  // NVLink, exactly the ring-allreduce volume cost_model.cpp:79-86 prices; each slice is computed
  // once (fixed member order), so every member holds bit-identical weights.  Momentum stays sharded:
  // dp_sync_state() completes it when the host reads it.
  struct DpRegion {
    size_t off, n;
  };
  virtual std::vector<DpRegion> dp_all_regions() const = 0;

  void dp_update(const std::vector<DpRegion>& regions, float* w, float* v, const float* g, void* shadow_bf16,
                 long long* counter, cudaStream_t st) {
    require_dp_params();
    const int G = dp_size_, me = dp_me_;
    for (const DpRegion& r : regions) {
      size_t lo = 0, hi = 0;
      pbdk::dp_slice(r.n, G, me, &lo, &hi);
      const auto src = dp_sources(g, r.off + lo);
      void* sh = shadow_bf16 != nullptr ? static_cast<void*>(static_cast<uint16_t*>(shadow_bf16) + r.off + lo) : nullptr;
      check(pbdk::sgd_momentum_sum(w + r.off + lo, v + r.off + lo, src.data(), G, sh, hi - lo, d_.lr, d_.momentum,
                                   counter, st),
            "dp reduce-scatter sgd");
      counter = nullptr;
    }
    pbdk::RelayReleaseArgs rel{};
    pbdk::RelayWaitArgs wt{};
    int n = 0;
    for (int j = 0; j < G; ++j) {
      if (j == me) continue;
      rel.flags[n] = dp_mail_[static_cast<size_t>(j)] + 64 + me;
      wt.flags[n] = mailbox_ + 64 + j;
      ++n;
    }
    rel.count = wt.count = n;
    rel.seq = relay_seq_ + 2;
    wt.seq = relay_seq_ + 2;
    rel.advance = 0;
    wt.bias = 0;
    check(pbdk::relay_release(rel, st), "dp updated");
    check(pbdk::relay_wait(wt, st), "dp wait updated");
    for (const DpRegion& r : regions) {
      std::vector<const float*> pw(static_cast<size_t>(G));
      for (int j = 0; j < G; ++j) pw[static_cast<size_t>(j)] = (j == me ? w : dp_params_[static_cast<size_t>(j)]) + r.off;
      void* sh = shadow_bf16 != nullptr ? static_cast<void*>(static_cast<uint16_t*>(shadow_bf16) + r.off) : nullptr;
      check(pbdk::dp_gather(w + r.off, sh, pw.data(), G, me, r.n, st), "dp all-gather");
    }
  }

  void require_dp_params() const {
    if (static_cast<int>(dp_params_.size()) != dp_size_) throw BadArg("dp group: peer params not set (pbdx_dp_set_params)");
  }

  // [0,16) relay ready, [16,32) relay consumed, [32,48) dp ready, [48,64) dp consumed, [64,80) dp updated
  static constexpr int kMailboxSlots = 80;
  int dp_size_ = 1, dp_me_ = 0;
  std::vector<const float*> dp_grads_;
  std::vector<const float*> dp_params_;
  std::vector<unsigned long long*> dp_mail_;

  void relay_wait_input(cudaStream_t st) {
    if (recv_consumed_.empty()) return;
    pbdk::RelayWaitArgs a{};
    for (size_t i = 0; i < recv_consumed_.size(); ++i) a.flags[i] = mailbox_ + i;
    a.seq = relay_seq_ + 0;  // receive sequence
    a.bias = 1;
    a.count = static_cast<int>(recv_consumed_.size());
    check(pbdk::relay_wait(a, st), "relay wait input");
  }

  void relay_send_output(cudaStream_t st) {
    if (send_.empty()) return;
    cuda(cudaEventRecord(relay_fork_, st), "event");
    cuda(cudaStreamWaitEvent(relay_stream_, relay_fork_, 0), "wait");
    pbdk::RelayWaitArgs w{};
    pbdk::RelayCopyArgs c{};
    const size_t row = relay_row_bytes();
    const char* out = static_cast<const char*>(relay_source());
    for (size_t i = 0; i < send_.size(); ++i) {
      w.flags[i] = mailbox_ + pbdk::kRelayMaxPeers + i;
      c.src[i] = out + row * static_cast<size_t>(send_[i].src_row);
      c.dst[i] = send_[i].dst;
      c.vec16[i] = static_cast<long long>(row * static_cast<size_t>(send_[i].rows) / 16);
      c.ready[i] = static_cast<unsigned long long*>(send_[i].remote_flag);
    }
    w.count = c.count = static_cast<int>(send_.size());
    w.seq = c.seq = relay_seq_ + 1;  // send sequence
    w.bias = 0;
    c.ticket = relay_ticket_;
    check(pbdk::relay_wait(w, relay_stream_), "relay wait consumed");
    check(pbdk::relay_copy(c, 64, relay_stream_), "relay copy");
    cuda(cudaEventRecord(relay_done_, relay_stream_), "event");
  }

  // after the last reader of the input (teacher block lo, student block lo) and the send
  void relay_finish(cudaStream_t st) {
    if (!send_.empty()) cuda(cudaStreamWaitEvent(st, relay_done_, 0), "join relay");
    if (recv_consumed_.empty()) return;
    pbdk::RelayReleaseArgs a{};
    for (size_t i = 0; i < recv_consumed_.size(); ++i)
      a.flags[i] = static_cast<unsigned long long*>(recv_consumed_[i]);
    a.seq = relay_seq_ + 0;
    a.count = static_cast<int>(recv_consumed_.size());
    check(pbdk::relay_release(a, st), "relay release");
  }

  bool trains(int i) const { return (train_mask_ >> i) & 1u; }
  bool all_train() const { return train_mask_ == 0xFFFFFFFFu || train_mask_ == ((1u << nblocks()) - 1u); }

  pbdx_desc d_;
  uint32_t train_mask_ = 0xFFFFFFFFu;
  int n_ = 0;
  int first_ = 0;
  int external_ = 0;  // 0 synthetic (Philox), 1 upload_images, 2 staged double buffer
  bool timing_ = false;
  Arena arena_;
  // K11 relay state: mailbox_ = flags written by peers ([0,16) ready per sender, [16,32) consumed
  // per receiver); relay_seq_ = {receive seq, send seq} (device-side, so graph replays advance them)
  unsigned long long* mailbox_ = nullptr;
  unsigned long long* relay_seq_ = nullptr;
  unsigned int* relay_ticket_ = nullptr;
  std::vector<cudaEvent_t> ev_t_, ev_s_;  // per block: {start, end} pairs
  cudaEvent_t trace_ref_ = nullptr;

 private:
  bool graph_valid_ = false;
  bool phases_valid_ = false;
  cudaGraphExec_t graph_exec_ = nullptr;
  cudaGraphExec_t phase_exec_[3] = {nullptr, nullptr, nullptr};
  cudaStream_t cap_stream_ = nullptr;
  std::vector<void*> recv_consumed_;
  std::vector<pbdx_relay_msg> send_;
  cudaStream_t relay_stream_ = nullptr;
  cudaEvent_t relay_fork_ = nullptr, relay_done_ = nullptr;
};

// model factories
PartitionBase* make_resnet_partition(const pbdx_desc& d);
PartitionBase* make_resnet_f32_partition(const pbdx_desc& d);
PartitionBase* make_mb_partition(const pbdx_desc& d);

}  // namespace pbd::exec
