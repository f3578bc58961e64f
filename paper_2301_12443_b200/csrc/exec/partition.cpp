// Per-GPU partition executor: the device body of Algorithm 1
// for a contiguous block range of the CIFAR ResNet-18 teacher / slim student
// chain.  The simulated counterpart is simulate.cpp:193-262;
// this runs the kernels for real and times them with CUDA events.
//
//   teacher_forward : [Philox input] -> per block: stem?, BasicBlock x2
//                     (tcgen05 conv + fused bias/residual/ReLU epilogues)
//   student_step    : per block: conv1, shortcut, BN1+ReLU, conv2, BN2/BNsc stats,
//                     fused MSE+ReLU-bwd+BN-bwd, wgrad x3 (split-K), dgrad (flipped
//                     weights, ReLU-mask epilogue), BN1 backward
//   apply_update    : one fused SGD-momentum launch over the partition's flat
//                     parameters (+ bf16 shadows) and one weight flip per block
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "bd_kernels.hpp"
#include "conv.hpp"
#include "pbdk.h"
#include "pbdx.h"
#include "relay.hpp"

namespace pbd::exec {

namespace {

constexpr int kBlocks = 4;
constexpr int T_CH[5] = {3, 64, 128, 256, 512};
constexpr int T_HW[5] = {32, 32, 16, 8, 4};

int stored(int c) { return c == 3 ? 16 : c; }

struct CudaFail : std::runtime_error {
  explicit CudaFail(const std::string& m) : std::runtime_error(m) {}
};
struct BadArg : std::runtime_error {
  explicit BadArg(const std::string& m) : std::runtime_error(m) {}
};

void check(int rc, const char* what) {
  if (rc == PBDK_EINVAL) throw BadArg(what);
  if (rc != PBDK_OK) throw CudaFail(std::string(what) + ": " + cudaGetErrorString(cudaGetLastError()));
}
void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail(std::string(what) + ": " + cudaGetErrorString(e));
}

float kaiming(int fan_in, float gain) { return std::sqrt(6.0f / static_cast<float>(fan_in)) * gain; }

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
    return static_cast<T*>(p);
  }

 private:
  std::vector<void*> ptrs_;
};

using bf16 = __nv_bfloat16;

struct TConv {
  int cin, cs, cout, r, stride, pad, hin, hout;
  float gain;
  uint32_t tensor;  // Philox tensor id of the weight (bias = +1)
  int epi;
  bf16* w = nullptr;
  float* bias = nullptr;
  const void* in = nullptr;
  void* out = nullptr;
  const void* aux = nullptr;
  pbdk::FpropPlan plan;
};

TConv tconv(int cin, int cs, int cout, int r, int stride, int pad, int hin, int hout, float gain, int epi) {
  TConv c;
  c.cin = cin;
  c.cs = cs;
  c.cout = cout;
  c.r = r;
  c.stride = stride;
  c.pad = pad;
  c.hin = hin;
  c.hout = hout;
  c.gain = gain;
  c.tensor = 0;
  c.epi = epi;
  return c;
}

struct TBlock {
  int k;
  std::vector<TConv> convs;  // execution order
  bf16* out = nullptr;       // t_k
};

// student parameter offsets inside the block's flat slice (padded storage)
struct SLayout {
  size_t w1, w2, wsc, g1, b1, g2, b2, gsc, bsc, total;
};

SLayout student_layout(int k) {
  const int cin = stored(T_CH[k]), cout = T_CH[k + 1], mid = cout / 2;
  SLayout l{};
  size_t o = 0;
  l.w1 = o;
  o += static_cast<size_t>(mid) * 9 * cin;
  l.w2 = o;
  o += static_cast<size_t>(cout) * 9 * mid;
  l.wsc = o;
  o += static_cast<size_t>(cout) * cin;
  l.g1 = o;
  o += mid;
  l.b1 = o;
  o += mid;
  l.g2 = o;
  o += cout;
  l.b2 = o;
  o += cout;
  l.gsc = o;
  o += cout;
  l.bsc = o;
  o += cout;
  l.total = o;
  return l;
}

struct SBlock {
  int k, cin, cs, cout, mid, stride, hin, hout;
  SLayout lay;
  size_t base = 0;  // offset of this block in the partition's flat vectors
  const bf16* in = nullptr;
  const bf16* target = nullptr;
  bf16 *y1, *a1, *y2, *ys, *dy2, *dys, *g1, *dy1, *w2flip;
  float *st1, *st2, *sts, *red, *red1;
  pbdk::FpropPlan p_conv1, p_sc, p_conv2, p_dgrad;
  pbdk::WgradPlan p_w2, p_wsc, p_w1;
  // per-block scratch + stream: student blocks only depend on teacher outputs, so each runs
  // on its own stream as soon as its teacher block is done (overlaps teacher k+1 and the
  // other student blocks; the late blocks alone do not fill 148 SMs).
  float* rws = nullptr;
  void* wws = nullptr;
  size_t wws_bytes = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
};

}  // namespace

class Partition {
 public:
  explicit Partition(const pbdx_desc& d) : d_(d) {
    if (d.block_lo < 0 || d.block_hi >= kBlocks || d.block_lo > d.block_hi) throw BadArg("bad block range");
    if (d.n_max < 1 || d.global_batch < 1) throw BadArg("bad batch");
    n_ = d.n_max;
    allocate();
    build_plans();
  }

  int nblocks() const { return d_.block_hi - d_.block_lo + 1; }

  void init_params(cudaStream_t st) {
    for (TBlock& tb : tblocks_)
      for (TConv& c : tb.convs) {
        check(pbdk::init_uniform(c.w, 1, c.cout, c.r, c.r, c.cs, c.cin, d_.seed_teacher, c.tensor,
                                 kaiming(c.cin * c.r * c.r, c.gain), st),
              "init teacher w");
        check(pbdk::init_uniform(c.bias, 0, c.cout, 1, 1, 1, 1, d_.seed_teacher, c.tensor + 1, 0.1f, st),
              "init teacher b");
      }
    for (SBlock& s : sblocks_) {
      float* p = params_ + s.base;
      check(pbdk::init_uniform(p + s.lay.w1, 0, s.mid, 3, 3, s.cs, s.cin, d_.seed_student, 10 * s.k + 0,
                               kaiming(9 * s.cin, 1.0f), st),
            "init w1");
      check(pbdk::init_uniform(p + s.lay.w2, 0, s.cout, 3, 3, s.mid, s.mid, d_.seed_student, 10 * s.k + 1,
                               kaiming(9 * s.mid, 1.0f), st),
            "init w2");
      check(pbdk::init_uniform(p + s.lay.wsc, 0, s.cout, 1, 1, s.cs, s.cin, d_.seed_student, 10 * s.k + 2,
                               kaiming(s.cin, 1.0f), st),
            "init wsc");
      check(pbdk::fill(p + s.lay.g1, s.mid, 1.0f, st), "fill");
      check(pbdk::fill(p + s.lay.b1, s.mid, 0.0f, st), "fill");
      check(pbdk::fill(p + s.lay.g2, s.cout, 1.0f, st), "fill");
      check(pbdk::fill(p + s.lay.b2, s.cout, 0.0f, st), "fill");
      check(pbdk::fill(p + s.lay.gsc, s.cout, 1.0f, st), "fill");
      check(pbdk::fill(p + s.lay.bsc, s.cout, 0.0f, st), "fill");
    }
    check(pbdk::fill(mom_, total_, 0.0f, st), "fill");
    check(pbdk::fill(grads_, total_, 0.0f, st), "fill");
    // shadows: an SGD step with zero gradient and lr 0 is an exact bf16 cast
    check(pbdk::sgd_momentum(params_, mom_, grads_, shadow_, total_, 0.0f, 0.0f, nullptr, st), "shadow");
    refresh_flips(st);
    cuda(cudaMemsetAsync(step_, 0, sizeof(long long), st), "memset");
  }

  void set_shard(int n, int first) {
    if (n < 1 || n > d_.n_max || first < 0 || first + n > d_.global_batch) throw BadArg("bad shard");
    first_ = first;
    if (n != n_) {
      n_ = n;
      build_plans();
      graph_valid_ = false;
      phases_valid_ = false;
    }
  }

  void set_external_input(bool ext) {
    external_ = ext;
    graph_valid_ = false;
    phases_valid_ = false;
  }

  void upload_images(const float* host, int n, cudaStream_t st) {
    if (d_.block_lo != 0) throw BadArg("only partition 0 loads data");
    if (n != n_) throw BadArg("upload size != shard size");
    cuda(cudaMemcpyAsync(stage_, host, static_cast<size_t>(n) * 32 * 32 * 3 * sizeof(float), cudaMemcpyHostToDevice,
                         st),
         "H2D images");
    check(pbdk::pack_image(stage_, input_, n, st), "pack image");
  }

  // ---- K11 peer relay (relay.cu): the receiver's input buffer is written by its senders
  void relay_set_recv(int n, void* const* remote_consumed) {
    if (n < 0 || n > pbdk::kRelayMaxPeers) throw BadArg("relay: too many senders");
    if (n > 0 && d_.block_lo == 0) throw BadArg("relay: partition 0 loads data, it receives nothing");
    recv_consumed_.assign(remote_consumed, remote_consumed + n);
    graph_valid_ = phases_valid_ = false;
  }

  void relay_set_send(int n, const pbdx_relay_msg* msgs) {
    if (n < 0 || n > pbdk::kRelayMaxPeers) throw BadArg("relay: too many receivers");
    const size_t row = tout_bytes_ / static_cast<size_t>(d_.n_max);
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
    graph_valid_ = phases_valid_ = false;
  }

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
    const size_t row = tout_bytes_ / static_cast<size_t>(d_.n_max);
    const char* out = reinterpret_cast<const char*>(tblocks_.back().out);
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

  void teacher_forward(cudaStream_t st) {
    relay_wait_input(st);
    if (d_.block_lo == 0 && !external_)
      check(pbdk::philox_image(input_, n_, first_, step_, d_.global_batch, d_.seed_data, st), "philox");
    for (size_t i = 0; i < tblocks_.size(); ++i) {
      if (timing_) cuda(cudaEventRecord(ev_t_[2 * i], st), "event");
      for (TConv& c : tblocks_[i].convs) check(pbdk::fprop_run(c.plan, st), "teacher conv");
      if (timing_) cuda(cudaEventRecord(ev_t_[2 * i + 1], st), "event");
      cuda(cudaEventRecord(tdone_[i], st), "event");
    }
    relay_send_output(st);
  }

  // Student block k runs on its own stream.  Fused step(): it starts once teacher block k is
  // done (event recorded by teacher_forward).  Standalone phase (multi-GPU driver, phase
  // graphs): the student streams fork from the caller's stream at entry.  The caller's
  // stream joins all of them before returning.
  void student_step(cudaStream_t caller) { student_step_impl(caller, true); }

  void student_step_impl(cudaStream_t caller, bool fork) {
    if (fork) cuda(cudaEventRecord(fork_, caller), "event");
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      SBlock& s = sblocks_[i];
      cudaStream_t st = s.stream;
      cuda(cudaStreamWaitEvent(st, fork ? fork_ : tdone_[i], 0), "wait teacher");
      if (timing_) cuda(cudaEventRecord(ev_s_[2 * i], st), "event");
      const float* p = params_ + s.base;
      float* g = grads_ + s.base;
      const int m = n_ * s.hout * s.hout;
      check(pbdk::fprop_run(s.p_conv1, st), "conv1");
      check(pbdk::fprop_run(s.p_sc, st), "shortcut");
      check(pbdk::bn_stats(s.y1, m, s.mid, s.rws, s.st1, st), "bn1 stats");
      check(pbdk::bn_apply_relu(s.y1, s.st1, p + s.lay.g1, p + s.lay.b1, s.a1, m, s.mid, st), "bn1 apply");
      check(pbdk::fprop_run(s.p_conv2, st), "conv2");
      check(pbdk::bn_stats2(s.y2, s.ys, m, s.cout, s.rws, s.st2, s.sts, st), "bn2/bnsc stats");
      const double norm = static_cast<double>(d_.global_batch) * s.cout * s.hout * s.hout;
      pbdk::MseArgs a{s.y2, s.ys, s.target, s.st2, s.sts, p + s.lay.g2, p + s.lay.b2, p + s.lay.gsc, p + s.lay.bsc,
                      m, s.cout, static_cast<float>(2.0 / norm), norm, s.rws, s.red, g + s.lay.g2, g + s.lay.b2,
                      g + s.lay.gsc, g + s.lay.bsc, losses_ + i, s.dy2, s.dys};
      check(pbdk::mse_bn_loss(a, st), "mse");
      check(pbdk::wgrad_run(s.p_w2, st), "wgrad2");
      check(pbdk::wgrad_run(s.p_wsc, st), "wgrad sc");
      check(pbdk::fprop_run(s.p_dgrad, st), "dgrad2");
      check(pbdk::bn_bwd(s.g1, s.y1, s.st1, p + s.lay.g1, m, s.mid, s.rws, s.red1, g + s.lay.g1, g + s.lay.b1, s.dy1,
                         st),
            "bn1 bwd");
      check(pbdk::wgrad_run(s.p_w1, st), "wgrad1");
      if (timing_) cuda(cudaEventRecord(ev_s_[2 * i + 1], st), "event");
      cuda(cudaEventRecord(s.done, st), "event");
    }
    for (SBlock& s : sblocks_) cuda(cudaStreamWaitEvent(caller, s.done, 0), "join");
    relay_finish(caller);
  }

  // bf16 shadows + flipped dgrad weights from the fp32 master weights (after a state migration)
  void refresh_shadows(cudaStream_t st) {
    check(pbdk::sgd_momentum(params_, mom_, grads_, shadow_, total_, 0.0f, 1.0f, nullptr, st), "shadow");
    refresh_flips(st);
  }

  void apply_update(cudaStream_t st) {
    check(pbdk::sgd_momentum(params_, mom_, grads_, shadow_, total_, d_.lr, d_.momentum, step_, st), "sgd");
    refresh_flips(st);
  }

  void step(cudaStream_t st) {
    teacher_forward(st);
    student_step_impl(st, false);
    apply_update(st);
  }

  // Three graphs (teacher_forward / student_step / apply_update) for the multi-GPU driver, which
  // interleaves NCCL relay and allreduce between them.
  // fuse_ts: phase 0 = teacher_forward + student_step with the per-block teacher->student
  // overlap of step(), phase 1 empty (ranks that send no relay: nothing to put in between).
  void capture_phases(cudaStream_t caller, bool fuse_ts) {
    if (cap_stream_ == nullptr) cuda(cudaStreamCreateWithFlags(&cap_stream_, cudaStreamNonBlocking), "stream");
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
      if (nodes > 0) cuda(cudaGraphInstantiate(&phase_exec_[ph], g, 0), "instantiate");
      cudaGraphDestroy(g);
    }
    timing_ = was_timing;
    phases_valid_ = true;
  }

  void replay_phase(int ph, cudaStream_t st) {
    if (ph < 0 || ph > 2 || !phases_valid_) throw BadArg("no captured phase graph");
    if (phase_exec_[ph] != nullptr) cuda(cudaGraphLaunch(phase_exec_[ph], st), "graph launch");
  }

  // Captures on a private non-blocking stream (the legacy default stream cannot be
  // captured); the instantiated graph is replayed on the caller's stream.
  void capture(cudaStream_t caller) {
    if (graph_exec_ != nullptr) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
    if (cap_stream_ == nullptr) cuda(cudaStreamCreateWithFlags(&cap_stream_, cudaStreamNonBlocking), "stream");
    cuda(cudaStreamSynchronize(caller), "sync");
    cudaStream_t st = cap_stream_;
    cudaGraph_t g = nullptr;
    cuda(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
    const bool was_timing = timing_;
    timing_ = false;
    try {
      step(st);
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      timing_ = was_timing;
      throw;
    }
    timing_ = was_timing;
    cuda(cudaStreamEndCapture(st, &g), "end capture");
    cuda(cudaGraphInstantiate(&graph_exec_, g, 0), "instantiate");
    cudaGraphDestroy(g);
    graph_valid_ = true;
  }

  void replay(cudaStream_t st) {
    if (!graph_valid_ || graph_exec_ == nullptr) throw BadArg("no captured graph for the current shard");
    cuda(cudaGraphLaunch(graph_exec_, st), "graph launch");
  }

  void set_timing(bool on) {
    timing_ = on;
    if (on && ev_t_.empty()) {
      ev_t_.resize(2 * tblocks_.size());
      ev_s_.resize(2 * sblocks_.size());
      for (auto& e : ev_t_) cuda(cudaEventCreate(&e), "event create");
      for (auto& e : ev_s_) cuda(cudaEventCreate(&e), "event create");
    }
  }

  void block_times(float* tms, float* sms) {
    if (ev_t_.empty()) throw BadArg("timing not enabled");
    for (size_t i = 0; i < tblocks_.size(); ++i) {
      cuda(cudaEventSynchronize(ev_t_[2 * i + 1]), "event sync");
      cuda(cudaEventElapsedTime(&tms[i], ev_t_[2 * i], ev_t_[2 * i + 1]), "elapsed");
      cuda(cudaEventSynchronize(ev_s_[2 * i + 1]), "event sync");
      cuda(cudaEventElapsedTime(&sms[i], ev_s_[2 * i], ev_s_[2 * i + 1]), "elapsed");
    }
  }

  void buffer(int which, void** ptr, size_t* bytes) {
    switch (which) {
      case PBDX_BUF_INPUT: *ptr = input_; *bytes = input_bytes_; break;
      case PBDX_BUF_TEACHER_OUT: *ptr = tblocks_.back().out; *bytes = tout_bytes_; break;
      case PBDX_BUF_GRADS: *ptr = grads_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_PARAMS: *ptr = params_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_MOMENTUM: *ptr = mom_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_LOSSES: *ptr = losses_; *bytes = nblocks() * sizeof(double); break;
      case PBDX_BUF_STEP: *ptr = step_; *bytes = sizeof(long long); break;
      case PBDX_BUF_TEACHER_PARAMS: *ptr = tparams_; *bytes = tparam_bytes_; break;
      case PBDX_BUF_MAILBOX: *ptr = mailbox_; *bytes = 2 * pbdk::kRelayMaxPeers * sizeof(unsigned long long); break;
      default: throw BadArg("unknown buffer");
    }
  }

  void teacher_act(int k, void** ptr, size_t* bytes) {
    if (k < d_.block_lo || k > d_.block_hi) throw BadArg("block outside partition");
    *ptr = tblocks_[static_cast<size_t>(k - d_.block_lo)].out;
    *bytes = act_bytes(T_HW[k + 1], T_CH[k + 1]);
  }

  int launches_per_step() const {
    int n = (d_.block_lo == 0 && !external_) ? 1 : 0;
    for (const TBlock& tb : tblocks_) n += static_cast<int>(tb.convs.size());
    for (const SBlock& s : sblocks_) {
      n += 3 + 3 + 2 + 3 + 1 + 3;  // convs, bn1 stats(2)+apply, bn2+bnsc stats(2), mse(3), dgrad, bn_bwd(3)
      n += (s.p_w2.splits > 1 ? 2 : 1) + (s.p_wsc.splits > 1 ? 2 : 1) + (s.p_w1.splits > 1 ? 2 : 1);
    }
    n += 1 + static_cast<int>(sblocks_.size());  // sgd + flips
    if (!recv_consumed_.empty()) n += 2;         // relay wait + release
    if (!send_.empty()) n += 2;                  // relay wait + copy
    return n;
  }

  ~Partition() {
    if (graph_exec_ != nullptr) cudaGraphExecDestroy(graph_exec_);
    if (cap_stream_ != nullptr) cudaStreamDestroy(cap_stream_);
    for (SBlock& s : sblocks_) {
      if (s.stream != nullptr) cudaStreamDestroy(s.stream);
      if (s.done != nullptr) cudaEventDestroy(s.done);
    }
    for (auto e : tdone_) cudaEventDestroy(e);
    for (auto g : phase_exec_)
      if (g != nullptr) cudaGraphExecDestroy(g);
    if (fork_ != nullptr) cudaEventDestroy(fork_);
    if (relay_stream_ != nullptr) cudaStreamDestroy(relay_stream_);
    if (relay_fork_ != nullptr) cudaEventDestroy(relay_fork_);
    if (relay_done_ != nullptr) cudaEventDestroy(relay_done_);
    for (auto e : ev_t_) cudaEventDestroy(e);
    for (auto e : ev_s_) cudaEventDestroy(e);
  }

 private:
  void refresh_flips(cudaStream_t st) {
    for (SBlock& s : sblocks_)
      check(pbdk_weight_flip(shadow_ + s.base + s.lay.w2, s.w2flip, s.cout, 3, 3, s.mid, st), "flip");
  }

  size_t act_bytes(int hw, int c) const { return static_cast<size_t>(d_.n_max) * hw * hw * c * sizeof(bf16); }

  void allocate() {
    const int lo = d_.block_lo, hi = d_.block_hi;
    input_bytes_ = act_bytes(T_HW[lo], stored(T_CH[lo]));
    input_ = arena_.get<bf16>(input_bytes_);
    if (lo == 0) stage_ = arena_.get<float>(static_cast<size_t>(d_.n_max) * 32 * 32 * 3 * sizeof(float));

    // ---- teacher program
    size_t tw = 0;
    std::vector<std::vector<TConv>> progs;
    for (int k = lo; k <= hi; ++k) {
      std::vector<TConv> convs;
      int j = 0;
      int cin = T_CH[k], hw = T_HW[k];
      if (k == 0) {
        convs.push_back(tconv(3, 16, 64, 3, 1, 1, 32, 32, 1.0f, PBDK_EPI_BIAS_RELU));
        convs.back().tensor = static_cast<uint32_t>(1000 * k + 10 * j++);
        cin = 64;
      }
      const int cout = T_CH[k + 1];
      const int s = T_HW[k] / T_HW[k + 1];
      for (int b = 0; b < 2; ++b) {
        const int stv = b == 0 ? s : 1;
        const int ci = b == 0 ? cin : cout;
        const int ohw = hw / stv;
        TConv c1 = tconv(ci, stored(ci), cout, 3, stv, 1, hw, ohw, 1.0f, PBDK_EPI_BIAS_RELU);
        TConv c2 = tconv(cout, cout, cout, 3, 1, 1, ohw, ohw, 0.5f, PBDK_EPI_BIAS_RES_RELU);
        c1.tensor = static_cast<uint32_t>(1000 * k + 10 * j);
        c2.tensor = static_cast<uint32_t>(1000 * k + 10 * (j + 1));
        convs.push_back(c1);
        if (stv != 1 || ci != cout) {
          TConv cp = tconv(ci, stored(ci), cout, 1, stv, 0, hw, ohw, 1.0f, PBDK_EPI_BIAS);
          cp.tensor = static_cast<uint32_t>(1000 * k + 10 * (j + 2));
          convs.push_back(cp);
          j += 3;
        } else {
          j += 2;
        }
        convs.push_back(c2);
        hw = ohw;
      }
      for (const TConv& c : convs) tw += static_cast<size_t>(c.cout) * c.r * c.r * c.cs;
      progs.push_back(std::move(convs));
    }
    tparam_bytes_ = tw * sizeof(bf16);
    tparams_ = arena_.get<bf16>(tparam_bytes_);
    bf16* wp = tparams_;
    const bf16* prev_out = input_;
    for (int k = lo; k <= hi; ++k) {
      TBlock tb;
      tb.k = k;
      tb.convs = std::move(progs[static_cast<size_t>(k - lo)]);
      const bf16* x = prev_out;
      const bf16* block_in = x;
      const bf16* sc = nullptr;
      for (TConv& c : tb.convs) {
        c.w = wp;
        wp += static_cast<size_t>(c.cout) * c.r * c.r * c.cs;
        c.bias = arena_.get<float>(static_cast<size_t>(c.cout) * sizeof(float));
        bf16* out = arena_.get<bf16>(act_bytes(c.hout, c.cout));
        if (c.epi == PBDK_EPI_BIAS) {  // projection shortcut: input of the BasicBlock
          c.in = block_in;
          c.out = out;
          sc = out;
        } else if (c.epi == PBDK_EPI_BIAS_RES_RELU) {  // conv2: residual = projection or block input
          c.in = x;
          c.out = out;
          c.aux = sc != nullptr ? sc : block_in;
          x = out;
          block_in = out;
          sc = nullptr;
        } else {  // stem / conv1
          c.in = x;
          c.out = out;
          if (c.r == 3 && c.cin == 3) {  // stem: its output is the first BasicBlock's input
            x = out;
            block_in = out;
          } else {
            x = out;
          }
        }
      }
      tb.out = const_cast<bf16*>(x);
      prev_out = tb.out;
      tblocks_.push_back(std::move(tb));
    }
    tout_bytes_ = act_bytes(T_HW[hi + 1], T_CH[hi + 1]);

    // ---- student blocks
    total_ = 0;
    for (int k = lo; k <= hi; ++k) {
      SBlock s{};
      s.k = k;
      s.cin = T_CH[k];
      s.cs = stored(T_CH[k]);
      s.cout = T_CH[k + 1];
      s.mid = s.cout / 2;
      s.hin = T_HW[k];
      s.hout = T_HW[k + 1];
      s.stride = s.hin / s.hout;
      s.lay = student_layout(k);
      s.base = total_;
      total_ += s.lay.total;
      s.in = (k == lo) ? input_ : tblocks_[static_cast<size_t>(k - lo - 1)].out;
      s.target = tblocks_[static_cast<size_t>(k - lo)].out;
      s.y1 = arena_.get<bf16>(act_bytes(s.hout, s.mid));
      s.a1 = arena_.get<bf16>(act_bytes(s.hout, s.mid));
      s.g1 = arena_.get<bf16>(act_bytes(s.hout, s.mid));
      s.dy1 = arena_.get<bf16>(act_bytes(s.hout, s.mid));
      s.y2 = arena_.get<bf16>(act_bytes(s.hout, s.cout));
      s.ys = arena_.get<bf16>(act_bytes(s.hout, s.cout));
      s.dy2 = arena_.get<bf16>(act_bytes(s.hout, s.cout));
      s.dys = arena_.get<bf16>(act_bytes(s.hout, s.cout));
      s.w2flip = arena_.get<bf16>(static_cast<size_t>(s.mid) * 9 * s.cout * sizeof(bf16));
      s.st1 = arena_.get<float>(2 * s.mid * sizeof(float));
      s.red1 = arena_.get<float>(2 * s.mid * sizeof(float));
      s.st2 = arena_.get<float>(2 * s.cout * sizeof(float));
      s.sts = arena_.get<float>(2 * s.cout * sizeof(float));
      s.red = arena_.get<float>(4 * s.cout * sizeof(float));
      sblocks_.push_back(s);
    }
    params_ = arena_.get<float>(total_ * sizeof(float));
    mom_ = arena_.get<float>(total_ * sizeof(float));
    grads_ = arena_.get<float>(total_ * sizeof(float));
    shadow_ = arena_.get<bf16>(total_ * sizeof(bf16));
    losses_ = arena_.get<double>(kBlocks * sizeof(double));
    step_ = arena_.get<long long>(sizeof(long long));
    mailbox_ = arena_.get<unsigned long long>(2 * pbdk::kRelayMaxPeers * sizeof(unsigned long long));
    relay_seq_ = arena_.get<unsigned long long>(2 * sizeof(unsigned long long));
    relay_ticket_ = arena_.get<unsigned int>(sizeof(unsigned int));

    // ---- per-block scratch sized for n_max, streams and events
    for (SBlock& s : sblocks_) {
      const int m = d_.n_max * s.hout * s.hout;
      size_t rws = std::max(pbdk::reduce_workspace_floats(m, s.cout, 3), pbdk::reduce_workspace_floats(m, s.mid, 3));
      size_t wws = 0;
      for (const pbdk_conv_desc& cd : {conv1_desc(s, d_.n_max), sc_desc(s, d_.n_max), conv2_desc(s, d_.n_max)})
        wws = std::max(wws, pbdk::wgrad_workspace_bytes(cd));
      s.rws = arena_.get<float>(rws * sizeof(float));
      s.wws_bytes = wws;
      s.wws = arena_.get<void>(wws);
      cuda(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "stream");
      cuda(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming), "event");
    }
    tdone_.resize(tblocks_.size());
    for (auto& e : tdone_) cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cuda(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "event");
  }

  static pbdk_conv_desc conv1_desc(const SBlock& s, int n) {
    return pbdk_conv_desc{n, s.hin, s.hin, s.cs, s.mid, 3, 3, s.stride, 1, s.hout, s.hout};
  }
  static pbdk_conv_desc sc_desc(const SBlock& s, int n) {
    return pbdk_conv_desc{n, s.hin, s.hin, s.cs, s.cout, 1, 1, s.stride, 0, s.hout, s.hout};
  }
  static pbdk_conv_desc conv2_desc(const SBlock& s, int n) {
    return pbdk_conv_desc{n, s.hout, s.hout, s.mid, s.cout, 3, 3, 1, 1, s.hout, s.hout};
  }

  void build_plans() {
    for (TBlock& tb : tblocks_)
      for (TConv& c : tb.convs) {
        const pbdk_conv_desc cd{n_, c.hin, c.hin, c.cs, c.cout, c.r, c.r, c.stride, c.pad, c.hout, c.hout};
        check(pbdk::fprop_plan(cd, c.in, c.w, c.out, c.bias, c.aux, c.epi, &c.plan), "teacher plan");
      }
    for (SBlock& s : sblocks_) {
      const bf16* sh = shadow_ + s.base;
      float* g = grads_ + s.base;
      check(pbdk::fprop_plan(conv1_desc(s, n_), s.in, sh + s.lay.w1, s.y1, nullptr, nullptr, PBDK_EPI_STORE,
                             &s.p_conv1),
            "conv1 plan");
      check(pbdk::fprop_plan(sc_desc(s, n_), s.in, sh + s.lay.wsc, s.ys, nullptr, nullptr, PBDK_EPI_STORE, &s.p_sc),
            "sc plan");
      check(pbdk::fprop_plan(conv2_desc(s, n_), s.a1, sh + s.lay.w2, s.y2, nullptr, nullptr, PBDK_EPI_STORE,
                             &s.p_conv2),
            "conv2 plan");
      const pbdk_conv_desc dg{n_, s.hout, s.hout, s.cout, s.mid, 3, 3, 1, 1, s.hout, s.hout};
      check(pbdk::fprop_plan(dg, s.dy2, s.w2flip, s.g1, nullptr, s.a1, PBDK_EPI_RELU_MASK, &s.p_dgrad), "dgrad plan");
      check(pbdk::wgrad_plan(conv2_desc(s, n_), s.a1, s.dy2, g + s.lay.w2, s.wws, s.wws_bytes, &s.p_w2), "wgrad2 plan");
      check(pbdk::wgrad_plan(sc_desc(s, n_), s.in, s.dys, g + s.lay.wsc, s.wws, s.wws_bytes, &s.p_wsc), "wgradsc plan");
      check(pbdk::wgrad_plan(conv1_desc(s, n_), s.in, s.dy1, g + s.lay.w1, s.wws, s.wws_bytes, &s.p_w1), "wgrad1 plan");
    }
  }

  pbdx_desc d_;
  int n_ = 0;
  int first_ = 0;
  bool external_ = false;
  bool timing_ = false;
  bool graph_valid_ = false;
  cudaGraphExec_t graph_exec_ = nullptr;
  cudaGraphExec_t phase_exec_[3] = {nullptr, nullptr, nullptr};
  bool phases_valid_ = false;
  cudaEvent_t fork_ = nullptr;
  cudaStream_t cap_stream_ = nullptr;
  Arena arena_;
  bf16* input_ = nullptr;
  size_t input_bytes_ = 0;
  float* stage_ = nullptr;
  size_t tout_bytes_ = 0;
  bf16* tparams_ = nullptr;
  size_t tparam_bytes_ = 0;
  std::vector<TBlock> tblocks_;
  std::vector<SBlock> sblocks_;
  size_t total_ = 0;
  float *params_ = nullptr, *mom_ = nullptr, *grads_ = nullptr;
  bf16* shadow_ = nullptr;
  double* losses_ = nullptr;
  long long* step_ = nullptr;
  std::vector<cudaEvent_t> tdone_;
  std::vector<cudaEvent_t> ev_t_, ev_s_;
  // K11 relay state: mailbox_ = flags written by peers ([0,16) ready per sender, [16,32) consumed
  // per receiver); relay_seq_ = {receive seq, send seq} (device-side, so graph replays advance them)
  unsigned long long* mailbox_ = nullptr;
  unsigned long long* relay_seq_ = nullptr;
  unsigned int* relay_ticket_ = nullptr;
  std::vector<void*> recv_consumed_;
  std::vector<pbdx_relay_msg> send_;
  cudaStream_t relay_stream_ = nullptr;
  cudaEvent_t relay_fork_ = nullptr, relay_done_ = nullptr;
};

}  // namespace pbd::exec

// ------------------------------------------------------------------ C ABI
namespace {

using pbd::exec::Partition;

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

Partition* P(void* h) { return static_cast<Partition*>(h); }
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int pbdx_create(const pbdx_desc* d, void** handle) {
  if (d == nullptr || handle == nullptr) return PBDK_EINVAL;
  return guard([&] { *handle = new Partition(*d); });
}

void pbdx_destroy(void* handle) { delete P(handle); }

int pbdx_init_params(void* h, void* st) { return guard([&] { P(h)->init_params(S(st)); }); }
int pbdx_set_shard(void* h, int n, int first) { return guard([&] { P(h)->set_shard(n, first); }); }
int pbdx_set_input_mode(void* h, int external) { return guard([&] { P(h)->set_external_input(external != 0); }); }
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

long pbdx_student_layout(int block, long* out) {
  if (block < 0 || block >= pbd::exec::kBlocks || out == nullptr) return -1;
  const auto l = pbd::exec::student_layout(block);
  const size_t v[9] = {l.w1, l.w2, l.wsc, l.g1, l.b1, l.g2, l.b2, l.gsc, l.bsc};
  for (int i = 0; i < 9; ++i) out[i] = static_cast<long>(v[i]);
  return static_cast<long>(l.total);
}

}  // extern "C"
