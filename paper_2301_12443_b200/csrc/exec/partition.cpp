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
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "knobs.hpp"
#include "bd_kernels.hpp"
#include "conv.hpp"
#include "pbdk.h"
#include "partition_base.hpp"
#include "pbdx.h"

namespace pbd::exec {

namespace {

constexpr int kBlocks = 4;
constexpr int T_CH[5] = {3, 64, 128, 256, 512};
constexpr int T_HW[5] = {32, 32, 16, 8, 4};

int stored(int c) { return c == 3 ? 16 : c; }

float kaiming(int fan_in, float gain) { return std::sqrt(6.0f / static_cast<float>(fan_in)) * gain; }

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
  pbdk::FixScratch fx[4];  // self-finalizing reductions: BN1 stats, BN2+BNsc stats, loss, BN1 backward
  pbdk::FpropPlan p_conv1, p_sc, p_conv2, p_dgrad;
  pbdk::WgradPlan p_w2, p_wsc, p_w1;
  // per-block scratch + stream: student blocks only depend on teacher outputs, so each runs
  // on its own stream as soon as its teacher block is done (overlaps teacher k+1 and the
  // other student blocks; the late blocks alone do not fill 148 SMs).
  void* wws = nullptr;
  void* wws2 = nullptr;  // workspace of the side stream's wgrads
  size_t wws_bytes = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  // backward fork: wgrad(conv2) + wgrad(shortcut) on `side` run beside dgrad(conv2) -> BN1 backward ->
  // wgrad(conv1), which is the block's critical chain
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

class ResNetPartition final : public PartitionBase {
 public:
  explicit ResNetPartition(const pbdx_desc& d) : PartitionBase(d) {
    if (d.block_lo < 0 || d.block_hi >= kBlocks || d.block_lo > d.block_hi) throw BadArg("bad block range");
    allocate();
    build_plans();
  }

  int nblocks() const override { return d_.block_hi - d_.block_lo + 1; }
  const void* relay_source() const override { return tblocks_.back().out; }
  size_t relay_row_bytes() const override { return tout_bytes_ / static_cast<size_t>(d_.n_max); }
  void rebuild_for_shard() override { build_plans(); }

  void init_params(cudaStream_t st) override {
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

  void upload_images(const float* host, int n, cudaStream_t st) override {
    if (d_.block_lo != 0) throw BadArg("only partition 0 loads data");
    if (n != n_) throw BadArg("upload size != shard size");
    cuda(cudaMemcpyAsync(stage_, host, static_cast<size_t>(n) * 32 * 32 * 3 * sizeof(float), cudaMemcpyHostToDevice,
                         st),
         "H2D images");
    check(pbdk::pack_image(stage_, input_, n, st), "pack image");
  }

  void stage_images(const float* host, int n, int slot, cudaStream_t st) override {
    if (d_.block_lo == 0 && n == n_ && (slot == 0 || slot == 1)) {
      const size_t bytes = static_cast<size_t>(n) * 32 * 32 * 3 * sizeof(float);
      cuda(cudaMemcpyAsync(slot == 0 ? stage_ : stage2_, host, bytes, cudaMemcpyHostToDevice, st), "H2D stage");
      return;
    }
    throw BadArg("stage_images: partition 0 only, n == shard size, slot 0/1");
  }

  void teacher_body(cudaStream_t st) override {
    if (d_.block_lo == 0 && external_ == 2)
      check(pbdk::pack_image_parity(stage_, stage2_, step_, input_, n_, st), "pack staged image");
    if (d_.block_lo == 0 && !external_)
      check(pbdk::philox_image(input_, n_, first_, step_, d_.global_batch, d_.seed_data, st), "philox");
    for (size_t i = 0; i < tblocks_.size(); ++i) {
      if (timing_) cuda(cudaEventRecord(ev_t_[2 * i], st), "event");
      for (TConv& c : tblocks_[i].convs) check(pbdk::fprop_run(c.plan, st), "teacher conv");
      if (timing_) cuda(cudaEventRecord(ev_t_[2 * i + 1], st), "event");
      cuda(cudaEventRecord(tdone_[i], st), "event");
    }
  }

  // Student block k runs on its own stream.  Fused step(): it starts once teacher block k is
  // done (event recorded by teacher_forward).  Standalone phase (multi-GPU driver, phase
  // graphs): the student streams fork from the caller's stream at entry.  The caller's
  // stream joins all of them before returning.
  void student_body(cudaStream_t caller, bool fork) override {
    // The BN / loss passes leave SMs to the other student streams' convs: one partial CTA per SM (for
    // every block count — the chunking fixes the summation order, so a block's results must not
    // depend on how many blocks the partition holds) and, with >= 3 concurrent streams, two apply
    // CTAs per SM.
    const pbdk::GridScope grids(148, sblocks_.size() >= 3 ? 296 : 0);
    if (fork) cuda(cudaEventRecord(fork_, caller), "event");
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      SBlock& s = sblocks_[i];
      cudaStream_t st = s.stream;
      cuda(cudaStreamWaitEvent(st, fork ? fork_ : tdone_[i], 0), "wait teacher");
      if (timing_) cuda(cudaEventRecord(ev_s_[2 * i], st), "event");
      if (!trains(static_cast<int>(i))) {  // DP-baseline mode: this block only feeds the teacher prefix
        if (timing_) cuda(cudaEventRecord(ev_s_[2 * i + 1], st), "event");
        cuda(cudaEventRecord(s.done, st), "event");
        continue;
      }
      const float* p = params_ + s.base;
      float* g = grads_ + s.base;
      const int m = n_ * s.hout * s.hout;
      check(pbdk::fprop_run(s.p_conv1, st), "conv1");
      check(pbdk::fprop_run(s.p_sc, st), "shortcut");
      check(pbdk::bn_stats_fix(s.y1, nullptr, m, s.mid, s.fx[0], s.st1, nullptr, st), "bn1 stats");
      check(pbdk::bn_apply_relu_fix(s.y1, s.st1, p + s.lay.g1, p + s.lay.b1, s.a1, m, s.mid, st), "bn1 apply");
      check(pbdk::fprop_run(s.p_conv2, st), "conv2");
      check(pbdk::bn_stats_fix(s.y2, s.ys, m, s.cout, s.fx[1], s.st2, s.sts, st), "bn2/bnsc stats");
      const double norm = static_cast<double>(d_.global_batch) * s.cout * s.hout * s.hout;
      pbdk::MseArgs a{s.y2, s.ys, s.target, s.st2, s.sts, p + s.lay.g2, p + s.lay.b2, p + s.lay.gsc, p + s.lay.bsc,
                      m, s.cout, static_cast<float>(2.0 / norm), norm, nullptr, s.red, g + s.lay.g2, g + s.lay.b2,
                      g + s.lay.gsc, g + s.lay.bsc, losses_ + i, s.dy2, s.dys};
      check(pbdk::mse_bn_loss_fix(a, s.fx[2], st), "mse");
      cudaStream_t ws = st;
      if (s.side != nullptr) {
        cuda(cudaEventRecord(s.fork, st), "event");
        cuda(cudaStreamWaitEvent(s.side, s.fork, 0), "fork");
        ws = s.side;
      }
      check(pbdk::wgrad_run(s.p_w2, ws), "wgrad2");
      check(pbdk::wgrad_run(s.p_wsc, ws), "wgrad sc");
      check(pbdk::fprop_run(s.p_dgrad, st), "dgrad2");
      check(pbdk::bn_bwd_fix(s.g1, s.y1, s.st1, p + s.lay.g1, m, s.mid, s.fx[3], s.red1, g + s.lay.g1, g + s.lay.b1,
                             s.dy1, st),
            "bn1 bwd");
      check(pbdk::wgrad_run(s.p_w1, st), "wgrad1");
      if (s.side != nullptr) {
        cuda(cudaEventRecord(s.join, s.side), "event");
        cuda(cudaStreamWaitEvent(st, s.join, 0), "join");
      }
      if (timing_) cuda(cudaEventRecord(ev_s_[2 * i + 1], st), "event");
      cuda(cudaEventRecord(s.done, st), "event");
    }
    for (SBlock& s : sblocks_) cuda(cudaStreamWaitEvent(caller, s.done, 0), "join");
  }

  // bf16 shadows + flipped dgrad weights from the fp32 master weights (after a state migration)
  void refresh_shadows(cudaStream_t st) override {
    check(pbdk::sgd_momentum(params_, mom_, grads_, shadow_, total_, 0.0f, 1.0f, nullptr, st), "shadow");
    refresh_flips(st);
  }

  void update_body(cudaStream_t st) override {
    if (dp_active()) {  // share_gradient + update: reduce-scatter + all-gather over peer memory
      dp_update({{0, total_}}, params_, mom_, grads_, shadow_, step_, st);
      refresh_flips(st);
      return;
    }
    if (all_train() && fused_flips()) {  // one launch: update + shadows + flipped dgrad filters
      pbdk::FlipSet fs;
      for (const SBlock& s : sblocks_) fs.reg[fs.count++] = flip_region(s, s.base);
      check(pbdk::sgd_momentum_flip(params_, mom_, grads_, shadow_, total_, d_.lr, d_.momentum, step_, fs, st),
            "sgd");
      return;
    }
    if (all_train()) {
      check(pbdk::sgd_momentum(params_, mom_, grads_, shadow_, total_, d_.lr, d_.momentum, step_, st), "sgd");
      refresh_flips(st);
      return;
    }
    long long* counter = step_;
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      if (!trains(static_cast<int>(i))) continue;
      const SBlock& s = sblocks_[i];
      pbdk::FlipSet fs;
      fs.reg[fs.count++] = flip_region(s, 0);
      check(pbdk::sgd_momentum_flip(params_ + s.base, mom_ + s.base, grads_ + s.base, shadow_ + s.base,
                                    s.lay.total, d_.lr, d_.momentum, counter, fs, st),
            "sgd");
      counter = nullptr;
    }
  }

  std::vector<DpRegion> dp_all_regions() const override { return {{0, total_}}; }

  void buffer(int which, void** ptr, size_t* bytes) override {
    switch (which) {
      case PBDX_BUF_INPUT: *ptr = input_; *bytes = input_bytes_; break;
      case PBDX_BUF_TEACHER_OUT: *ptr = tblocks_.back().out; *bytes = tout_bytes_; break;
      case PBDX_BUF_GRADS: *ptr = grads_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_PARAMS: *ptr = params_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_MOMENTUM: *ptr = mom_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_LOSSES: *ptr = losses_; *bytes = nblocks() * sizeof(double); break;
      case PBDX_BUF_STEP: *ptr = step_; *bytes = sizeof(long long); break;
      case PBDX_BUF_TEACHER_PARAMS: *ptr = tparams_; *bytes = tparam_bytes_; break;
      case PBDX_BUF_MAILBOX: *ptr = mailbox_; *bytes = kMailboxSlots * sizeof(unsigned long long); break;
      default: throw BadArg("unknown buffer");
    }
  }

  void teacher_act(int k, void** ptr, size_t* bytes) override {
    if (k < d_.block_lo || k > d_.block_hi) throw BadArg("block outside partition");
    *ptr = tblocks_[static_cast<size_t>(k - d_.block_lo)].out;
    *bytes = act_bytes(T_HW[k + 1], T_CH[k + 1]);
  }

  int body_launches_per_step() const override {
    int n = (d_.block_lo == 0 && external_ != 1) ? 1 : 0;  // philox or staged pack
    for (const TBlock& tb : tblocks_) n += static_cast<int>(tb.convs.size());
    int trained = 0;
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      if (!trains(static_cast<int>(i))) continue;
      const SBlock& s = sblocks_[i];
      ++trained;
      n += 3 + 2 + 1 + 2 + 1 + 2;  // convs, bn1 stats+apply, bn2+bnsc stats, mse(2), dgrad, bn_bwd(2)
      n += (s.p_w2.splits > 1 ? 2 : 1) + (s.p_wsc.splits > 1 ? 2 : 1) + (s.p_w1.splits > 1 ? 2 : 1);
    }
    if (dp_active() || (all_train() && !fused_flips()))
      n += all_train() ? 1 + static_cast<int>(sblocks_.size()) : 2 * trained;  // sgd + flips
    else
      n += all_train() ? 1 : trained;  // sgd with the flips fused (sgd_momentum_flip)
    return n;
  }

  static bool student_fork() {
    static const bool on = [] {
      const char* e = pbd::knob_env("PBD_STUDENT_FORK");
      return e == nullptr || e[0] != '0';
    }();
    return on;
  }

  ~ResNetPartition() override {
    for (SBlock& s : sblocks_) {
      if (s.stream != nullptr) cudaStreamDestroy(s.stream);
      if (s.done != nullptr) cudaEventDestroy(s.done);
      if (s.side != nullptr) cudaStreamDestroy(s.side);
      if (s.fork != nullptr) cudaEventDestroy(s.fork);
      if (s.join != nullptr) cudaEventDestroy(s.join);
    }
    for (auto e : tdone_) cudaEventDestroy(e);
    if (fork_ != nullptr) cudaEventDestroy(fork_);
  }

 private:
  bool fused_flips() const { return sblocks_.size() <= static_cast<size_t>(pbdk::FlipSet::kMax); }

  // conv2's filter [cout][3][3][mid] at offset base + lay.w2 of the updated vector -> w2flip
  static pbdk::FlipRegion flip_region(const SBlock& s, size_t base) {
    return pbdk::FlipRegion{base + s.lay.w2, s.cout, 3, 3, s.mid, s.w2flip};
  }

  void refresh_flips(cudaStream_t st) {
    for (SBlock& s : sblocks_)
      check(pbdk_weight_flip(shadow_ + s.base + s.lay.w2, s.w2flip, s.cout, 3, 3, s.mid, st), "flip");
  }

  size_t act_bytes(int hw, int c) const { return static_cast<size_t>(d_.n_max) * hw * hw * c * sizeof(bf16); }

  void allocate() {
    const int lo = d_.block_lo, hi = d_.block_hi;
    input_bytes_ = act_bytes(T_HW[lo], stored(T_CH[lo]));
    input_ = arena_.get<bf16>(input_bytes_);
    if (lo == 0) {
      stage_ = arena_.get<float>(static_cast<size_t>(d_.n_max) * 32 * 32 * 3 * sizeof(float));
      stage2_ = arena_.get<float>(static_cast<size_t>(d_.n_max) * 32 * 32 * 3 * sizeof(float));
    }

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
      {  // zero-initialised once; each reduction's last CTA re-zeroes its scratch
        const size_t words = pbdk::fix_acc_words(s.cout);
        auto* acc = arena_.get<unsigned long long>(4 * words * sizeof(unsigned long long));
        auto* tickets = arena_.get<unsigned int>(4 * sizeof(unsigned int));
        cuda(cudaMemset(acc, 0, 4 * words * sizeof(unsigned long long)), "memset");
        cuda(cudaMemset(tickets, 0, 4 * sizeof(unsigned int)), "memset");
        for (int j = 0; j < 4; ++j) s.fx[j] = pbdk::FixScratch{acc + j * words, tickets + j};
      }
      sblocks_.push_back(s);
    }
    // master weights and momentum in ONE allocation (momentum at +total_): a DP peer reaches both
    // through the one IPC mapping of PBDX_BUF_PARAMS (PartitionBase::dp_sync_state)
    params_ = arena_.get<float>(2 * total_ * sizeof(float));
    mom_ = params_ + total_;
    grads_ = arena_.get<float>(total_ * sizeof(float));
    shadow_ = arena_.get<bf16>(total_ * sizeof(bf16));
    losses_ = arena_.get<double>(kBlocks * sizeof(double));
    step_ = arena_.get<long long>(sizeof(long long));
    allocate_relay();

    // ---- per-block scratch sized for n_max, streams and events
    for (SBlock& s : sblocks_) {
      size_t wws = 0;
      for (const pbdk_conv_desc& cd : {conv1_desc(s, d_.n_max), sc_desc(s, d_.n_max), conv2_desc(s, d_.n_max)})
        wws = std::max(wws, pbdk::wgrad_workspace_bytes(cd));
      s.wws_bytes = wws;
      s.wws = arena_.get<void>(wws);
      const bool last = s.k == d_.block_hi;
      // Three levels: the teacher (capture stream) and the last block's student chain highest, the other
      // student chains in the middle, the side streams (wgrads off the critical chain) lowest.
      // Measured 0.907 -> 0.895 ms vs two levels (PBD_PRIO_MODE=0: side streams share their block's).
      static const int prio_mode = [] {
        const char* e = pbd::knob_env("PBD_PRIO_MODE");
        return e != nullptr ? std::atoi(e) : 2;
      }();
      const int hi = priority_high(), lo = priority_low();
      const int mid = (hi + lo) / 2;
      const int p_main = last ? hi : (prio_mode == 2 ? mid : lo);
      const int p_side = prio_mode == 2 ? lo : p_main;
      cuda(cudaStreamCreateWithPriority(&s.stream, cudaStreamNonBlocking, p_main), "stream");
      cuda(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming), "event");
      if (student_fork()) {
        s.wws2 = arena_.get<void>(wws);
        cuda(cudaStreamCreateWithPriority(&s.side, cudaStreamNonBlocking, p_side), "stream");
        cuda(cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming), "event");
        cuda(cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming), "event");
      }
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

  static int env_ctas(const char* name) {
    const char* e = pbd::knob_env(name);
    return e != nullptr ? std::atoi(e) : 0;
  }
  // PBDK_TCONV_CTAS_LIST / PBDK_SCONV_CTAS_LIST = "a,b,c,d": per-block grid caps (experiments)
  static int env_list(const char* name, size_t i, int dflt) {
    const char* e = pbd::knob_env(name);
    if (e == nullptr) return dflt;
    std::string v(e);
    size_t pos = 0;
    for (size_t k = 0; k < i; ++k) {
      pos = v.find(',', pos);
      if (pos == std::string::npos) return dflt;
      ++pos;
    }
    return std::atoi(v.c_str() + pos);
  }

  void build_plans() {
    // Every ResNet conv (teacher and student) gets two epilogue warps per TMEM lane quarter whatever
    // its K — slightly slower alone (64->64 @32x32: 26.7 -> 27.1 us) but the step, where the convs
    // share SMs, gains 0.892 -> 0.886 ms (teacher-only or student-only: no gain).  PBDK_EPW=1
    // disables it everywhere.
    for (size_t i = 0; i < tblocks_.size(); ++i) {
      const pbdk::ConvGridScope scope(env_list("PBDK_TCONV_CTAS_LIST", i, env_ctas("PBDK_TCONV_CTAS")), 2);
      for (TConv& c : tblocks_[i].convs) {
        const pbdk_conv_desc cd{n_, c.hin, c.hin, c.cs, c.cout, c.r, c.r, c.stride, c.pad, c.hout, c.hout};
        check(pbdk::fprop_plan(cd, c.in, c.w, c.out, c.bias, c.aux, c.epi, &c.plan), "teacher plan");
      }
    }
    // With >= 3 student blocks their streams run concurrently: each student conv spreads over at most
    // 64 SMs so the streams share the GPU spatially instead of queueing behind each other's full-GPU
    // persistent grids (measured, 4 blocks at b=256: 0.934 -> 0.907 ms per step; capping the teacher
    // convs, which run mostly alone, costs time).  PBDK_SCONV_CTAS overrides (0 = all SMs).
    const int sconv = pbd::knob_env("PBDK_SCONV_CTAS") != nullptr ? env_ctas("PBDK_SCONV_CTAS")
                                                                : (sblocks_.size() >= 3 ? 64 : 0);
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      SBlock& s = sblocks_[i];
      const pbdk::ConvGridScope scope(env_list("PBDK_SCONV_CTAS_LIST", i, sconv), 2);
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
      void* ws2 = s.wws2 != nullptr ? s.wws2 : s.wws;
      check(pbdk::wgrad_plan(conv2_desc(s, n_), s.a1, s.dy2, g + s.lay.w2, ws2, s.wws_bytes, &s.p_w2), "wgrad2 plan");
      check(pbdk::wgrad_plan(sc_desc(s, n_), s.in, s.dys, g + s.lay.wsc, ws2, s.wws_bytes, &s.p_wsc), "wgradsc plan");
      check(pbdk::wgrad_plan(conv1_desc(s, n_), s.in, s.dy1, g + s.lay.w1, s.wws, s.wws_bytes, &s.p_w1), "wgrad1 plan");
    }
    // programmatic dependent launch for every conv: its prologue overlaps the previous kernel's tail
    if (pbd::pdl_enabled()) {
      for (TBlock& tb : tblocks_)
        for (TConv& c : tb.convs) c.plan.pdl = true;
      for (SBlock& s : sblocks_) {
        for (pbdk::FpropPlan* f : {&s.p_conv1, &s.p_sc, &s.p_conv2, &s.p_dgrad}) f->pdl = true;
        for (pbdk::WgradPlan* w : {&s.p_w2, &s.p_wsc, &s.p_w1}) w->pdl = true;
      }
    }
  }

  cudaEvent_t fork_ = nullptr;
  bf16* input_ = nullptr;
  size_t input_bytes_ = 0;
  float* stage_ = nullptr;
  float* stage2_ = nullptr;  // second staging slot (input mode 2)
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
};

}  // namespace

PartitionBase* make_resnet_partition(const pbdx_desc& d) { return new ResNetPartition(d); }

}  // namespace pbd::exec

// ------------------------------------------------------------------ C ABI (ResNet layout query)
extern "C" long pbdx_student_layout(int block, long* out) {
  if (block < 0 || block >= pbd::exec::kBlocks || out == nullptr) return -1;
  const auto l = pbd::exec::student_layout(block);
  const size_t v[9] = {l.w1, l.w2, l.wsc, l.g1, l.b1, l.g2, l.b2, l.gsc, l.bsc};
  for (int i = 0; i < 9; ++i) out[i] = static_cast<long>(v[i]);
  return static_cast<long>(l.total);
}
