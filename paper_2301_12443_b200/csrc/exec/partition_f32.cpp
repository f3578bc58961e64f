// Per-GPU partition executor of the fp32 CIFAR workload (BASELINE configs[0]: the reference's
// smallest case, 4-block teacher / student, batch 64, fp32): the device body of Algorithm 1
// with the same model as partition.cpp and fp32 numerics — the
// oracle's bf16_mode = 0 (oracle/bd_oracle.c).
//
// Every convolution runs on the tensor cores as 3xTF32 (conv_tf32.hpp): operands that feed a
// convolution are stored split, [rows][hi(c) | lo(c)] with hi + lo == the fp32 value; outputs that only
// feed elementwise kernels stay plain fp32.  Per tensor:
//   split : image (32 stored channels, 3 real), teacher activations (conv outputs, relay payload,
//           distillation targets), a1 = relu(BN1(y1)), dy2 / dysc / dy1 (backward operands), the
//           conv weights shadows and the flipped dgrad weights (refreshed from the fp32 masters by
//           the update)
//   plain : y1, y2, ysc, g1 (BN inputs / masks), fp32 master weights, momentum, gradients
// Elementwise kernels are the bf16 workload's with fp32 / split row I/O (bd_kernels.cu IoF32 /
// IoSplit): the same operand order and fixed-order reductions.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "bd_kernels.hpp"
#include "conv_tf32.hpp"
#include "partition_base.hpp"
#include "pbdk.h"
#include "pbdx.h"

namespace pbd::exec {

namespace {

constexpr int kBlocks = 4;
constexpr int T_CH[5] = {3, 64, 128, 256, 512};
constexpr int T_HW[5] = {32, 32, 16, 8, 4};
constexpr int kImageC = 32;  // stored image channels per half (MN-major tf32 operands come in 32-channel atoms)

int stored(int c) { return c == 3 ? kImageC : c; }
float kaiming(int fan_in, float gain) { return std::sqrt(6.0f / static_cast<float>(fan_in)) * gain; }

struct SLayout {
  size_t w1, w2, wsc, g1, b1, g2, b2, gsc, bsc, total;
};

SLayout layout_f32(int k) {
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

struct TConv {
  int cin, cs, cout, r, stride, pad, hin, hout;
  float gain;
  uint32_t tensor;
  int epi;
  float* w = nullptr;  // split [cout][r][r][2cs]
  float* bias = nullptr;
  const float* in = nullptr;
  float* out = nullptr;  // split [m][2cout]
  const float* aux = nullptr;
  pbdk::F3FpropPlan plan;
};

struct SBlock {
  int k, cin, cs, cout, mid, stride, hin, hout;
  SLayout lay;
  size_t base = 0;
  const float* in = nullptr;      // split
  const float* target = nullptr;  // split
  float *w1s, *w2s, *wscs, *w2flip;  // split weight shadows
  float *y1, *a1, *y2, *ys, *dy2, *dys, *g1, *dy1;
  float *st1, *st2, *sts, *red, *red1, *rws;
  void* wws = nullptr;
  size_t wws_bytes = 0;
  pbdk::F3FpropPlan p_conv1, p_sc, p_conv2, p_dgrad;
  pbdk::F3WgradPlan p_w1, p_wsc, p_w2;
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
};

class ResNetF32Partition final : public PartitionBase {
 public:
  explicit ResNetF32Partition(const pbdx_desc& d) : PartitionBase(d) {
    if (d.block_lo < 0 || d.block_hi >= kBlocks || d.block_lo > d.block_hi) throw BadArg("bad block range");
    allocate();
    build_plans();
  }

  ~ResNetF32Partition() override {
    for (SBlock& s : sblocks_) {
      if (s.stream != nullptr) cudaStreamDestroy(s.stream);
      if (s.done != nullptr) cudaEventDestroy(s.done);
    }
    for (auto e : tdone_) cudaEventDestroy(e);
    if (fork_ != nullptr) cudaEventDestroy(fork_);
  }

  int nblocks() const override { return d_.block_hi - d_.block_lo + 1; }
  const void* relay_source() const override { return tout_; }
  size_t relay_row_bytes() const override { return tout_bytes_ / static_cast<size_t>(d_.n_max); }
  void rebuild_for_shard() override { build_plans(); }

  void init_params(cudaStream_t st) override {
    for (TConv& c : tconvs_) {
      check(pbdk::init_uniform(c.w, 2, c.cout, c.r, c.r, c.cs, c.cin, d_.seed_teacher, c.tensor,
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
      for (size_t o : {s.lay.g1, s.lay.g2, s.lay.gsc}) check(pbdk::fill(p + o, o == s.lay.g1 ? s.mid : s.cout, 1.0f, st), "fill");
      for (size_t o : {s.lay.b1, s.lay.b2, s.lay.bsc}) check(pbdk::fill(p + o, o == s.lay.b1 ? s.mid : s.cout, 0.0f, st), "fill");
    }
    check(pbdk::fill(mom_, total_, 0.0f, st), "fill");
    check(pbdk::fill(grads_, total_, 0.0f, st), "fill");
    refresh_shadows(st);
    cuda(cudaMemsetAsync(step_, 0, sizeof(long long), st), "memset");
  }

  void upload_images(const float* host, int n, cudaStream_t st) override {
    if (d_.block_lo != 0) throw BadArg("only partition 0 loads data");
    if (n != n_) throw BadArg("upload size != shard size");
    cuda(cudaMemcpyAsync(stage_, host, static_cast<size_t>(n) * 32 * 32 * 3 * sizeof(float), cudaMemcpyHostToDevice,
                         st),
         "H2D images");
    check(pbdk::pack_image(stage_, input_, n, st, 32, 1), "pack image");
  }

  void stage_images(const float* host, int n, int slot, cudaStream_t st) override {
    if (d_.block_lo == 0 && n == n_ && (slot == 0 || slot == 1)) {
      cuda(cudaMemcpyAsync(slot == 0 ? stage_ : stage2_, host, static_cast<size_t>(n) * 32 * 32 * 3 * sizeof(float),
                           cudaMemcpyHostToDevice, st),
           "H2D stage");
      return;
    }
    throw BadArg("stage_images: partition 0 only, n == shard size, slot 0/1");
  }

  void teacher_body(cudaStream_t st) override {
    if (d_.block_lo == 0 && external_ == 2)
      check(pbdk::pack_image_parity(stage_, stage2_, step_, input_, n_, st, 32, 1), "pack staged image");
    if (d_.block_lo == 0 && !external_)
      check(pbdk::philox_image(input_, n_, first_, step_, d_.global_batch, d_.seed_data, st, 32, 1), "philox");
    for (size_t i = 0; i < tblock_convs_.size(); ++i) {
      if (timing_) cuda(cudaEventRecord(ev_t_[2 * i], st), "event");
      for (size_t j = tblock_convs_[i].first; j < tblock_convs_[i].second; ++j)
        check(pbdk::f3_fprop_run(tconvs_[j].plan, st), "teacher conv");
      if (timing_) cuda(cudaEventRecord(ev_t_[2 * i + 1], st), "event");
      cuda(cudaEventRecord(tdone_[i], st), "event");
    }
  }

  void student_body(cudaStream_t caller, bool fork) override {
    if (fork) cuda(cudaEventRecord(fork_, caller), "event");
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      SBlock& s = sblocks_[i];
      cudaStream_t st = s.stream;
      cuda(cudaStreamWaitEvent(st, fork ? fork_ : tdone_[i], 0), "wait teacher");
      if (timing_) cuda(cudaEventRecord(ev_s_[2 * i], st), "event");
      if (trains(static_cast<int>(i))) {
        const float* p = params_ + s.base;
        float* g = grads_ + s.base;
        const int m = n_ * s.hout * s.hout;
        check(pbdk::f3_fprop_run(s.p_conv1, st), "conv1");
        check(pbdk::f3_fprop_run(s.p_sc, st), "shortcut");
        check(pbdk::bn_stats(s.y1, m, s.mid, s.rws, s.st1, st, 1), "bn1 stats");
        check(pbdk::bn_apply_relu(s.y1, s.st1, p + s.lay.g1, p + s.lay.b1, s.a1, m, s.mid, st, 1), "bn1 apply");
        check(pbdk::f3_fprop_run(s.p_conv2, st), "conv2");
        check(pbdk::bn_stats2(s.y2, s.ys, m, s.cout, s.rws, s.st2, s.sts, st, 1), "bn2/bnsc stats");
        const double norm = static_cast<double>(d_.global_batch) * s.cout * s.hout * s.hout;
        pbdk::MseArgs a{s.y2, s.ys, s.target, s.st2, s.sts, p + s.lay.g2, p + s.lay.b2, p + s.lay.gsc,
                        p + s.lay.bsc, m, s.cout, static_cast<float>(2.0 / norm), norm, s.rws, s.red,
                        g + s.lay.g2, g + s.lay.b2, g + s.lay.gsc, g + s.lay.bsc, losses_ + i, s.dy2, s.dys, 1};
        check(pbdk::mse_bn_loss(a, st), "mse");
        check(pbdk::f3_wgrad_run(s.p_w2, st), "wgrad2");
        check(pbdk::f3_wgrad_run(s.p_wsc, st), "wgrad sc");
        check(pbdk::f3_fprop_run(s.p_dgrad, st), "dgrad2");
        check(pbdk::bn_bwd(s.g1, s.y1, s.st1, p + s.lay.g1, m, s.mid, s.rws, s.red1, g + s.lay.g1, g + s.lay.b1, s.dy1,
                           st, 1),
              "bn1 bwd");
        check(pbdk::f3_wgrad_run(s.p_w1, st), "wgrad1");
      }
      if (timing_) cuda(cudaEventRecord(ev_s_[2 * i + 1], st), "event");
      cuda(cudaEventRecord(s.done, st), "event");
    }
    for (SBlock& s : sblocks_) cuda(cudaStreamWaitEvent(caller, s.done, 0), "join");
  }

  // split weight shadows and flipped dgrad weights from the fp32 masters
  void refresh_shadows(cudaStream_t st) override {
    for (SBlock& s : sblocks_) refresh_block(s, st);
  }

  void update_body(cudaStream_t st) override {
    if (dp_active()) {  // reduce-scatter + all-gather over peer memory (PartitionBase::dp_update)
      dp_update({{0, total_}}, params_, mom_, grads_, nullptr, step_, st);
    } else if (all_train()) {
      check(pbdk::sgd_momentum(params_, mom_, grads_, nullptr, total_, d_.lr, d_.momentum, step_, st), "sgd");
    } else {
      long long* counter = step_;
      for (size_t i = 0; i < sblocks_.size(); ++i) {
        if (!trains(static_cast<int>(i))) continue;
        const SBlock& s = sblocks_[i];
        check(pbdk::sgd_momentum(params_ + s.base, mom_ + s.base, grads_ + s.base, nullptr, s.lay.total, d_.lr,
                                 d_.momentum, counter, st),
              "sgd");
        counter = nullptr;
      }
    }
    for (size_t i = 0; i < sblocks_.size(); ++i)
      if (trains(static_cast<int>(i))) refresh_block(sblocks_[i], st);
  }

  std::vector<DpRegion> dp_all_regions() const override { return {{0, total_}}; }

  void buffer(int which, void** ptr, size_t* bytes) override {
    switch (which) {
      case PBDX_BUF_INPUT: *ptr = input_; *bytes = input_bytes_; break;
      case PBDX_BUF_TEACHER_OUT: *ptr = tout_; *bytes = tout_bytes_; break;
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
    *ptr = tact_[static_cast<size_t>(k - d_.block_lo)];
    *bytes = act_bytes(T_HW[k + 1], T_CH[k + 1]);
  }

  int body_launches_per_step() const override {
    int n = (d_.block_lo == 0 && external_ != 1) ? 1 : 0;
    n += static_cast<int>(tconvs_.size());
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      if (!trains(static_cast<int>(i))) continue;
      const SBlock& s = sblocks_[i];
      n += 4 + 2 + 2 + 3 + 3;  // convs (3 + dgrad), bn1 stats + apply, bn2 stats, mse, bn bwd
      n += (s.p_w2.splits > 1 ? 2 : 1) + (s.p_wsc.splits > 1 ? 2 : 1) + (s.p_w1.splits > 1 ? 2 : 1);
      n += 4;  // shadow split x3 + flip
    }
    return n + (all_train() || dp_active() ? 1 : 0) + (all_train() || dp_active() ? 0 : nblocks());
  }

 private:
  size_t act_bytes(int hw, int c) const { return static_cast<size_t>(d_.n_max) * hw * hw * c * sizeof(float); }

  void refresh_block(SBlock& s, cudaStream_t st) {
    const float* p = params_ + s.base;
    check(pbdk::f3_split(p + s.lay.w1, s.w1s, static_cast<size_t>(s.mid) * 9, s.cs, st), "split w1");
    check(pbdk::f3_split(p + s.lay.w2, s.w2s, static_cast<size_t>(s.cout) * 9, s.mid, st), "split w2");
    check(pbdk::f3_split(p + s.lay.wsc, s.wscs, static_cast<size_t>(s.cout), s.cs, st), "split wsc");
    check(pbdk::f3_flip_split(p + s.lay.w2, s.w2flip, s.cout, 3, 3, s.mid, st), "flip w2");
  }

  void allocate() {
    const int lo = d_.block_lo, hi = d_.block_hi;
    input_bytes_ = act_bytes(T_HW[lo], 2 * stored(T_CH[lo]));
    input_ = arena_.get<float>(input_bytes_);
    if (lo == 0) {
      stage_ = arena_.get<float>(static_cast<size_t>(d_.n_max) * 32 * 32 * 3 * sizeof(float));
      stage2_ = arena_.get<float>(static_cast<size_t>(d_.n_max) * 32 * 32 * 3 * sizeof(float));
    }
    // ---- teacher program (same chain as partition.cpp; Philox tensor ids = 1000*block + 10*j)
    for (int k = lo; k <= hi; ++k) {
      const size_t first = tconvs_.size();
      int j = 0;
      int cin = T_CH[k], hw = T_HW[k];
      auto add = [&](int ci, int co, int r, int stv, int pad, int h, int ho, float gain, int epi, int tid) {
        TConv c{};
        c.cin = ci;
        c.cs = stored(ci);
        c.cout = co;
        c.r = r;
        c.stride = stv;
        c.pad = pad;
        c.hin = h;
        c.hout = ho;
        c.gain = gain;
        c.tensor = static_cast<uint32_t>(1000 * k + 10 * tid);
        c.epi = epi;
        tconvs_.push_back(c);
      };
      if (k == 0) {
        add(3, 64, 3, 1, 1, 32, 32, 1.0f, PBDK_EPI_BIAS_RELU, j++);
        cin = 64;
      }
      const int cout = T_CH[k + 1];
      const int s = T_HW[k] / T_HW[k + 1];
      for (int b = 0; b < 2; ++b) {
        const int stv = b == 0 ? s : 1;
        const int ci = b == 0 ? cin : cout;
        const int ohw = hw / stv;
        add(ci, cout, 3, stv, 1, hw, ohw, 1.0f, PBDK_EPI_BIAS_RELU, j);
        const bool proj = stv != 1 || ci != cout;
        if (proj) add(ci, cout, 1, stv, 0, hw, ohw, 1.0f, PBDK_EPI_BIAS, j + 2);
        add(cout, cout, 3, 1, 1, ohw, ohw, 0.5f, PBDK_EPI_BIAS_RES_RELU, j + 1);
        j += proj ? 3 : 2;
        hw = ohw;
      }
      tblock_convs_.emplace_back(first, tconvs_.size());
    }
    // execution order per BasicBlock: conv1, projection, conv2
    size_t tw = 0;
    for (const TConv& c : tconvs_) tw += static_cast<size_t>(c.cout) * c.r * c.r * 2 * c.cs;
    tparam_bytes_ = tw * sizeof(float);
    tparams_ = arena_.get<float>(tparam_bytes_);
    float* wp = tparams_;
    const float* x = input_;
    for (size_t b = 0; b < tblock_convs_.size(); ++b) {
      const float* block_in = x;
      const float* sc = nullptr;
      for (size_t j = tblock_convs_[b].first; j < tblock_convs_[b].second; ++j) {
        TConv& c = tconvs_[j];
        c.w = wp;
        wp += static_cast<size_t>(c.cout) * c.r * c.r * 2 * c.cs;
        c.bias = arena_.get<float>(static_cast<size_t>(c.cout) * sizeof(float));
        c.out = arena_.get<float>(act_bytes(c.hout, 2 * c.cout));
        if (c.epi == PBDK_EPI_BIAS) {  // projection shortcut of the BasicBlock input
          c.in = block_in;
          sc = c.out;
        } else if (c.epi == PBDK_EPI_BIAS_RES_RELU) {  // conv2: + projection or the block input
          c.in = x;
          c.aux = sc != nullptr ? sc : block_in;
          x = c.out;
          block_in = c.out;
          sc = nullptr;
        } else {  // stem / conv1
          c.in = x;
          x = c.out;
          if (c.cin == 3) block_in = c.out;
        }
      }
      tact_.push_back(const_cast<float*>(x));
    }
    tout_ = tact_.back();
    tout_bytes_ = act_bytes(T_HW[hi + 1], 2 * T_CH[hi + 1]);

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
      s.lay = layout_f32(k);
      s.base = total_;
      total_ += s.lay.total;
      s.in = (k == lo) ? input_ : tact_[static_cast<size_t>(k - lo - 1)];
      s.target = tact_[static_cast<size_t>(k - lo)];
      s.w1s = arena_.get<float>(static_cast<size_t>(s.mid) * 9 * 2 * s.cs * sizeof(float));
      s.w2s = arena_.get<float>(static_cast<size_t>(s.cout) * 9 * 2 * s.mid * sizeof(float));
      s.wscs = arena_.get<float>(static_cast<size_t>(s.cout) * 2 * s.cs * sizeof(float));
      s.w2flip = arena_.get<float>(static_cast<size_t>(s.mid) * 9 * 2 * s.cout * sizeof(float));
      s.y1 = arena_.get<float>(act_bytes(s.hout, s.mid));
      s.a1 = arena_.get<float>(act_bytes(s.hout, 2 * s.mid));
      s.g1 = arena_.get<float>(act_bytes(s.hout, s.mid));
      s.dy1 = arena_.get<float>(act_bytes(s.hout, 2 * s.mid));
      s.y2 = arena_.get<float>(act_bytes(s.hout, s.cout));
      s.ys = arena_.get<float>(act_bytes(s.hout, s.cout));
      s.dy2 = arena_.get<float>(act_bytes(s.hout, 2 * s.cout));
      s.dys = arena_.get<float>(act_bytes(s.hout, 2 * s.cout));
      s.st1 = arena_.get<float>(2 * s.mid * sizeof(float));
      s.red1 = arena_.get<float>(2 * s.mid * sizeof(float));
      s.st2 = arena_.get<float>(2 * s.cout * sizeof(float));
      s.sts = arena_.get<float>(2 * s.cout * sizeof(float));
      s.red = arena_.get<float>(4 * s.cout * sizeof(float));
      const int m = d_.n_max * s.hout * s.hout;
      s.rws = arena_.get<float>(std::max(pbdk::reduce_workspace_floats(m, s.cout, 3),
                                         pbdk::reduce_workspace_floats(m, s.mid, 3)) *
                                sizeof(float));
      size_t wws = 0;
      for (const pbdk_conv_desc& cd : {conv1_desc(s, d_.n_max), sc_desc(s, d_.n_max), conv2_desc(s, d_.n_max)})
        wws = std::max(wws, pbdk::f3_wgrad_workspace_bytes(cd));
      s.wws_bytes = wws;
      s.wws = arena_.get<void>(wws);
      cuda(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "stream");
      cuda(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming), "event");
      sblocks_.push_back(s);
    }
    // master weights and momentum in ONE allocation (momentum at +total_): a DP peer reaches both
    // through the one IPC mapping of PBDX_BUF_PARAMS (PartitionBase::dp_sync_state)
    params_ = arena_.get<float>(2 * total_ * sizeof(float));
    mom_ = params_ + total_;
    grads_ = arena_.get<float>(total_ * sizeof(float));
    losses_ = arena_.get<double>(kBlocks * sizeof(double));
    step_ = arena_.get<long long>(sizeof(long long));
    allocate_relay();
    tdone_.resize(tblock_convs_.size());
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
    for (TConv& c : tconvs_) {
      const pbdk_conv_desc cd{n_, c.hin, c.hin, c.cs, c.cout, c.r, c.r, c.stride, c.pad, c.hout, c.hout};
      check(pbdk::f3_fprop_plan(cd, c.in, c.w, c.out, 1, c.bias, c.aux, c.epi, &c.plan), "teacher plan");
    }
    for (SBlock& s : sblocks_) {
      float* g = grads_ + s.base;
      check(pbdk::f3_fprop_plan(conv1_desc(s, n_), s.in, s.w1s, s.y1, 0, nullptr, nullptr, PBDK_EPI_STORE, &s.p_conv1),
            "conv1 plan");
      check(pbdk::f3_fprop_plan(sc_desc(s, n_), s.in, s.wscs, s.ys, 0, nullptr, nullptr, PBDK_EPI_STORE, &s.p_sc),
            "sc plan");
      check(pbdk::f3_fprop_plan(conv2_desc(s, n_), s.a1, s.w2s, s.y2, 0, nullptr, nullptr, PBDK_EPI_STORE, &s.p_conv2),
            "conv2 plan");
      const pbdk_conv_desc dg{n_, s.hout, s.hout, s.cout, s.mid, 3, 3, 1, 1, s.hout, s.hout};
      check(pbdk::f3_fprop_plan(dg, s.dy2, s.w2flip, s.g1, 0, nullptr, s.a1, PBDK_EPI_RELU_MASK, &s.p_dgrad),
            "dgrad plan");
      check(pbdk::f3_wgrad_plan(conv2_desc(s, n_), s.a1, s.dy2, g + s.lay.w2, s.wws, s.wws_bytes, &s.p_w2),
            "wgrad2 plan");
      check(pbdk::f3_wgrad_plan(sc_desc(s, n_), s.in, s.dys, g + s.lay.wsc, s.wws, s.wws_bytes, &s.p_wsc),
            "wgradsc plan");
      check(pbdk::f3_wgrad_plan(conv1_desc(s, n_), s.in, s.dy1, g + s.lay.w1, s.wws, s.wws_bytes, &s.p_w1),
            "wgrad1 plan");
    }
  }

  cudaEvent_t fork_ = nullptr;
  float* input_ = nullptr;
  size_t input_bytes_ = 0;
  float* stage_ = nullptr;
  float* stage2_ = nullptr;
  float* tout_ = nullptr;
  size_t tout_bytes_ = 0;
  float* tparams_ = nullptr;
  size_t tparam_bytes_ = 0;
  std::vector<TConv> tconvs_;
  std::vector<std::pair<size_t, size_t>> tblock_convs_;  // [first, last) conv of each teacher block
  std::vector<float*> tact_;                             // teacher output of each block (split)
  std::vector<SBlock> sblocks_;
  size_t total_ = 0;
  float *params_ = nullptr, *mom_ = nullptr, *grads_ = nullptr;
  double* losses_ = nullptr;
  long long* step_ = nullptr;
  std::vector<cudaEvent_t> tdone_;
};

}  // namespace

PartitionBase* make_resnet_f32_partition(const pbdx_desc& d) { return new ResNetF32Partition(d); }

}  // namespace pbd::exec

extern "C" long pbdx_student_layout_fp32(int block, long* out) {
  if (block < 0 || block >= pbd::exec::kBlocks || out == nullptr) return -1;
  const auto l = pbd::exec::layout_f32(block);
  const size_t v[9] = {l.w1, l.w2, l.wsc, l.g1, l.b1, l.g2, l.b2, l.gsc, l.bsc};
  for (int i = 0; i < 9; ++i) out[i] = static_cast<long>(v[i]);
  return static_cast<long>(l.total);
}
