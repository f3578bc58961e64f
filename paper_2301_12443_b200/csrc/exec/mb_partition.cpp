// Per-GPU partition executor of the MobileNetV2 -> ProxylessNAS workload (BASELINE.json configs[2],
// DESIGN.md §10): the device body of Algorithm 1 for a contiguous range of the
// 6-block chain, teacher = MobileNetV2 (BN folded, frozen), student = single-path supernet whose
// searchable MBConv layers hold the candidates {k3,k5,k7} x {e3,e6}.
//
//   teacher_body : [Philox image] -> per block: [stem], per MBConv: expand 1x1 (+bias+ReLU6 epilogue),
//                  depthwise k x k (+bias+ReLU6), project 1x1 (+bias [+residual] epilogue)
//   student_body : per block on its own stream, the active path: forward with training-mode BN,
//                  MSE on the block output, backward (BN backward, 1x1 dgrad with ReLU6-mask / residual
//                  epilogues on tcgen05, depthwise dgrad/wgrad on CUDA cores, 1x1 wgrad on tcgen05)
//   update_body  : fused SGD-momentum over the active candidates only, then their bf16 shadows,
//                  transposed 1x1 weights (dgrad operands) and flipped depthwise weights.
// The 1x1 convolutions run on the tcgen05 implicit-GEMM engine as plain GEMMs: rows = pixels,
// described as ceil(m/128) "images" of 128 x 1 pixels, so activation buffers hold m rounded up to
// 128 rows; padded rows are zero wherever a row reduction could see them.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "knobs.hpp"
#include "bd_kernels.hpp"
#include "conv.hpp"
#include "mb_kernels.hpp"
#include "partition_base.hpp"
#include "pbdk.h"
#include "pbdx.h"

namespace pbd::exec {

namespace {

using bf16 = __nv_bfloat16;

constexpr int kBlocks = 6;
constexpr int kCands = 6;
constexpr int DIV[7] = {1, 4, 8, 16, 16, 32, 32};

// Teacher families: MobileNetV2 (ReLU6; configs[2]) and EfficientNet-B0 (swish,
// squeeze-excite, k5 stages; configs[3]); the student is the same ProxylessNAS supernet over the
// family's block / layer structure.  Channels are stored rounded up to the tensor-tile granularity
// (CH); the architecture's true widths (CT) are the only non-zero ones — the extra stored channels
// have zero weights and receive zero gradients, so the network computed is the true-width one.
struct Family {
  int CH[7];
  int CT[7];
  int NL[6];
  int K[6];
  int act;  // teacher activation code (mb_kernels.hpp): 1 ReLU6, 2 swish
  bool se;  // squeeze-excite in every teacher MBConv
};
constexpr Family kMbv2{{3, 32, 32, 64, 128, 192, 320}, {3, 24, 32, 64, 96, 160, 320}, {3, 3, 4, 3, 3, 1},
                      {3, 3, 3, 3, 3, 3}, 1, false};
constexpr Family kEffb0{{3, 32, 64, 128, 128, 192, 320}, {3, 24, 40, 80, 112, 192, 320}, {3, 2, 3, 3, 4, 1},
                       {3, 5, 3, 5, 5, 3}, 2, true};
const Family& family(int model) { return model == PBDX_MODEL_EFFB0_PROXYLESS ? kEffb0 : kMbv2; }

// the family in effect for the layout helpers below (set by every public entry point)
thread_local const Family* g_fam = &kMbv2;
struct FamScope {
  const Family* prev;
  explicit FamScope(const Family& f) : prev(g_fam) { g_fam = &f; }
  ~FamScope() { g_fam = prev; }
};
#define CH (g_fam->CH)
#define CT (g_fam->CT)
#define NL (g_fam->NL)

struct MbLayer {
  int t, k, cin, cout, stride;  // stored widths
  int cin_t, cout_t;            // true widths
};

MbLayer teacher_layer(int b, int l) {
  static const MbLayer B0[3] = {{1, 3, 32, 16, 1, 32, 16}, {6, 3, 16, 32, 2, 16, 24}, {6, 3, 32, 32, 1, 24, 24}};
  if (b == 0) return B0[l];
  const int cin = CH[b], cout = CH[b + 1];
  const int s = DIV[b + 1] / DIV[b];
  const int k = g_fam->K[b];
  return l == 0 ? MbLayer{6, k, cin, cout, s, CT[b], CT[b + 1]} : MbLayer{6, k, cout, cout, 1, CT[b + 1], CT[b + 1]};
}

int se_ch(const MbLayer& m) { return g_fam->se ? std::max(1, m.cin / 4) : 0; }
int se_ch_t(const MbLayer& m) { return g_fam->se ? std::max(1, m.cin_t / 4) : 0; }
int round_ch(int c) { return c <= 16 ? 16 : c <= 32 ? 32 : (c + 63) / 64 * 64; }
int expand_ch(int cin, int t) { return t == 1 ? cin : round_ch(cin * t); }
int expand_ch_t(int cin_t, int t) { return t == 1 ? cin_t : cin_t * t; }
// a residual joins input and output when the stride is 1 and the TRUE widths agree
bool has_res(const MbLayer& m) { return m.stride == 1 && m.cin_t == m.cout_t; }
int student_layers(int b) { return NL[b] + (b == 0 ? 1 : 0); }
int layer_cands(int b, int l) { return (b == 0 && l < 2) ? 1 : kCands; }
bool is_stem(int b, int l) { return b == 0 && l == 0; }

// per-candidate parameter layout (element offsets inside the candidate) — mb_oracle.c cand_lay
struct CandLayout {
  size_t we = 0, wd = 0, wp = 0, g1 = 0, b1 = 0, g2 = 0, b2 = 0, g3 = 0, b3 = 0, total = 0;
  int E = 0, k = 0, e = 0;
  int Et = 0;  // true expanded width
};

MbLayer student_mb(int b, int l) { return teacher_layer(b, b == 0 ? l - 1 : l); }

CandLayout cand_layout(int b, int l, int c) {
  CandLayout L;
  if (is_stem(b, l)) {
    L.g2 = 32 * 9 * 16;
    L.b2 = L.g2 + 32;
    L.total = L.b2 + 32;
    L.E = 32;
    L.Et = 32;
    L.k = 3;
    return L;
  }
  const MbLayer m = student_mb(b, l);
  if (b == 0 && l < 2) {
    L.k = 3;
    L.e = 1;
  } else {
    static const int KS[3] = {3, 5, 7}, ES[2] = {3, 6};
    L.k = KS[c % 3];
    L.e = ES[c / 3];
  }
  L.E = expand_ch(m.cin, L.e);
  L.Et = expand_ch_t(m.cin_t, L.e);
  size_t o = 0;
  if (L.e != 1) {
    L.we = o;
    o += static_cast<size_t>(L.E) * m.cin;
  }
  L.wd = o;
  o += static_cast<size_t>(L.E) * L.k * L.k;
  L.wp = o;
  o += static_cast<size_t>(m.cout) * L.E;
  if (L.e != 1) {
    L.g1 = o;
    o += L.E;
    L.b1 = o;
    o += L.E;
  }
  L.g2 = o;
  o += L.E;
  L.b2 = o;
  o += L.E;
  L.g3 = o;
  o += m.cout;
  L.b3 = o;
  o += m.cout;
  L.total = o;
  return L;
}

size_t cand_offset(int b, int l, int c, size_t* count) {
  size_t off = 0;
  for (int i = 0; i < student_layers(b); ++i)
    for (int j = 0; j < layer_cands(b, i); ++j) {
      const CandLayout L = cand_layout(b, i, j);
      if (i == l && j == c) {
        if (count) *count = L.total;
        return off;
      }
      off += L.total;
    }
  if (count) *count = 0;
  return off;
}

size_t block_params(int b) { return cand_offset(b, student_layers(b), 0, nullptr); }

float kaiming(int fan_in, float gain) { return std::sqrt(6.0f / static_cast<float>(fan_in)) * gain; }
size_t pad128(size_t m) { return (m + 127) / 128 * 128; }

// 1x1 convolution as a tcgen05 GEMM over m pixels (rows padded to 128)
pbdk_conv_desc pw_desc(size_t m, int cin, int cout) {
  return pbdk_conv_desc{static_cast<int>(pad128(m) / 128), 1, 128, cin, cout, 1, 1, 1, 0, 1, 128};
}

// ---- teacher program
struct TOp {
  enum Kind { STEM, PW, DW, SE } kind;
  int cs = 0;                                  // SE width
  int cin_t = 0, cout_t = 0, cs_t = 0;         // true widths (weights beyond them are zero)
  bf16 *w2 = nullptr;                          // SE: w = W1 [cs][E], w2 = W2 [E][cs]
  float* b2 = nullptr;                         // SE: bias = b1 [cs], b2 [E]
  int cin = 0, cout = 0, k = 0, stride = 1, hin = 0, hout = 0, epi = 0;
  uint32_t tensor = 0;
  float gain = 1.0f;
  bf16* w = nullptr;      // [cout][cin] (PW), [32][3][3][16] (STEM), [E][k][k] (DW, as initialised)
  bf16* wflip = nullptr;  // DW: flipped tap-major copy
  float* bias = nullptr;
  const bf16* in = nullptr;
  bf16* out = nullptr;
  const bf16* aux = nullptr;
  pbdk::FpropPlan plan;
};

struct TBlock {
  std::vector<TOp> ops;
  bf16* out = nullptr;
};

// ---- student
struct SCand {
  CandLayout L;
  size_t off = 0;  // inside the partition's flat vectors
  bf16* weT = nullptr;  // [cin][E]   expand dgrad operand
  bf16* wpT = nullptr;  // [E][cout]  project dgrad operand
  bf16* wdF = nullptr;  // [k][k][E]  flipped depthwise
  pbdk::FpropPlan p_exp, p_proj, p_proj_dgrad, p_exp_dgrad;
  pbdk::WgradPlan w_exp, w_proj;
};

struct SLayer {
  int cin = 0, cout = 0, stride = 1, hin = 0, hout = 0, Emax = 0;
  int cin_t = 0, cout_t = 0;  // true widths
  bool res = false, stem = false, need_dx = false, last = false;
  std::vector<SCand> cands;
  int active = 0;
  const bf16* x = nullptr;  // layer input
  bf16 *y1 = nullptr, *a1 = nullptr, *g1 = nullptr, *dy1 = nullptr;
  bf16 *y2 = nullptr, *a2 = nullptr, *g2 = nullptr, *dy2 = nullptr;
  bf16 *y3 = nullptr, *dy3 = nullptr, *z = nullptr;
  bf16* gz = nullptr;        // gradient w.r.t. this layer's output
  bf16* gx = nullptr;        // gradient w.r.t. this layer's input (= previous layer's gz)
  float *st1 = nullptr, *st2 = nullptr, *st3 = nullptr;
  float *red1 = nullptr, *red2 = nullptr, *red3 = nullptr;
};

struct SBlock {
  int k = 0;
  size_t base = 0;  // offset of the block in the flat vectors
  std::vector<SLayer> layers;
  const bf16* in = nullptr;
  const bf16* target = nullptr;
  float* rws = nullptr;  // loss reductions
  size_t rws_floats = 0;
  pbdk::FixScratch fx{};  // self-finalizing BN reductions of this block's stream (sequential: one scratch)
  float* dws = nullptr;  // depthwise / stem wgrad partials
  size_t dws_floats = 0;
  void* wws = nullptr;  // 1x1 wgrad split-K partials
  size_t wws_bytes = 0;
  double* lws = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
};

class MbPartition final : public PartitionBase {
 public:
  explicit MbPartition(const pbdx_desc& d) : PartitionBase(d), fam_(family(d.model)) {
    if (d.block_lo < 0 || d.block_hi >= kBlocks || d.block_lo > d.block_hi) throw BadArg("bad block range");
    if (d.image < 32 || d.image % 32 != 0) throw BadArg("image side must be a multiple of 32");
    S_ = d.image;
    FamScope fs(fam_);
    allocate();
    build_plans();
  }

  ~MbPartition() override {
    for (SBlock& s : sblocks_) {
      if (s.stream != nullptr) cudaStreamDestroy(s.stream);
      if (s.done != nullptr) cudaEventDestroy(s.done);
    }
    for (auto e : tdone_) cudaEventDestroy(e);
    if (fork_ != nullptr) cudaEventDestroy(fork_);
  }

  int nblocks() const override { return d_.block_hi - d_.block_lo + 1; }
  const void* relay_source() const override { return tblocks_.back().out; }
  size_t relay_row_bytes() const override { return act_row_bytes(d_.block_hi + 1); }
  void rebuild_for_shard() override {
    FamScope fs(fam_);
    build_plans();
  }

  void init_params(cudaStream_t st) override {
    for (TBlock& tb : tblocks_)
      for (TOp& op : tb.ops) {
        if (op.kind == TOp::SE) {
          check(pbdk::init_uniform(op.w, 1, op.cs, 1, 1, op.cout, op.cout_t, d_.seed_teacher, op.tensor,
                                   kaiming(op.cout_t, 1.0f), st, op.cs_t),
                "init");
          check(pbdk::init_uniform(op.bias, 0, op.cs, 1, 1, 1, 1, d_.seed_teacher, op.tensor + 1, 0.1f, st, op.cs_t),
                "init");
          check(pbdk::init_uniform(op.w2, 1, op.cout, 1, 1, op.cs, op.cs_t, d_.seed_teacher, op.tensor + 10,
                                   kaiming(op.cs_t, 1.0f), st, op.cout_t),
                "init");
          check(pbdk::init_uniform(op.b2, 0, op.cout, 1, 1, 1, 1, d_.seed_teacher, op.tensor + 11, 0.1f, st, op.cout_t),
                "init");
          continue;
        }
        if (op.kind == TOp::STEM) {
          check(pbdk::init_uniform(op.w, 1, 32, 3, 3, 16, 3, d_.seed_teacher, op.tensor, kaiming(27, 1.0f), st), "init");
        } else if (op.kind == TOp::PW) {
          check(pbdk::init_uniform(op.w, 1, op.cout, 1, 1, op.cin, op.cin_t, d_.seed_teacher, op.tensor,
                                   kaiming(op.cin_t, op.gain), st, op.cout_t),
                "init");
        } else {
          check(pbdk::init_uniform(op.w, 1, op.cout, op.k, op.k, 1, 1, d_.seed_teacher, op.tensor,
                                   kaiming(op.k * op.k, 1.0f), st, op.cout_t),
                "init");
          check(pbdk_weight_flip(op.w, op.wflip, op.cout, op.k, op.k, 1, st), "flip");
        }
        check(pbdk::init_uniform(op.bias, 0, op.cout, 1, 1, 1, 1, d_.seed_teacher, op.tensor + 1, 0.1f, st,
                                 op.cout_t),
              "init");
      }
    for (SBlock& sb : sblocks_)
      for (size_t l = 0; l < sb.layers.size(); ++l) {
        SLayer& L = sb.layers[l];
        for (size_t c = 0; c < L.cands.size(); ++c) {
          const SCand& C = L.cands[c];
          float* q = params_ + C.off;
          const uint32_t tid = 40000u + 1000u * static_cast<uint32_t>(sb.k) + 100u * static_cast<uint32_t>(l) +
                               10u * static_cast<uint32_t>(c);
          if (L.stem) {
            check(pbdk::init_uniform(q, 0, 32, 3, 3, 16, 3, d_.seed_student, tid, kaiming(27, 1.0f), st), "init");
            check(pbdk::fill(q + C.L.g2, 32, 1.0f, st), "fill");
            check(pbdk::fill(q + C.L.b2, 32, 0.0f, st), "fill");
            continue;
          }
          if (C.L.e != 1)
            check(pbdk::init_uniform(q + C.L.we, 0, C.L.E, 1, 1, L.cin, L.cin_t, d_.seed_student, tid,
                                     kaiming(L.cin_t, 1.0f), st, C.L.Et),
                  "init");
          check(pbdk::init_uniform(q + C.L.wd, 0, C.L.E, C.L.k, C.L.k, 1, 1, d_.seed_student, tid + 1u,
                                   kaiming(C.L.k * C.L.k, 1.0f), st, C.L.Et),
                "init");
          check(pbdk::init_uniform(q + C.L.wp, 0, L.cout, 1, 1, C.L.E, C.L.Et, d_.seed_student, tid + 2u,
                                   kaiming(C.L.Et, 1.0f), st, L.cout_t),
                "init");
          if (C.L.e != 1) {
            check(pbdk::fill(q + C.L.g1, C.L.E, 1.0f, st), "fill");
            check(pbdk::fill(q + C.L.b1, C.L.E, 0.0f, st), "fill");
          }
          check(pbdk::fill(q + C.L.g2, C.L.E, 1.0f, st), "fill");
          check(pbdk::fill(q + C.L.b2, C.L.E, 0.0f, st), "fill");
          check(pbdk::fill(q + C.L.g3, L.cout, 1.0f, st), "fill");
          check(pbdk::fill(q + C.L.b3, L.cout, 0.0f, st), "fill");
        }
      }
    check(pbdk::fill(mom_, total_, 0.0f, st), "fill");
    check(pbdk::fill(grads_, total_, 0.0f, st), "fill");
    check(pbdk::sgd_momentum(params_, mom_, grads_, shadow_, total_, 0.0f, 0.0f, nullptr, st), "shadow");
    for (SBlock& sb : sblocks_)
      for (SLayer& L : sb.layers)
        for (SCand& C : L.cands) refresh_derived(L, C, st);
    cuda(cudaMemsetAsync(step_, 0, sizeof(long long), st), "memset");
  }

  void set_path(int block, const int* path, int n) override {
    if (block < d_.block_lo || block > d_.block_hi) throw BadArg("block outside partition");
    SBlock& sb = sblocks_[static_cast<size_t>(block - d_.block_lo)];
    if (n != static_cast<int>(sb.layers.size())) throw BadArg("path length != student layers");
    for (int l = 0; l < n; ++l)
      if (path[l] < 0 || path[l] >= static_cast<int>(sb.layers[static_cast<size_t>(l)].cands.size()))
        throw BadArg("candidate out of range");
    for (int l = 0; l < n; ++l) sb.layers[static_cast<size_t>(l)].active = path[l];
    // inactive candidates carry no gradient (a DP allreduce then sums zeros)
    FamScope fs(fam_);
    cuda(cudaMemset(grads_ + sb.base, 0, block_params(sb.k) * sizeof(float)), "memset");
    invalidate_graphs();
  }

  void upload_images(const float* host, int n, cudaStream_t st) override {
    if (d_.block_lo != 0) throw BadArg("only partition 0 loads data");
    if (n != n_) throw BadArg("upload size != shard size");
    cuda(cudaMemcpyAsync(stage_, host, static_cast<size_t>(n) * S_ * S_ * 3 * sizeof(float), cudaMemcpyHostToDevice,
                         st),
         "H2D images");
    check(pbdk::pack_image(stage_, input_, n, st, S_), "pack image");
  }

  void stage_images(const float* host, int n, int slot, cudaStream_t st) override {
    if (d_.block_lo != 0 || n != n_ || (slot != 0 && slot != 1))
      throw BadArg("stage_images: partition 0 only, n == shard size, slot 0/1");
    const size_t bytes = static_cast<size_t>(n) * S_ * S_ * 3 * sizeof(float);
    cuda(cudaMemcpyAsync(slot == 0 ? stage_ : stage2_, host, bytes, cudaMemcpyHostToDevice, st), "H2D stage");
  }

  void teacher_body(cudaStream_t st) override {
    if (d_.block_lo == 0 && external_ == 2)
      check(pbdk::pack_image_parity(stage_, stage2_, step_, input_, n_, st, S_), "pack staged image");
    if (d_.block_lo == 0 && !external_)
      check(pbdk::philox_image(input_, n_, first_, step_, d_.global_batch, d_.seed_data, st, S_), "philox");
    for (size_t i = 0; i < tblocks_.size(); ++i) {
      if (timing_) cuda(cudaEventRecord(ev_t_[2 * i], st), "event");
      for (TOp& op : tblocks_[i].ops) run_teacher_op(op, st);
      if (timing_) cuda(cudaEventRecord(ev_t_[2 * i + 1], st), "event");
      cuda(cudaEventRecord(tdone_[i], st), "event");
    }
  }

  void student_body(cudaStream_t caller, bool fork) override {
    // measured (scripts/ab_mb_grids2.sh, profiles/r02_ab_mb_grids.txt): one reduction CTA per SM, 296-CTA
    // applies and >= 1 MB per reduction CTA beside the six concurrent student streams: MobileNetV2 step
    // 16.20 -> 15.81 ms, EfficientNet-B0 19.90 -> 19.58 ms
    static const int red = [] { const char* e = pbd::knob_env("PBDK_MB_RED"); return e ? std::atoi(e) : 148; }();
    static const int app = [] { const char* e = pbd::knob_env("PBDK_MB_APPLY"); return e ? std::atoi(e) : 296; }();
    const pbdk::GridScope grids(red, app, 1 << 20);
    if (fork) cuda(cudaEventRecord(fork_, caller), "event");
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      SBlock& sb = sblocks_[i];
      cudaStream_t st = sb.stream;
      cuda(cudaStreamWaitEvent(st, fork ? fork_ : tdone_[i], 0), "wait teacher");
      if (timing_) cuda(cudaEventRecord(ev_s_[2 * i], st), "event");
      if (trains(static_cast<int>(i))) student_block(sb, i, st);
      if (timing_) cuda(cudaEventRecord(ev_s_[2 * i + 1], st), "event");
      cuda(cudaEventRecord(sb.done, st), "event");
    }
    for (SBlock& sb : sblocks_) cuda(cudaStreamWaitEvent(caller, sb.done, 0), "join");
  }

  void update_body(cudaStream_t st) override {
    if (dp_active()) {  // reduce-scatter + all-gather of the active candidates (PartitionBase::dp_update)
      std::vector<DpRegion> regions;
      for (size_t i = 0; i < sblocks_.size(); ++i) {
        if (!trains(static_cast<int>(i))) continue;
        for (SLayer& L : sblocks_[i].layers) {
          const SCand& C = L.cands[static_cast<size_t>(L.active)];
          regions.push_back({C.off, C.L.total});
        }
      }
      dp_update(regions, params_, mom_, grads_, shadow_, step_, st);
      for (size_t i = 0; i < sblocks_.size(); ++i) {
        if (!trains(static_cast<int>(i))) continue;
        for (SLayer& L : sblocks_[i].layers) refresh_derived(L, L.cands[static_cast<size_t>(L.active)], st);
      }
      return;
    }
    long long* counter = step_;
    for (size_t i = 0; i < sblocks_.size(); ++i) {
      if (!trains(static_cast<int>(i))) continue;
      SBlock& sb = sblocks_[i];
      for (SLayer& L : sb.layers) {
        SCand& C = L.cands[static_cast<size_t>(L.active)];
        if (L.stem) {
          check(pbdk::sgd_momentum(params_ + C.off, mom_ + C.off, grads_ + C.off, shadow_ + C.off, C.L.total,
                                   d_.lr, d_.momentum, counter, st),
                "sgd");
        } else {  // one launch: update + shadow + the three derived dgrad operands (refresh_derived)
          check(pbdk::sgd_momentum_flip(params_ + C.off, mom_ + C.off, grads_ + C.off, shadow_ + C.off, C.L.total,
                                        d_.lr, d_.momentum, counter, derived_regions(L, C), st),
                "sgd");
        }
        counter = nullptr;  // advance the step counter once
      }
    }
  }

  std::vector<DpRegion> dp_all_regions() const override {  // every candidate: each keeps its own slicing
    std::vector<DpRegion> r;
    for (const SBlock& sb : sblocks_)
      for (const SLayer& L : sb.layers)
        for (const SCand& C : L.cands) r.push_back({C.off, C.L.total});
    return r;
  }

  void refresh_shadows(cudaStream_t st) override {
    check(pbdk::sgd_momentum(params_, mom_, grads_, shadow_, total_, 0.0f, 1.0f, nullptr, st), "shadow");
    for (SBlock& sb : sblocks_)
      for (SLayer& L : sb.layers)
        for (SCand& C : L.cands) refresh_derived(L, C, st);
  }

  void buffer(int which, void** ptr, size_t* bytes) override {
    switch (which) {
      case PBDX_BUF_INPUT: *ptr = input_; *bytes = input_bytes_; break;
      case PBDX_BUF_TEACHER_OUT: *ptr = tblocks_.back().out; *bytes = act_bytes(d_.block_hi + 1); break;
      case PBDX_BUF_GRADS: *ptr = grads_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_PARAMS: *ptr = params_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_MOMENTUM: *ptr = mom_; *bytes = total_ * sizeof(float); break;
      case PBDX_BUF_LOSSES: *ptr = losses_; *bytes = nblocks() * sizeof(double); break;
      case PBDX_BUF_STEP: *ptr = step_; *bytes = sizeof(long long); break;
      case PBDX_BUF_TEACHER_PARAMS: *ptr = nullptr; *bytes = 0; break;
      case PBDX_BUF_MAILBOX: *ptr = mailbox_; *bytes = kMailboxSlots * sizeof(unsigned long long); break;
      default: throw BadArg("unknown buffer");
    }
  }

  void teacher_act(int k, void** ptr, size_t* bytes) override {
    if (k < d_.block_lo || k > d_.block_hi) throw BadArg("block outside partition");
    *ptr = tblocks_[static_cast<size_t>(k - d_.block_lo)].out;
    *bytes = act_bytes(k + 1);
  }

  int body_launches_per_step() const override {
    int n = (d_.block_lo == 0 && external_ != 1) ? 1 : 0;
    for (const TBlock& tb : tblocks_) n += static_cast<int>(tb.ops.size());
    for (size_t bi = 0; bi < sblocks_.size(); ++bi) {
      if (!trains(static_cast<int>(bi))) continue;
      for (const SLayer& L : sblocks_[bi].layers) {
        const SCand& C = L.cands[static_cast<size_t>(L.active)];
        if (L.stem) {
          n += (1 + 1 + 1) + (2 + 2) + 1;  // conv, stats, apply | bn bwd, wgrad | sgd
          continue;
        }
        const bool e = C.L.e != 1;
        n += (e ? 3 : 0) + 1 + 1 + 1 + 1 + 1 + (L.last ? 2 : 1);                      // forward
        n += 2 + (C.w_proj.splits > 1 ? 2 : 1) + 1 + 2 + 2;                            // bn3, wgrad, dgrad, bn2, dw wgrad
        n += e ? (1 + 2 + (C.w_exp.splits > 1 ? 2 : 1) + (L.need_dx ? 1 : 0)) : (L.need_dx ? 1 : 0);
        n += dp_active() ? 1 + (e ? 2 : 1) + 1 : 1;  // sgd (+ transposes, flip unless fused into it)
      }
    }
    return n;
  }

  long long total_params() const { return static_cast<long long>(total_); }

 private:
  size_t act_row_bytes(int boundary) const {
    const int hw = S_ / DIV[boundary];
    const int c = boundary == 0 ? 16 : CH[boundary];
    return static_cast<size_t>(hw) * hw * c * sizeof(bf16);
  }
  size_t act_rows(int boundary, int n) const {
    const int hw = S_ / DIV[boundary];
    return static_cast<size_t>(n) * hw * hw;
  }
  size_t act_bytes(int boundary) const { return pad128(act_rows(boundary, d_.n_max)) * act_row_bytes(boundary) /
                                                (static_cast<size_t>(S_ / DIV[boundary]) * (S_ / DIV[boundary])); }
  // bf16 buffer of (m rows padded to 128) x c
  bf16* act(size_t m, int c) { return arena_.get<bf16>(pad128(m) * static_cast<size_t>(c) * sizeof(bf16)); }

  // refresh_derived's three transposes / flips as regions of the candidate's slice (offsets from C.off)
  static pbdk::FlipSet derived_regions(const SLayer& L, const SCand& C) {
    pbdk::FlipSet fs;
    if (C.L.e != 1) fs.reg[fs.count++] = pbdk::FlipRegion{C.L.we, C.L.E, 1, 1, L.cin, C.weT};
    fs.reg[fs.count++] = pbdk::FlipRegion{C.L.wp, L.cout, 1, 1, C.L.E, C.wpT};
    fs.reg[fs.count++] = pbdk::FlipRegion{C.L.wd, C.L.E, C.L.k, C.L.k, 1, C.wdF};
    return fs;
  }

  void refresh_derived(SLayer& L, SCand& C, cudaStream_t st) {
    if (L.stem) return;
    const bf16* sh = shadow_ + C.off;
    if (C.L.e != 1) check(pbdk_weight_flip(sh + C.L.we, C.weT, C.L.E, 1, 1, L.cin, st), "transpose we");
    check(pbdk_weight_flip(sh + C.L.wp, C.wpT, L.cout, 1, 1, C.L.E, st), "transpose wp");
    check(pbdk_weight_flip(sh + C.L.wd, C.wdF, C.L.E, C.L.k, C.L.k, 1, st), "flip wd");
  }

  void run_teacher_op(TOp& op, cudaStream_t st) {
    if (op.kind == TOp::STEM) {
      check(pbdk::stem_fwd(op.in, op.w, op.bias, op.out, n_, S_, fam_.act, st), "teacher stem");
    } else if (op.kind == TOp::PW) {
      check(pbdk::fprop_run(op.plan, st), "teacher 1x1");
    } else if (op.kind == TOp::SE) {
      check(pbdk::se_apply(op.out, n_, op.hout * op.hout, op.cout, op.cs, op.w, op.bias, op.w2, op.b2, se_pool_,
                           se_gate_, st),
            "teacher squeeze-excite");
    } else {
      const pbdk::DwArgs a{n_, op.hin, op.hin, op.cout, op.k, op.stride, op.hout, op.hout};
      check(pbdk::dw_fwd(a, op.in, op.wflip, op.bias, op.out, fam_.act, st), "teacher dw");
    }
  }

  void student_block(SBlock& sb, size_t i, cudaStream_t st) {
    const int nl = static_cast<int>(sb.layers.size());
    // ---- forward
    for (int l = 0; l < nl; ++l) {
      SLayer& L = sb.layers[static_cast<size_t>(l)];
      SCand& C = L.cands[static_cast<size_t>(L.active)];
      const float* p = params_ + C.off;
      const size_t mi = act_rows_hw(L.hin), mo = act_rows_hw(L.hout);
      if (L.stem) {
        check(pbdk::stem_fwd(L.x, shadow_ + C.off, nullptr, L.y2, n_, S_, 0, st), "student stem");
        check(pbdk::bn_stats_fix(L.y2, nullptr, static_cast<int>(mo), 32, sb.fx, L.st2, nullptr, st), "stem stats");
        check(pbdk::bn_apply_act(L.y2, L.st2, p + C.L.g2, p + C.L.b2, nullptr, L.a2, static_cast<long long>(mo), 32,
                                 1, st),
              "stem apply");
        continue;
      }
      const bf16* a_in = L.x;
      if (C.L.e != 1) {
        check(pbdk::fprop_run(C.p_exp, st), "expand");
        check(pbdk::bn_stats_fix(L.y1, nullptr, static_cast<int>(mi), C.L.E, sb.fx, L.st1, nullptr, st), "bn1 stats");
        check(pbdk::bn_apply_act(L.y1, L.st1, p + C.L.g1, p + C.L.b1, nullptr, L.a1, static_cast<long long>(mi), C.L.E,
                                 1, st),
              "bn1 apply");
        a_in = L.a1;
      }
      const pbdk::DwArgs dw{n_, L.hin, L.hin, C.L.E, C.L.k, L.stride, L.hout, L.hout};
      check(pbdk::dw_fwd(dw, a_in, C.wdF, nullptr, L.y2, 0, st), "dw");
      check(pbdk::bn_stats_fix(L.y2, nullptr, static_cast<int>(mo), C.L.E, sb.fx, L.st2, nullptr, st), "bn2 stats");
      check(pbdk::bn_apply_act(L.y2, L.st2, p + C.L.g2, p + C.L.b2, nullptr, L.a2, static_cast<long long>(mo), C.L.E, 1,
                               st),
            "bn2 apply");
      check(pbdk::fprop_run(C.p_proj, st), "project");
      check(pbdk::bn_stats_fix(L.y3, nullptr, static_cast<int>(mo), L.cout, sb.fx, L.st3, nullptr, st), "bn3 stats");
      if (!L.last) {
        check(pbdk::bn_apply_act(L.y3, L.st3, p + C.L.g3, p + C.L.b3, L.res ? L.x : nullptr, L.z,
                                 static_cast<long long>(mo), L.cout, 0, st),
              "bn3 apply");
      } else {
        const double norm = static_cast<double>(d_.global_batch) * L.cout_t * L.hout * L.hout;  // true widths
        check(pbdk::mse_affine(L.y3, L.st3, p + C.L.g3, p + C.L.b3, L.res ? L.x : nullptr, sb.target,
                               static_cast<long long>(mo), L.cout, static_cast<float>(2.0 / norm), norm, L.gz, sb.lws,
                               losses_ + i, st),
              "mse");
      }
    }
    // ---- backward
    for (int l = nl - 1; l >= 0; --l) {
      SLayer& L = sb.layers[static_cast<size_t>(l)];
      SCand& C = L.cands[static_cast<size_t>(L.active)];
      const float* p = params_ + C.off;
      float* g = grads_ + C.off;
      const size_t mi = act_rows_hw(L.hin), mo = act_rows_hw(L.hout);
      if (L.stem) {
        check(pbdk::bn_bwd_fix(L.gz, L.y2, L.st2, p + C.L.g2, static_cast<int>(mo), 32, sb.fx, L.red2, g + C.L.g2,
                           g + C.L.b2, L.dy2, st),
              "stem bn bwd");
        check(pbdk::stem_wgrad(L.x, L.dy2, n_, S_, sb.dws, sb.dws_floats, g, st), "stem wgrad");
        continue;
      }
      check(pbdk::bn_bwd_fix(L.gz, L.y3, L.st3, p + C.L.g3, static_cast<int>(mo), L.cout, sb.fx, L.red3, g + C.L.g3,
                         g + C.L.b3, L.dy3, st),
            "bn3 bwd");
      check(pbdk::wgrad_run(C.w_proj, st), "wgrad project");
      check(pbdk::fprop_run(C.p_proj_dgrad, st), "dgrad project");
      check(pbdk::bn_bwd_fix(L.g2, L.y2, L.st2, p + C.L.g2, static_cast<int>(mo), C.L.E, sb.fx, L.red2, g + C.L.g2,
                         g + C.L.b2, L.dy2, st),
            "bn2 bwd");
      const pbdk::DwArgs dw{n_, L.hin, L.hin, C.L.E, C.L.k, L.stride, L.hout, L.hout};
      const bf16* a_in = C.L.e != 1 ? L.a1 : L.x;
      check(pbdk::dw_wgrad(dw, a_in, L.dy2, sb.dws, sb.dws_floats, g + C.L.wd, st), "dw wgrad");
      if (C.L.e != 1) {
        check(pbdk::dw_dgrad(dw, L.dy2, C.wdF, L.a1, L.g1, st), "dw dgrad");
        check(pbdk::bn_bwd_fix(L.g1, L.y1, L.st1, p + C.L.g1, static_cast<int>(mi), C.L.E, sb.fx, L.red1, g + C.L.g1,
                           g + C.L.b1, L.dy1, st),
              "bn1 bwd");
        check(pbdk::wgrad_run(C.w_exp, st), "wgrad expand");
        if (L.need_dx) check(pbdk::fprop_run(C.p_exp_dgrad, st), "dgrad expand");
      } else if (L.need_dx) {
        // MBConv1 directly on the stem activation: its ReLU6 mask
        check(pbdk::dw_dgrad(dw, L.dy2, C.wdF, L.x, L.gx, st), "dw dgrad (stem)");
      }
    }
  }

  size_t act_rows_hw(int hw) const { return static_cast<size_t>(n_) * hw * hw; }
  size_t rows_max(int hw) const { return static_cast<size_t>(d_.n_max) * hw * hw; }

  void allocate() {
    const int lo = d_.block_lo, hi = d_.block_hi;
    const int N = d_.n_max;
    // input of block lo: the padded image or a relayed activation
    input_bytes_ = act_bytes(lo);
    input_ = arena_.get<bf16>(input_bytes_);
    if (lo == 0) {
      stage_ = arena_.get<float>(static_cast<size_t>(N) * S_ * S_ * 3 * sizeof(float));
      stage2_ = arena_.get<float>(static_cast<size_t>(N) * S_ * S_ * 3 * sizeof(float));
    }

    // ---- teacher program
    const bf16* prev = input_;
    size_t se_elems = 0;
    for (int b = lo; b <= hi; ++b) {
      TBlock tb;
      int j = 0;
      int hw = S_ / DIV[b];
      const uint32_t base = 20000u + 1000u * static_cast<uint32_t>(b);
      const bf16* x = prev;
      if (b == 0) {
        TOp op{};
        op.kind = TOp::STEM;
        op.cin = 3;
        op.cout = 32;
        op.cin_t = 3;
        op.cout_t = 32;
        op.k = 3;
        op.stride = 2;
        op.hin = S_;
        op.hout = S_ / 2;
        op.tensor = base + 10u * j++;
        op.in = x;
        op.out = act(rows_max(op.hout), 32);
        op.w = arena_.get<bf16>(32 * 9 * 16 * sizeof(bf16));
        op.bias = arena_.get<float>(32 * sizeof(float));
        tb.ops.push_back(op);
        x = op.out;
        hw = S_ / 2;
      }
      for (int l = 0; l < NL[b]; ++l) {
        const MbLayer m = teacher_layer(b, l);
        const int E = expand_ch(m.cin, m.t), Et = expand_ch_t(m.cin_t, m.t);
        const int ho = (hw + 2 * (m.k / 2) - m.k) / m.stride + 1;
        const bf16* a = x;
        if (m.t != 1) {
          TOp e{};
          e.kind = TOp::PW;
          e.cin = m.cin;
          e.cout = E;
          e.cin_t = m.cin_t;
          e.cout_t = Et;
          e.hin = e.hout = hw;
          e.epi = fam_.act == 2 ? PBDK_EPI_BIAS_SWISH : PBDK_EPI_BIAS_RELU6;
          e.tensor = base + 10u * j++;
          e.in = x;
          e.out = act(rows_max(hw), E);
          e.w = arena_.get<bf16>(static_cast<size_t>(E) * m.cin * sizeof(bf16));
          e.bias = arena_.get<float>(E * sizeof(float));
          tb.ops.push_back(e);
          a = e.out;
        }
        TOp d{};
        d.kind = TOp::DW;
        d.cin = d.cout = E;
        d.cin_t = d.cout_t = Et;
        d.k = m.k;
        d.stride = m.stride;
        d.hin = hw;
        d.hout = ho;
        d.tensor = base + 10u * j++;
        d.in = a;
        d.out = act(rows_max(ho), E);
        d.w = arena_.get<bf16>(static_cast<size_t>(E) * m.k * m.k * sizeof(bf16));
        d.wflip = arena_.get<bf16>(static_cast<size_t>(E) * m.k * m.k * sizeof(bf16));
        d.bias = arena_.get<float>(E * sizeof(float));
        tb.ops.push_back(d);
        if (const int cs = se_ch(m); cs > 0) {  // squeeze-excite in place on the depthwise output
          TOp q{};
          q.kind = TOp::SE;
          q.cout = E;
          q.cs = cs;
          q.cout_t = Et;
          q.cs_t = se_ch_t(m);
          q.hin = q.hout = ho;
          q.tensor = base + 10u * j;
          j += 2;
          q.out = d.out;
          q.w = arena_.get<bf16>(static_cast<size_t>(cs) * E * sizeof(bf16));
          q.bias = arena_.get<float>(cs * sizeof(float));
          q.w2 = arena_.get<bf16>(static_cast<size_t>(E) * cs * sizeof(bf16));
          q.b2 = arena_.get<float>(E * sizeof(float));
          tb.ops.push_back(q);
          se_elems = std::max(se_elems, static_cast<size_t>(N) * E);
        }
        const bool res = has_res(m);
        TOp pj{};
        pj.kind = TOp::PW;
        pj.cin = E;
        pj.cout = m.cout;
        pj.cin_t = Et;
        pj.cout_t = m.cout_t;
        pj.hin = pj.hout = ho;
        pj.epi = res ? PBDK_EPI_BIAS_RES : PBDK_EPI_BIAS;
        pj.gain = res ? 0.5f : 1.0f;
        pj.tensor = base + 10u * j++;
        pj.in = d.out;
        pj.aux = res ? x : nullptr;
        pj.out = act(rows_max(ho), m.cout);
        pj.w = arena_.get<bf16>(static_cast<size_t>(m.cout) * E * sizeof(bf16));
        pj.bias = arena_.get<float>(m.cout * sizeof(float));
        tb.ops.push_back(pj);
        x = pj.out;
        hw = ho;
      }
      tb.out = const_cast<bf16*>(x);
      prev = tb.out;
      tblocks_.push_back(std::move(tb));
    }
    if (se_elems > 0) {
      se_pool_ = arena_.get<float>(se_elems * sizeof(float));
      se_gate_ = arena_.get<float>(se_elems * sizeof(float));
    }

    // ---- student blocks
    total_ = 0;
    for (int b = lo; b <= hi; ++b) {
      SBlock sb;
      sb.k = b;
      sb.base = total_;
      sb.in = b == lo ? input_ : tblocks_[static_cast<size_t>(b - lo - 1)].out;
      sb.target = tblocks_[static_cast<size_t>(b - lo)].out;
      const int nl = student_layers(b);
      int hw = S_ / DIV[b];
      size_t rws = 0, dws = 0, wws = 0, lws = 0;
      const bf16* x = sb.in;
      for (int l = 0; l < nl; ++l) {
        SLayer L;
        L.stem = is_stem(b, l);
        L.last = l == nl - 1;
        if (L.stem) {
          L.cin = 3;
          L.cout = 32;
          L.cin_t = 3;
          L.cout_t = 32;
          L.stride = 2;
          L.hin = S_;
          L.hout = S_ / 2;
          L.Emax = 32;
        } else {
          const MbLayer m = student_mb(b, l);
          L.cin = m.cin;
          L.cout = m.cout;
          L.cin_t = m.cin_t;
          L.cout_t = m.cout_t;
          L.stride = m.stride;
          L.hin = hw;
          L.hout = (hw - 1) / m.stride + 1;
          L.res = has_res(m);
        }
        L.need_dx = l > 0;
        const size_t mi = rows_max(L.hin), mo = rows_max(L.hout);
        for (int c = 0; c < layer_cands(b, l); ++c) {
          SCand C;
          C.L = cand_layout(b, l, c);
          C.off = sb.base + cand_offset(b, l, c, nullptr);
          L.Emax = std::max(L.Emax, C.L.E);
          if (!L.stem) {
            if (C.L.e != 1) C.weT = arena_.get<bf16>(static_cast<size_t>(C.L.E) * L.cin * sizeof(bf16));
            C.wpT = arena_.get<bf16>(static_cast<size_t>(C.L.E) * L.cout * sizeof(bf16));
            C.wdF = arena_.get<bf16>(static_cast<size_t>(C.L.E) * C.L.k * C.L.k * sizeof(bf16));
            dws = std::max(dws, pbdk::dw_wgrad_workspace_floats(
                                    pbdk::DwArgs{N, L.hin, L.hin, C.L.E, C.L.k, L.stride, L.hout, L.hout}));
            if (C.L.e != 1) wws = std::max(wws, pbdk::wgrad_workspace_bytes(pw_desc(mi, L.cin, C.L.E)));
            wws = std::max(wws, pbdk::wgrad_workspace_bytes(pw_desc(mo, C.L.E, L.cout)));
          }
          L.cands.push_back(C);
        }
        L.x = x;
        if (L.stem) {
          L.y2 = act(mo, 32);
          L.a2 = act(mo, 32);
          L.dy2 = act(mo, 32);
          L.st2 = arena_.get<float>(2 * 32 * sizeof(float));
          L.red2 = arena_.get<float>(2 * 32 * sizeof(float));
          dws = std::max(dws, pbdk::stem_wgrad_workspace_floats(N, S_));
          rws = std::max(rws, pbdk::reduce_workspace_floats(static_cast<int>(mo), 32, 3));
          L.z = L.a2;
        } else {
          if (!(b == 0 && l == 1)) {  // every layer but MBConv1 has an expand conv
            L.y1 = act(mi, L.Emax);
            L.a1 = act(mi, L.Emax);
            L.g1 = act(mi, L.Emax);
            L.dy1 = act(mi, L.Emax);
            L.st1 = arena_.get<float>(2 * L.Emax * sizeof(float));
            L.red1 = arena_.get<float>(2 * L.Emax * sizeof(float));
          }
          L.y2 = act(mo, L.Emax);
          L.a2 = act(mo, L.Emax);
          L.g2 = act(mo, L.Emax);
          L.dy2 = act(mo, L.Emax);
          L.y3 = act(mo, L.cout);
          L.dy3 = act(mo, L.cout);
          L.st2 = arena_.get<float>(2 * L.Emax * sizeof(float));
          L.red2 = arena_.get<float>(2 * L.Emax * sizeof(float));
          L.st3 = arena_.get<float>(2 * L.cout * sizeof(float));
          L.red3 = arena_.get<float>(2 * L.cout * sizeof(float));
          if (!L.last) L.z = act(mo, L.cout);
          rws = std::max({rws, pbdk::reduce_workspace_floats(static_cast<int>(mi), L.Emax, 3),
                          pbdk::reduce_workspace_floats(static_cast<int>(mo), L.Emax, 3),
                          pbdk::reduce_workspace_floats(static_cast<int>(mo), L.cout, 3)});
          if (L.last) lws = pbdk::mse_affine_workspace_doubles(static_cast<long long>(mo), L.cout);
        }
        L.gz = act(mo, L.cout);
        x = L.z;
        hw = L.hout;
        for (const SCand& C : L.cands) total_ += C.L.total;
        sb.layers.push_back(std::move(L));
      }
      // gradient w.r.t. each layer's input = the previous layer's output gradient
      for (int l = 1; l < nl; ++l) sb.layers[static_cast<size_t>(l)].gx = sb.layers[static_cast<size_t>(l - 1)].gz;
      sb.rws_floats = rws;
      sb.rws = arena_.get<float>(rws * sizeof(float));
      {  // zero-initialised once; every reduction's last CTA re-zeroes it
        int cmax = 32;
        for (const SLayer& L : sb.layers) cmax = std::max({cmax, L.Emax, L.cout});
        const size_t words = pbdk::fix_acc_words(cmax);
        sb.fx.acc = arena_.get<unsigned long long>(words * sizeof(unsigned long long));
        sb.fx.ticket = arena_.get<unsigned int>(sizeof(unsigned int));
        cuda(cudaMemset(sb.fx.acc, 0, words * sizeof(unsigned long long)), "memset");
        cuda(cudaMemset(sb.fx.ticket, 0, sizeof(unsigned int)), "memset");
      }
      sb.dws_floats = dws;
      sb.dws = arena_.get<float>(dws * sizeof(float));
      sb.wws_bytes = wws;
      sb.wws = arena_.get<void>(wws);
      sb.lws = arena_.get<double>(std::max<size_t>(lws, 1) * sizeof(double));
      cuda(cudaStreamCreateWithPriority(&sb.stream, cudaStreamNonBlocking,
                                        b == hi ? priority_high() : priority_low()),
           "stream");
      cuda(cudaEventCreateWithFlags(&sb.done, cudaEventDisableTiming), "event");
      sblocks_.push_back(std::move(sb));
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
    tdone_.resize(tblocks_.size());
    for (auto& e : tdone_) cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cuda(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "event");
  }

  void build_plans() {
    for (TBlock& tb : tblocks_)
      for (TOp& op : tb.ops)
        if (op.kind == TOp::PW)
          check(pbdk::fprop_plan(pw_desc(act_rows_hw(op.hin), op.cin, op.cout), op.in, op.w, op.out, op.bias, op.aux,
                                 op.epi, &op.plan),
                "teacher 1x1 plan");
    const char* sc = pbd::knob_env("PBDK_MB_SCONV");  // student conv grid cap (experiments; 0 = all SMs)
    const pbdk::ConvGridScope scope(sc != nullptr ? std::atoi(sc) : 0);
    for (SBlock& sb : sblocks_)
      for (SLayer& L : sb.layers) {
        if (L.stem) continue;
        const size_t mi = act_rows_hw(L.hin), mo = act_rows_hw(L.hout);
        for (SCand& C : L.cands) {
          const bf16* sh = shadow_ + C.off;
          float* g = grads_ + C.off;
          if (C.L.e != 1) {
            check(pbdk::fprop_plan(pw_desc(mi, L.cin, C.L.E), L.x, sh + C.L.we, L.y1, nullptr, nullptr, PBDK_EPI_STORE,
                                   &C.p_exp),
                  "expand plan");
            check(pbdk::wgrad_plan(pw_desc(mi, L.cin, C.L.E), L.x, L.dy1, g + C.L.we, sb.wws, sb.wws_bytes, &C.w_exp),
                  "expand wgrad plan");
            if (L.need_dx)
              check(pbdk::fprop_plan(pw_desc(mi, C.L.E, L.cin), L.dy1, C.weT, L.gx, nullptr, L.res ? L.gz : nullptr,
                                     L.res ? PBDK_EPI_ADD : PBDK_EPI_STORE, &C.p_exp_dgrad),
                    "expand dgrad plan");
          }
          check(pbdk::fprop_plan(pw_desc(mo, C.L.E, L.cout), L.a2, sh + C.L.wp, L.y3, nullptr, nullptr, PBDK_EPI_STORE,
                                 &C.p_proj),
                "project plan");
          check(pbdk::wgrad_plan(pw_desc(mo, C.L.E, L.cout), L.a2, L.dy3, g + C.L.wp, sb.wws, sb.wws_bytes, &C.w_proj),
                "project wgrad plan");
          check(pbdk::fprop_plan(pw_desc(mo, L.cout, C.L.E), L.dy3, C.wpT, L.g2, nullptr, L.a2, PBDK_EPI_RELU6_MASK,
                                 &C.p_proj_dgrad),
                "project dgrad plan");
          if (pbd::pdl_enabled())
            for (pbdk::FpropPlan* f : {&C.p_exp, &C.p_exp_dgrad, &C.p_proj, &C.p_proj_dgrad}) f->pdl = true;
          if (pbd::pdl_enabled()) C.w_exp.pdl = C.w_proj.pdl = true;
        }
      }
    if (pbd::pdl_enabled())
      for (TBlock& tb : tblocks_)
        for (TOp& op : tb.ops)
          if (op.kind == TOp::PW) op.plan.pdl = true;
  }

  const Family& fam_;
  float* se_pool_ = nullptr;
  float* se_gate_ = nullptr;
  int S_ = 224;
  bf16* input_ = nullptr;
  size_t input_bytes_ = 0;
  float* stage_ = nullptr;
  float* stage2_ = nullptr;
  std::vector<TBlock> tblocks_;
  std::vector<SBlock> sblocks_;
  size_t total_ = 0;
  float *params_ = nullptr, *mom_ = nullptr, *grads_ = nullptr;
  bf16* shadow_ = nullptr;
  double* losses_ = nullptr;
  long long* step_ = nullptr;
  std::vector<cudaEvent_t> tdone_;
  cudaEvent_t fork_ = nullptr;
};

}  // namespace

PartitionBase* make_mb_partition(const pbdx_desc& d) { return new MbPartition(d); }

// layout queries for the C-ABI
int mb_layers(int model, int b) {
  FamScope fs(family(model));
  return student_layers(b);
}
int mb_cands(int model, int b, int l) {
  FamScope fs(family(model));
  return layer_cands(b, l);
}
size_t mb_offset(int model, int b, int l, int c, size_t* n) {
  FamScope fs(family(model));
  return cand_offset(b, l, c, n);
}
size_t mb_block_params(int model, int b) {
  FamScope fs(family(model));
  return block_params(b);
}

}  // namespace pbd::exec

// ------------------------------------------------------------------ C ABI: supernet layout
namespace {
bool mb_model(int m) { return m == PBDX_MODEL_MBV2_PROXYLESS || m == PBDX_MODEL_EFFB0_PROXYLESS; }
}  // namespace

extern "C" {

int pbdx_mb_layers(int model, int block) {
  if (!mb_model(model) || block < 0 || block >= pbd::exec::kBlocks) return -1;
  return pbd::exec::mb_layers(model, block);
}

int pbdx_mb_candidates(int model, int block, int layer) {
  if (pbdx_mb_layers(model, block) <= layer || layer < 0) return -1;
  return pbd::exec::mb_cands(model, block, layer);
}

long pbdx_mb_candidate_offset(int model, int block, int layer, int cand, long* count) {
  if (pbdx_mb_candidates(model, block, layer) <= cand || cand < 0) return -1;
  size_t n = 0;
  const size_t off = pbd::exec::mb_offset(model, block, layer, cand, &n);
  if (count != nullptr) *count = static_cast<long>(n);
  return static_cast<long>(off);
}

long pbdx_mb_block_params(int model, int block) {
  if (!mb_model(model) || block < 0 || block >= pbd::exec::kBlocks) return -1;
  return static_cast<long>(pbd::exec::mb_block_params(model, block));
}

}  // extern "C"
