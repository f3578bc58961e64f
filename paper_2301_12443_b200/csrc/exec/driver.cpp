// Single-process multi-GPU driver (include/pbdr.h): a whole Pipe-BD schedule in one host process,
// over the pbdx C-ABI (include/pbdx.h) and the host core's schedule type (include/pbd/core.hpp).
//
// Per schedule device ("rank"): one executor on its CUDA device with its DP shard of the global
// batch (SPEC.md:231 remainder rule), the K11 peer relay to the next partition's ranks (every
// overlapping row range of the two groups' shards) and, inside a partition with |G| > 1, the
// reduce-scatter + all-gather gradient exchange — both over CUDA peer memory with device-side
// sequence flags, so a step is one CUDA graph per rank and the host only enqueues them.
// This is the C++ form of runtime.PipeBD (placements / relay_plan / peer_wiring, runtime.py:40-199)
// for one node; the simulated counterpart is simulate.cpp:193-264.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbd/core.hpp"
#include "pbdk.h"
#include "pbdr.h"
#include "pbdx.h"

namespace {

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(int rc, const char* what) {
  if (rc != PBDK_OK) throw Fail(rc, what);
}
void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Fail(PBDK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// (first, count) of member i of a g-member group (runtime.shard)
void shard(int gb, int g, int i, int* first, int* count) {
  const int base = gb / g, extra = gb % g;
  *count = base + (i < extra ? 1 : 0);
  *first = i * base + std::min(i, extra);
}

struct Place {
  int part = -1, lo = 0, hi = 0, index = 0, first = 0, count = 0, n_max = 0;
  std::vector<int> group;
};

std::vector<Place> placements(const pbd::ScheduleConfig& s, int gb, int nranks) {
  std::vector<Place> out(static_cast<size_t>(nranks));
  for (int j = 0; j < s.num_partitions(); ++j) {
    const pbd::PartitionSpec& p = s.partitions[static_cast<size_t>(j)];
    for (int i = 0; i < p.group_size(); ++i) {
      const int r = p.devices[static_cast<size_t>(i)];
      if (r < 0 || r >= nranks || out[static_cast<size_t>(r)].part >= 0)
        throw Fail(PBDK_EINVAL, "schedule devices must be the ranks 0..R-1, each once");
      Place& pl = out[static_cast<size_t>(r)];
      pl.part = j;
      pl.lo = p.block_lo;
      pl.hi = p.block_hi;
      pl.index = i;
      pl.group = p.devices;
      shard(gb, p.group_size(), i, &pl.first, &pl.count);
      pl.n_max = std::max(pl.count, p.per_device_batch);
    }
  }
  for (const Place& pl : out)
    if (pl.part < 0) throw Fail(PBDK_EINVAL, "a rank has no slot in the schedule");
  return out;
}

struct Msg {
  int src, dst;
  long long src_row, dst_row, rows;
};

// messages across `boundary` (partition boundary-1 -> boundary), sender-major (runtime.relay_plan)
std::vector<Msg> relay_plan(const pbd::ScheduleConfig& s, int gb, int boundary) {
  const std::vector<int>& up = s.partitions[static_cast<size_t>(boundary - 1)].devices;
  const std::vector<int>& down = s.partitions[static_cast<size_t>(boundary)].devices;
  std::vector<Msg> msgs;
  for (size_t a = 0; a < up.size(); ++a) {
    int fa, ca;
    shard(gb, static_cast<int>(up.size()), static_cast<int>(a), &fa, &ca);
    for (size_t c = 0; c < down.size(); ++c) {
      int fc, cc;
      shard(gb, static_cast<int>(down.size()), static_cast<int>(c), &fc, &cc);
      const int lo = std::max(fa, fc), hi = std::min(fa + ca, fc + cc);
      if (hi > lo) msgs.push_back(Msg{up[a], down[c], lo - fa, lo - fc, hi - lo});
    }
  }
  return msgs;
}

pbd::ScheduleConfig parse(const char* json) {
  if (json == nullptr) throw Fail(PBDK_EINVAL, "no schedule");
  try {
    return pbd::load_schedule(std::string(json)).first;
  } catch (const std::exception& e) {
    throw Fail(PBDK_EINVAL, e.what());
  }
}

struct Rank {
  Place pl;
  int device = 0;
  void* ex = nullptr;
  cudaStream_t stream = nullptr;
  void *input = nullptr, *mailbox = nullptr, *grads = nullptr, *params = nullptr;
  size_t row_out = 0;
};

class Driver {
 public:
  Driver(const char* json, const pbdr_desc& d, const int* dev, int nranks) : d_(d) {
    sched_ = parse(json);
    if (nranks < 1 || dev == nullptr) throw Fail(PBDK_EINVAL, "no ranks");
    const std::vector<Place> place = placements(sched_, d.global_batch, nranks);
    ranks_.resize(static_cast<size_t>(nranks));
    for (int r = 0; r < nranks; ++r) {
      Rank& k = ranks_[static_cast<size_t>(r)];
      k.pl = place[static_cast<size_t>(r)];
      k.device = dev[r];
      cu(cudaSetDevice(k.device), "set device");
      cu(cudaStreamCreateWithFlags(&k.stream, cudaStreamNonBlocking), "stream");
      const pbdx_desc pd{k.pl.lo, k.pl.hi, k.pl.n_max, d.global_batch, d.seed_data, d.seed_teacher,
                         d.seed_student, d.lr, d.momentum, d.model, d.image};
      ck(pbdx_create(&pd, &k.ex), "pbdx_create");
      ck(pbdx_set_shard(k.ex, k.pl.count, k.pl.first), "set_shard");
      ck(pbdx_init_params(k.ex, k.stream), "init_params");
      size_t bytes = 0;
      ck(pbdx_buffer(k.ex, PBDX_BUF_INPUT, &k.input, &bytes), "buffer");
      ck(pbdx_buffer(k.ex, PBDX_BUF_MAILBOX, &k.mailbox, &bytes), "buffer");
      ck(pbdx_buffer(k.ex, PBDX_BUF_GRADS, &k.grads, &bytes), "buffer");
      ck(pbdx_buffer(k.ex, PBDX_BUF_PARAMS, &k.params, &bytes), "buffer");
      k.row_out = pbdx_relay_row_bytes(k.ex);
    }
    wire();
    for (Rank& k : ranks_) {
      cu(cudaSetDevice(k.device), "set device");
      cu(cudaStreamSynchronize(k.stream), "init");
    }
    if (d.graphs)
      for (Rank& k : ranks_) {
        cu(cudaSetDevice(k.device), "set device");
        ck(pbdx_capture(k.ex, k.stream), "capture");
      }
  }

  ~Driver() {
    for (Rank& k : ranks_) {
      if (k.ex == nullptr) continue;
      cudaSetDevice(k.device);
      cudaStreamSynchronize(k.stream);
      pbdx_destroy(k.ex);
      cudaStreamDestroy(k.stream);
    }
  }

  void step() {
    for (Rank& k : ranks_) {
      cu(cudaSetDevice(k.device), "set device");
      ck(d_.graphs ? pbdx_replay(k.ex, k.stream) : pbdx_step(k.ex, k.stream), "step");
    }
  }

  void sync() {
    for (Rank& k : ranks_) {
      cu(cudaSetDevice(k.device), "set device");
      cu(cudaStreamSynchronize(k.stream), "sync");
    }
  }

  int num_blocks() const {
    int hi = 0;
    for (const pbd::PartitionSpec& p : sched_.partitions) hi = std::max(hi, p.block_hi);
    return hi + 1;
  }

  void losses(double* out) {
    sync();
    std::fill(out, out + num_blocks(), 0.0);
    for (Rank& k : ranks_) {
      void* p = nullptr;
      size_t bytes = 0;
      ck(pbdx_buffer(k.ex, PBDX_BUF_LOSSES, &p, &bytes), "buffer");
      std::vector<double> v(bytes / sizeof(double));
      cu(cudaSetDevice(k.device), "set device");
      cu(cudaMemcpy(v.data(), p, bytes, cudaMemcpyDeviceToHost), "losses");
      for (size_t i = 0; i < v.size(); ++i) out[k.pl.lo + static_cast<int>(i)] += v[i];
    }
  }

  const Rank& rank(int r) const { return ranks_.at(static_cast<size_t>(r)); }

 private:
  void peer(const Rank& a, const Rank& b) {  // a reads / writes b's memory
    if (a.device == b.device) return;
    int can = 0;
    cu(cudaDeviceCanAccessPeer(&can, a.device, b.device), "peer query");
    if (!can) throw Fail(PBDK_ECUDA, "no peer access between the devices of two communicating ranks");
    cu(cudaSetDevice(a.device), "set device");
    const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      (void)cudaGetLastError();
      return;
    }
    cu(e, "enable peer access");
  }

  // runtime.peer_wiring: a receiver's ready slot for a sender = the sender's index among its senders;
  // a sender's consumed slot for a receiver = the receiver's index among its receivers
  void wire() {
    const int P = sched_.num_partitions();
    const int gb = d_.global_batch;
    for (int r = 0; r < static_cast<int>(ranks_.size()); ++r) {
      Rank& k = ranks_[static_cast<size_t>(r)];
      std::vector<void*> recv;
      if (k.pl.part > 0) {
        const std::vector<Msg> in = relay_plan(sched_, gb, k.pl.part);
        for (const Msg& m : in) {
          if (m.dst != r) continue;
          const Rank& src = ranks_[static_cast<size_t>(m.src)];
          int slot = 0;
          for (const Msg& o : in)  // the same boundary's messages, sender-major: src's receivers
            if (o.src == m.src) {
              if (o.dst == r) break;
              ++slot;
            }
          peer(k, src);
          recv.push_back(static_cast<unsigned long long*>(src.mailbox) + 16 + slot);
        }
      }
      ck(pbdx_relay_set_recv(k.ex, static_cast<int>(recv.size()), recv.data()), "relay_set_recv");
      std::vector<pbdx_relay_msg> send;
      if (k.pl.part + 1 < P) {
        const std::vector<Msg> out = relay_plan(sched_, gb, k.pl.part + 1);
        for (const Msg& m : out) {
          if (m.src != r) continue;
          const Rank& dst = ranks_[static_cast<size_t>(m.dst)];
          int slot = 0;
          for (const Msg& o : out)  // dst's senders in ascending order of the sender list
            if (o.dst == m.dst) {
              if (o.src == r) break;
              ++slot;
            }
          peer(k, dst);
          send.push_back(pbdx_relay_msg{m.src_row, m.rows, static_cast<char*>(dst.input) + m.dst_row * k.row_out,
                                        static_cast<unsigned long long*>(dst.mailbox) + slot});
        }
      }
      ck(pbdx_relay_set_send(k.ex, static_cast<int>(send.size()), send.data()), "relay_set_send");
      const std::vector<int>& g = k.pl.group;
      if (g.size() > 1) {
        std::vector<void*> grads, mail, params;
        for (int m : g) {
          const Rank& o = ranks_[static_cast<size_t>(m)];
          peer(k, o);
          grads.push_back(o.grads);
          mail.push_back(o.mailbox);
          params.push_back(o.params);
        }
        const int G = static_cast<int>(g.size());
        ck(pbdx_dp_set_group(k.ex, G, k.pl.index, grads.data(), mail.data()), "dp_set_group");
        ck(pbdx_dp_set_params(k.ex, G, params.data()), "dp_set_params");
      }
    }
  }

  pbdr_desc d_;
  pbd::ScheduleConfig sched_;
  std::vector<Rank> ranks_;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return PBDK_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (const std::bad_alloc&) {
    return PBDK_ECUDA;
  } catch (const std::exception&) {
    return PBDK_EINVAL;
  }
}

}  // namespace

extern "C" {

int pbdr_create(const char* schedule_json, const pbdr_desc* d, const int* device_of_rank, int nranks,
                void** handle) {
  if (d == nullptr || handle == nullptr) return PBDK_EINVAL;
  return guard([&] { *handle = new Driver(schedule_json, *d, device_of_rank, nranks); });
}

void pbdr_destroy(void* handle) { delete static_cast<Driver*>(handle); }

int pbdr_step(void* h) { return guard([&] { static_cast<Driver*>(h)->step(); }); }
int pbdr_sync(void* h) { return guard([&] { static_cast<Driver*>(h)->sync(); }); }
int pbdr_num_blocks(void* h) { return h == nullptr ? -1 : static_cast<Driver*>(h)->num_blocks(); }
int pbdr_block_losses(void* h, double* out) {
  if (h == nullptr || out == nullptr) return PBDK_EINVAL;
  return guard([&] { static_cast<Driver*>(h)->losses(out); });
}
int pbdr_rank(void* h, int r, void** ex, int* device) {
  if (h == nullptr) return PBDK_EINVAL;
  return guard([&] {
    const Rank& k = static_cast<Driver*>(h)->rank(r);
    if (ex != nullptr) *ex = k.ex;
    if (device != nullptr) *device = k.device;
  });
}

int pbdr_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

int pbdr_relay_plan(const char* schedule_json, int global_batch, int boundary, long long* out, int max_msgs) {
  try {
    const pbd::ScheduleConfig s = parse(schedule_json);
    if (boundary < 1 || boundary >= s.num_partitions() || global_batch < 1) return -PBDK_EINVAL;
    const std::vector<Msg> msgs = relay_plan(s, global_batch, boundary);
    for (size_t i = 0; i < msgs.size() && static_cast<int>(i) < max_msgs; ++i) {
      const Msg& m = msgs[i];
      const long long v[5] = {m.src, m.dst, m.src_row, m.dst_row, m.rows};
      std::memcpy(out + 5 * i, v, sizeof(v));
    }
    return static_cast<int>(msgs.size());
  } catch (const Fail& e) {
    return -e.code;
  } catch (const std::exception&) {
    return -PBDK_EINVAL;
  }
}

}  // extern "C"
