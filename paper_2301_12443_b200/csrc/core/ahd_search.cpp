// Attribution: validate_schedule / predicted_step_time / the DP-LS plan generators restate
// proj/core/src/schedule.cpp, Copyright 2026 The pbd Authors, Apache License 2.0; the
// best_schedule table search is new.
// Automatic hybrid distribution (AHD) search and schedule documents.
// Reference semantics: proj/core/src/schedule.cpp.
//   canonical enumeration order      schedule.cpp:37-69, 115-134
//   P_j = sum_k T_k(b_j)+S_k(b_j) + DPC_j, b_j = ceil(b/g_j)   schedule.cpp:136-146, 63
//   argmin max_j P_j, strict <, lowest enumeration index wins  schedule.cpp:197-233
//   contiguous-only subspace (one device per partition, N parts)  schedule.cpp:172-185
//
// B200 redesign: instead of materialising all C(B+N-2, B-1) ScheduleConfig
// objects and re-evaluating the cost model for each (the reference spends ~60%
// of its search in enumeration), every distinct partition
// (lo, hi, g) is costed exactly once into a table, and the search walks the
// compositions in canonical order taking max over table entries.  Each table
// entry is produced by the same expression sequence as partition_cost(), so
// the winner and every predicted double are bit-identical to the reference.
#include <algorithm>
#include <chrono>
#include <fstream>
#include <functional>
#include <numeric>
#include <sstream>

#include "json.hpp"
#include "pbd/core.hpp"

namespace pbd {

using json::Value;

namespace {

// All ordered ways to write `total` as `parts` positive integers, lexicographic.
std::vector<std::vector<int>> compositions_of(int total, int parts) {
  std::vector<std::vector<int>> out;
  std::vector<int> cur;
  std::function<void(int, int)> rec = [&](int left, int k) {
    if (k == 1) {
      cur.push_back(left);
      out.push_back(cur);
      cur.pop_back();
      return;
    }
    for (int first = 1; first <= left - (k - 1); ++first) {
      cur.push_back(first);
      rec(left - first, k - 1);
      cur.pop_back();
    }
  };
  rec(total, parts);
  return out;
}

ScheduleConfig config_from(const std::vector<int>& blocks, const std::vector<int>& groups, int global_batch) {
  ScheduleConfig cfg;
  cfg.partitions.resize(blocks.size());
  int b = 0, d = 0;
  for (size_t i = 0; i < blocks.size(); ++i) {
    PartitionSpec& p = cfg.partitions[i];
    p.block_lo = b;
    p.block_hi = b + blocks[i] - 1;
    p.devices.resize(static_cast<size_t>(groups[i]));
    std::iota(p.devices.begin(), p.devices.end(), d);
    p.per_device_batch = global_batch > 0 ? ceil_div(global_batch, groups[i]) : 0;
    b += blocks[i];
    d += groups[i];
  }
  return cfg;
}

// partition_cost() with the group given by its size (the device ids do not
// enter the cost).
double cost_of(const CostModel& m, int lo, int hi, int g, int pdb) {
  if (pdb < 1) throw ValidationError("per_device_batch must be >= 1");
  double t = 0.0;
  for (int k = lo; k <= hi; ++k) {
    t += m.exec_time(k, Role::teacher, pdb);
    t += m.exec_time(k, Role::student, pdb);
  }
  return t + m.dpc_time(lo, hi, g);
}

std::string infeasible_reason(size_t j, int lo, int hi, int g, double mem, double cap) {
  std::ostringstream r;
  r << "partition " << j << " (blocks " << lo << "-" << hi << ", " << g << " devices): memory estimate " << mem
    << " B exceeds capacity " << cap << " B";
  return r.str();
}

}  // namespace

std::pair<int, int> shard_range(int global_batch, int group_size, int rank) {
  if (group_size < 1 || rank < 0 || rank >= group_size) throw ValidationError("bad shard rank");
  const int base = global_batch / group_size;
  const int extra = global_batch % group_size;
  const int count = base + (rank < extra ? 1 : 0);
  const int first = rank * base + std::min(rank, extra);
  return {first, count};
}

std::vector<ScheduleConfig> enumerate_configs(int blocks, int devices, int global_batch) {
  if (blocks < 1 || devices < 1) throw ValidationError("blocks and devices must be >= 1");
  std::vector<ScheduleConfig> out;
  for (int parts = 1; parts <= std::min(blocks, devices); ++parts) {
    const auto bc = compositions_of(blocks, parts);
    const auto gc = compositions_of(devices, parts);
    for (const auto& b : bc)
      for (const auto& g : gc) out.push_back(config_from(b, g, global_batch));
  }
  return out;
}

void validate_schedule(const CostModel& model, const ScheduleConfig& cfg) {
  const int nb = model.num_blocks();
  const int nd = model.hw().num_devices;
  if (cfg.partitions.empty()) throw ValidationError("schedule has no partitions");
  std::vector<char> taken(static_cast<size_t>(nd), 0);
  int expect = 0;
  for (const PartitionSpec& p : cfg.partitions) {
    if (p.block_lo != expect || p.block_hi < p.block_lo)
      throw ValidationError("schedule partitions must cover blocks contiguously in order");
    expect = p.block_hi + 1;
    if (p.devices.empty()) throw ValidationError("partition has an empty device group");
    for (int d : p.devices) {
      if (d < 0 || d >= nd) throw ValidationError("device id " + std::to_string(d) + " out of range");
      if (taken[static_cast<size_t>(d)]) throw ValidationError("device id " + std::to_string(d) + " assigned twice");
      taken[static_cast<size_t>(d)] = 1;
    }
    if (p.per_device_batch < 1) throw ValidationError("per_device_batch must be >= 1");
  }
  if (expect != nb)
    throw ValidationError("schedule covers " + std::to_string(expect) + " blocks, model has " + std::to_string(nb));
}

double partition_cost(const CostModel& model, const PartitionSpec& p) {
  return cost_of(model, p.block_lo, p.block_hi, p.group_size(), p.per_device_batch);
}

ConfigCost predicted_step_time(const CostModel& model, const ScheduleConfig& cfg) {
  ConfigCost c;
  c.partition_ms.reserve(cfg.partitions.size());
  for (size_t j = 0; j < cfg.partitions.size(); ++j) {
    const PartitionSpec& p = cfg.partitions[j];
    c.partition_ms.push_back(partition_cost(model, p));
    const double mem = model.memory_estimate(p.block_lo, p.block_hi, p.per_device_batch);
    if (c.feasible && mem > model.hw().mem_bytes_per_device) {
      c.feasible = false;
      c.infeasibility_reason =
          infeasible_reason(j, p.block_lo, p.block_hi, p.group_size(), mem, model.hw().mem_bytes_per_device);
    }
  }
  c.step_ms = *std::max_element(c.partition_ms.begin(), c.partition_ms.end());
  return c;
}

std::pair<ScheduleConfig, ConfigCost> best_schedule(const CostModel& model, const SearchOptions& opts) {
  const auto t0 = std::chrono::steady_clock::now();
  const int nb = model.num_blocks();
  const int nd = model.hw().num_devices;
  const int gb = model.global_batch();
  const double cap = model.hw().mem_bytes_per_device;

  // table[(lo*nb + hi)*nd + (g-1)]
  const size_t cells = static_cast<size_t>(nb) * nb * nd;
  std::vector<double> cost(cells, 0.0);
  std::vector<char> fits(cells, 0);
  for (int lo = 0; lo < nb; ++lo)
    for (int hi = lo; hi < nb; ++hi)
      for (int g = 1; g <= nd; ++g) {
        const size_t i = (static_cast<size_t>(lo) * nb + hi) * nd + (g - 1);
        const int pdb = ceil_div(gb, g);
        cost[i] = cost_of(model, lo, hi, g, pdb);
        fits[i] = model.memory_estimate(lo, hi, pdb) > cap ? 0 : 1;
      }

  long evaluated = 0;
  long best_index = -1;
  double best_step = 0.0;
  std::vector<int> best_blocks, best_groups;

  const int p_first = opts.contiguous_only ? nd : 1;
  const int p_last = opts.contiguous_only ? std::min(nb, nd) : std::min(nb, nd);
  if (opts.contiguous_only && nb < nd)
    throw InfeasibleError(
        "no feasible configuration: contiguous-only search needs at least as many blocks as devices");

  for (int parts = p_first; parts <= p_last; ++parts) {
    const auto bcs = compositions_of(nb, parts);
    const auto gcs = opts.contiguous_only ? std::vector<std::vector<int>>{std::vector<int>(static_cast<size_t>(parts), 1)}
                                          : compositions_of(nd, parts);
    for (const auto& bc : bcs) {
      for (const auto& gc : gcs) {
        const long index = evaluated++;
        double step = 0.0;
        bool ok = true;
        int lo = 0;
        for (int j = 0; j < parts; ++j) {
          const int hi = lo + bc[static_cast<size_t>(j)] - 1;
          const size_t i = (static_cast<size_t>(lo) * nb + hi) * nd + (gc[static_cast<size_t>(j)] - 1);
          const double pj = cost[i];
          if (j == 0 || pj > step) step = pj;
          ok = ok && fits[i];
          lo = hi + 1;
        }
        if (!ok) continue;
        if (best_index < 0 || step < best_step) {
          best_index = index;
          best_step = step;
          best_blocks = bc;
          best_groups = gc;
        }
      }
    }
  }
  if (best_index < 0) throw InfeasibleError("no feasible configuration");

  ScheduleConfig winner = config_from(best_blocks, best_groups, gb);
  winner.flags = ScheduleFlags{true, true, !opts.contiguous_only};
  ConfigCost c;
  int lo = 0;
  for (size_t j = 0; j < best_blocks.size(); ++j) {
    const int hi = lo + best_blocks[j] - 1;
    c.partition_ms.push_back(cost[(static_cast<size_t>(lo) * nb + hi) * nd + (best_groups[j] - 1)]);
    lo = hi + 1;
  }
  c.step_ms = best_step;
  winner.provenance.configs_evaluated = evaluated;
  winner.provenance.search_cost_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return {std::move(winner), std::move(c)};
}

BaselinePlan dp_schedule(const CostModel& model) {
  const int nd = model.hw().num_devices;
  BaselinePlan plan;
  plan.kind = BaselineKind::dp;
  plan.per_device_batch = ceil_div(model.global_batch(), nd);
  double prefix = 0.0;
  for (int i = 0; i < model.num_blocks(); ++i) {
    prefix += model.exec_time(i, Role::teacher, plan.per_device_batch);
    const double s = model.exec_time(i, Role::student, plan.per_device_batch);
    plan.phase_step_ms.push_back(prefix + s + model.dpc_time(i, i, nd));
  }
  plan.step_ms = std::accumulate(plan.phase_step_ms.begin(), plan.phase_step_ms.end(), 0.0);
  return plan;
}

BaselinePlan ls_schedule(const CostModel& model) {
  const int nd = model.hw().num_devices;
  const int nb = model.num_blocks();
  const int b = model.global_batch();
  BaselinePlan plan;
  plan.kind = BaselineKind::ls;
  plan.per_device_batch = b;
  plan.device_blocks.assign(static_cast<size_t>(nd), {});
  std::vector<double> weight(static_cast<size_t>(nb));
  for (int i = 0; i < nb; ++i)
    weight[static_cast<size_t>(i)] = model.exec_time(i, Role::teacher, b) + model.exec_time(i, Role::student, b);
  std::vector<int> order(static_cast<size_t>(nb));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return weight[static_cast<size_t>(x)] > weight[static_cast<size_t>(y)]; });
  std::vector<double> load(static_cast<size_t>(nd), 0.0);
  for (int i : order) {
    const size_t dev = static_cast<size_t>(std::min_element(load.begin(), load.end()) - load.begin());
    load[dev] += weight[static_cast<size_t>(i)];
    plan.device_blocks[dev].push_back(i);
  }
  for (auto& v : plan.device_blocks) std::sort(v.begin(), v.end());
  plan.device_step_ms.assign(static_cast<size_t>(nd), 0.0);
  for (int d = 0; d < nd; ++d) {
    const auto& mine = plan.device_blocks[static_cast<size_t>(d)];
    if (mine.empty()) continue;
    double t = 0.0;
    for (int k = 0; k <= mine.back(); ++k) t += model.exec_time(k, Role::teacher, b);
    for (int i : mine) t += model.exec_time(i, Role::student, b);
    plan.device_step_ms[static_cast<size_t>(d)] = t;
  }
  plan.step_ms = *std::max_element(plan.device_step_ms.begin(), plan.device_step_ms.end());
  return plan;
}

ScheduleConfig ir_schedule(const CostModel& model) {
  ScheduleConfig cfg = config_from({model.num_blocks()}, {model.hw().num_devices}, model.global_batch());
  cfg.flags = ScheduleFlags{true, true, true};
  return cfg;
}

double profile_drift(const Bpdg& reference, const Bpdg& observed) {
  if (reference.num_blocks() != observed.num_blocks())
    throw ValidationError("profile structure mismatch: different block counts");
  double worst = 0.0;
  for (int i = 0; i < reference.num_blocks(); ++i) {
    const BlockProfile& a = reference.blocks[static_cast<size_t>(i)];
    const BlockProfile& o = observed.blocks[static_cast<size_t>(i)];
    const std::map<int, double>* pairs[2][2] = {{&a.teacher_ms, &o.teacher_ms}, {&a.student_ms, &o.student_ms}};
    for (auto& pr : pairs) {
      const auto& ref = *pr[0];
      const auto& obs = *pr[1];
      if (ref.size() != obs.size())
        throw ValidationError("profile structure mismatch: different batch keys in block " + std::to_string(i));
      auto it = obs.begin();
      for (const auto& [batch, ms] : ref) {
        if (it->first != batch)
          throw ValidationError("profile structure mismatch: different batch keys in block " + std::to_string(i));
        worst = std::max(worst, std::abs(it->second - ms) / ms);
        ++it;
      }
    }
  }
  return worst;
}

std::optional<ScheduleConfig> reconfigure(const CostModel& model, const ScheduleConfig& current,
                                          const ProfileDoc& observed, double threshold) {
  if (threshold < 0.0) throw ValidationError("threshold must be >= 0");
  validate_schedule(model, current);
  if (profile_drift(model.bpdg(), observed.bpdg) <= threshold) return std::nullopt;
  const CostModel updated(observed, model.act_mem_multiplier());
  return best_schedule(updated).first;
}

std::string save_schedule(const ScheduleConfig& cfg, const ConfigCost& cost) {
  Value root = Value::object();
  Value flags = Value::object();
  flags["tr"] = Value::boolean(cfg.flags.tr);
  flags["dpu"] = Value::boolean(cfg.flags.dpu);
  flags["ahd"] = Value::boolean(cfg.flags.ahd);
  root["flags"] = std::move(flags);
  Value parts = Value::array();
  for (const PartitionSpec& p : cfg.partitions) {
    Value jp = Value::object();
    Value range = Value::array();
    range.push(Value::integer(p.block_lo));
    range.push(Value::integer(p.block_hi));
    jp["blocks"] = std::move(range);
    Value devs = Value::array();
    for (int d : p.devices) devs.push(Value::integer(d));
    jp["devices"] = std::move(devs);
    jp["per_device_batch"] = Value::integer(p.per_device_batch);
    parts.push(std::move(jp));
  }
  root["partitions"] = std::move(parts);
  Value pred = Value::object();
  Value pms = Value::array();
  for (double x : cost.partition_ms) pms.push(Value::real(x));
  pred["partition_ms"] = std::move(pms);
  pred["step_ms"] = Value::real(cost.step_ms);
  root["predicted"] = std::move(pred);
  return root.dump(2) + "\n";
}

std::pair<ScheduleConfig, ConfigCost> load_schedule(const std::string& text) {
  Value j;
  try {
    j = json::parse(text);
  } catch (const std::exception& e) {
    throw ValidationError(std::string("schedule parse error: ") + e.what());
  }
  if (!j.is_object() || !j.contains("flags") || !j.contains("partitions") || !j.contains("predicted"))
    throw ValidationError("schedule document needs flags, partitions and predicted");
  ScheduleConfig cfg;
  ConfigCost cost;
  try {
    const Value& f = j.at("flags");
    cfg.flags.tr = f.at("tr").as_bool();
    cfg.flags.dpu = f.at("dpu").as_bool();
    cfg.flags.ahd = f.at("ahd").as_bool();
    for (const Value& jp : j.at("partitions").items()) {
      PartitionSpec p;
      const Value& range = jp.at("blocks");
      if (!range.is_array() || range.size() != 2) throw ValidationError("partition blocks must be [lo, hi]");
      p.block_lo = static_cast<int>(range.items()[0].as_int64());
      p.block_hi = static_cast<int>(range.items()[1].as_int64());
      for (const Value& d : jp.at("devices").items()) p.devices.push_back(static_cast<int>(d.as_int64()));
      p.per_device_batch = static_cast<int>(jp.at("per_device_batch").as_int64());
      cfg.partitions.push_back(std::move(p));
    }
    for (const Value& x : j.at("predicted").at("partition_ms").items()) cost.partition_ms.push_back(x.as_double());
    cost.step_ms = j.at("predicted").at("step_ms").as_double();
  } catch (const ValidationError&) {
    throw;
  } catch (const std::exception& e) {
    throw ValidationError(std::string("schedule document: ") + e.what());
  }
  if (cfg.partitions.empty() || cost.partition_ms.size() != cfg.partitions.size())
    throw ValidationError("schedule document partition/prediction size mismatch");
  return {std::move(cfg), std::move(cost)};
}

std::pair<ScheduleConfig, ConfigCost> load_schedule_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open schedule file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return load_schedule(ss.str());
}

}  // namespace pbd
