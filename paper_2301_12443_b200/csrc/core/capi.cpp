// Flat C-ABI over the host core (declarations and reference mapping: include/pbd_capi.h).
#include "pbd_capi.h"

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "json.hpp"
#include "pbd/core.hpp"

namespace {

using pbd::json::Value;

char* heap_copy(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (p != nullptr) std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class Fn>
int shielded(char** err, Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const pbd::ValidationError& e) {
    if (err) *err = heap_copy(e.what());
    return 1;
  } catch (const pbd::InfeasibleError& e) {
    if (err) *err = heap_copy(e.what());
    return 2;
  } catch (const pbd::IoError& e) {
    if (err) *err = heap_copy(e.what());
    return 3;
  } catch (const std::exception& e) {
    if (err) *err = heap_copy(e.what());
    return 4;
  }
}

pbd::SimConfig sim_config(const char* text) {
  pbd::SimConfig s;
  if (text == nullptr || *text == '\0') return s;
  Value j;
  try {
    j = pbd::json::parse(text);
  } catch (const std::exception& e) {
    throw pbd::ValidationError(std::string("sim config parse error: ") + e.what());
  }
  if (j.contains("steps_per_epoch")) s.steps_per_epoch = static_cast<int>(j.at("steps_per_epoch").as_int64());
  if (j.contains("epochs")) s.epochs = static_cast<int>(j.at("epochs").as_int64());
  if (j.contains("dpu")) s.dpu = j.at("dpu").as_bool();
  if (j.contains("overlap_send")) s.overlap_send = j.at("overlap_send").as_bool();
  if (j.contains("overlap_load")) s.overlap_load = j.at("overlap_load").as_bool();
  if (j.contains("epoch_sync_ms")) s.epoch_sync_ms = j.at("epoch_sync_ms").as_double();
  if (j.contains("weight_update_ms")) s.weight_update_ms = j.at("weight_update_ms").as_double();
  return s;
}

}  // namespace

extern "C" {

void pbd_free(char* p) { std::free(p); }

long pbd_enumerate_count(int blocks, int devices) {
  try {
    return static_cast<long>(pbd::enumerate_configs(blocks, devices).size());
  } catch (...) {
    return -1;
  }
}

int pbd_best_schedule(const char* profile_json, int contiguous_only, int threads, char** schedule_out,
                      char** meta_out, char** err_out) {
  return shielded(err_out, [&] {
    const pbd::CostModel m(pbd::load_profile(profile_json));
    pbd::SearchOptions o;
    o.contiguous_only = contiguous_only != 0;
    o.threads = threads;
    const auto [cfg, cost] = pbd::best_schedule(m, o);
    *schedule_out = heap_copy(pbd::save_schedule(cfg, cost));
    if (meta_out != nullptr) {
      Value meta = Value::object();
      meta["configs_evaluated"] = Value::integer(cfg.provenance.configs_evaluated);
      meta["search_cost_ms"] = Value::real(cfg.provenance.search_cost_ms);
      *meta_out = heap_copy(meta.dump(-1));
    }
  });
}

int pbd_baseline_plan(const char* profile_json, int kind, char** plan_out, char** err_out) {
  return shielded(err_out, [&] {
    const pbd::CostModel m(pbd::load_profile(profile_json));
    if (kind != 0 && kind != 1) throw pbd::ValidationError("baseline kind must be 0 (dp) or 1 (ls)");
    const pbd::BaselinePlan p = kind == 0 ? pbd::dp_schedule(m) : pbd::ls_schedule(m);
    Value j = Value::object();
    j["kind"] = Value::string(kind == 0 ? "dp" : "ls");
    j["per_device_batch"] = Value::integer(p.per_device_batch);
    Value ph = Value::array();
    for (double x : p.phase_step_ms) ph.push(Value::real(x));
    j["phase_step_ms"] = std::move(ph);
    Value db = Value::array();
    for (const auto& blocks : p.device_blocks) {
      Value b = Value::array();
      for (int k : blocks) b.push(Value::integer(k));
      db.push(std::move(b));
    }
    j["device_blocks"] = std::move(db);
    Value ds = Value::array();
    for (double x : p.device_step_ms) ds.push(Value::real(x));
    j["device_step_ms"] = std::move(ds);
    j["step_ms"] = Value::real(p.step_ms);
    *plan_out = heap_copy(j.dump(-1));
  });
}

int pbd_predicted_step_time(const char* profile_json, const char* schedule_json, char** cost_out, char** err_out) {
  return shielded(err_out, [&] {
    const pbd::CostModel m(pbd::load_profile(profile_json));
    const auto sched = pbd::load_schedule(schedule_json);
    const pbd::ConfigCost c = pbd::predicted_step_time(m, sched.first);
    Value j = Value::object();
    Value pm = Value::array();
    for (double x : c.partition_ms) pm.push(Value::real(x));
    j["partition_ms"] = std::move(pm);
    j["step_ms"] = Value::real(c.step_ms);
    j["feasible"] = Value::boolean(c.feasible);
    j["reason"] = Value::string(c.infeasibility_reason);
    *cost_out = heap_copy(j.dump(-1));
  });
}

int pbd_simulate(const char* profile_json, const char* schedule_json, const char* sim_json, char** report_out,
                 char** err_out) {
  return shielded(err_out, [&] {
    const pbd::CostModel m(pbd::load_profile(profile_json));
    const auto sched = pbd::load_schedule(schedule_json);
    *report_out = heap_copy(pbd::save_report(pbd::simulate(m, sched.first, sim_config(sim_json))));
  });
}

int pbd_reconfigure(const char* profile_json, const char* schedule_json, const char* observed_json, double threshold,
                    char** schedule_out, char** err_out) {
  return shielded(err_out, [&] {
    const pbd::CostModel m(pbd::load_profile(profile_json));
    const auto sched = pbd::load_schedule(schedule_json);
    const pbd::ProfileDoc observed = pbd::load_profile(observed_json);
    const auto next = pbd::reconfigure(m, sched.first, observed, threshold);
    if (!next) {
      *schedule_out = heap_copy("");
      return;
    }
    const pbd::CostModel m2(observed, m.act_mem_multiplier());
    *schedule_out = heap_copy(pbd::save_schedule(*next, pbd::predicted_step_time(m2, *next)));
  });
}

int pbd_profile_drift(const char* reference_json, const char* observed_json, double* drift_out, char** err_out) {
  return shielded(err_out, [&] {
    *drift_out = pbd::profile_drift(pbd::load_profile(reference_json).bpdg, pbd::load_profile(observed_json).bpdg);
  });
}

int pbd_exec_time(const char* profile_json, int block, int role, int batch, double* ms_out, char** err_out) {
  return shielded(err_out, [&] {
    const pbd::CostModel m(pbd::load_profile(profile_json));
    *ms_out = m.exec_time(block, role == 0 ? pbd::Role::teacher : pbd::Role::student, batch);
  });
}

int pbd_load_save_profile(const char* profile_json, char** profile_out, char** err_out) {
  return shielded(err_out, [&] { *profile_out = heap_copy(pbd::save_profile(pbd::load_profile(profile_json))); });
}

int pbd_synth_profile(const char* spec_json, char** profile_out, char** err_out) {
  return shielded(err_out, [&] {
    Value j;
    try {
      j = pbd::json::parse(spec_json);
    } catch (const std::exception& e) {
      throw pbd::ValidationError(std::string("synth spec parse error: ") + e.what());
    }
    pbd::SynthSpec s;
    if (j.contains("shape")) s.shape = pbd::synth_shape_from_string(j.at("shape").as_string());
    if (j.contains("blocks")) s.blocks = static_cast<int>(j.at("blocks").as_int64());
    if (j.contains("scale_ms")) s.scale_ms = j.at("scale_ms").as_double();
    if (j.contains("front_weight")) s.front_weight = j.at("front_weight").as_double();
    if (j.contains("custom_weights"))
      for (const Value& w : j.at("custom_weights").items()) s.custom_weights.push_back(w.as_double());
    if (j.contains("curvature")) s.curvature = j.at("curvature").as_double();
    if (j.contains("jitter")) s.jitter = j.at("jitter").as_double();
    if (j.contains("seed")) s.seed = static_cast<std::uint64_t>(j.at("seed").as_int64());
    if (j.contains("reference_batch")) s.reference_batch = static_cast<int>(j.at("reference_batch").as_int64());
    if (j.contains("student_teacher_ratio")) s.student_teacher_ratio = j.at("student_teacher_ratio").as_double();
    if (j.contains("num_devices")) s.hardware.num_devices = static_cast<int>(j.at("num_devices").as_int64());
    if (j.contains("global_batch")) s.global_batch = static_cast<int>(j.at("global_batch").as_int64());
    *profile_out = heap_copy(pbd::save_profile(pbd::synth_profile(s)));
  });
}

int pbd_shard_range(int global_batch, int group_size, int rank, int* first_out, int* count_out) {
  char* err = nullptr;
  const int rc = shielded(&err, [&] {
    const auto [first, count] = pbd::shard_range(global_batch, group_size, rank);
    *first_out = first;
    *count_out = count;
  });
  std::free(err);
  return rc;
}

int pbd_time_best_schedule(const char* profile_json, int reps, double* ms_out, char** err_out) {
  return shielded(err_out, [&] {
    const pbd::CostModel m(pbd::load_profile(profile_json));
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) (void)pbd::best_schedule(m);
    *ms_out = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / reps;
  });
}

int pbd_report_steady_state(const char* report_json, double* out, char** err_out) {
  return shielded(err_out, [&] { *out = pbd::steady_state_step_time(pbd::load_report(report_json)); });
}

int pbd_validate_prediction(const char* report_json, const char* profile_json, const char* schedule_json,
                            double* out, char** err_out) {
  return shielded(err_out, [&] {
    const pbd::CostModel m(pbd::load_profile(profile_json));
    const auto sched = pbd::load_schedule(schedule_json);
    *out = pbd::validate_prediction(pbd::load_report(report_json), pbd::predicted_step_time(m, sched.first));
  });
}

int pbd_gantt_svg(const char* report_json, const char* title, char** svg_out, char** err_out) {
  return shielded(err_out, [&] {
    *svg_out = heap_copy(pbd::gantt(pbd::load_report(report_json), title != nullptr ? title : ""));
  });
}

}  // extern "C"
