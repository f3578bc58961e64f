// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the *unmodified* reference core library (compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into oracle/_ref/).
// It lets the Python tests and bench.py's cpu_baseline leg call the reference
// partitioner / simulator with JSON documents and compare the product's
// results bit for bit.  Status codes follow the reference CLI exit codes
// (pbd_cli.cpp:29-32): 0 ok, 1 validation, 2 infeasible, 3 io.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "json.hpp"
#include "pbd/cost_model.hpp"
#include "pbd/profile.hpp"
#include "pbd/report.hpp"
#include "pbd/schedule.hpp"
#include "pbd/simulate.hpp"

using nlohmann::json;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class F>
int guarded(char** err, F&& f) {
  try {
    f();
    return 0;
  } catch (const pbd::ValidationError& e) {
    if (err) *err = dup(e.what());
    return 1;
  } catch (const pbd::InfeasibleError& e) {
    if (err) *err = dup(e.what());
    return 2;
  } catch (const pbd::IoError& e) {
    if (err) *err = dup(e.what());
    return 3;
  } catch (const std::exception& e) {
    if (err) *err = dup(e.what());
    return 4;
  }
}

pbd::SimConfig sim_from_json(const std::string& text) {
  pbd::SimConfig s;
  const json j = json::parse(text);
  if (j.contains("steps_per_epoch")) s.steps_per_epoch = j.at("steps_per_epoch").get<int>();
  if (j.contains("epochs")) s.epochs = j.at("epochs").get<int>();
  if (j.contains("dpu")) s.dpu = j.at("dpu").get<bool>();
  if (j.contains("overlap_send")) s.overlap_send = j.at("overlap_send").get<bool>();
  if (j.contains("overlap_load")) s.overlap_load = j.at("overlap_load").get<bool>();
  if (j.contains("epoch_sync_ms")) s.epoch_sync_ms = j.at("epoch_sync_ms").get<double>();
  if (j.contains("weight_update_ms")) s.weight_update_ms = j.at("weight_update_ms").get<double>();
  return s;
}

}  // namespace

extern "C" {

void ref_free(char* p) { std::free(p); }

long ref_enumerate_count(int blocks, int devices) {
  try {
    return static_cast<long>(pbd::enumerate_configs(blocks, devices).size());
  } catch (...) {
    return -1;
  }
}

// Every enumerated config as "lo-hi:g;..." lines, in enumeration order.
int ref_enumerate(int blocks, int devices, int global_batch, char** out, char** err) {
  return guarded(err, [&] {
    std::string s;
    for (const auto& c : pbd::enumerate_configs(blocks, devices, global_batch)) {
      for (const auto& p : c.partitions) {
        s += std::to_string(p.block_lo) + "-" + std::to_string(p.block_hi) + ":" + std::to_string(p.group_size()) +
             "/" + std::to_string(p.per_device_batch) + ";";
      }
      s += "\n";
    }
    *out = dup(s);
  });
}

int ref_exec_time(const char* profile, int block, int role, int batch, double* out, char** err) {
  return guarded(err, [&] {
    const pbd::CostModel m(pbd::load_profile(profile));
    *out = m.exec_time(block, role == 0 ? pbd::Role::teacher : pbd::Role::student, batch);
  });
}

// Returns the winning schedule document plus {"configs_evaluated", "search_cost_ms"} in *meta.
int ref_best_schedule(const char* profile, int contiguous_only, int threads, char** out, char** meta, char** err) {
  return guarded(err, [&] {
    const pbd::CostModel m(pbd::load_profile(profile));
    pbd::SearchOptions o;
    o.contiguous_only = contiguous_only != 0;
    o.threads = threads;
    const auto [cfg, cost] = pbd::best_schedule(m, o);
    *out = dup(pbd::save_schedule(cfg, cost));
    json jm;
    jm["configs_evaluated"] = cfg.provenance.configs_evaluated;
    jm["search_cost_ms"] = cfg.provenance.search_cost_ms;
    *meta = dup(jm.dump());
  });
}

// Times best_schedule `reps` times in-process; returns mean ms per search.
int ref_time_best_schedule(const char* profile, int threads, int reps, double* ms, char** err) {
  return guarded(err, [&] {
    const pbd::CostModel m(pbd::load_profile(profile));
    pbd::SearchOptions o;
    o.threads = threads;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) (void)pbd::best_schedule(m, o);
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / reps;
  });
}

int ref_predicted_step_time(const char* profile, const char* schedule, char** out, char** err) {
  return guarded(err, [&] {
    const pbd::CostModel m(pbd::load_profile(profile));
    const auto [cfg, unused] = pbd::load_schedule(schedule);
    (void)unused;
    const pbd::ConfigCost c = pbd::predicted_step_time(m, cfg);
    json j;
    j["partition_ms"] = c.partition_ms;
    j["step_ms"] = c.step_ms;
    j["feasible"] = c.feasible;
    j["reason"] = c.infeasibility_reason;
    *out = dup(j.dump());
  });
}

int ref_simulate(const char* profile, const char* schedule, const char* sim, char** out, char** err) {
  return guarded(err, [&] {
    const pbd::CostModel m(pbd::load_profile(profile));
    const auto [cfg, unused] = pbd::load_schedule(schedule);
    (void)unused;
    *out = dup(pbd::save_report(pbd::simulate(m, cfg, sim_from_json(sim))));
  });
}

int ref_reconfigure(const char* profile, const char* schedule, const char* observed, double threshold, char** out,
                    char** err) {
  return guarded(err, [&] {
    const pbd::CostModel m(pbd::load_profile(profile));
    const auto [cfg, unused] = pbd::load_schedule(schedule);
    (void)unused;
    const auto r = pbd::reconfigure(m, cfg, pbd::load_profile(observed), threshold);
    if (!r) {
      *out = dup("");
    } else {
      const pbd::CostModel m2(pbd::load_profile(observed), m.act_mem_multiplier());
      *out = dup(pbd::save_schedule(*r, pbd::predicted_step_time(m2, *r)));
    }
  });
}

int ref_profile_drift(const char* a, const char* b, double* out, char** err) {
  return guarded(err, [&] { *out = pbd::profile_drift(pbd::load_profile(a).bpdg, pbd::load_profile(b).bpdg); });
}

int ref_load_save_profile(const char* profile, char** out, char** err) {
  return guarded(err, [&] { *out = dup(pbd::save_profile(pbd::load_profile(profile))); });
}

// spec: {"shape","blocks","scale_ms","front_weight","custom_weights","curvature","jitter","seed",
//        "reference_batch","student_teacher_ratio","num_devices","global_batch"}
int ref_synth_profile(const char* spec_json, char** out, char** err) {
  return guarded(err, [&] {
    const json j = json::parse(spec_json);
    pbd::SynthSpec s;
    if (j.contains("shape")) s.shape = pbd::synth_shape_from_string(j.at("shape").get<std::string>());
    if (j.contains("blocks")) s.blocks = j.at("blocks").get<int>();
    if (j.contains("scale_ms")) s.scale_ms = j.at("scale_ms").get<double>();
    if (j.contains("front_weight")) s.front_weight = j.at("front_weight").get<double>();
    if (j.contains("custom_weights")) s.custom_weights = j.at("custom_weights").get<std::vector<double>>();
    if (j.contains("curvature")) s.curvature = j.at("curvature").get<double>();
    if (j.contains("jitter")) s.jitter = j.at("jitter").get<double>();
    if (j.contains("seed")) s.seed = j.at("seed").get<std::uint64_t>();
    if (j.contains("reference_batch")) s.reference_batch = j.at("reference_batch").get<int>();
    if (j.contains("student_teacher_ratio")) s.student_teacher_ratio = j.at("student_teacher_ratio").get<double>();
    if (j.contains("num_devices")) s.hardware.num_devices = j.at("num_devices").get<int>();
    if (j.contains("global_batch")) s.global_batch = j.at("global_batch").get<int>();
    *out = dup(pbd::save_profile(pbd::synth_profile(s)));
  });
}

// The reference's report API on one profile: Comparison {dp (baseline), ir, tr+dpu+ahd}, its
// speedup / breakdown tables in text, CSV and JSON, and gantt_svg of the AHD run with default and
// non-default options, concatenated with "\n@@\n" separators (tests/test_report.py renders the
// same with libpbd.so and compares the bytes).
int ref_report_render(const char* profile, const char* sim, char** out, char** err) {
  return guarded(err, [&] {
    const pbd::CostModel m(pbd::load_profile(profile));
    const pbd::SimConfig sc = sim_from_json(sim);
    const pbd::SimReport ahd = pbd::simulate(m, pbd::best_schedule(m).first, sc);
    pbd::Comparison c({{"dp", pbd::simulate_baseline(m, pbd::dp_schedule(m), sc)},
                       {"ir", pbd::simulate(m, pbd::ir_schedule(m), sc)},
                       {"tr+dpu+ahd", ahd}},
                      "dp");
    pbd::GanttOptions o;
    o.title = "pipeline";
    o.legend = false;
    o.show_overlapped_sends = false;
    o.plot_width_px = 700.0;
    o.lane_height_px = 20.0;
    const std::string sep = "\n@@\n";
    *out = dup(pbd::speedup_table(c).to_text() + sep + pbd::speedup_table(c).to_csv() + sep +
               pbd::speedup_table(c).to_json() + sep + pbd::breakdown_table(c).to_text() + sep +
               pbd::breakdown_table(c).to_csv() + sep + pbd::breakdown_table(c).to_json() + sep +
               pbd::gantt_svg(ahd) + sep + pbd::gantt_svg(ahd, o));
  });
}

}  // extern "C"
