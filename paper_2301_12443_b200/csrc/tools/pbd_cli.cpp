// pbd — command line over the host core (the drop-in for proj/tools/pbd_cli.cpp:109-379; CLI11 is
// not in this image, so arguments are parsed by hand).  Subcommands and the exit-code contract
// (pbd_cli.cpp:29-32: 0 ok, 1 validation, 2 infeasible, 3 I/O):
//
//   pbd schedule <profile|-> [--no-ahd] [--devices N] [--threads N] [--out F] [--format text|json]
//   pbd simulate <schedule|-> <profile> [--steps N] [--epochs N] [--dpu on|off] [--overlap-send on|off]
//                [--overlap-load on|off] [--epoch-sync-ms X] [--weight-update-ms X] [--gantt F.svg]
//                [--out F] [--format text|json]
//   pbd compare <profile|-> --against dp,ls,ir [--ablation tr,tr+dpu,tr+dpu+ahd] [sim flags]
//               [--out F] [--format text|csv|json]
//   pbd profile-gen --blocks N [--shape uniform|front-heavy|custom] [--scale X] [--weight X]
//               [--weights a,b,..] [--curve X] [--jitter X] [--seed N] [--student-ratio X]
//               [--devices N] [--global-batch N] [--reference-batch N] [--load-ms X] [--mem-bytes X]
//               [--out F]
//   pbd report <report.json> [--gantt F.svg] [--profile P --schedule S]   (measured runs, §8f)
//   pbd run <schedule|-> --global-batch N [--steps N] [--warmup N] [--devices d0,d1,..]
//           [--model resnet|resnet_fp32|mbv2|effb0] [--image S] [--eager]
//       runs the schedule on the GPUs of this node in ONE process through the C++ driver
//       (include/pbdr.h): rank r of the schedule on CUDA device d_r (default: rank r % #devices),
//       peer relay + peer DP exchange, one CUDA graph per rank; prints ms/step and block losses.
//
// The torch.distributed flavour (one process per GPU, measured profiles, checkpoints) is
// `python -m paper_2301_12443_b200.cli profile|run`.
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <iterator>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include <chrono>

#include "pbd/core.hpp"
#include "pbd/report.hpp"
#include "pbdr.h"
#include "pbdx.h"

namespace {

constexpr int kOk = 0, kValidation = 1, kInfeasible = 2, kIo = 3;

struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    const auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
};

Args parse(int argc, char** argv, int first, const std::set<std::string>& bool_flags) {
  Args a;
  for (int i = first; i < argc; ++i) {
    const std::string s = argv[i];
    if (s.size() > 2 && s.rfind("--", 0) == 0) {
      std::string key = s.substr(2), val;
      const auto eq = key.find('=');
      if (eq != std::string::npos) {
        val = key.substr(eq + 1);
        key = key.substr(0, eq);
        a.opt[key] = val;
      } else if (bool_flags.count(key)) {
        a.flags.insert(key);
      } else {
        if (i + 1 >= argc) throw pbd::ValidationError("option --" + key + " needs a value");
        a.opt[key] = argv[++i];
      }
    } else {
      a.pos.push_back(s);
    }
  }
  return a;
}

std::string read_all(std::istream& in) { return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()}; }

std::string read_doc(const std::string& path) {
  if (path == "-") return read_all(std::cin);
  std::ifstream f(path);
  if (!f) throw pbd::IoError("cannot read " + path);
  return read_all(f);
}

void write_doc(const std::string& text, const std::string& path) {
  if (path.empty() || path == "-") {
    std::cout << text;
    return;
  }
  std::ofstream f(path);
  if (!f || !(f << text)) throw pbd::IoError("cannot write " + path);
}

double num(const std::string& s, const char* what) {
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (s.empty() || *end != '\0') throw pbd::ValidationError(std::string("bad number for ") + what + ": " + s);
  return v;
}

bool on_off(const std::string& s, const char* what) {
  if (s == "on") return true;
  if (s == "off") return false;
  throw pbd::ValidationError(std::string(what) + " must be on|off");
}

std::vector<std::string> csv(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

pbd::SimConfig sim_config(const Args& a, bool dpu_default) {
  pbd::SimConfig c;
  c.steps_per_epoch = static_cast<int>(num(a.get("steps", "16"), "--steps"));
  c.epochs = static_cast<int>(num(a.get("epochs", "1"), "--epochs"));
  c.dpu = a.has("dpu") ? on_off(a.get("dpu"), "--dpu") : dpu_default;
  c.overlap_send = on_off(a.get("overlap-send", "on"), "--overlap-send");
  c.overlap_load = on_off(a.get("overlap-load", "on"), "--overlap-load");
  c.epoch_sync_ms = num(a.get("epoch-sync-ms", "0"), "--epoch-sync-ms");
  c.weight_update_ms = num(a.get("weight-update-ms", "0"), "--weight-update-ms");
  return c;
}

// shortest round-trip form, integral values with ".0" (the JSON documents' number format)
std::string shortest(double v) {
  char b[64];
  const auto r = std::to_chars(b, b + sizeof(b), v);
  std::string t(b, r.ptr);
  if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
  return t;
}

std::string fixed(double v, int digits = 6) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.*f", digits, v);
  return b;
}

int cmd_schedule(const Args& a) {
  if (a.pos.size() != 1) throw pbd::ValidationError("usage: pbd schedule <profile|-> [options]");
  pbd::ProfileDoc doc = pbd::load_profile(read_doc(a.pos[0]));
  if (a.has("devices")) doc.hardware.num_devices = static_cast<int>(num(a.get("devices"), "--devices"));
  const pbd::CostModel model(doc);
  pbd::SearchOptions o;
  o.contiguous_only = a.flags.count("no-ahd") != 0;
  o.threads = static_cast<int>(num(a.get("threads", "0"), "--threads"));
  const auto [cfg, cost] = pbd::best_schedule(model, o);
  const std::string document = pbd::save_schedule(cfg, cost);
  const std::string summary = "configs evaluated: " + std::to_string(cfg.provenance.configs_evaluated) +
                              "\npredicted step time: " + fixed(cost.step_ms) + " ms\npartitions: " +
                              std::to_string(cfg.num_partitions()) + "\n";
  std::fprintf(stderr, "search took %.3f ms\n", cfg.provenance.search_cost_ms);
  const std::string fmt = a.get("format", "text");
  if (a.has("out")) {
    write_doc(document, a.get("out"));
    std::cout << summary;
  } else if (fmt == "json") {
    std::cout << document;
    std::cerr << summary;
  } else {
    std::cout << summary << document;
  }
  return kOk;
}

int cmd_simulate(const Args& a) {
  if (a.pos.size() != 2) throw pbd::ValidationError("usage: pbd simulate <schedule|-> <profile> [options]");
  const auto [cfg, predicted] = pbd::load_schedule(read_doc(a.pos[0]));
  const pbd::CostModel model(pbd::load_profile(read_doc(a.pos[1])));
  const pbd::SimReport r = pbd::simulate(model, cfg, sim_config(a, cfg.flags.dpu));
  if (a.has("gantt")) write_doc(pbd::gantt(r), a.get("gantt"));
  if (a.get("format", "text") == "json" || a.has("out")) {
    write_doc(pbd::save_report(r), a.get("out"));
    return kOk;
  }
  std::cout << "makespan: " << r.makespan_ms << " ms\nsteady-state step: " << r.steady_state_step_ms
            << " ms\npredicted step: " << predicted.step_ms << " ms\nbubble ratio: " << r.bubble_ratio
            << "\nper-device totals (ms):\n";
  for (const auto& [k, v] : r.category_totals_ms) std::cout << "  " << k << ": " << v / r.num_devices << "\n";
  return kOk;
}

int cmd_compare(const Args& a) {
  if (a.pos.size() != 1) throw pbd::ValidationError("usage: pbd compare <profile|-> --against dp,ls,ir");
  const pbd::CostModel model(pbd::load_profile(read_doc(a.pos[0])));
  const auto base = csv(a.get("against"));
  const auto abl = csv(a.get("ablation"));
  if (base.empty()) throw pbd::ValidationError("--against needs at least one of dp,ls,ir");
  std::vector<std::string> labels = base;
  labels.insert(labels.end(), abl.begin(), abl.end());
  std::set<std::string> seen;
  for (const auto& l : labels) {
    static const std::set<std::string> known{"dp", "ls", "ir", "tr", "tr+dpu", "tr+dpu+ahd"};
    if (!known.count(l)) throw pbd::ValidationError("unknown comparison label \"" + l + "\"");
    if (!seen.insert(l).second) throw pbd::ValidationError("duplicate comparison label \"" + l + "\"");
  }
  std::optional<pbd::ScheduleConfig> contiguous;
  auto run = [&](const std::string& l) {
    if (l == "dp") return pbd::simulate_baseline(model, pbd::dp_schedule(model), sim_config(a, true));
    if (l == "ls") return pbd::simulate_baseline(model, pbd::ls_schedule(model), sim_config(a, true));
    if (l == "ir") return pbd::simulate(model, pbd::ir_schedule(model), sim_config(a, true));
    if (l == "tr+dpu+ahd") {
      pbd::SimConfig c = sim_config(a, true);
      c.dpu = true;
      return pbd::simulate(model, pbd::best_schedule(model).first, c);
    }
    if (!contiguous) contiguous = pbd::best_schedule(model, pbd::SearchOptions{true, 0}).first;
    pbd::SimConfig c = sim_config(a, l == "tr+dpu");
    c.dpu = l == "tr+dpu";
    return pbd::simulate(model, *contiguous, c);
  };
  std::vector<std::pair<std::string, pbd::SimReport>> rows;
  for (const auto& l : labels) rows.emplace_back(l, run(l));
  // the reference's report API (pbd/report.hpp, pbd_cli.cpp:238-252 of the reference)
  const pbd::Comparison cmp(std::move(rows), base.front());
  const pbd::Table speed = pbd::speedup_table(cmp), split = pbd::breakdown_table(cmp);
  const std::string fmt = a.get("format", "text");
  std::ostringstream o;
  if (fmt == "json") {  // {"baseline", "breakdown": rows of breakdown_table, "speedup": label -> ratio}
    std::string rows_json = split.to_json();
    rows_json.pop_back();
    for (size_t p = rows_json.find('\n'); p != std::string::npos; p = rows_json.find('\n', p + 3))
      rows_json.replace(p, 1, "\n  ");
    o << "{\n  \"baseline\": \"" << cmp.baseline_label << "\",\n  \"breakdown\": " << rows_json
      << ",\n  \"speedup\": {";
    bool first = true;
    for (const auto& [l, v] : pbd::speedup(cmp)) {
      o << (first ? "\n" : ",\n") << "    \"" << l << "\": " << shortest(v);
      first = false;
    }
    o << "\n  }\n}\n";
  } else if (fmt == "csv") {
    o << speed.to_csv() << "\n" << split.to_csv();
  } else {
    o << "== speedup vs " << cmp.baseline_label << " ==\n"
      << speed.to_text() << "\n== breakdown (per-device ms) ==\n" << split.to_text();
  }
  write_doc(o.str(), a.get("out"));
  return kOk;
}

int cmd_profile_gen(const Args& a) {
  pbd::SynthSpec s;
  if (!a.has("blocks")) throw pbd::ValidationError("--blocks is required");
  s.blocks = static_cast<int>(num(a.get("blocks"), "--blocks"));
  s.shape = pbd::synth_shape_from_string(a.get("shape", "uniform"));
  if (a.has("scale")) s.scale_ms = num(a.get("scale"), "--scale");
  if (a.has("weight")) s.front_weight = num(a.get("weight"), "--weight");
  for (const auto& w : csv(a.get("weights"))) s.custom_weights.push_back(num(w, "--weights"));
  if (a.has("curve")) s.curvature = num(a.get("curve"), "--curve");
  if (a.has("jitter")) s.jitter = num(a.get("jitter"), "--jitter");
  if (a.has("seed")) s.seed = static_cast<std::uint64_t>(num(a.get("seed"), "--seed"));
  if (a.has("student-ratio")) s.student_teacher_ratio = num(a.get("student-ratio"), "--student-ratio");
  if (a.has("devices")) s.hardware.num_devices = static_cast<int>(num(a.get("devices"), "--devices"));
  if (a.has("global-batch")) s.global_batch = static_cast<int>(num(a.get("global-batch"), "--global-batch"));
  if (a.has("reference-batch")) s.reference_batch = static_cast<int>(num(a.get("reference-batch"), "--reference-batch"));
  if (a.has("load-ms")) s.hardware.data_load_ms_per_batch = num(a.get("load-ms"), "--load-ms");
  if (a.has("mem-bytes")) s.hardware.mem_bytes_per_device = num(a.get("mem-bytes"), "--mem-bytes");
  write_doc(pbd::save_profile(pbd::synth_profile(s)), a.get("out"));
  return kOk;
}

int cmd_report(const Args& a) {
  if (a.pos.size() != 1) throw pbd::ValidationError("usage: pbd report <report.json> [--gantt F] [--profile P --schedule S]");
  const pbd::SimReport r = pbd::load_report(read_doc(a.pos[0]));
  if (a.has("gantt")) write_doc(pbd::gantt(r, a.get("title")), a.get("gantt"));
  std::cout << "devices: " << r.num_devices << "\nmakespan: " << r.makespan_ms << " ms\n";
  if (r.sim.steps_per_epoch >= 4) std::cout << "steady-state step: " << pbd::steady_state_step_time(r) << " ms\n";
  if (a.has("profile") && a.has("schedule")) {
    const pbd::CostModel m(pbd::load_profile(read_doc(a.get("profile"))));
    const auto sched = pbd::load_schedule(read_doc(a.get("schedule")));
    const pbd::ConfigCost c = pbd::predicted_step_time(m, sched.first);
    std::cout << "predicted step: " << c.step_ms << " ms\nrelative error: " << pbd::validate_prediction(r, c) << "\n";
  }
  return kOk;
}

int cmd_run(const Args& a) {
  if (a.pos.size() != 1 || !a.has("global-batch"))
    throw pbd::ValidationError("usage: pbd run <schedule|-> --global-batch N [--steps N] [--devices d0,d1,..]");
  const std::string text = read_doc(a.pos[0]);
  const auto sched = pbd::load_schedule(text).first;
  int nranks = 0;
  for (const auto& p : sched.partitions) nranks += p.group_size();
  const int ndev = pbdr_device_count();
  if (ndev < 1) throw pbd::IoError("no CUDA device");
  std::vector<int> dev(static_cast<size_t>(nranks));
  for (int r = 0; r < nranks; ++r) dev[static_cast<size_t>(r)] = r % ndev;
  if (a.has("devices")) {
    std::stringstream ss(a.get("devices"));
    std::string item;
    for (int r = 0; std::getline(ss, item, ','); ++r) {
      if (r >= nranks) throw pbd::ValidationError("--devices: more entries than schedule ranks");
      dev[static_cast<size_t>(r)] = static_cast<int>(num(item, "--devices"));
    }
  }
  const std::string model = a.get("model", "resnet");
  const int m = model == "resnet" ? PBDX_MODEL_RESNET_CIFAR : model == "resnet_fp32" ? PBDX_MODEL_RESNET_CIFAR_FP32
              : model == "mbv2" ? PBDX_MODEL_MBV2_PROXYLESS : model == "effb0" ? PBDX_MODEL_EFFB0_PROXYLESS : -1;
  if (m < 0) throw pbd::ValidationError("--model resnet|resnet_fp32|mbv2|effb0");
  const int image = a.has("image") ? static_cast<int>(num(a.get("image"), "--image"))
                                   : (m == PBDX_MODEL_RESNET_CIFAR || m == PBDX_MODEL_RESNET_CIFAR_FP32 ? 32 : 224);
  const pbdr_desc d{static_cast<int>(num(a.get("global-batch"), "--global-batch")), m, image, 1234u, 1u, 2u, 0.1f,
                    0.9f, a.flags.count("eager") ? 0 : 1};
  void* h = nullptr;
  if (pbdr_create(text.c_str(), &d, dev.data(), nranks, &h) != 0) throw pbd::IoError("driver setup failed (device)");
  const int steps = static_cast<int>(num(a.get("steps", "20"), "--steps"));
  const int warmup = static_cast<int>(num(a.get("warmup", "3"), "--warmup"));
  int rc = 0;
  for (int i = 0; i < warmup && rc == 0; ++i) rc = pbdr_step(h);
  if (rc == 0) rc = pbdr_sync(h);
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps && rc == 0; ++i) rc = pbdr_step(h);
  if (rc == 0) rc = pbdr_sync(h);
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::vector<double> losses(static_cast<size_t>(std::max(1, pbdr_num_blocks(h))));
  if (rc == 0) rc = pbdr_block_losses(h, losses.data());
  pbdr_destroy(h);
  if (rc != 0) throw pbd::IoError("device step failed");
  std::cout << "ranks: " << nranks << "\nms/step: " << ms / std::max(1, steps) << " (host wall clock, " << steps
            << " steps)\nsamples/s: " << d.global_batch * std::max(1, steps) / (ms * 1e-3) << "\nblock losses:";
  for (double l : losses) std::cout << " " << l;
  std::cout << "\n";
  return kOk;
}

void usage() {
  std::cerr << "usage: pbd <schedule|simulate|compare|profile-gen|report|run> ...  (see the header of csrc/tools/pbd_cli.cpp)\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return kValidation;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "schedule") return cmd_schedule(parse(argc, argv, 2, {"no-ahd"}));
    if (cmd == "simulate") return cmd_simulate(parse(argc, argv, 2, {}));
    if (cmd == "compare") return cmd_compare(parse(argc, argv, 2, {}));
    if (cmd == "profile-gen") return cmd_profile_gen(parse(argc, argv, 2, {}));
    if (cmd == "report") return cmd_report(parse(argc, argv, 2, {}));
    if (cmd == "run") return cmd_run(parse(argc, argv, 2, {"eager"}));
    if (cmd == "-h" || cmd == "--help") {
      usage();
      return kOk;
    }
    usage();
    return kValidation;
  } catch (const pbd::ValidationError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kValidation;
  } catch (const pbd::InfeasibleError& e) {
    std::cerr << "infeasible: " << e.what() << "\n";
    return kInfeasible;
  } catch (const pbd::IoError& e) {
    std::cerr << "io error: " << e.what() << "\n";
    return kIo;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kValidation;
  }
}
