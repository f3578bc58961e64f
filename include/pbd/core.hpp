/*
 * pbd/core.hpp — host-side API of the B200 blockwise-distillation framework.
 *
 * Drop-in for the reference's `pbd::core` C++ library: the same type names,
 * fields, function names, argument meanings and exception types as
 * proj/core/include/pbd/{errors,profile,cost_model,schedule,simulate}.hpp, so
 * reference callers (pbd_cli.cpp, the reference tests) compile against it
 * unchanged through the forwarding headers next to this file (plus pbd/report.hpp for the
 * reporting API).  Provenance of the implementation (csrc/core/): the AHD search is new — it
 * precomputes every (block range, group size) partition cost once and scans compositions over
 * that table instead of materialising ScheduleConfig objects, keeping the reference's
 * floating-point evaluation order so the chosen partition and its predicted times are
 * bit-identical.  The profile validation / JSON I/O / synth_profile (bpdg.cpp), the cost model
 * (costs.cpp) and the simulator (pipeline_sim.cpp) are close restatements of the reference's
 * profile.cpp, cost_model.cpp and simulate.cpp (Apache-2.0, The pbd Authors), because their
 * error strings and operand order are the bit-exact contract.
 *
 * Additions beyond the reference API are marked [B200].
 */
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace pbd {

// ----------------------------------------------------------------- errors
// Reference: errors.hpp:23-38.  CLI exit codes 1 / 2 / 3.
struct ValidationError : std::runtime_error {
  explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
struct InfeasibleError : std::runtime_error {
  explicit InfeasibleError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
  explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
// [B200] a CUDA / driver failure inside a device call (pbdk status PBDK_ECUDA).
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

// ----------------------------------------------------------------- BPDG / profile
// Reference: profile.hpp:30-86.  Times in ms keyed by batch (samples).
struct BlockProfile {
  int block_id = 0;
  std::map<int, double> teacher_ms;
  std::map<int, double> student_ms;
  double act_bytes_per_sample = 0.0;
  double param_bytes = 0.0;
  double teacher_param_bytes = 0.0;
  std::optional<double> dpc_ms_override;
  bool operator==(const BlockProfile&) const = default;
};

struct BpdgEdge {
  int from_block = 0;
  int to_block = 0;
  double act_bytes_per_sample = 0.0;
  bool operator==(const BpdgEdge&) const = default;
};

struct Bpdg {
  std::vector<BlockProfile> blocks;
  std::vector<BpdgEdge> edges;
  int num_blocks() const { return static_cast<int>(blocks.size()); }
  const BlockProfile& block(int id) const;
  bool operator==(const Bpdg&) const = default;
};

struct HardwareSpec {
  int num_devices = 1;
  double link_bytes_per_ms = 1.0;
  double allreduce_bytes_per_ms = 1.0;
  double mem_bytes_per_device = 1.0;
  double data_load_ms_per_batch = 0.0;
  double min_utilization_floor = 1.0;
  bool operator==(const HardwareSpec&) const = default;
};

struct ProfileDoc {
  Bpdg bpdg;
  HardwareSpec hardware;
  int global_batch = 1;
  bool operator==(const ProfileDoc&) const = default;
};

Bpdg make_bpdg(std::vector<BlockProfile> blocks);
void validate_hardware(const HardwareSpec& hw);
ProfileDoc load_profile(const std::string& text);
ProfileDoc load_profile_file(const std::string& path);
std::string save_profile(const ProfileDoc& doc);

enum class SynthShape { uniform, front_heavy, custom };
SynthShape synth_shape_from_string(const std::string& s);

struct SynthSpec {
  SynthShape shape = SynthShape::uniform;
  int blocks = 1;
  double scale_ms = 1.0;
  double front_weight = 4.0;
  std::vector<double> custom_weights;
  double curvature = 0.0;
  double jitter = 0.0;
  std::uint64_t seed = 0;
  int reference_batch = 256;
  double student_teacher_ratio = 1.0;
  double act_bytes_per_sample = 4096.0;
  double param_bytes = 1.0e6;
  double teacher_param_bytes = 2.0e6;
  HardwareSpec hardware{4, 1.0e8, 4.0e7, 1.0e15, 0.05, 0.25};
  int global_batch = 256;
};
ProfileDoc synth_profile(const SynthSpec& spec);

// ----------------------------------------------------------------- cost model
// Reference: cost_model.hpp:26-66.
enum class Role { teacher, student };

class CostModel {
 public:
  CostModel(Bpdg bpdg, HardwareSpec hw, int global_batch, double act_mem_multiplier = 3.0);
  explicit CostModel(const ProfileDoc& doc, double act_mem_multiplier = 3.0)
      : CostModel(doc.bpdg, doc.hardware, doc.global_batch, act_mem_multiplier) {}

  const Bpdg& bpdg() const { return g_; }
  const HardwareSpec& hw() const { return hw_; }
  int global_batch() const { return batch_; }
  int num_blocks() const { return g_.num_blocks(); }
  double act_mem_multiplier() const { return act_mult_; }

  double exec_time(int block, Role role, int batch) const;
  double comm_time(int block, int batch) const;
  double allreduce_time(double param_bytes, int group_size) const;
  double dpc_time(int lo, int hi, int group_size) const;
  double memory_estimate(int lo, int hi, int per_device_batch) const;

 private:
  Bpdg g_;
  HardwareSpec hw_;
  int batch_;
  double act_mult_;
};

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ----------------------------------------------------------------- schedule
// Reference: schedule.hpp:28-150.
struct PartitionSpec {
  int block_lo = 0;
  int block_hi = 0;  // inclusive
  std::vector<int> devices;
  int per_device_batch = 0;
  int num_blocks() const { return block_hi - block_lo + 1; }
  int group_size() const { return static_cast<int>(devices.size()); }
  bool operator==(const PartitionSpec&) const = default;
};

struct ScheduleFlags {
  bool tr = true;
  bool dpu = true;
  bool ahd = true;
  bool operator==(const ScheduleFlags&) const = default;
};

struct SearchProvenance {
  double search_cost_ms = 0.0;
  long configs_evaluated = 0;
};

struct ScheduleConfig {
  std::vector<PartitionSpec> partitions;
  ScheduleFlags flags;
  SearchProvenance provenance;
  int num_partitions() const { return static_cast<int>(partitions.size()); }
  bool operator==(const ScheduleConfig& o) const { return partitions == o.partitions && flags == o.flags; }
};

struct ConfigCost {
  std::vector<double> partition_ms;
  double step_ms = 0.0;
  bool feasible = true;
  std::string infeasibility_reason;
  bool operator==(const ConfigCost&) const = default;
};

enum class BaselineKind { dp, ls };

struct BaselinePlan {
  BaselineKind kind = BaselineKind::dp;
  int per_device_batch = 0;
  std::vector<double> phase_step_ms;
  std::vector<std::vector<int>> device_blocks;
  std::vector<double> device_step_ms;
  double step_ms = 0.0;
};

std::vector<ScheduleConfig> enumerate_configs(int blocks, int devices, int global_batch = 0);
void validate_schedule(const CostModel& model, const ScheduleConfig& cfg);
double partition_cost(const CostModel& model, const PartitionSpec& p);
ConfigCost predicted_step_time(const CostModel& model, const ScheduleConfig& cfg);

struct SearchOptions {
  bool contiguous_only = false;
  int threads = 0;  // accepted for API compatibility; the table search is single-pass
};

std::pair<ScheduleConfig, ConfigCost> best_schedule(const CostModel& model, const SearchOptions& opts = {});
BaselinePlan dp_schedule(const CostModel& model);
BaselinePlan ls_schedule(const CostModel& model);
ScheduleConfig ir_schedule(const CostModel& model);
double profile_drift(const Bpdg& reference, const Bpdg& observed);
std::optional<ScheduleConfig> reconfigure(const CostModel& model, const ScheduleConfig& current,
                                          const ProfileDoc& observed, double threshold);
std::string save_schedule(const ScheduleConfig& cfg, const ConfigCost& cost);
std::pair<ScheduleConfig, ConfigCost> load_schedule(const std::string& text);
std::pair<ScheduleConfig, ConfigCost> load_schedule_file(const std::string& path);

// [B200] Sample range [first, first+count) of device `rank` (0-based within its group)
// under the remainder rule of SPEC.md:231: the first (b mod g) devices take one extra.
std::pair<int, int> shard_range(int global_batch, int group_size, int rank);

// ----------------------------------------------------------------- simulator / timelines
// Reference: simulate.hpp:27-127.  The executor fills the same Event/SimReport
// types from measured CUDA-event timelines [B200].
struct SimConfig {
  int steps_per_epoch = 1;
  int epochs = 1;
  bool dpu = true;
  bool overlap_send = true;
  bool overlap_load = true;
  double epoch_sync_ms = 0.0;
  double weight_update_ms = 0.0;
  bool operator==(const SimConfig&) const = default;
};

enum class EventCategory {
  data_load,
  teacher_fwd,
  student_fwd_bwd,
  send,
  recv_wait,
  grad_share,
  weight_update,
  barrier_wait,
  idle,
};

constexpr std::array<EventCategory, 9> kAllCategories = {
    EventCategory::data_load,     EventCategory::teacher_fwd,  EventCategory::student_fwd_bwd,
    EventCategory::send,          EventCategory::recv_wait,    EventCategory::grad_share,
    EventCategory::weight_update, EventCategory::barrier_wait, EventCategory::idle,
};

const char* to_string(EventCategory c);

struct Event {
  int device = 0;
  EventCategory category = EventCategory::idle;
  std::optional<int> block;
  double start_ms = 0.0;
  double end_ms = 0.0;
  int step = 0;
  int epoch = 0;
  bool overlapped = false;
  double duration() const { return end_ms - start_ms; }
  bool operator==(const Event&) const = default;
};

struct SimReport {
  int num_devices = 0;
  SimConfig sim;
  double makespan_ms = 0.0;
  double steady_state_step_ms = 0.0;
  double bubble_ratio = 0.0;
  std::map<std::string, double> category_totals_ms;
  double overlapped_send_ms = 0.0;
  std::vector<double> peak_mem_bytes;
  std::vector<std::vector<Event>> timelines;
};

SimReport simulate(const CostModel& model, const ScheduleConfig& cfg, const SimConfig& sim);
SimReport simulate_baseline(const CostModel& model, const BaselinePlan& plan, const SimConfig& sim);
double steady_state_step_time(const SimReport& report);
double validate_prediction(const SimReport& report, const ConfigCost& cost);
std::string save_report(const SimReport& report);
// Parse a save_report() document (simulated or measured) back into a SimReport.
SimReport load_report(const std::string& text);
// Per-device Gantt chart (SVG) of a report (the role of report.cpp:93-165 gantt_svg).
std::string gantt(const SimReport& report, const std::string& title = "");

}  // namespace pbd
