/*
 * pbd_capi.h — C-ABI over the host-side Pipe-BD core (libpbd.so).
 *
 * The reference exposes its partitioner / simulator only as a C++ library
 * (pbd::core, proj/core/include/pbd/ headers) driven by the CLI
 * (proj/tools/pbd_cli.cpp:109-255).  This flat ABI carries the same documents
 * the CLI reads and writes (profile JSON, schedule JSON, report JSON) so any
 * FFI (ctypes here) can drive the same calls:
 *
 *   pbd_best_schedule        <- pbd::best_schedule       schedule.hpp:119-122 / pbd_cli.cpp:109-141
 *   pbd_predicted_step_time  <- pbd::predicted_step_time schedule.hpp:105
 *   pbd_simulate             <- pbd::simulate            simulate.hpp:106 / pbd_cli.cpp:143-170
 *   pbd_reconfigure          <- pbd::reconfigure         schedule.hpp:142-143
 *   pbd_profile_drift        <- pbd::profile_drift       schedule.hpp:137
 *   pbd_exec_time            <- pbd::CostModel::exec_time cost_model.hpp:41
 *   pbd_synth_profile        <- pbd::synth_profile       profile.hpp:136 / pbd_cli.cpp profile-gen
 *   pbd_report_steady_state  <- pbd::steady_state_step_time simulate.hpp:120 (on any report document)
 *   pbd_validate_prediction  <- pbd::validate_prediction simulate.hpp:123 (measured report vs the plan)
 *   pbd_gantt_svg            <- pbd::gantt_svg           report.hpp:44 (per-device Gantt chart)
 *
 * Return codes mirror the CLI exit codes (pbd_cli.cpp:29-32):
 *   0 ok, 1 ValidationError, 2 InfeasibleError, 3 IoError, 4 other.
 * Output strings are malloc'ed; release them with pbd_free().
 */
#ifndef PBD_CAPI_H_
#define PBD_CAPI_H_

#ifdef __cplusplus
extern "C" {
#endif

void pbd_free(char* p);

long pbd_enumerate_count(int blocks, int devices);

/* schedule_out: schedule document; meta_out: {"configs_evaluated": n, "search_cost_ms": t} */
int pbd_best_schedule(const char* profile_json, int contiguous_only, int threads, char** schedule_out,
                      char** meta_out, char** err_out);

/* cost_out: {"partition_ms": [...], "step_ms": x, "feasible": b, "reason": s} */
/* Baseline plans of the paper's comparison (schedule.cpp:246-303): kind 0 = DP (every block in turn on all
 * devices with the teacher prefix recomputed), 1 = LS (LPT block assignment, full batch per device).
 * JSON {"kind", "per_device_batch", "phase_step_ms", "device_blocks", "device_step_ms", "step_ms"}. */
int pbd_baseline_plan(const char* profile_json, int kind, char** plan_out, char** err_out);
int pbd_predicted_step_time(const char* profile_json, const char* schedule_json, char** cost_out, char** err_out);

/* sim_json: SimConfig fields (any subset); report_out: save_report() document */
int pbd_simulate(const char* profile_json, const char* schedule_json, const char* sim_json, char** report_out,
                 char** err_out);

/* schedule_out = "" when the current schedule stands */
int pbd_reconfigure(const char* profile_json, const char* schedule_json, const char* observed_json, double threshold,
                    char** schedule_out, char** err_out);

int pbd_profile_drift(const char* reference_json, const char* observed_json, double* drift_out, char** err_out);

/* role: 0 teacher, 1 student */
int pbd_exec_time(const char* profile_json, int block, int role, int batch, double* ms_out, char** err_out);

/* round-trip through load_profile/save_profile (validation) */
int pbd_load_save_profile(const char* profile_json, char** profile_out, char** err_out);

int pbd_synth_profile(const char* spec_json, char** profile_out, char** err_out);

/* shard of device `rank` in a group of `group_size` (remainder rule SPEC.md:231) */
int pbd_shard_range(int global_batch, int group_size, int rank, int* first_out, int* count_out);

/* mean wall ms of `reps` best_schedule searches (bench: host-side search cost) */
int pbd_time_best_schedule(const char* profile_json, int reps, double* ms_out, char** err_out);

/* Reports from real runs: steady-state step of a report document (simulated, or
 * measured by runtime.measured_report), |steady - predicted| / predicted for a schedule on a profile,
 * and an SVG Gantt chart of the report. */
int pbd_report_steady_state(const char* report_json, double* out, char** err_out);
int pbd_validate_prediction(const char* report_json, const char* profile_json, const char* schedule_json,
                            double* out, char** err_out);
int pbd_gantt_svg(const char* report_json, const char* title, char** svg_out, char** err_out);

#ifdef __cplusplus
}
#endif

#endif /* PBD_CAPI_H_ */
