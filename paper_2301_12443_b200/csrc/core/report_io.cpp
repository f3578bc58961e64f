// Report documents beyond the simulator: parse a save_report() document —
// simulated, or built from measured CUDA-event timelines by runtime.measured_report — back into a
// SimReport, so steady_state_step_time / validate_prediction (simulate.cpp:388-429) apply to real
// runs, and render a per-device Gantt chart of it (the role of report.cpp:93-165).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <string>

#include "json.hpp"
#include "pbd/core.hpp"

namespace pbd {

namespace {

using json::Value;

EventCategory category_from(const std::string& s) {
  for (EventCategory c : kAllCategories)
    if (s == to_string(c)) return c;
  throw ValidationError("unknown event category '" + s + "'");
}

const Value& need(const Value& o, const char* k) {
  if (!o.is_object() || !o.contains(k)) throw ValidationError(std::string("report: missing '") + k + "'");
  return o.at(k);
}

// Tableau-10 colors per category (idle is not drawn: the lane background shows through)
const char* fill_of(EventCategory c) {
  switch (c) {
    case EventCategory::data_load: return "#76b7b2";
    case EventCategory::teacher_fwd: return "#4e79a7";
    case EventCategory::student_fwd_bwd: return "#e15759";
    case EventCategory::send: return "#f28e2b";
    case EventCategory::recv_wait: return "#edc948";
    case EventCategory::grad_share: return "#b07aa1";
    case EventCategory::weight_update: return "#59a14f";
    case EventCategory::barrier_wait: return "#ff9da7";
    case EventCategory::idle: return "#bab0ac";
  }
  return "#9c755f";
}

std::string num(double v, int digits) {
  char b[48];
  std::snprintf(b, sizeof(b), "%.*f", digits, v);
  return b;
}

// "nice" axis step: 1, 2 or 5 x 10^k giving about `target` intervals
double tick_step(double span, int target) {
  const double raw = span / target;
  const double mag = std::pow(10.0, std::floor(std::log10(raw)));
  for (double m : {1.0, 2.0, 5.0, 10.0})
    if (m * mag >= raw) return m * mag;
  return 10.0 * mag;
}

}  // namespace

SimReport load_report(const std::string& text) {
  Value root;
  try {
    root = json::parse(text);
  } catch (const std::exception& e) {
    throw IoError(std::string("report: ") + e.what());
  }
  SimReport r;
  r.num_devices = static_cast<int>(need(root, "num_devices").as_int64());
  r.makespan_ms = need(root, "makespan_ms").as_double();
  if (root.contains("steady_state_step_ms")) r.steady_state_step_ms = root.at("steady_state_step_ms").as_double();
  if (root.contains("bubble_ratio")) r.bubble_ratio = root.at("bubble_ratio").as_double();
  if (root.contains("overlapped_send_ms")) r.overlapped_send_ms = root.at("overlapped_send_ms").as_double();
  if (root.contains("category_totals_ms"))
    for (const auto& [k, v] : root.at("category_totals_ms").members()) r.category_totals_ms[k] = v.as_double();
  if (root.contains("peak_mem_bytes"))
    for (const Value& v : root.at("peak_mem_bytes").items()) r.peak_mem_bytes.push_back(v.as_double());
  const Value& sim = need(root, "sim");
  r.sim.steps_per_epoch = static_cast<int>(need(sim, "steps_per_epoch").as_int64());
  r.sim.epochs = static_cast<int>(need(sim, "epochs").as_int64());
  if (sim.contains("dpu")) r.sim.dpu = sim.at("dpu").as_bool();
  if (sim.contains("overlap_send")) r.sim.overlap_send = sim.at("overlap_send").as_bool();
  if (sim.contains("overlap_load")) r.sim.overlap_load = sim.at("overlap_load").as_bool();
  if (sim.contains("epoch_sync_ms")) r.sim.epoch_sync_ms = sim.at("epoch_sync_ms").as_double();
  if (sim.contains("weight_update_ms")) r.sim.weight_update_ms = sim.at("weight_update_ms").as_double();
  int d = 0;
  for (const Value& line : need(root, "timelines").items()) {
    std::vector<Event> evs;
    for (const Value& je : line.items()) {
      Event e;
      e.device = d;
      e.category = category_from(need(je, "category").as_string());
      const Value& b = need(je, "block");
      if (!b.is_null()) e.block = static_cast<int>(b.as_int64());
      e.start_ms = need(je, "start_ms").as_double();
      e.end_ms = need(je, "end_ms").as_double();
      e.step = static_cast<int>(need(je, "step").as_int64());
      e.epoch = static_cast<int>(need(je, "epoch").as_int64());
      if (je.contains("overlapped")) e.overlapped = je.at("overlapped").as_bool();
      if (e.end_ms < e.start_ms) throw ValidationError("report: event ends before it starts");
      evs.push_back(e);
    }
    r.timelines.push_back(std::move(evs));
    ++d;
  }
  if (static_cast<int>(r.timelines.size()) != r.num_devices) throw ValidationError("report: timelines != num_devices");
  return r;
}

std::string gantt(const SimReport& r, const std::string& title) {
  if (r.timelines.empty() || r.makespan_ms <= 0.0) throw ValidationError("gantt: empty report");
  const double label_w = 72.0, plot_w = 1000.0, row_h = 26.0, pad = 10.0;
  const double head = title.empty() ? pad : 30.0;
  const int lanes = static_cast<int>(r.timelines.size());
  const double axis_y = head + lanes * row_h;
  const double legend_y = axis_y + 34.0;
  const double W = label_w + plot_w + 2 * pad, H = legend_y + 22.0;
  const double sx = plot_w / r.makespan_ms;
  std::ostringstream o;
  o << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << num(W, 0) << "\" height=\"" << num(H, 0)
    << "\" font-family=\"Helvetica,Arial,sans-serif\" font-size=\"11\">\n";
  if (!title.empty()) o << "<text x=\"" << num(label_w, 1) << "\" y=\"20\" font-size=\"13\">" << title << "</text>\n";
  for (int d = 0; d < lanes; ++d) {
    const double y = head + d * row_h;
    o << "<rect x=\"" << num(label_w, 1) << "\" y=\"" << num(y, 1) << "\" width=\"" << num(plot_w, 1)
      << "\" height=\"" << num(row_h - 2, 1) << "\" fill=\"" << (d % 2 ? "#f7f7f7" : "#eeeeee") << "\"/>\n";
    o << "<text x=\"" << num(pad, 1) << "\" y=\"" << num(y + row_h * 0.62, 1) << "\">GPU " << d << "</text>\n";
    for (const Event& e : r.timelines[static_cast<size_t>(d)]) {
      if (e.category == EventCategory::idle || e.duration() <= 0.0) continue;
      const double x = label_w + e.start_ms * sx, w = std::max(0.5, e.duration() * sx);
      // overlapped work (relay sends, concurrent student streams) is drawn as a thin band
      const double yy = e.overlapped ? y + row_h * 0.62 : y + 1.0;
      const double hh = e.overlapped ? row_h * 0.3 : row_h - 4.0;
      o << "<rect x=\"" << num(x, 2) << "\" y=\"" << num(yy, 1) << "\" width=\"" << num(w, 2) << "\" height=\""
        << num(hh, 1) << "\" fill=\"" << fill_of(e.category) << "\"><title>" << to_string(e.category);
      if (e.block) o << " b" << *e.block;
      o << " step " << e.step << ": " << num(e.start_ms, 3) << "-" << num(e.end_ms, 3) << " ms</title></rect>\n";
    }
  }
  o << "<line x1=\"" << num(label_w, 1) << "\" y1=\"" << num(axis_y, 1) << "\" x2=\"" << num(label_w + plot_w, 1)
    << "\" y2=\"" << num(axis_y, 1) << "\" stroke=\"#444\"/>\n";
  const double step = tick_step(r.makespan_ms, 8);
  for (double t = 0.0; t <= r.makespan_ms + 1e-9; t += step) {
    const double x = label_w + t * sx;
    o << "<line x1=\"" << num(x, 2) << "\" y1=\"" << num(axis_y, 1) << "\" x2=\"" << num(x, 2) << "\" y2=\""
      << num(axis_y + 5, 1) << "\" stroke=\"#444\"/>\n";
    o << "<text x=\"" << num(x, 2) << "\" y=\"" << num(axis_y + 17, 1) << "\" text-anchor=\"middle\">"
      << num(t, step < 1.0 ? 2 : 1) << "</text>\n";
  }
  o << "<text x=\"" << num(label_w + plot_w, 1) << "\" y=\"" << num(axis_y + 30, 1)
    << "\" text-anchor=\"end\">ms</text>\n";
  double lx = label_w;
  for (EventCategory c : kAllCategories) {
    if (c == EventCategory::idle) continue;
    o << "<rect x=\"" << num(lx, 1) << "\" y=\"" << num(legend_y, 1) << "\" width=\"10\" height=\"10\" fill=\""
      << fill_of(c) << "\"/><text x=\"" << num(lx + 14, 1) << "\" y=\"" << num(legend_y + 9, 1) << "\">"
      << to_string(c) << "</text>\n";
    lx += 24.0 + 6.5 * std::string(to_string(c)).size();
  }
  o << "</svg>\n";
  return o.str();
}

}  // namespace pbd
