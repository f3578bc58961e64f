"""pbd/report.hpp drop-in (reference: proj/core/include/pbd/report.hpp:26-64).

* a consumer written like proj/tests/report_test.cpp (same headers, names and calls) compiles
  against include/ and links libpbd.so alone; it re-asserts that test file's golden values;
* the tables (text / CSV / JSON) and the Gantt SVGs are byte-identical to the reference core
  compiled unmodified (oracle/_ref) on the same profiles.
"""
import os
import subprocess

import pytest

from oracle import ref
from tests.profiles import random_doc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2301_12443_b200", "lib", "libpbd.so")

CONSUMER = r'''
#include "pbd/report.hpp"
#include "pbd/schedule.hpp"
#include "pbd/simulate.hpp"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>

#define CHECK(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); return 1; } } while (0)

using namespace pbd;

// proportional_doc of proj/tests/testutil.hpp:51-83: T_k(b) = t_k * b / ref at keys {ref/4, ref/2, ref}
ProfileDoc proportional(std::vector<double> t, std::vector<double> s, int devices, int batch) {
  std::vector<BlockProfile> blocks;
  for (size_t k = 0; k < t.size(); ++k) {
    BlockProfile b;
    b.block_id = static_cast<int>(k);
    for (int key : {batch / 4, batch / 2, batch}) {
      b.teacher_ms[key] = t[k] * key / batch;
      b.student_ms[key] = s[k] * key / batch;
    }
    b.act_bytes_per_sample = 0.0;
    b.param_bytes = 0.0;
    b.teacher_param_bytes = 0.0;
    blocks.push_back(b);
  }
  ProfileDoc d;
  d.bpdg = make_bpdg(blocks);
  d.hardware.num_devices = devices;
  d.hardware.link_bytes_per_ms = 1e9;
  d.hardware.allreduce_bytes_per_ms = 1e9;
  d.hardware.mem_bytes_per_device = 1e18;
  d.hardware.data_load_ms_per_batch = 0.0;
  d.hardware.min_utilization_floor = 1.0;
  d.global_batch = batch;
  return d;
}

SimReport balanced(bool dpu) {
  const CostModel model(proportional({2.0, 2.0}, {3.0, 3.0}, 2, 256));
  ScheduleConfig cfg;
  cfg.partitions = {{0, 0, {0}, 256}, {1, 1, {1}, 256}};
  SimConfig sim;
  sim.steps_per_epoch = 10;
  sim.dpu = dpu;
  return simulate(model, cfg, sim);
}

int main(int argc, char** argv) {
  {  // report_test.cpp:88-107 DrawsEveryBusyEvent
    ProfileDoc doc = proportional({2.0}, {3.0}, 1, 256);
    doc.hardware.data_load_ms_per_batch = 1.0;
    const CostModel model(doc);
    ScheduleConfig cfg;
    cfg.partitions = {{0, 0, {0}, 256}};
    const std::string svg = gantt_svg(simulate(model, cfg, SimConfig{}));
    size_t rects = 0;
    for (size_t p = svg.find("<rect"); p != std::string::npos; p = svg.find("<rect", p + 1)) ++rects;
    CHECK(rects >= 3);
    CHECK(svg.find("#8dd3c7") != std::string::npos);
    CHECK(svg.find("#80b1d3") != std::string::npos);
    CHECK(svg.find("#fb8072") != std::string::npos);
  }
  {  // :114-135 SecondLaneStartsAtTheRelayOffset, OutputIsDeterministic
    const SimReport r = balanced(true);
    CHECK(gantt_svg(r) == gantt_svg(r));
    char want[64];
    std::snprintf(want, sizeof(want), "x=\"%.2f\"", 64.0 + 2.0 * (960.0 / r.makespan_ms));
    CHECK(gantt_svg(r).find(want) != std::string::npos);
    GanttOptions o;
    o.title = "pipeline";
    o.legend = false;
    CHECK(gantt_svg(balanced(false), o).find("pipeline") != std::string::npos);
    SimReport empty;
    bool threw = false;
    try { gantt_svg(empty); } catch (const ValidationError&) { threw = true; }
    CHECK(threw);
  }
  {  // :146-163 Breakdown
    Comparison c({{"dpu", balanced(true)}, {"barrier", balanced(false)}}, "barrier");
    const auto totals = breakdown_totals(c);
    for (const auto& [label, r] : c.entries)
      for (const auto& [cat, ms] : r.category_totals_ms) CHECK(std::fabs(totals.at(label).at(cat) * r.num_devices - ms) < 1e-9);
    CHECK(breakdown_table(c).rows.size() == 2 && breakdown_table(c).columns.front() == "label");
    Comparison one({{"pbd", balanced(true)}}, "pbd");
    CHECK(std::fabs(breakdown_totals(one).at("pbd").at("idle")) < 1e-9);
  }
  {  // :165-193 Speedup
    Comparison c({{"dp", balanced(false)}, {"pbd", balanced(true)}}, "dp");
    CHECK(speedup(c).at("dp") == 1.0);
    CHECK(std::fabs(speedup(c).at("pbd") - 1.3461538461538463) < 1e-12);
    SimReport dp = balanced(false), pb = balanced(true);
    dp.makespan_ms = 31520.0;
    pb.makespan_ms = 10230.0;
    CHECK(std::fabs(speedup(Comparison({{"dp", dp}, {"pbd", pb}}, "dp")).at("pbd") - 3.081) < 1e-3);
    pb.makespan_ms = 0.0;
    bool threw = false;
    try { speedup(Comparison({{"dp", dp}, {"broken", pb}}, "dp")); } catch (const ValidationError&) { threw = true; }
    CHECK(threw);
  }
  {  // :195-199 ValidatesLabels
    int n = 0;
    try { Comparison({{"a", balanced(true)}, {"a", balanced(true)}}, "a"); } catch (const ValidationError&) { ++n; }
    try { Comparison({{"a", balanced(true)}}, "missing"); } catch (const ValidationError&) { ++n; }
    CHECK(n == 2);
  }
  {  // :201-212 RenderInEveryFormat
    Comparison c({{"dp", balanced(false)}, {"pbd", balanced(true)}}, "dp");
    const Table t = speedup_table(c);
    CHECK(t.to_text().find("speedup") != std::string::npos);
    const std::string csv = t.to_csv();
    int lines = 0;
    for (char ch : csv) lines += ch == '\n';
    CHECK(lines == 3);
    CHECK(t.to_json().find("\"label\": \"pbd\"") != std::string::npos);
  }
  {  // :214-231 TeacherRedundancyIsVisible
    const CostModel m(proportional({2.0, 2.0}, {3.0, 3.0}, 2, 256));
    SimConfig sim;
    sim.steps_per_epoch = 10;
    Comparison c({{"dp", simulate_baseline(m, dp_schedule(m), sim)}, {"pbd", simulate(m, ir_schedule(m), sim)}}, "dp");
    const auto t = breakdown_totals(c);
    CHECK(std::fabs(t.at("dp").at("teacher_fwd") - t.at("pbd").at("teacher_fwd") -
                    10.0 * m.exec_time(0, Role::teacher, 128)) < 1e-9);
  }
  if (argc == 3) {  // render the same documents as oracle/ref_shim.cpp:ref_report_render
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    const CostModel m(load_profile(ss.str()));
    SimConfig sc;
    sc.steps_per_epoch = std::atoi(argv[2]);
    const SimReport ahd = simulate(m, best_schedule(m).first, sc);
    Comparison c({{"dp", simulate_baseline(m, dp_schedule(m), sc)}, {"ir", simulate(m, ir_schedule(m), sc)},
                  {"tr+dpu+ahd", ahd}}, "dp");
    GanttOptions o;
    o.title = "pipeline";
    o.legend = false;
    o.show_overlapped_sends = false;
    o.plot_width_px = 700.0;
    o.lane_height_px = 20.0;
    const std::string sep = "\n@@\n";
    const std::string s = speedup_table(c).to_text() + sep + speedup_table(c).to_csv() + sep + speedup_table(c).to_json() +
                          sep + breakdown_table(c).to_text() + sep + breakdown_table(c).to_csv() + sep +
                          breakdown_table(c).to_json() + sep + gantt_svg(ahd) + sep + gantt_svg(ahd, o);
    std::fwrite(s.data(), 1, s.size(), stdout);
    return 0;
  }
  std::printf("ok\n");
  return 0;
}
'''


@pytest.fixture(scope="module")
def consumer(tmp_path_factory):
    d = tmp_path_factory.mktemp("report")
    src = d / "consumer.cpp"
    src.write_text(CONSUMER)
    exe = d / "consumer"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", str(src), "-o", str(exe), LIB,
                    f"-Wl,-rpath,{os.path.dirname(LIB)}"], check=True)
    return exe


def test_reference_report_test_assertions(consumer):
    r = subprocess.run([str(consumer)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(8))
def test_tables_and_gantt_byte_identical_to_reference(consumer, tmp_path, seed):
    import json
    import random
    doc = random_doc(random.Random(seed), max_blocks=6, max_devices=8, overrides=seed % 2 == 1)
    p = tmp_path / "p.json"
    p.write_text(json.dumps(doc))
    steps = 3 + seed
    ours = subprocess.run([str(consumer), str(p), str(steps)], capture_output=True, text=True, check=True).stdout
    theirs = ref.report_render(doc, {"steps_per_epoch": steps})
    ours_parts, their_parts = ours.split("\n@@\n"), theirs.split("\n@@\n")
    assert len(ours_parts) == len(their_parts) == 8
    for i, (a, b) in enumerate(zip(ours_parts, their_parts)):
        assert a == b, f"part {i} differs"
