"""Host core (libpbd.so: profile / cost model / AHD partitioner / simulator) parity.

Three layers of evidence:
  1. golden values restated from the reference's own tests (file:line cited);
  2. bit-exact agreement with the reference compiled unmodified (oracle/_ref)
     on fuzzed documents: same winning partition, identical predicted doubles;
  3. agreement with the pure-Python restatement (oracle/sched_oracle.py).
"""
import json
import math
import random
import struct

import pytest

from paper_2301_12443_b200 import core
from oracle import ref, sched_oracle
from tests.profiles import proportional_doc, random_doc

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (needs /root/reference)")


def bits(x):
    return struct.pack("<d", float(x))


def sched_doc(parts, gb):
    """parts: list of (lo, hi, devices)."""
    return {"flags": {"tr": True, "dpu": True, "ahd": True},
            "partitions": [{"blocks": [lo, hi], "devices": devs, "per_device_batch": -(-gb // len(devs))}
                           for lo, hi, devs in parts],
            "predicted": {"partition_ms": [0.0] * len(parts), "step_ms": 0.0}}


# ---------------------------------------------------------------- golden values (reference tests)

def test_enumerate_counts_closed_form():
    # schedule_test.cpp:28-42: counts 1/4/56 and C(B+N-2, B-1) for B,N <= 8
    assert core.enumerate_count(1, 1) == 1
    assert core.enumerate_count(4, 2) == 4
    assert core.enumerate_count(6, 4) == 56
    for B in range(1, 9):
        for N in range(1, 9):
            assert core.enumerate_count(B, N) == math.comb(B + N - 2, B - 1)


def test_partition_cost_equation():
    # schedule_test.cpp:76-97: T+S = 4 and 6 ms at full batch; DPC(g=2) = 1 -> (4+6)/2+1 = 6; g=1 -> 10
    doc = proportional_doc([2.0, 3.0], [2.0, 3.0], 2, 256, param_bytes=2.0e4, allreduce_bytes_per_ms=4.0e4)
    c = core.predicted_step_time(doc, sched_doc([(0, 1, [0, 1])], 256))
    assert c["step_ms"] == pytest.approx(6.0, abs=1e-9)
    c = core.predicted_step_time(doc, sched_doc([(0, 1, [0])], 256))
    assert c["step_ms"] == pytest.approx(10.0, abs=1e-9)
    # max over partitions: 4 and 6 -> 6 (schedule_test.cpp:139-150)
    c = core.predicted_step_time(doc, sched_doc([(0, 0, [0]), (1, 1, [1])], 256))
    assert c["partition_ms"] == pytest.approx([4.0, 6.0], abs=1e-9)
    assert c["step_ms"] == pytest.approx(6.0, abs=1e-9)
    assert c["feasible"]


def test_memory_infeasibility_flag():
    # schedule_test.cpp:152-161
    doc = proportional_doc([2.0, 3.0], [2.0, 3.0], 2, 256, param_bytes=2.0e4, allreduce_bytes_per_ms=4.0e4)
    doc["hardware"]["mem_bytes_per_device"] = 100.0
    c = core.predicted_step_time(doc, sched_doc([(0, 1, [0, 1])], 256))
    assert not c["feasible"] and "partition 0" in c["reason"]
    with pytest.raises(core.InfeasibleError):
        core.best_schedule(doc)


@pytest.mark.parametrize("t,n_parts,g0,step", [([5.0, 1.0], 1, 2, 7.0), ([2.5, 2.5], 2, 1, 5.0)])
def test_best_schedule_merge_vs_split(t, n_parts, g0, step):
    # schedule_test.cpp:163-180
    doc = proportional_doc(t, t, 2, 256, param_bytes=2.0e4, allreduce_bytes_per_ms=4.0e4)
    s, meta = core.best_schedule(doc)
    assert len(s["partitions"]) == n_parts
    assert len(s["partitions"][0]["devices"]) == g0
    assert s["predicted"]["step_ms"] == pytest.approx(step, abs=1e-9)


def test_best_schedule_degenerate():
    # schedule_test.cpp:182-188
    s, meta = core.best_schedule(proportional_doc([2.0], [3.0], 1, 256))
    assert s["predicted"]["step_ms"] == pytest.approx(5.0, abs=1e-9)
    assert meta["configs_evaluated"] == 1


def test_exec_time_interpolation_floor_extrapolation():
    # cost_model_test.cpp:51-65
    def doc(times, floor=0.3):
        b = {"id": 0, "teacher_ms": times, "student_ms": times, "act_bytes_per_sample": 0.0, "param_bytes": 0.0,
             "teacher_param_bytes": 0.0}
        return {"blocks": [b], "global_batch": 256,
                "hardware": {"num_devices": 2, "link_bytes_per_ms": 1048576.0, "allreduce_bytes_per_ms": 1.0e5,
                             "mem_bytes_per_device": 1.0e12, "data_load_ms_per_batch": 0.0,
                             "min_utilization_floor": floor}}
    assert core.exec_time(doc({"64": 1.0, "128": 2.0}), 0, "teacher", 96) == pytest.approx(1.5, abs=1e-9)
    assert core.exec_time(doc({"64": 1.0}), 0, "teacher", 16) == pytest.approx(0.3, abs=1e-9)
    assert core.exec_time(doc({"64": 1.0, "128": 2.0}), 0, "teacher", 256) == pytest.approx(4.0, abs=1e-9)
    with pytest.raises(core.ValidationError):
        core.exec_time(doc({"64": 1.0}), 1, "teacher", 64)
    with pytest.raises(core.ValidationError):
        core.exec_time(doc({"64": 1.0}), 0, "teacher", 0)


def test_profile_validation_errors():
    # profile_test.cpp / SPEC.md:30-33: gaps, non-monotone, unknown keys
    good = proportional_doc([1.0, 1.0], [1.0, 1.0], 2, 256)
    core.load_save_profile(good)
    bad = json.loads(json.dumps(good))
    bad["blocks"][1]["id"] = 2
    with pytest.raises(core.ValidationError, match="non-contiguous block ids"):
        core.load_save_profile(bad)
    bad = json.loads(json.dumps(good))
    bad["blocks"][0]["teacher_ms"] = {"128": 2.0, "64": 3.0}
    bad["blocks"][0]["student_ms"] = {"128": 2.0, "64": 3.0}
    with pytest.raises(core.ValidationError, match="non-monotone"):
        core.load_save_profile(bad)
    bad = json.loads(json.dumps(good))
    bad["blocks"][0]["bogus"] = 1
    with pytest.raises(core.ValidationError, match="unknown key"):
        core.load_save_profile(bad)
    bad = json.loads(json.dumps(good))
    bad["blocks"][0]["student_ms"] = {"64": 1.0}
    with pytest.raises(core.ValidationError, match="missing batch key"):
        core.load_save_profile(bad)


def test_profile_round_trip_is_byte_stable():
    rng = random.Random(5)
    for _ in range(50):
        d = random_doc(rng, overrides=True)
        once = core.load_save_profile(d)
        assert core.load_save_profile(once) == once
        assert json.loads(once) == json.loads(core.load_save_profile(json.loads(once)))


def test_simulate_hand_traced():
    # simulate_test.cpp:47-102
    doc = proportional_doc([2.0, 2.0], [3.0, 3.0], 2, 256)
    s = sched_doc([(0, 0, [0]), (1, 1, [1])], 256)
    r = core.simulate(doc, s, {"steps_per_epoch": 10, "dpu": True})
    assert r["makespan_ms"] == pytest.approx(52.0, abs=1e-9)
    assert r["steady_state_step_ms"] == pytest.approx(5.0, abs=1e-9)
    r = core.simulate(doc, s, {"steps_per_epoch": 10, "dpu": False})
    assert r["makespan_ms"] == pytest.approx(70.0, abs=1e-9)
    assert r["steady_state_step_ms"] == pytest.approx(7.0, abs=1e-9)
    one = proportional_doc([2.0], [3.0], 1, 256)
    one["hardware"]["data_load_ms_per_batch"] = 1.5
    s1 = sched_doc([(0, 0, [0])], 256)
    r = core.simulate(one, s1, {"steps_per_epoch": 10, "epoch_sync_ms": 2.5})
    assert r["makespan_ms"] == pytest.approx(54.0, abs=1e-9)
    assert r["category_totals_ms"]["data_load"] == pytest.approx(1.5, abs=1e-9)
    r = core.simulate(one, s1, {"steps_per_epoch": 10, "epoch_sync_ms": 2.5, "epochs": 2})
    assert r["makespan_ms"] == pytest.approx(108.0, abs=1e-9)
    assert r["category_totals_ms"]["data_load"] == pytest.approx(3.0, abs=1e-9)
    bott = proportional_doc([3.0, 2.5], [3.0, 2.5], 2, 256)
    r = core.simulate(bott, s, {"steps_per_epoch": 10})
    assert r["steady_state_step_ms"] == pytest.approx(6.0, abs=1e-9)


def test_readme_front_heavy_profile():
    # proj/README.md:55-64 (+ SURVEY.md §6, measured): 56 configs, step 6.0, 3 partitions
    doc = core.synth_profile(shape="front-heavy", blocks=6, front_weight=4.0, curvature=0.4, num_devices=4)
    s, meta = core.best_schedule(doc)
    assert meta["configs_evaluated"] == 56
    assert [p["blocks"] for p in s["partitions"]] == [[0, 0], [1, 2], [3, 5]]
    assert [len(p["devices"]) for p in s["partitions"]] == [2, 1, 1]
    assert s["partitions"][0]["per_device_batch"] == 128
    assert bits(s["predicted"]["step_ms"]) == bits(6.0)
    assert [bits(x) for x in s["predicted"]["partition_ms"]] == [bits(5.699999999999999), bits(4.0), bits(6.0)]


def test_shard_ranges_remainder_rule():
    # first (b mod g) devices take one extra sample
    for b in (1, 7, 64, 255, 256):
        for g in range(1, 9):
            if g > b:
                continue
            ranges = [core.shard_range(b, g, r) for r in range(g)]
            assert sum(c for _, c in ranges) == b
            assert ranges[0][0] == 0
            for (f0, c0), (f1, _) in zip(ranges, ranges[1:]):
                assert f1 == f0 + c0
            assert max(c for _, c in ranges) == -(-b // g)


# ---------------------------------------------------------------- bit-exact vs the compiled reference

def _same_schedule(a, b):
    assert a["partitions"] == b["partitions"]
    assert a["flags"] == b["flags"]
    assert bits(a["predicted"]["step_ms"]) == bits(b["predicted"]["step_ms"])
    assert [bits(x) for x in a["predicted"]["partition_ms"]] == [bits(x) for x in b["predicted"]["partition_ms"]]


@needs_ref
@pytest.mark.parametrize("seed", range(4))
def test_best_schedule_bit_exact_fuzz(seed):
    rng = random.Random(1000 + seed)
    n = 2500
    for i in range(n):
        mem = 1.0e18 if rng.random() < 0.7 else rng.uniform(1e6, 2e7)
        d = random_doc(rng, max_blocks=8, max_devices=8, mem=mem, overrides=True)
        contiguous = rng.random() < 0.2
        try:
            want, wmeta = ref.best_schedule(d, contiguous_only=contiguous)
        except ref.RefError as e:
            with pytest.raises((core.InfeasibleError, core.ValidationError)):
                core.best_schedule(d, contiguous_only=contiguous)
            continue
        got, gmeta = core.best_schedule(d, contiguous_only=contiguous)
        _same_schedule(got, want)
        assert gmeta["configs_evaluated"] == wmeta["configs_evaluated"]


@needs_ref
def test_python_oracle_matches_reference():
    rng = random.Random(77)
    for _ in range(300):
        d = random_doc(rng, max_blocks=6, max_devices=6, overrides=True)
        want, _ = ref.best_schedule(d)
        cfg, pms, step, count = sched_oracle.best_schedule(d)
        assert [[lo, hi] for lo, hi, _, _ in cfg] == [p["blocks"] for p in want["partitions"]]
        assert [g for _, _, g, _ in cfg] == [len(p["devices"]) for p in want["partitions"]]
        assert bits(step) == bits(want["predicted"]["step_ms"])
        assert [bits(x) for x in pms] == [bits(x) for x in want["predicted"]["partition_ms"]]
        assert count == ref.enumerate_count(len(d["blocks"]), d["hardware"]["num_devices"])


@needs_ref
def test_exec_time_bit_exact():
    rng = random.Random(9)
    for _ in range(200):
        d = random_doc(rng, overrides=True)
        for blk in range(len(d["blocks"])):
            for role in ("teacher", "student"):
                for batch in (1, 3, 8, 17, 64, 100, 255, 1024):
                    a = core.exec_time(d, blk, role, batch)
                    assert bits(a) == bits(ref.exec_time(d, blk, role, batch))
                    assert bits(a) == bits(sched_oracle.Model(d).exec_time(blk, role, batch))


@needs_ref
def test_simulate_matches_reference():
    rng = random.Random(11)
    for i in range(120):
        d = random_doc(rng, max_blocks=6, max_devices=6)
        s, _ = ref.best_schedule(d)
        sim = {"steps_per_epoch": rng.choice([1, 3, 4, 8, 16]), "epochs": rng.choice([1, 2]),
               "dpu": rng.random() < 0.7, "overlap_send": rng.random() < 0.8, "overlap_load": rng.random() < 0.8,
               "epoch_sync_ms": rng.random(), "weight_update_ms": rng.choice([0.0, 0.05])}
        want = ref.simulate(d, s, sim)
        got = core.simulate(d, s, sim)
        for key in ("makespan_ms", "steady_state_step_ms", "bubble_ratio", "overlapped_send_ms"):
            assert bits(got[key]) == bits(want[key]), key
        assert {k: bits(v) for k, v in got["category_totals_ms"].items()} == \
            {k: bits(v) for k, v in want["category_totals_ms"].items()}
        assert got["timelines"] == want["timelines"]
        assert got["peak_mem_bytes"] == want["peak_mem_bytes"]


@needs_ref
def test_reconfigure_and_drift_match_reference():
    rng = random.Random(13)
    for _ in range(100):
        d = random_doc(rng, max_blocks=6, max_devices=6)
        s, _ = ref.best_schedule(d)
        obs = json.loads(json.dumps(d))
        for b in obs["blocks"]:
            f = 1.0 + rng.uniform(-0.5, 0.5)
            b["teacher_ms"] = {k: v * f for k, v in b["teacher_ms"].items()}
        thr = rng.choice([0.0, 0.1, 0.3])
        assert bits(core.profile_drift(d, obs)) == bits(ref.profile_drift(d, obs))
        got = core.reconfigure(d, s, obs, thr)
        want = ref.reconfigure(d, s, obs, thr)
        assert (got is None) == (want is None)
        if got is not None:
            _same_schedule(got, want)


@needs_ref
def test_synth_profile_matches_reference():
    for spec in (dict(shape="front-heavy", blocks=6, front_weight=4.0, curvature=0.4, num_devices=4),
                 dict(shape="uniform", blocks=4, jitter=0.2, seed=17),
                 dict(shape="custom", blocks=6, custom_weights=[1, 1, 1, 2, 4, 6], curvature=0.2, jitter=0.1,
                      seed=5, num_devices=8)):
        got = core.synth_profile(**spec)
        want = ref.synth_profile(**spec)
        assert json.dumps(got, sort_keys=True) == json.dumps(want, sort_keys=True)


def test_report_roundtrip_steady_state_validation_and_gantt():
    """§8f: reports of real runs — any save_report document (simulated here; measured ones come from
    runtime.measured_report) parses back, yields the reference's steady-state step and prediction
    error, and renders a per-device Gantt chart."""
    from paper_2301_12443_b200 import core
    prof = core.synth_profile(shape="front-heavy", blocks=6, front_weight=3.0, curvature=0.4, num_devices=4)
    sched, _ = core.best_schedule(prof)
    rep = core.simulate(prof, sched, {"steps_per_epoch": 8, "epochs": 1})
    assert core.report_steady_state(rep) == rep["steady_state_step_ms"]
    assert core.validate_prediction(rep, prof, sched) < 1e-12
    # a "measured" run 10% slower than planned
    slow = json.loads(json.dumps(rep))
    for line in slow["timelines"]:
        for e in line:
            e["start_ms"] *= 1.1
            e["end_ms"] *= 1.1
    slow["makespan_ms"] *= 1.1
    assert core.validate_prediction(slow, prof, sched) == pytest.approx(0.1, rel=1e-9)
    svg = core.gantt_svg(rep, "plan")
    assert svg.startswith("<svg") and svg.count("<rect") > 4 * 8 and "GPU 3" in svg
    with pytest.raises(core.ValidationError):
        core.report_steady_state({**rep, "sim": {**rep["sim"], "steps_per_epoch": 2}})
