"""The `pbd` command line (csrc/tools/pbd_cli.cpp, drop-in for proj/tools/pbd_cli.cpp): subcommands,
documents and the exit-code contract 0/1/2/3 (pbd_cli.cpp:29-32).  Golden: `profile-gen --blocks 4`
then `schedule` evaluates 20 configs (cli_test.cpp:38)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PBD = os.path.join(ROOT, "paper_2301_12443_b200", "lib", "pbd")


def run(*args, stdin=None):
    return subprocess.run([PBD, *args], capture_output=True, text=True, input=stdin, timeout=60)


@pytest.fixture(scope="module")
def profile(tmp_path_factory):
    if not os.path.exists(PBD):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2301_12443_b200"), "-j8"], check=True)
    p = tmp_path_factory.mktemp("cli") / "profile.json"
    r = run("profile-gen", "--blocks", "4", "--out", str(p))
    assert r.returncode == 0, r.stderr
    return p


def test_schedule_golden_config_count(profile, tmp_path):
    r = run("schedule", str(profile))
    assert r.returncode == 0 and "configs evaluated: 20" in r.stdout
    out = tmp_path / "s.json"
    assert run("schedule", str(profile), "--out", str(out)).returncode == 0
    doc = json.loads(out.read_text())
    from paper_2301_12443_b200 import core
    want, _ = core.best_schedule(json.loads(profile.read_text()))
    assert doc["partitions"] == want["partitions"]
    # stdin and --format json
    r = run("schedule", "-", "--format", "json", stdin=profile.read_text())
    assert r.returncode == 0 and json.loads(r.stdout)["partitions"] == want["partitions"]


def test_simulate_report_gantt_and_compare(profile, tmp_path):
    s = tmp_path / "s.json"
    assert run("schedule", str(profile), "--out", str(s)).returncode == 0
    rep, svg = tmp_path / "r.json", tmp_path / "g.svg"
    r = run("simulate", str(s), str(profile), "--steps", "8", "--out", str(rep), "--gantt", str(svg))
    assert r.returncode == 0, r.stderr
    report = json.loads(rep.read_text())
    assert report["sim"]["steps_per_epoch"] == 8 and svg.read_text().startswith("<svg")
    r = run("report", str(rep), "--profile", str(profile), "--schedule", str(s))
    assert r.returncode == 0 and "relative error: 0" in r.stdout
    r = run("compare", str(profile), "--against", "dp,ls,ir", "--ablation", "tr,tr+dpu,tr+dpu+ahd", "--format", "json")
    assert r.returncode == 0, r.stderr
    cmp = json.loads(r.stdout)
    assert cmp["baseline"] == "dp" and cmp["speedup"]["dp"] == 1.0 and {row["label"] for row in cmp["breakdown"]} == {
        "dp", "ls", "ir", "tr", "tr+dpu", "tr+dpu+ahd"}
    assert run("compare", str(profile), "--against", "dp,xx").returncode == 1


def test_exit_codes(profile, tmp_path):
    assert run("schedule", str(tmp_path / "missing.json")).returncode == 3        # IoError
    assert run("profile-gen", "--blocks", "x").returncode == 1                    # ValidationError
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert run("schedule", str(bad)).returncode in (1, 3)
    # infeasible: memory too small for any partition
    tiny = tmp_path / "tiny.json"
    assert run("profile-gen", "--blocks", "4", "--mem-bytes", "1", "--out", str(tiny)).returncode == 0
    assert run("schedule", str(tiny)).returncode == 2                             # InfeasibleError
    assert run("nonsense").returncode == 1
