"""`python -m paper_2301_12443_b200.cli` GPU subcommands end to end (one rank): profile -> schedule
(lib/pbd) -> run with --save, then --resume continues the data stream and the student state."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args, timeout=600):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29600 + os.getpid() % 300))
    return subprocess.run([sys.executable, "-m", "paper_2301_12443_b200.cli", *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def test_profile_run_save_resume(tmp_path):
    prof = tmp_path / "profile.json"
    r = _cli("profile", "--global-batch", "32", "--devices", "1", "--out", str(prof))
    assert r.returncode == 0, r.stderr
    doc = json.loads(prof.read_text())
    assert len(doc["blocks"]) == 4 and doc["global_batch"] == 32
    sched = {"flags": {"tr": True, "dpu": True, "ahd": True},
             "partitions": [{"blocks": [0, 3], "devices": [0], "per_device_batch": 32}],
             "predicted": {"partition_ms": [0.0], "step_ms": 0.0}}
    sp = tmp_path / "schedule.json"
    sp.write_text(json.dumps(sched))
    ck = tmp_path / "ck"
    full = _cli("run", "--schedule", str(sp), "--global-batch", "32", "--steps", "4")
    first = _cli("run", "--schedule", str(sp), "--global-batch", "32", "--steps", "2", "--save", str(ck))
    second = _cli("run", "--schedule", str(sp), "--global-batch", "32", "--steps", "2", "--resume", str(ck))
    for r in (full, first, second):
        assert r.returncode == 0, r.stderr
    assert json.loads((ck / "meta.json").read_text())["step"] == 2
    assert "resumed at step 2" in second.stderr
    last = lambda r: json.loads(r.stdout.strip().splitlines()[-1])["block_losses"]  # noqa: E731
    assert last(second) == last(full)
    assert last(first) != last(full)
