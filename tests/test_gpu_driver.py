"""The C++ single-process driver (include/pbdr.h): a whole schedule in one process, executors wired
over peer memory by C++ (csrc/exec/driver.cpp), one CUDA graph per rank per step.  On the one GPU of
the test box all ranks share device 0 (the same kernels, flag protocol and slot wiring as across
NVLink).  It must be BITWISE identical to the Python-wired runs of test_gpu_relay.py."""
import os
import subprocess

import pytest
import torch

from tests.test_gpu_relay import _single, run_inprocess, sched

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ex():
    from paper_2301_12443_b200 import executor
    return executor


def drive(schedule, b, steps, graphs=True):
    from paper_2301_12443_b200 import driver
    d = driver.Driver(schedule, b, graphs=graphs)
    for _ in range(steps):
        d.step()
    d.sync()
    return d, {r: d.rank_state(r) for r in range(d.nranks)}


@pytest.mark.parametrize("graphs", [True, False])
def test_driver_pure_pipeline_bitwise(ex, graphs):
    b, steps = 8, 3
    s = sched([(0, 1, [0]), (2, 3, [1])], b)
    d, got = drive(s, b, steps, graphs)
    ref = _single(ex, b, steps)
    assert torch.equal(torch.cat([got[0]["params"], got[1]["params"]]), ref.params().cpu())
    assert torch.equal(torch.cat([got[0]["momentum"], got[1]["momentum"]]), ref.momentum().cpu())
    assert d.block_losses() == ref.losses()


@pytest.mark.parametrize("parts,b", [([(0, 3, [0, 1])], 8), ([(0, 0, [0]), (1, 2, [1, 2]), (3, 3, [3])], 10),
                                     ([(0, 1, [0, 1, 2]), (2, 3, [3, 4])], 7)])
def test_driver_hybrid_dp_bitwise(ex, parts, b):
    """Resharded relay (1->2, 2->1, 3->2) + DP groups over peer memory, vs host copies + host gradient sum."""
    s = sched(parts, b)
    d, got = drive(s, b, 3)
    want = run_inprocess(ex, s, b, 3, "copy")
    for r in want:
        assert torch.equal(got[r]["params"], want[r][0]), r
        assert torch.equal(got[r]["momentum"], want[r][1]), r
        assert got[r]["losses"].tolist() == want[r][2], r
    for _, _, devs in parts:
        for r in devs[1:]:
            assert torch.equal(got[r]["params"], got[devs[0]]["params"])


def test_driver_many_steps_full_batch(ex):
    """b = 256, four single-block partitions (the bench configuration's pure pipeline), 20 graph steps:
    equal to one partition holding all blocks."""
    b = 256
    s = sched([(0, 0, [0]), (1, 1, [1]), (2, 2, [2]), (3, 3, [3])], b)
    d, got = drive(s, b, 20)
    ref = _single(ex, b, 20)
    assert torch.equal(torch.cat([got[r]["params"] for r in range(4)]), ref.params().cpu())
    assert d.block_losses() == ref.losses()


def test_cli_run(tmp_path):
    import json
    b = 16
    s = sched([(0, 1, [0]), (2, 3, [1, 2])], b)
    f = tmp_path / "s.json"
    f.write_text(json.dumps(s))
    out = subprocess.run([os.path.join(ROOT, "paper_2301_12443_b200", "lib", "pbd"), "run", str(f), "--global-batch",
                          str(b), "--steps", "4", "--devices", "0,0,0"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "ms/step" in out.stdout and "block losses" in out.stdout
    losses = [float(v) for v in out.stdout.split("block losses:")[1].split()]
    assert len(losses) == 4 and all(0 < v < 10 for v in losses)
