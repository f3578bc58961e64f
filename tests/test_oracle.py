"""Pin the C oracle (oracle/bd_oracle.c) before trusting it as the GPU checker:
  * Philox4x32-10 known-answer vectors (Random123 kat_vectors);
  * bf16 rounding == torch's round-to-nearest-even conversion;
  * the full blockwise-distillation step (teacher fwd, student fwd/bwd with
    per-shard BN, MSE, SGD-momentum) vs an independent torch-fp32 + autograd
    implementation (tests/golden/bd_torch_fp32.npz, made by make_golden.py);
  * thread-count independence (bit-identical under 1 and 8 OpenMP threads).
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import bd

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bd_torch_fp32.npz")


def test_philox_known_answers():
    assert bd.philox([0, 0, 0, 0], [0, 0]) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert bd.philox([0xffffffff] * 4, [0xffffffff] * 2) == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert bd.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0]) == \
        [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 10,
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3.4e38, 1e-40], np.float32)])
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(bd.bf16(x), want)
    for v in x[:2000]:
        assert np.float32(bd.lib().bdo_bf16(float(v))) == np.float32(bd.bf16(np.array([v]))[0])


def test_inputs_in_range_and_bf16_exact():
    x = bd.make_input(4, 10, bf16_mode=0)
    assert x.shape == (4, 32, 32, 3)
    assert x.min() >= -1.0 and x.max() < 1.0
    assert abs(float(x.mean())) < 0.05
    xb = bd.make_input(4, 10, bf16_mode=1)
    np.testing.assert_array_equal(xb, bd.bf16(x))
    # sample identity depends only on the global index
    np.testing.assert_array_equal(bd.make_input(2, 12, bf16_mode=0), x[2:4])


def test_oracle_matches_torch_fp32_golden():
    g = np.load(GOLD)
    B, steps, sub = (int(v) for v in g["meta"][:3])
    groups = {k: int(g["meta"][3 + k]) for k in range(4)}
    tr = bd.Trainer(B, bf16_mode=0)
    for step in range(steps):
        x = bd.make_input(B, step * B, bf16_mode=0)
        act = x
        for k in range(4):
            t = bd.teacher_fwd(k, tr.tp[k], act, bf16_mode=0)
            assert np.isclose(t.astype(np.float64).sum(), g[f"s{step}_b{k}_teacher_sum"], rtol=1e-5, atol=1e-3)
            assert np.isclose((t.astype(np.float64) ** 2).sum(), g[f"s{step}_b{k}_teacher_sq"], rtol=1e-5)
            np.testing.assert_allclose(t.reshape(-1)[::sub], g[f"s{step}_b{k}_teacher_sub"], rtol=1e-4, atol=1e-4)
            total = np.zeros_like(tr.sp[k])
            loss = 0.0
            base, extra = divmod(B, groups[k])
            first = 0
            for r in range(groups[k]):
                cnt = base + (1 if r < extra else 0)
                l, gr = bd.student_fwd_bwd(k, tr.sp[k], act[first:first + cnt], t[first:first + cnt], B, 0)
                total += gr
                loss += l
                first += cnt
            assert loss == pytest.approx(float(g[f"s{step}_b{k}_loss"]), rel=1e-5)
            for name, (o, n) in bd.student_layout(k).items():
                want = float(g[f"s{step}_b{k}_gnorm_{name}"])
                got = float(np.linalg.norm(total[o:o + n].astype(np.float64)))
                assert got == pytest.approx(want, rel=2e-4, abs=1e-9), (step, k, name)
            gs = g[f"s{step}_b{k}_grad_sub"]
            np.testing.assert_allclose(total[::sub], gs, rtol=0, atol=2e-4 * np.abs(gs).max() + 1e-12)
            bd.sgd(tr.sp[k], tr.mom[k], total)
            act = t
    for k in range(4):
        want = g[f"final_b{k}_param_sub"]
        np.testing.assert_allclose(tr.sp[k][::sub], want, rtol=0, atol=1e-5 * np.abs(want).max())


def test_oracle_thread_count_invariant():
    code = ("from oracle import bd; tr = bd.Trainer(3); l = tr.step(0, {1: 2}); "
            "import hashlib; h = hashlib.sha256(); [h.update(tr.sp[k].tobytes()) for k in range(4)]; "
            "print(h.hexdigest(), repr(l))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for threads in ("1", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=threads)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, check=True)
        outs.append(r.stdout.strip())
    assert outs[0] == outs[1]
