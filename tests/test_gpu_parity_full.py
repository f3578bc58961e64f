"""GPU parity at the BENCHMARKED configurations (BASELINE.json configs[1..3]).

The step bench.py times is Partition(0, 3, n=256, gb=256) for CIFAR and Partition(0, 5, 256) at 224²
for the MBConv families.  Tile shape, m2/halo selection, split-K counts and the pass grids all depend
on n (conv.cu fprop_plan / wgrad_plan), so the small-batch parity of test_gpu_parity.py does not
cover them.  Here the exact plans the bench runs are compared with the oracle (oracle/bd_oracle.c,
oracle/mb_oracle.c) on identical inputs, per stage:

  * teacher block k on the GPU's own t_{k-1}: bf16 tolerance of tests/gpu_helpers.py (max
    depth*2^-7, mean depth*2^-11 of the output scale);
  * student block k fwd+bwd on the GPU's own (t_{k-1}, t_k): loss 1e-4 relative (CIFAR) / 1e-3
    (MBConv); every gradient tensor within max(5e-3 relative, the oracle's own bf16-vs-fp32 distance)
    (MBConv: 2e-2 / 2x that distance, as test_gpu_mb.py) — i.e. inside the bf16 quantisation noise.

End to end (several chained steps), the student trajectory is checked with the teacher noise
removed: the oracle trains its own copy of every student block on the GPU's teacher activations of
each step, so the only difference left is the student path's own accumulation order.  The weight
deltas must agree within 1e-2 relative L2 (or 2x the oracle's bf16-vs-fp32 trajectory spread) —
round 1's test allowed up to 2.5e-1 because it let the 20-conv teacher chain's bf16 noise
compound into the targets.
"""
import numpy as np
import pytest
import torch

from oracle import bd
from tests.gpu_helpers import compare_bf16_tensors, to_oracle_layout

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex():
    from paper_2301_12443_b200 import executor
    return executor


def _grad_checks(k, gg, g, g32, rel=5e-3, noise_mult=1.0):
    for name, (o, n) in bd.student_layout(k).items():
        a, w, w32 = gg[o:o + n], g[o:o + n], g32[o:o + n]
        noise = np.linalg.norm(w - w32)
        err = np.linalg.norm(a - w)
        assert err <= max(rel * np.linalg.norm(w), noise_mult * noise) + 1e-12, (k, name, err, noise)


@pytest.fixture(scope="module")
def cifar256(ex):
    """The bench's configs[1] executor (IR point, b=256) after one eager step body."""
    b = 256
    p = ex.Partition(0, 3, b, b)
    p.init_params()
    p.teacher_forward()
    p.student_step()
    torch.cuda.synchronize()
    return p


def test_cifar_b256_input_bit_exact(cifar256):
    from tests.gpu_helpers import pad_image
    got = cifar256.input_act().float().cpu().numpy()
    np.testing.assert_array_equal(got, pad_image(bd.make_input(256, 0, 1)))


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_cifar_b256_teacher_block(cifar256, k):
    b = 256
    prev = bd.make_input(b, 0, 1) if k == 0 else cifar256.teacher_act(k - 1)[:b].float().cpu().numpy()
    got = cifar256.teacher_act(k)[:b].float().cpu().numpy()
    want = bd.teacher_fwd(k, bd.teacher_params(k, 1), prev, 1)
    compare_bf16_tensors(got, want, depth=5)


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_cifar_b256_student_block(cifar256, k):
    """Loss and every gradient tensor of student block k at the benchmarked batch."""
    b = 256
    prev = bd.make_input(b, 0, 1) if k == 0 else cifar256.teacher_act(k - 1)[:b].float().cpu().numpy()
    tk = cifar256.teacher_act(k)[:b].float().cpu().numpy()
    loss, g = bd.student_fwd_bwd(k, bd.student_params(k), prev, tk, b, 1)
    _, g32 = bd.student_fwd_bwd(k, bd.student_params(k), prev, tk, b, 0)
    assert cifar256.losses()[k] == pytest.approx(loss, rel=1e-4), k
    base, _, total = cifar256.layouts[k]
    gg = to_oracle_layout(k, cifar256.grads()[base:base + total].cpu().numpy())
    _grad_checks(k, gg, g, g32)


def test_cifar_b256_graph_replay_equals_eager(ex):
    """The bench replays one captured graph of the whole step; at b=256 it equals eager steps bit for bit."""
    b = 256
    res = []
    for graph in (False, True):
        p = ex.Partition(0, 3, b, b)
        p.init_params()
        losses = []
        for s in range(2):
            if graph:
                if s == 0:
                    p.capture()
                p.replay()
            else:
                p.step()
            torch.cuda.synchronize()
            losses.append(p.losses())
        res.append((losses, p.params().cpu()))
    assert res[0][0] == res[1][0]
    assert torch.equal(res[0][1], res[1][1])


def _student_trajectory(ex, b, steps, lo=0, hi=3):
    """GPU steps (eager phases) + the oracle's student chain trained on the GPU's teacher activations."""
    p = ex.Partition(lo, hi, b, b)
    p.init_params()
    blocks = list(range(lo, hi + 1))
    w = {k: bd.student_params(k) for k in blocks}
    v = {k: np.zeros_like(w[k]) for k in blocks}
    w32 = {k: w[k].copy() for k in blocks}
    v32 = {k: np.zeros_like(w[k]) for k in blocks}
    w0 = {k: w[k].copy() for k in blocks}
    for s in range(steps):
        p.teacher_forward()
        p.student_step()
        torch.cuda.synchronize()
        gl = p.losses()
        prev = bd.make_input(b, s * b, 1)
        for i, k in enumerate(blocks):
            tk = p.teacher_act(k)[:b].float().cpu().numpy()
            loss, g = bd.student_fwd_bwd(k, w[k], prev, tk, b, 1)
            _, g32 = bd.student_fwd_bwd(k, w32[k], prev, tk, b, 0)
            assert gl[i] == pytest.approx(loss, rel=1e-3), (s, k, gl[i], loss)
            bd.sgd(w[k], v[k], g)
            bd.sgd(w32[k], v32[k], g32)
            prev = tk
        p.apply_update()
    torch.cuda.synchronize()
    return p, w0, w, w32


@pytest.mark.parametrize("b,steps", [(64, 4), (256, 2)])
def test_cifar_student_trajectory_tight(ex, b, steps):
    """Chained SGD steps: student weights after `steps` updates vs the oracle trained on the GPU's own
    teacher activations.  A wrong update (lr, momentum, a missing gradient term, a stale shadow) moves
    dw by O(1) relative; bf16 accumulation-order noise stays at the oracle's own bf16-vs-fp32 spread."""
    p, w0, w, w32 = _student_trajectory(ex, b, steps)
    for k in range(4):
        base, _, total = p.layouts[k]
        got = to_oracle_layout(k, p.params()[base:base + total].cpu().numpy())
        dg, do, d32 = got - w0[k], w[k] - w0[k], w32[k] - w0[k]
        err = np.linalg.norm(dg - do)
        spread = np.linalg.norm(do - d32)
        assert err <= max(1e-2 * np.linalg.norm(do), 2 * spread), (k, err / np.linalg.norm(do),
                                                                   spread / np.linalg.norm(do))


# --------------------------------------------------------------------------- MBConv at 224²
S224 = 224


@pytest.fixture(params=[("mbv2", 0), ("effb0", 1)], ids=["mbv2", "effb0"])
def mbfam(request):
    from oracle import mb
    mb.set_family(request.param[1])
    yield request.param[0], mb
    mb.set_family(0)


def test_mbconv_224_b32_per_stage(ex, mbfam):
    """configs[2]/[3] image size (224²) at b=32: every block (one per stage boundary) vs the oracle."""
    fam, mb = mbfam
    b = 32
    paths = {k: mb.sample_path(k, 5) for k in range(6)}
    p = ex.Partition(0, 5, b, b, model=fam, image=S224)
    p.init_params()
    for k in range(6):
        p.set_path(k, paths[k])
    p.teacher_forward()
    p.student_step()
    torch.cuda.synchronize()
    gl = p.losses()
    prev = mb.image(b, 0, S224)
    got_img = p.input_act()[:b].float().cpu().numpy()[..., :3]
    np.testing.assert_array_equal(got_img, prev)
    for k in range(6):
        gpu_t = p.teacher_act(k)[:b].float().cpu().numpy()
        want_t = mb.teacher_fwd(k, mb.teacher_params(k), prev, S224)
        depth = (3 if fam == "mbv2" else 4) * mb.NL[k] + (1 if k == 0 else 0)
        compare_bf16_tensors(gpu_t, want_t, depth=depth)
        norm = float(b) * mb.true_channels(k + 1) * mb.hw(k + 1, S224) ** 2
        sp = mb.student_params(k)
        g, loss = mb.student_fwd_bwd(k, sp, paths[k], prev, gpu_t, S224, norm, bf16=True)
        g32, _ = mb.student_fwd_bwd(k, sp, paths[k], prev, gpu_t, S224, norm, bf16=False)
        assert gl[k] == pytest.approx(loss, rel=1e-3), (k, gl[k], loss)
        base, _, total = p.layouts[k]
        gg = p.grads()[base:base + total].cpu().numpy()
        active = np.zeros(gg.size, bool)
        for l in range(mb.layers(k)):
            c = int(paths[k][l])
            off, n = mb.candidate_span(k, l, c)
            active[off:off + n] = True
            for name, (o, cnt) in mb.candidate_layout(k, l, c).items():
                a, w, w32 = gg[off + o: off + o + cnt], g[off + o: off + o + cnt], g32[off + o: off + o + cnt]
                err = np.linalg.norm(a - w)
                noise = np.linalg.norm(w - w32)
                assert err <= max(2e-2 * np.linalg.norm(w), 2 * noise) + 1e-9, (k, l, name, err, noise)
        assert not gg[~active].any(), k
        prev = gpu_t
