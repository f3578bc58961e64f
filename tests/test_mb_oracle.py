"""MBConv oracle (oracle/mb_oracle.c) pinned against the independent torch float64 + autograd
implementation (tests/golden/mb_torch_fp64.npz, make_golden_mb.py), plus its own invariants:
layout, determinism across thread counts, single-path sparsity of gradients and updates.

Tolerances: the oracle runs fp32 (bf16 off) against a float64 reference at S=64 (blocks 4-5 at
2x2 pixels, m = 12 BN samples); teacher outputs 1e-5 relative L2 / 1e-4 per element of the output
scale; losses 1e-5 relative; gradient tensors: norm 5e-3 relative (an fp32-vs-fp64 flip of a ReLU6 mask element moves
the expand-layer gradients by ~3e-3), subsampled elements 2e-2
relative L2 (a few elements sit on BN-backward cancellations); gradients that cancel to < 1e-4 of
the block's gradient scale (gamma behind a following BN) to 1e-5 of that scale."""
import os

import numpy as np
import pytest

from oracle import mb

GOLD = {0: os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mb_torch_fp64.npz"),
        1: os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "effb0_torch_fp64.npz")}
B, S, SUB, DRAW = 3, 64, 53, 5


@pytest.fixture(scope="module", params=[0, 1], ids=["mbv2", "effb0"])
def family(request):
    """teacher family: MobileNetV2 (configs[2]) / EfficientNet-B0 with swish + squeeze-excite (configs[3])"""
    mb.set_family(request.param)
    yield request.param
    mb.set_family(0)


@pytest.fixture(scope="module")
def gold(family):
    return np.load(GOLD[family])


@pytest.fixture(scope="module")
def chain(family):
    x = mb.image(B, 0, S, bf16=False)
    acts = [x]
    for b in range(mb.BLOCKS):
        acts.append(mb.teacher_fwd(b, mb.teacher_params(b, bf16=False), acts[-1], S, bf16=False))
    return acts


def test_teacher_matches_torch(gold, chain):
    for b in range(mb.BLOCKS):
        y = chain[b + 1]
        assert y.shape == mb.act_shape(b + 1, B, S)
        assert abs(np.linalg.norm(y) - gold[f"t{b}_norm"]) <= 1e-5 * gold[f"t{b}_norm"]
        sub = y.reshape(-1)[::SUB]
        np.testing.assert_allclose(sub, gold[f"t{b}"], rtol=0, atol=1e-4 * np.abs(gold[f"t{b}"]).max())


def test_student_matches_torch(gold, chain):
    for b in range(mb.BLOCKS):
        sp = mb.student_params(b)
        path = mb.sample_path(b, DRAW)
        assert (path == gold[f"s{b}_path"]).all()
        c, hh = mb.true_channels(b + 1), mb.hw(b + 1, S)
        norm = float(B) * c * hh * hh
        g, loss = mb.student_fwd_bwd(b, sp, path, chain[b], chain[b + 1], S, norm, bf16=False)
        assert loss == pytest.approx(float(gold[f"s{b}_loss"]), rel=1e-5)
        top = max(float(v) for k_, v in gold.items() if k_.startswith(f"s{b}_l") and k_.endswith("_norm"))
        for l in range(mb.layers(b)):
            off, _ = mb.candidate_span(b, l, int(path[l]))
            for name, (o, n) in mb.candidate_layout(b, l, int(path[l])).items():
                v = g[off + o: off + o + n]
                want_norm = float(gold[f"s{b}_l{l}_{name}_norm"])
                if want_norm < 1e-4 * top:
                    # BN gamma gradients that cancel to ~1e-6 of the block's gradient scale
                    # (sum g*xhat after a following BN): fp32-vs-fp64 noise only
                    assert abs(np.linalg.norm(v) - want_norm) <= 1e-5 * top, (b, l, name)
                    continue
                assert abs(np.linalg.norm(v) - want_norm) <= 5e-3 * want_norm, (b, l, name)
                sub = v.reshape(-1)[::SUB] if v.size > 64 else v
                ref = gold[f"s{b}_l{l}_{name}"]
                err = np.linalg.norm(sub - ref) / np.linalg.norm(ref)
                assert err <= 2e-2, (b, l, name, err)


def test_gradients_only_on_active_path_and_sgd_touches_only_it():
    b = 2
    sp = mb.student_params(b)
    path = mb.sample_path(b, 11)
    x = mb.image(2, 0, S)
    acts = [x]
    for k in range(b + 1):
        acts.append(mb.teacher_fwd(k, mb.teacher_params(k), acts[-1], S))
    g, _ = mb.student_fwd_bwd(b, sp, path, acts[b], acts[b + 1], S, 1.0)
    active = np.zeros(sp.size, bool)
    for l in range(mb.layers(b)):
        off, n = mb.candidate_span(b, l, int(path[l]))
        active[off:off + n] = True
    assert not g[~active].any()
    w, v = sp.copy(), np.zeros_like(sp)
    v[~active] = 0.25  # stale momentum of inactive candidates must not move their weights
    mb.sgd_path(b, path, w, v, g)
    assert (w[~active] == sp[~active]).all() and (v[~active] == 0.25).all()
    assert not np.array_equal(w[active], sp[active])


def test_layout_and_path_sampler():
    for b in range(mb.BLOCKS):
        tot = 0
        for l in range(mb.layers(b)):
            for c in range(mb.candidates(b, l)):
                off, n = mb.candidate_span(b, l, c)
                assert off == tot and n == sum(v[1] for v in mb.candidate_layout(b, l, c).values())
                tot += n
        assert tot == mb.student_param_count(b)
        seen = set()
        for d in range(64):
            p = mb.sample_path(b, d)
            assert (p >= 0).all() and (p < mb.CANDIDATES).all()
            seen.add(tuple(p))
        assert len(seen) > 1
    assert [mb.hw(k, 224) for k in range(7)] == [224, 56, 28, 14, 14, 7, 7]


def test_oracle_bf16_mode_close_to_fp32(chain):
    """bf16 rounding points change the loss only at the bf16 noise level."""
    b = 1
    sp = mb.student_params(b)
    path = mb.sample_path(b, 3)
    norm = float(B) * mb.true_channels(b + 1) * mb.hw(b + 1, S) ** 2
    _, l32 = mb.student_fwd_bwd(b, sp, path, chain[b], chain[b + 1], S, norm, bf16=False)
    _, l16 = mb.student_fwd_bwd(b, sp, path, chain[b], chain[b + 1], S, norm, bf16=True)
    assert l16 == pytest.approx(l32, rel=2e-2)


def test_true_widths_extra_channels_stay_zero():
    """The stored extra channels (tensor-tile rounding) are identically zero: teacher activations,
    student gradients and, after SGD, student weights — so the network is the true-width one."""
    for fam in (0, 1):
        mb.set_family(fam)
        try:
            x = mb.image(2, 0, S)
            acts = [x]
            for k in range(mb.BLOCKS):
                acts.append(mb.teacher_fwd(k, mb.teacher_params(k), acts[-1], S))
                ct, cs = mb.true_channels(k + 1), mb.channels(k + 1)
                assert cs >= ct
                assert not acts[-1][..., ct:].any(), (fam, k)
                assert np.abs(acts[-1][..., :ct]).max() > 0
            for b in range(mb.BLOCKS):
                sp = mb.student_params(b)
                path = mb.sample_path(b, 4)
                g, _ = mb.student_fwd_bwd(b, sp, path, acts[b], acts[b + 1], S, 1.0)
                for l in range(mb.layers(b)):
                    geo = mb.student_layer(b, l, int(path[l]))
                    if geo["kind"] == "stem":
                        continue
                    off, _ = mb.candidate_span(b, l, int(path[l]))
                    lay = mb.candidate_layout(b, l, int(path[l]))
                    E, Et, cin, ci, cout, co = geo["E"], geo["Et"], geo["cin"], geo["cin_t"], geo["cout"], geo["cout_t"]
                    wp = sp[off + lay["wp"][0]: off + sum(lay["wp"])].reshape(cout, E)
                    gp = g[off + lay["wp"][0]: off + sum(lay["wp"])].reshape(cout, E)
                    assert not wp[co:].any() and not wp[:, Et:].any()
                    assert not gp[co:].any() and not gp[:, Et:].any()
                    assert np.abs(gp[:co, :Et]).max() > 0
                    if "we" in lay:
                        ge = g[off + lay["we"][0]: off + sum(lay["we"])].reshape(E, cin)
                        assert not ge[Et:].any() and not ge[:, ci:].any()
                    for bn in ("b2", "g2"):
                        gb = g[off + lay[bn][0]: off + sum(lay[bn])]
                        assert not gb[Et:].any()
        finally:
            mb.set_family(0)


def test_teacher_is_mobilenetv2_1_0():
    """The MobileNetV2 teacher body at its true widths has the published MobileNetV2-1.0 cost:
    300.77 M MACs at 224^2 = body + final 1x1 conv 320->1280 at 7^2 + 1280->1000 FC."""
    from paper_2301_12443_b200 import mb_models
    mb_models.set_family("mbv2")
    head = 7 * 7 * 320 * 1280 + 1280 * 1000
    assert mb_models.teacher_true_macs(224) + head == pytest.approx(300.77e6, abs=0.01e6)
    mb_models.set_family("effb0")
    try:  # EfficientNet-B0: 0.39 B FLOPs (multiply-adds) in its paper, incl. the same head
        assert (mb_models.teacher_true_macs(224) + head) / 1e9 == pytest.approx(0.39, abs=0.005)
    finally:
        mb_models.set_family("mbv2")
