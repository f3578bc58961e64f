"""ProxylessNAS step on the GPU (paper_2301_12443_b200/nas.py over the MBConv executor) vs the oracle:
the same sampled paths replayed on oracle/mb_oracle.c (architecture round: fwd/bwd without update,
weight round: fwd/bwd + path-sparse SGD).  Tolerances of tests/test_gpu_mb.py."""
import numpy as np
import pytest
import torch

from oracle import mb
from paper_2301_12443_b200 import mb_models, nas

pytestmark = pytest.mark.gpu
S = 64


@pytest.fixture(params=[("mbv2", 0), ("effb0", 1)], ids=["mbv2", "effb0"])
def fam(request):
    mb.set_family(request.param[1])
    mb_models.set_family(request.param[0])
    yield request.param[0]
    mb.set_family(0)
    mb_models.set_family("mbv2")


def test_nas_steps_match_oracle(fam):
    from paper_2301_12443_b200 import executor
    b, steps = 4, 3
    p = executor.Partition(0, 5, b, b, model=fam, image=S)
    p.init_params()
    arch = nas.ArchParams(range(6), lr=0.05)
    rec = []
    for s in range(steps):
        w0 = p.params().cpu().numpy().copy()
        out = nas.nas_step(p, arch, s)
        torch.cuda.synchronize()
        rec.append((dict(p.paths), out))
        # the architecture round never touches weights: candidates active only in it are unchanged
        w1 = p.params().cpu().numpy()
        changed = np.flatnonzero(w1 != w0)
        for k in range(6):
            base, _, total = p.layouts[k]
            for l, c in enumerate(p.paths[k]):
                off, n = mb.candidate_span(k, l, c)
                changed = changed[(changed < base + off) | (changed >= base + off + n)]
        assert changed.size == 0  # only the weight round's active candidates were updated
    # oracle replay of the same rounds
    tp = {k: mb.teacher_params(k) for k in range(6)}
    sp = {k: mb.student_params(k) for k in range(6)}
    sv = {k: np.zeros_like(sp[k]) for k in range(6)}
    ref = nas.ArchParams(range(6), lr=0.05)
    for s in range(steps):
        x = mb.image(b, s * b, S)
        acts = [x]
        for k in range(6):
            acts.append(mb.teacher_fwd(k, tp[k], acts[-1], S))
        wpaths, out = rec[s]
        for k in range(6):
            apath = np.array(ref.sample(k, 2 * s), dtype=np.int32)
            norm = float(b) * mb.true_channels(k + 1) * mb.hw(k + 1, S) ** 2
            _, la = mb.student_fwd_bwd(k, sp[k], apath, acts[k], acts[k + 1], S, norm)
            assert out["arch"][k] == pytest.approx(la, rel=2e-2), (s, k)
            ref.update(k, list(apath), out["arch"][k])  # the GPU's losses: identical alpha, identical paths
            wpath = np.array(ref.sample(k, 2 * s + 1), dtype=np.int32)
            assert list(wpath) == wpaths[k], (s, k)
            g, lw = mb.student_fwd_bwd(k, sp[k], wpath, acts[k], acts[k + 1], S, norm)
            assert out["weight"][k] == pytest.approx(lw, rel=2e-2), (s, k)
            mb.sgd_path(k, wpath, sp[k], sv[k], g)
    for k in range(6):
        np.testing.assert_array_equal(arch.alpha[k], ref.alpha[k])
        base, _, total = p.layouts[k]
        got = p.params()[base:base + total].cpu().numpy()
        assert np.linalg.norm(got - sp[k]) <= 2e-2 * np.linalg.norm(sp[k])
