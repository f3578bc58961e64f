"""ProxylessNAS architecture-parameter round (paper_2301_12443_b200/nas.py), host logic (CPU)."""
import numpy as np
import pytest

from paper_2301_12443_b200 import mb_models, nas


@pytest.fixture(autouse=True)
def _family():
    mb_models.set_family("mbv2")
    yield
    mb_models.set_family("mbv2")


def test_sampling_follows_softmax_and_is_deterministic():
    a = nas.ArchParams(range(6))
    assert a.sample(3, 5) == a.sample(3, 5)
    assert a.sample(0, 1)[:2] == [0, 0]  # stem + fixed MBConv1
    a.alpha[2][:, 4] = 6.0  # p(4) = e^6 / (e^6 + 5) ~ 0.988
    hits = sum(a.sample(2, d)[l] == 4 for d in range(400) for l in range(nas.student_layers(2)))
    assert hits / (400 * nas.student_layers(2)) > 0.95
    uni = nas.ArchParams([1])
    counts = np.bincount([uni.sample(1, d)[0] for d in range(3000)], minlength=6) / 3000
    assert np.abs(counts - 1 / 6).max() < 0.03


def test_reinforce_moves_alpha_towards_lower_loss():
    a = nas.ArchParams([1], lr=0.05)
    path = [2, 2, 2]
    a.update(1, path, 1.0)  # first round sets the baseline: zero advantage, no move
    assert not a.alpha[1].any()
    a.update(1, path, 0.5)  # lower loss than the baseline: the sampled candidates gain probability
    assert (a.alpha[1][:, 2] > 0).all() and (a.alpha[1][:, [0, 1, 3, 4, 5]] < 0).all()
    p_before = a.probs(1)[0, 2]
    a.update(1, [3, 3, 3], 2.0)  # higher loss: candidate 3 loses probability
    assert a.probs(1)[0, 3] < 1 / 6 and a.probs(1)[0, 2] > 1 / 6 and p_before > 1 / 6
    assert a.derived()[1] == [2, 2, 2]


def test_fixed_layers_never_move():
    a = nas.ArchParams([0], lr=0.1)
    a.update(0, [0, 0, 5, 5], 1.0)
    a.update(0, [0, 0, 5, 5], 0.1)
    assert not a.alpha[0][:2].any() and a.alpha[0][2:].any()
    assert 0.0 < a.entropy(0) <= 1.0
