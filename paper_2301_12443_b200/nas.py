"""ProxylessNAS architecture-parameter round for the supernet students (configs[2] / configs[3]).

PAPER.md:407-411: "each step periodically requires two rounds of forward/backward passes for students:
one for the architecture parameters and another for the weight parameters ... each round can be
regarded as a single training step", with ProxylessNAS (Cai et al., ICLR 2019) as the search backbone.

Every searchable MBConv layer l of student block k carries architecture parameters alpha[k][l] over its
6 candidates ({k3,k5,k7} x {e3,e6}); the path of a round is sampled from softmax(alpha) (binarised
path, one candidate active).  The architecture update is ProxylessNAS's REINFORCE form (Cai et al. §3.3:
grad_alpha J = E[R * grad_alpha log p(path)], R = -L_k the block's distillation loss, an exponential
moving-average baseline), applied with Adam as ProxylessNAS's architecture optimiser (beta1 = 0,
beta2 = 0.999, lr 6e-3).  Blockwise: block k's alpha follows block k's loss only.  The gradient form
needs only the loss of the sampled path, so the architecture round is one more student forward /
backward whose weight gradients are discarded — exactly the "single training step" the paper counts.

Per NAS step (nas_step): teacher forward once, architecture round (path ~ softmax(alpha), student
forward/backward, losses -> alpha update), weight round (a new path ~ softmax(alpha), student
forward/backward, SGD update of the active candidates).  Path sampling is a Philox inverse-CDF draw,
so the oracle side of the tests replays the identical paths.  Host logic only: the kernels are the
executor's (include/pbdx.h pbdx_set_path / pbdx_student_step / pbdx_apply_update).
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence

import numpy as np

from . import mb_models

CANDIDATES = 6
KEY_ARCH = 0xA5C4A4C4


def searchable(block: int, layer: int) -> bool:
    """block 0: stem and the fixed MBConv1 are not searchable (mb_oracle.c mbo_layer_candidates)."""
    return not (block == 0 and layer < 2)


def student_layers(block: int) -> int:
    return mb_models.NL[block] + (1 if block == 0 else 0)


def _uniform(draw: int, layer: int, block: int, seed: int) -> float:
    o = mb_models._philox((draw & 0xFFFFFFFF, (draw >> 32) & 0xFFFFFFFF, layer, block), (seed, KEY_ARCH))
    return (o >> 8) * (1.0 / 16777216.0)


class ArchParams:
    """alpha, Adam state and REINFORCE baseline of the searchable layers of `blocks`."""

    def __init__(self, blocks: Sequence[int], lr: float = 6e-3, beta1: float = 0.0, beta2: float = 0.999,
                 eps: float = 1e-8, baseline_decay: float = 0.9, seed: int = 11):
        self.blocks = list(blocks)
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.decay = baseline_decay
        self.seed = seed
        self.alpha = {k: np.zeros((student_layers(k), CANDIDATES)) for k in self.blocks}
        self.m = {k: np.zeros_like(a) for k, a in self.alpha.items()}
        self.v = {k: np.zeros_like(a) for k, a in self.alpha.items()}
        self.t = {k: 0 for k in self.blocks}
        self.baseline: Dict[int, float] = {}

    def probs(self, k: int) -> np.ndarray:
        a = self.alpha[k]
        e = np.exp(a - a.max(axis=1, keepdims=True))
        return e / e.sum(axis=1, keepdims=True)

    def sample(self, k: int, draw: int) -> List[int]:
        """path[l] ~ softmax(alpha[k][l]) by inverse CDF of a Philox uniform (fixed layers: 0)."""
        p = self.probs(k)
        path = []
        for l in range(student_layers(k)):
            if not searchable(k, l):
                path.append(0)
                continue
            u = _uniform(draw, l, k, self.seed)
            c = int(np.searchsorted(np.cumsum(p[l]), u, side="right"))
            path.append(min(c, CANDIDATES - 1))
        return path

    def update(self, k: int, path: Sequence[int], loss: float):
        """REINFORCE with an EMA baseline: d(-J)/d alpha[l] = -(R - b) (onehot(path[l]) - p[l]), Adam step."""
        reward = -float(loss)
        base = self.baseline.get(k, reward)  # first round: zero advantage
        adv = reward - base
        self.baseline[k] = self.decay * base + (1.0 - self.decay) * reward
        p = self.probs(k)
        g = np.zeros_like(self.alpha[k])
        for l, c in enumerate(path):
            if searchable(k, l):
                onehot = np.zeros(CANDIDATES)
                onehot[c] = 1.0
                g[l] = -adv * (onehot - p[l])
        self.t[k] += 1
        t = self.t[k]
        self.m[k] = self.beta1 * self.m[k] + (1.0 - self.beta1) * g
        self.v[k] = self.beta2 * self.v[k] + (1.0 - self.beta2) * g * g
        mh = self.m[k] / (1.0 - self.beta1 ** t)
        vh = self.v[k] / (1.0 - self.beta2 ** t)
        self.alpha[k] -= self.lr * mh / (np.sqrt(vh) + self.eps)

    def derived(self) -> Dict[int, List[int]]:
        """The searched architecture: the most probable candidate of every layer."""
        return {k: [int(np.argmax(self.alpha[k][l])) if searchable(k, l) else 0 for l in range(student_layers(k))]
                for k in self.blocks}

    def entropy(self, k: int) -> float:
        p = self.probs(k)
        rows = [l for l in range(student_layers(k)) if searchable(k, l)]
        return float(-sum((p[l] * np.log(p[l])).sum() for l in rows)) / max(1, len(rows)) / math.log(CANDIDATES)


def nas_step(part, arch: ArchParams, step: int, stream=None) -> Dict[str, Dict[int, float]]:
    """One ProxylessNAS step of a partition (executor.Partition over an MBConv model): teacher forward,
    architecture round (alpha update from the block losses), weight round (SGD).  Returns both rounds'
    block losses."""
    blocks = arch.blocks
    arch_paths = {k: arch.sample(k, 2 * step) for k in blocks}
    for k in blocks:
        part.set_path(k, arch_paths[k])
    part.teacher_forward(stream)
    part.student_step(stream)  # architecture round: weight gradients are discarded
    la = dict(zip(blocks, part.losses()))
    for k in blocks:
        arch.update(k, arch_paths[k], la[k])
    for k in blocks:
        part.set_path(k, arch.sample(k, 2 * step + 1))
    part.student_step(stream)  # weight round on the same teacher targets
    part.apply_update(stream)
    lw = dict(zip(blocks, part.losses()))
    return {"arch": la, "weight": lw}
