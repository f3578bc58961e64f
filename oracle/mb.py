"""TEST INFRASTRUCTURE ONLY — numpy face of the MobileNetV2 -> ProxylessNAS oracle
(oracle/_build/libmb_oracle.so, mb_oracle.h).  Used by tests/, smoke() and bench.py's baseline
legs as the checker; never imported by the product package."""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libmb_oracle.so")
BLOCKS = 6
CANDIDATES = 6
SEED_DATA, SEED_TEACHER, SEED_STUDENT, SEED_PATH = 1234, 1, 2, 7
LR, MOMENTUM = 0.1, 0.9

_L = None
F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def lib():
    global _L
    if _L is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
        L = ctypes.CDLL(LIB)
        I, S, U, D = ctypes.c_int, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_double
        for f in ("mbo_channels", "mbo_true_channels", "mbo_student_layers"):
            getattr(L, f).argtypes = [I]
            getattr(L, f).restype = I
        L.mbo_hw.argtypes = [I, I]
        L.mbo_hw.restype = I
        L.mbo_layer_candidates.argtypes = [I, I]
        L.mbo_layer_candidates.restype = I
        for f in ("mbo_teacher_param_count", "mbo_student_param_count"):
            getattr(L, f).argtypes = [I]
            getattr(L, f).restype = S
        L.mbo_candidate_offset.argtypes = [I, I, I, ctypes.POINTER(S)]
        L.mbo_candidate_offset.restype = S
        L.mbo_input.argtypes = [I, ctypes.c_int64, I, U, F32P, I]
        L.mbo_teacher_init.argtypes = [I, U, F32P, I]
        L.mbo_student_init.argtypes = [I, U, F32P]
        L.mbo_sample_path.argtypes = [I, U, ctypes.c_int64, I32P]
        L.mbo_teacher_fwd.argtypes = [I, F32P, I, I, F32P, F32P, I]
        L.mbo_student_fwd_bwd.argtypes = [I, F32P, I32P, I, I, F32P, F32P, D, I, F32P, ctypes.POINTER(D)]
        L.mbo_sgd_path.argtypes = [I, I32P, F32P, F32P, F32P, ctypes.c_float, ctypes.c_float]
        L.mbo_set_family.argtypes = [I]
        L.mbo_family.restype = I
        _L = L
    return _L


def set_family(f: int):
    """0 = MobileNetV2 teacher (configs[2]), 1 = EfficientNet-B0 teacher (configs[3])."""
    global FAMILY
    lib().mbo_set_family(int(f))
    FAMILY = int(f)


FAMILY = 0


def channels(b: int) -> int:
    """stored channels at boundary b (tensor-tile granularity)"""
    return lib().mbo_channels(b)


def true_channels(b: int) -> int:
    """the architecture's channels at boundary b (the stored extra channels are identically zero)"""
    return lib().mbo_true_channels(b)


def hw(b: int, S: int) -> int:
    return lib().mbo_hw(b, S)


def layers(b: int) -> int:
    return lib().mbo_student_layers(b)


def candidates(b: int, l: int) -> int:
    return lib().mbo_layer_candidates(b, l)


def candidate_span(b: int, l: int, c: int):
    n = ctypes.c_size_t()
    off = lib().mbo_candidate_offset(b, l, c, ctypes.byref(n))
    return int(off), int(n.value)


def student_param_count(b: int) -> int:
    return int(lib().mbo_student_param_count(b))


def teacher_param_count(b: int) -> int:
    return int(lib().mbo_teacher_param_count(b))


def act_shape(b: int, n: int, S: int):
    c = channels(b)
    return (n, hw(b, S), hw(b, S), c)


def image(n: int, first: int, S: int, seed: int = SEED_DATA, bf16: bool = True) -> np.ndarray:
    out = np.empty((n, S, S, 3), np.float32)
    lib().mbo_input(n, first, S, seed, out, int(bf16))
    return out


def teacher_params(b: int, seed: int = SEED_TEACHER, bf16: bool = True) -> np.ndarray:
    p = np.empty(teacher_param_count(b), np.float32)
    lib().mbo_teacher_init(b, seed, p, int(bf16))
    return p


def student_params(b: int, seed: int = SEED_STUDENT) -> np.ndarray:
    p = np.empty(student_param_count(b), np.float32)
    lib().mbo_student_init(b, seed, p)
    return p


def sample_path(b: int, draw: int, seed: int = SEED_PATH) -> np.ndarray:
    p = np.zeros(layers(b), np.int32)
    lib().mbo_sample_path(b, seed, draw, p)
    return p


def teacher_fwd(b: int, tp: np.ndarray, x: np.ndarray, S: int, bf16: bool = True) -> np.ndarray:
    n = x.shape[0]
    out = np.empty(act_shape(b + 1, n, S), np.float32)
    rc = lib().mbo_teacher_fwd(b, tp, n, S, np.ascontiguousarray(x, np.float32), out, int(bf16))
    assert rc == 0
    return out


def student_fwd_bwd(b: int, sp: np.ndarray, path: np.ndarray, x: np.ndarray, t: np.ndarray, S: int, norm: float,
                    bf16: bool = True):
    g = np.empty_like(sp)
    loss = ctypes.c_double()
    rc = lib().mbo_student_fwd_bwd(b, sp, np.ascontiguousarray(path, np.int32), x.shape[0], S,
                                   np.ascontiguousarray(x, np.float32), np.ascontiguousarray(t, np.float32),
                                   float(norm), int(bf16), g, ctypes.byref(loss))
    assert rc == 0
    return g, loss.value


def sgd_path(b: int, path: np.ndarray, w: np.ndarray, v: np.ndarray, g: np.ndarray, lr=LR, mu=MOMENTUM):
    lib().mbo_sgd_path(b, np.ascontiguousarray(path, np.int32), w, v, g, lr, mu)


class Trainer:
    """Whole-chain oracle of the MBConv workload: every block on the full batch (or DP shards)."""

    def __init__(self, b: int, S: int, bf16: bool = True, blocks: Optional[List[int]] = None):
        self.b, self.S, self.bf16 = b, S, bf16
        self.blocks = list(range(BLOCKS)) if blocks is None else blocks
        self.tp = {k: teacher_params(k, bf16=bf16) for k in range(BLOCKS)}
        self.sp = {k: student_params(k) for k in self.blocks}
        self.sv = {k: np.zeros_like(self.sp[k]) for k in self.blocks}

    def step(self, step: int, paths: Dict[int, np.ndarray], groups: Optional[Dict[int, int]] = None):
        groups = groups or {}
        x = image(self.b, step * self.b, self.S, bf16=self.bf16)
        acts = [x]
        for k in range(max(self.blocks) + 1):
            acts.append(teacher_fwd(k, self.tp[k], acts[-1], self.S, self.bf16))
        losses = {}
        for k in self.blocks:
            c, hh = true_channels(k + 1), hw(k + 1, self.S)
            norm = float(self.b) * c * hh * hh
            g_total = np.zeros_like(self.sp[k])
            loss = 0.0
            gsz = groups.get(k, 1)
            base, extra = divmod(self.b, gsz)
            first = 0
            for i in range(gsz):
                cnt = base + (1 if i < extra else 0)
                g, l_ = student_fwd_bwd(k, self.sp[k], paths[k], acts[k][first:first + cnt],
                                        acts[k + 1][first:first + cnt], self.S, norm, self.bf16)
                g_total += g
                loss += l_
                first += cnt
            sgd_path(k, paths[k], self.sp[k], self.sv[k], g_total)
            losses[k] = loss
        self.acts = acts
        return losses


# ---------------------------------------------------------------- per-candidate layout (mb_oracle.c cand_lay)
KS, ES = (3, 5, 7), (3, 6)
NLF = ((3, 3, 4, 3, 3, 1), (3, 2, 3, 3, 4, 1))
CHF = ((3, 32, 32, 64, 128, 192, 320), (3, 32, 64, 128, 128, 192, 320))
CTF = ((3, 24, 32, 64, 96, 160, 320), (3, 24, 40, 80, 112, 192, 320))  # true widths
KF = ((3, 3, 3, 3, 3, 3), (3, 5, 3, 5, 5, 3))
DIV = (1, 4, 8, 16, 16, 32, 32)


class _FamTable:
    def __init__(self, t):
        self.t = t

    def __getitem__(self, i):
        return self.t[FAMILY][i]

    def __len__(self):
        return len(self.t[FAMILY])


NL = _FamTable(NLF)
CH = _FamTable(CHF)
CT = _FamTable(CTF)


def se_ch(cin: int) -> int:
    return max(1, cin // 4) if FAMILY == 1 else 0


def round_ch(c: int) -> int:
    return 16 if c <= 16 else 32 if c <= 32 else (c + 63) // 64 * 64


def teacher_layer(b: int, l: int):
    """(t, k, cin, cout, stride) of teacher MBConv layer l of block b (stored widths)."""
    return teacher_layer_t(b, l)[:5]


def teacher_layer_t(b: int, l: int):
    """(t, k, cin, cout, stride, cin_true, cout_true)."""
    if b == 0:
        return ((1, 3, 32, 16, 1, 32, 16), (6, 3, 16, 32, 2, 16, 24), (6, 3, 32, 32, 1, 24, 24))[l]
    cin, cout = CH[b], CH[b + 1]
    s = DIV[b + 1] // DIV[b]
    k = KF[FAMILY][b]
    return (6, k, cin, cout, s, CT[b], CT[b + 1]) if l == 0 else (6, k, cout, cout, 1, CT[b + 1], CT[b + 1])


def student_layer(b: int, l: int, c: int):
    """dict(kind, k, e, E, cin, cout, stride, res, Et, cin_t, cout_t) of candidate c of student layer l
    (stored widths E / cin / cout, true widths *_t; residual by the true widths)."""
    if b == 0 and l == 0:
        return dict(kind="stem", k=3, e=0, E=32, cin=3, cout=32, stride=2, res=False, Et=32, cin_t=3, cout_t=32)
    t, _, cin, cout, s, cin_t, cout_t = teacher_layer_t(b, l - 1 if b == 0 else l)
    if b == 0 and l == 1:
        k, e = 3, 1
    else:
        k, e = KS[c % 3], ES[c // 3]
    E = cin if e == 1 else round_ch(cin * e)
    Et = cin_t if e == 1 else cin_t * e
    return dict(kind="mb", k=k, e=e, E=E, cin=cin, cout=cout, stride=s, res=(s == 1 and cin_t == cout_t), Et=Et,
                cin_t=cin_t, cout_t=cout_t)


def candidate_layout(b: int, l: int, c: int) -> Dict[str, tuple]:
    """{tensor: (offset within the candidate, count)}."""
    g = student_layer(b, l, c)
    if g["kind"] == "stem":
        return {"w": (0, 32 * 9 * 16), "g2": (32 * 9 * 16, 32), "b2": (32 * 9 * 16 + 32, 32)}
    E, k, cin, cout = g["E"], g["k"], g["cin"], g["cout"]
    out, o = {}, 0
    sizes = ([("we", E * cin)] if g["e"] != 1 else []) + [("wd", E * k * k), ("wp", cout * E)] + \
        ([("g1", E), ("b1", E)] if g["e"] != 1 else []) + [("g2", E), ("b2", E), ("g3", cout), ("b3", cout)]
    for name, n in sizes:
        out[name] = (o, n)
        o += n
    return out
