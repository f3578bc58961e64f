"""TEST INFRASTRUCTURE ONLY — numpy face of the C oracle (oracle/_build/libbd_oracle.so).

Used by tests/ (parity checker), __graft_entry__.smoke() and bench.py's
cpu_baseline leg.  Never imported by the product package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libbd_oracle.so")
BLOCKS = 4
SEED_DATA, SEED_TEACHER, SEED_STUDENT = 1234, 1, 2
LR, MOMENTUM = 0.1, 0.9

_L = None
F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def lib():
    global _L
    if _L is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
        L = ctypes.CDLL(LIB)
        for f in ("bdo_in_channels", "bdo_out_channels", "bdo_in_hw", "bdo_out_hw"):
            getattr(L, f).argtypes = [ctypes.c_int]
            getattr(L, f).restype = ctypes.c_int
        for f in ("bdo_student_param_count", "bdo_teacher_param_count"):
            getattr(L, f).argtypes = [ctypes.c_int]
            getattr(L, f).restype = ctypes.c_size_t
        L.bdo_philox.argtypes = [ctypes.POINTER(ctypes.c_uint32)] * 3
        L.bdo_input.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, F32P, ctypes.c_int]
        L.bdo_teacher_init.argtypes = [ctypes.c_int, ctypes.c_uint32, F32P, ctypes.c_int]
        L.bdo_student_init.argtypes = [ctypes.c_int, ctypes.c_uint32, F32P]
        L.bdo_teacher_fwd.argtypes = [ctypes.c_int, F32P, ctypes.c_int, F32P, F32P, ctypes.c_int]
        L.bdo_student_fwd_bwd.argtypes = [ctypes.c_int, F32P, ctypes.c_int, F32P, F32P, ctypes.c_double,
                                          ctypes.c_int, F32P, ctypes.POINTER(ctypes.c_double)]
        L.bdo_sgd.argtypes = [ctypes.c_size_t, F32P, F32P, F32P, ctypes.c_float, ctypes.c_float]
        L.bdo_bf16.argtypes = [ctypes.c_float]
        L.bdo_bf16.restype = ctypes.c_float
        L.bdo_threads.restype = ctypes.c_int
        _L = L
    return _L


def geom(k):
    L = lib()
    return dict(cin=L.bdo_in_channels(k), cout=L.bdo_out_channels(k), hin=L.bdo_in_hw(k), hout=L.bdo_out_hw(k))


def student_layout(k):
    """Offsets of the flat student parameter vector (bd_oracle.c sgeom)."""
    g = geom(k)
    cin, cout = g["cin"], g["cout"]
    mid = cout // 2
    sizes = [("w1", mid * 9 * cin), ("w2", cout * 9 * mid), ("wsc", cout * cin), ("g1", mid), ("b1", mid),
             ("g2", cout), ("b2", cout), ("gsc", cout), ("bsc", cout)]
    out, o = {}, 0
    for name, n in sizes:
        out[name] = (o, n)
        o += n
    return out


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().bdo_philox(c, k, o)
    return list(o)


def bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16 (vectorised, same rule as bdo_bf16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)


def make_input(n, first, bf16_mode=1, seed=SEED_DATA):
    out = np.empty((n, 32, 32, 3), np.float32)
    lib().bdo_input(n, first, seed, out, bf16_mode)
    return out


def teacher_params(k, bf16_mode=1, seed=SEED_TEACHER):
    p = np.empty(lib().bdo_teacher_param_count(k), np.float32)
    lib().bdo_teacher_init(k, seed, p, bf16_mode)
    return p


def student_params(k, seed=SEED_STUDENT):
    p = np.empty(lib().bdo_student_param_count(k), np.float32)
    lib().bdo_student_init(k, seed, p)
    return p


def teacher_fwd(k, tparams, x, bf16_mode=1):
    g = geom(k)
    n = x.shape[0]
    out = np.empty((n, g["hout"], g["hout"], g["cout"]), np.float32)
    lib().bdo_teacher_fwd(k, tparams, n, np.ascontiguousarray(x, np.float32), out, bf16_mode)
    return out


def student_fwd_bwd(k, sparams, x, t_out, global_batch, bf16_mode=1):
    g = geom(k)
    norm = float(global_batch) * g["cout"] * g["hout"] * g["hout"]
    grads = np.empty_like(sparams)
    loss = ctypes.c_double()
    lib().bdo_student_fwd_bwd(k, sparams, x.shape[0], np.ascontiguousarray(x, np.float32),
                              np.ascontiguousarray(t_out, np.float32), norm, bf16_mode, grads, ctypes.byref(loss))
    return loss.value, grads


def sgd(w, v, g, lr=LR, mu=MOMENTUM):
    lib().bdo_sgd(w.size, w, v, np.ascontiguousarray(g, np.float32), lr, mu)


class Trainer:
    """Whole-model CPU step (all blocks on one 'device' = the IR point) with the
    DP-group semantics of a partition: shards follow the remainder rule and
    their gradients are summed before one SGD step (DDP-style allreduce)."""

    def __init__(self, global_batch, bf16_mode=1, blocks=range(BLOCKS)):
        self.b = global_batch
        self.bf16 = bf16_mode
        self.blocks = list(blocks)
        self.tp = {k: teacher_params(k, bf16_mode) for k in range(BLOCKS)}
        self.sp = {k: student_params(k) for k in self.blocks}
        self.mom = {k: np.zeros_like(self.sp[k]) for k in self.blocks}

    def step(self, step_idx, groups=None):
        """groups: {block: g} DP degree per block (default 1). Returns per-block losses."""
        groups = groups or {}
        x = make_input(self.b, step_idx * self.b, self.bf16)
        act = x
        losses = {}
        for k in range(BLOCKS):
            t = teacher_fwd(k, self.tp[k], act, self.bf16)
            if k in self.blocks:
                g = groups.get(k, 1)
                total = np.zeros_like(self.sp[k])
                loss = 0.0
                base, extra = divmod(self.b, g)
                first = 0
                for r in range(g):
                    cnt = base + (1 if r < extra else 0)
                    l, gr = student_fwd_bwd(k, self.sp[k], act[first:first + cnt], t[first:first + cnt], self.b,
                                            self.bf16)
                    total += gr
                    loss += l
                    first += cnt
                losses[k] = loss
                sgd(self.sp[k], self.mom[k], total)
            act = t
        return losses
