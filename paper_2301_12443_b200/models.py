"""Block definitions of the CIFAR workload and its algorithmic work accounting.

Teacher (frozen, BN folded): ResNet-18-CIFAR in 4 BPDG blocks —
  B0 = stem 3x3 3->64 + 2 BasicBlocks(64) @32x32, B1..B3 = 2 BasicBlocks each
  at 128@16x16, 256@8x8, 512@4x4 (first one strided, 1x1 projection shortcut).
Student (trained): one residual unit per block —
  conv3x3(Cin->Cout/2, stride s) BN ReLU, conv3x3(->Cout) BN, 1x1(Cin->Cout, s) BN, add, ReLU.
Mirrors csrc/exec/partition.cpp and oracle/bd_oracle.c.  The
FLOP and byte counts here define the roofline denominators.
"""
from __future__ import annotations

from typing import List, Tuple

T_CH = (3, 64, 128, 256, 512)
T_HW = (32, 32, 16, 8, 4)
BLOCKS = 4
BF16, F32 = 2, 4

Conv = Tuple[int, int, int, int, int, int]  # cin, cout, r, stride, hin, hout


def teacher_convs(k: int) -> List[Tuple[Conv, bool]]:
    """(conv, has_residual_read) in execution order."""
    out = []
    cin, hw = T_CH[k], T_HW[k]
    if k == 0:
        out.append(((3, 64, 3, 1, 32, 32), False))
        cin = 64
    cout = T_CH[k + 1]
    s = T_HW[k] // T_HW[k + 1]
    for b in range(2):
        st = s if b == 0 else 1
        ci = cin if b == 0 else cout
        ohw = hw // st
        out.append(((ci, cout, 3, st, hw, ohw), False))
        if st != 1 or ci != cout:
            out.append(((ci, cout, 1, st, hw, ohw), False))
        out.append(((cout, cout, 3, 1, ohw, ohw), True))
        hw = ohw
    return out


def student_geom(k: int):
    cin, cout = T_CH[k], T_CH[k + 1]
    return dict(cin=cin, cout=cout, mid=cout // 2, hin=T_HW[k], hout=T_HW[k + 1], stride=T_HW[k] // T_HW[k + 1])


def conv_flops(n: int, c: Conv) -> float:
    cin, cout, r, _, _, hout = c
    return 2.0 * n * hout * hout * cout * r * r * cin


def student_param_count(k: int) -> int:
    g = student_geom(k)
    return g["mid"] * 9 * g["cin"] + g["cout"] * 9 * g["mid"] + g["cout"] * g["cin"] + 2 * g["mid"] + 4 * g["cout"]


def teacher_flops(n: int, k: int) -> float:
    return sum(conv_flops(n, c) for c, _ in teacher_convs(k))


def student_flops(n: int, k: int) -> float:
    g = student_geom(k)
    c1 = (g["cin"], g["mid"], 3, g["stride"], g["hin"], g["hout"])
    c2 = (g["mid"], g["cout"], 3, 1, g["hout"], g["hout"])
    sc = (g["cin"], g["cout"], 1, g["stride"], g["hin"], g["hout"])
    fwd = conv_flops(n, c1) + conv_flops(n, c2) + conv_flops(n, sc)
    bwd = conv_flops(n, c2) * 2 + conv_flops(n, sc) + conv_flops(n, c1)  # dgrad2 + wgrad2 + wgradsc + wgrad1
    return fwd + bwd


def step_flops(n: int, blocks=range(BLOCKS)) -> float:
    return sum(teacher_flops(n, k) + student_flops(n, k) for k in blocks)


def _act(n, hw, c):
    return n * hw * hw * c * BF16


def step_bytes(n: int, blocks=range(BLOCKS), act_bytes: int = BF16) -> float:
    """ALGORITHMIC HBM bytes of one step (the roofline denominator): every logical tensor
    of the step written once and read once — the 3-channel input image, each teacher conv output, the
    student's y1, a1, y2, ysc (forward) and dy2, dysc, g1, dy1 (backward) — every weight read once, the
    student gradients written once, and the momentum SGD's minimal traffic (w, v read+write, g read,
    bf16 shadow write).  Independent of how the kernels are split: re-reads, recomputation and padded
    channels of the implementation are NOT counted (step_bytes_decomposition counts those)."""
    def act(hw, c):
        return n * hw * hw * c * act_bytes

    total = 0.0
    for k in blocks:
        if k == 0:
            total += 2 * act(32, 3)  # the image: written (load_data), read
        for (cin, cout, r, st, hin, hout), _ in teacher_convs(k):
            total += 2 * act(hout, cout) + cout * r * r * cin * act_bytes  # output w+r, weights r
        g = student_geom(k)
        m, o = act(g["hout"], g["mid"]), act(g["hout"], g["cout"])
        total += 2 * (2 * m + 2 * o)  # forward: y1, a1, y2, ysc written + read
        total += 2 * (2 * o + 2 * m)  # backward: dy2, dysc, g1, dy1 written + read
        p = student_param_count(k)
        total += p * act_bytes + p * F32 + p * (4 * F32 + F32 + BF16)  # weights r, grads w, SGD
    return total


def step_bytes_decomposition(n: int, blocks=range(BLOCKS)) -> float:
    """HBM traffic of the implemented (round-1) kernel decomposition: every kernel reads its operands
    once and writes its results once (weights once per step) — counts the BN statistics passes, the
    loss reduce + recompute and the 16-channel padded image, so it is larger than step_bytes()."""
    total = 0.0
    for k in blocks:
        if k == 0:
            total += _act(n, 32, 16)  # synthetic input written
        for (cin, cout, r, st, hin, hout), res in teacher_convs(k):
            cs = 16 if cin == 3 else cin
            total += _act(n, hin, cs) + _act(n, hout, cout) + cout * r * r * cs * BF16
            if res:
                total += _act(n, hout, cout)
        g = student_geom(k)
        cs = 16 if g["cin"] == 3 else g["cin"]
        x = _act(n, g["hin"], cs)
        m = _act(n, g["hout"], g["mid"])
        o = _act(n, g["hout"], g["cout"])
        total += (x + m) + (x + o)             # conv1, shortcut
        total += m + (m + m)                   # bn1 stats, bn1 apply
        total += (m + o)                       # conv2
        total += 2 * o                         # bn2 / bnsc stats
        total += 3 * o + (3 * o + 2 * o)       # loss reduce, loss bwd apply (recompute)
        total += (m + o) + (x + o)             # wgrad2, wgrad sc
        total += (o + m + m)                   # dgrad2 (+ relu mask read), g1 write
        total += 2 * m + (2 * m + m)           # bn1 bwd reduce + apply
        total += (x + m)                       # wgrad1
        total += student_param_count(k) * (3 * F32 + 2 * F32 + BF16)  # SGD: w,v rw; g r; shadow w
    return total


def step_working_set_bytes(n: int, blocks=range(BLOCKS)) -> int:
    """Distinct device bytes touched per step (activations + parameters)."""
    total = 0
    for k in blocks:
        if k == 0:
            total += _act(n, 32, 16)
        for (cin, cout, r, st, hin, hout), _ in teacher_convs(k):
            total += _act(n, hout, cout)
        g = student_geom(k)
        total += 4 * _act(n, g["hout"], g["mid"]) + 4 * _act(n, g["hout"], g["cout"])
        total += student_param_count(k) * (3 * F32 + BF16)
    return int(total)
