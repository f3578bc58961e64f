"""Generate tests/golden/bd_torch_fp32.npz — pins the C oracle (oracle/bd_oracle.c)
against an independent implementation: the same blockwise-distillation step
written with torch fp32 ops + autograd (the paper's implementation framework,
PAPER.md:393-398, 456-458).  Inputs (data, teacher and student weights) come
from the oracle's Philox generator in fp32 mode; everything computed here is
torch's.  Run from the repo root:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import bd  # noqa: E402

torch.set_num_threads(8)
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bd_torch_fp32.npz")
B = 3          # odd: exercises the remainder rule
GROUPS = {0: 1, 1: 2, 2: 1, 3: 3}   # DP degree per block (per-shard BN statistics, summed grads)
STEPS = 2
SUB = 97       # subsample stride for stored tensors


def nchw(x):
    return torch.from_numpy(np.ascontiguousarray(x)).permute(0, 3, 1, 2)


def conv_w(flat, k, r, c):
    return torch.from_numpy(flat.reshape(k, r, r, c).copy()).permute(0, 3, 1, 2).contiguous()


def teacher_fwd(k, tp, x):
    """ResNet-18-CIFAR block k with folded BN."""
    p = torch.from_numpy(tp)
    off = [0]

    def take(n):
        t = p[off[0]:off[0] + n]
        off[0] += n
        return t

    def conv(x, cin, cout, r, s):
        w = take(cout * r * r * cin).reshape(cout, r, r, cin).permute(0, 3, 1, 2)
        b = take(cout)
        return F.conv2d(x, w, b, stride=s, padding=r // 2)

    cin = bd.geom(k)["cin"]
    if k == 0:
        x = F.relu(conv(x, 3, 64, 3, 1))
        cin = 64
    cout = bd.geom(k)["cout"]
    s = bd.geom(k)["hin"] // bd.geom(k)["hout"]
    for blk in range(2):
        st = s if blk == 0 else 1
        ci = cin if blk == 0 else cout
        h = F.relu(conv(x, ci, cout, 3, st))
        y2 = conv(h, cout, cout, 3, 1)  # consumed in order: conv1, conv2, proj
        sc = conv(x, ci, cout, 1, st) if (st != 1 or ci != cout) else x
        x = F.relu(y2 + sc)
    assert off[0] == tp.size
    return x


def student_loss(k, sp, x, t, norm):
    g = bd.geom(k)
    lay = bd.student_layout(k)
    cin, cout = g["cin"], g["cout"]
    mid = cout // 2
    s = g["hin"] // g["hout"]

    def part(name):
        o, n = lay[name]
        return sp[o:o + n]

    w1 = part("w1").reshape(mid, 3, 3, cin).permute(0, 3, 1, 2)
    w2 = part("w2").reshape(cout, 3, 3, mid).permute(0, 3, 1, 2)
    wsc = part("wsc").reshape(cout, 1, 1, cin).permute(0, 3, 1, 2)
    y1 = F.conv2d(x, w1, stride=s, padding=1)
    a1 = F.relu(F.batch_norm(y1, None, None, part("g1"), part("b1"), training=True, eps=1e-5))
    y2 = F.conv2d(a1, w2, padding=1)
    ys = F.conv2d(x, wsc, stride=s)
    z = F.batch_norm(y2, None, None, part("g2"), part("b2"), training=True, eps=1e-5) + \
        F.batch_norm(ys, None, None, part("gsc"), part("bsc"), training=True, eps=1e-5)
    return ((F.relu(z) - t) ** 2).sum() / norm


def main():
    tps = {k: bd.teacher_params(k, bf16_mode=0) for k in range(4)}
    sps = {k: torch.from_numpy(bd.student_params(k)).clone() for k in range(4)}
    moms = {k: torch.zeros_like(sps[k]) for k in range(4)}
    rec = {}
    for step in range(STEPS):
        x = bd.make_input(B, step * B, bf16_mode=0)
        act = nchw(x)
        for k in range(4):
            with torch.no_grad():
                t = teacher_fwd(k, tps[k], act)
            g = bd.geom(k)
            norm = float(B) * g["cout"] * g["hout"] * g["hout"]
            p = sps[k].clone().requires_grad_(True)
            loss = 0.0
            base, extra = divmod(B, GROUPS[k])
            first = 0
            for r in range(GROUPS[k]):
                cnt = base + (1 if r < extra else 0)
                loss = loss + student_loss(k, p, act[first:first + cnt], t[first:first + cnt], norm)
                first += cnt
            loss.backward()
            grad = p.grad.detach()
            with torch.no_grad():   # torch.optim.SGD(momentum=0.9) semantics
                moms[k] = moms[k] * bd.MOMENTUM + grad
                sps[k] = sps[k] - bd.LR * moms[k]
            tnhwc = t.permute(0, 2, 3, 1).contiguous().numpy()
            rec[f"s{step}_b{k}_loss"] = np.float64(loss.item())
            rec[f"s{step}_b{k}_grad_sub"] = grad.numpy()[::SUB].copy()
            rec[f"s{step}_b{k}_teacher_sum"] = np.float64(tnhwc.astype(np.float64).sum())
            rec[f"s{step}_b{k}_teacher_sq"] = np.float64((tnhwc.astype(np.float64) ** 2).sum())
            rec[f"s{step}_b{k}_teacher_sub"] = tnhwc.reshape(-1)[::SUB].copy()
            for name, (o, n) in bd.student_layout(k).items():
                rec[f"s{step}_b{k}_gnorm_{name}"] = np.float64(grad[o:o + n].double().norm().item())
            act = t
    for k in range(4):
        rec[f"final_b{k}_param_sub"] = sps[k].numpy()[::SUB].copy()
    rec["meta"] = np.array([B, STEPS, SUB] + [GROUPS[k] for k in range(4)], np.int64)
    np.savez_compressed(OUT, **rec)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
