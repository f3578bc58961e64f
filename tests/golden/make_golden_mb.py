"""Generate tests/golden/mb_torch_fp64.npz — pins the MBConv C oracle (oracle/mb_oracle.c) against an
independent implementation: the MobileNetV2 teacher / ProxylessNAS student blockwise-distillation
step written with torch ops + autograd (PyTorch is the paper's framework), in
float64 so the fixture is a clean reference for the oracle's fp32 mode.  The torch model runs at the
architectures' TRUE channel widths (MobileNetV2-1.0: 24/32/64/96/160/320, EfficientNet-B0:
24/40/80/112/192/320), slicing the oracle's zero-padded storage — so the fixture also pins that the
padded layout computes exactly the true-width network.  Inputs (data, teacher and
student weights, the sampled path) come from the oracle's Philox generators; everything computed
here is torch's (F.conv2d with groups for depthwise, F.batch_norm in training mode, hardtanh as
ReLU6, autograd).  Run from the repo root:  python tests/golden/make_golden_mb.py [0|1]   (1 = EfficientNet-B0 teacher:
swish, squeeze-excite -> effb0_torch_fp64.npz)
"""
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import mb  # noqa: E402

torch.set_num_threads(8)
FAMILY = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # 0 MobileNetV2, 1 EfficientNet-B0 teacher
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                   "mb_torch_fp64.npz" if FAMILY == 0 else "effb0_torch_fp64.npz")
B, S = 3, 64
SUB = 53
DRAW = 5  # path sampling index
DT = torch.float64


def nchw(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DT).permute(0, 3, 1, 2)


def nhwc(x):
    return x.permute(0, 2, 3, 1).contiguous()


def relu6(x):
    return F.hardtanh(x, 0.0, 6.0)


def tact(x):
    """the teacher's activation: ReLU6 (MobileNetV2) or swish = x * sigmoid(x) (EfficientNet-B0)"""
    return x * torch.sigmoid(x) if FAMILY == 1 else relu6(x)


def teacher_fwd(b, tp, x):
    """The teacher at its TRUE widths (MobileNetV2-1.0 / EfficientNet-B0): the stored parameter
    vector is sliced to the true channels, the stored extra channels of x are ignored and the output
    is zero-padded back to the stored width (the layout the oracle uses)."""
    p = torch.from_numpy(tp).to(DT)
    off = [0]

    def take(n):
        t = p[off[0]:off[0] + n]
        off[0] += n
        return t

    if b == 0:
        w = take(32 * 9 * 16).reshape(32, 3, 3, 16)[..., :3].permute(0, 3, 1, 2)
        x = tact(F.conv2d(x[:, :3], w, take(32), stride=2, padding=1))
    else:
        x = x[:, :mb.CT[b]]
    for l in range(mb.NL[b]):
        t, k, cin, cout, s, ci, co = mb.teacher_layer_t(b, l)
        E = cin if t == 1 else mb.round_ch(cin * t)
        Et = ci * t
        h = x
        if t != 1:
            w = take(E * cin).reshape(E, cin)[:Et, :ci].reshape(Et, ci, 1, 1)
            h = tact(F.conv2d(h, w, take(E)[:Et]))
        wd = take(E * k * k).reshape(E, 1, k, k)[:Et]
        h = tact(F.conv2d(h, wd, take(E)[:Et], stride=s, padding=k // 2, groups=Et))
        cs = mb.se_ch(cin)
        if cs:  # squeeze-excite, reduce width 0.25 x the true input channels
            cst = mb.se_ch(ci)
            w1, b1 = take(cs * E).reshape(cs, E)[:cst, :Et], take(cs)[:cst]
            w2, b2 = take(E * cs).reshape(E, cs)[:Et, :cst], take(E)[:Et]
            z = h.mean(dim=(2, 3))
            z = z @ w1.T + b1
            z = z * torch.sigmoid(z)
            gate = torch.sigmoid(z @ w2.T + b2)
            h = h * gate[:, :, None, None]
        wp = take(cout * E).reshape(cout, E)[:co, :Et].reshape(co, Et, 1, 1)
        y = F.conv2d(h, wp, take(cout)[:co])
        x = y + x if (s == 1 and ci == co) else y
    return F.pad(x, (0, 0, 0, 0, 0, mb.CH[b + 1] - x.shape[1]))


def student(b, sp, path, x, t, norm):
    """loss, {(layer, tensor): grad} of the active path.  The network runs at the TRUE widths: every
    parameter is a leaf in the stored layout and enters through its true-width slice, so the stored
    extra entries get exactly zero gradient (as in the oracle / product)."""
    params = {}
    for l in range(mb.layers(b)):
        c = int(path[l])
        off, _ = mb.candidate_span(b, l, c)
        for name, (o, n) in mb.candidate_layout(b, l, c).items():
            params[(l, name)] = torch.tensor(sp[off + o: off + o + n], dtype=DT, requires_grad=True)

    def bn(y, l, g, be, n):
        return F.batch_norm(y, None, None, params[(l, g)][:n], params[(l, be)][:n], training=True, eps=1e-5)

    h = x[:, :3] if b == 0 else x[:, :mb.CT[b]]
    for l in range(mb.layers(b)):
        g = mb.student_layer(b, l, int(path[l]))
        if g["kind"] == "stem":
            w = params[(l, "w")].reshape(32, 3, 3, 16)[..., :3].permute(0, 3, 1, 2)
            h = relu6(bn(F.conv2d(h, w, stride=2, padding=1), l, "g2", "b2", 32))
            continue
        E, k, cin, cout = g["E"], g["k"], g["cin"], g["cout"]
        Et, ci, co = g["Et"], g["cin_t"], g["cout_t"]
        a = h
        if g["e"] != 1:
            we = params[(l, "we")].reshape(E, cin)[:Et, :ci].reshape(Et, ci, 1, 1)
            a = relu6(bn(F.conv2d(h, we), l, "g1", "b1", Et))
        wd = params[(l, "wd")].reshape(E, 1, k, k)[:Et]
        a = relu6(bn(F.conv2d(a, wd, stride=g["stride"], padding=k // 2, groups=Et), l, "g2", "b2", Et))
        wp = params[(l, "wp")].reshape(cout, E)[:co, :Et].reshape(co, Et, 1, 1)
        z = bn(F.conv2d(a, wp), l, "g3", "b3", co)
        h = z + h if g["res"] else z
    loss = ((h - t[:, :h.shape[1]]) ** 2).sum() / norm
    loss.backward()
    return float(loss), {key: v.grad.numpy() for key, v in params.items()}


def main():
    mb.set_family(FAMILY)
    out = {}
    x = mb.image(B, 0, S, bf16=False)
    acts = [x]
    for b in range(mb.BLOCKS):
        tp = mb.teacher_params(b, bf16=False)
        y = nhwc(teacher_fwd(b, tp, nchw(acts[-1]))).numpy()
        acts.append(y)
        out[f"t{b}"] = y.reshape(-1)[::SUB]
        out[f"t{b}_norm"] = np.linalg.norm(y)
    for b in range(mb.BLOCKS):
        sp = mb.student_params(b)
        path = mb.sample_path(b, DRAW)
        c, hh = mb.true_channels(b + 1), mb.hw(b + 1, S)
        norm = float(B) * c * hh * hh
        loss, grads = student(b, sp, path, nchw(acts[b]), nchw(acts[b + 1]), norm)
        out[f"s{b}_path"] = path
        out[f"s{b}_loss"] = loss
        for (l, name), gv in grads.items():
            out[f"s{b}_l{l}_{name}_norm"] = np.linalg.norm(gv)
            out[f"s{b}_l{l}_{name}"] = gv.reshape(-1)[::SUB] if gv.size > 64 else gv
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
