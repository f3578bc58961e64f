"""Algorithmic work of the MobileNetV2 -> ProxylessNAS step for the roofline.

Mirrors csrc/exec/mb_partition.cpp: per kernel of the implemented decomposition, FLOPs count
2*MACs (1x1 convs as GEMMs, depthwise and stem convs as direct convolutions; dgrad and wgrad like
the forward), bytes count every operand read once and every result written once (bf16
activations, fp32 parameters/gradients).  The workload is HBM-bound (arithmetic intensity well
below the B200 ridge), so the step roofline is bytes / measured HBM bandwidth.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

FAMILIES = {
    # stored channels per boundary, teacher MBConv layers per block, teacher kernel per block,
    # squeeze-excite, true channels per boundary (MobileNetV2-1.0 / EfficientNet-B0; the stored extra
    # channels are identically zero)
    "mbv2": ((3, 32, 32, 64, 128, 192, 320), (3, 3, 4, 3, 3, 1), (3, 3, 3, 3, 3, 3), False,
             (3, 24, 32, 64, 96, 160, 320)),
    "effb0": ((3, 32, 64, 128, 128, 192, 320), (3, 2, 3, 3, 4, 1), (3, 5, 3, 5, 5, 3), True,
              (3, 24, 40, 80, 112, 192, 320)),
}
CH, NL, KT, SE, CT = FAMILIES["mbv2"]
DIV = (1, 4, 8, 16, 16, 32, 32)
KS, ES = (3, 5, 7), (3, 6)


def set_family(model: str):
    """Select the teacher family the helpers below describe ("mbv2" | "effb0")."""
    global CH, NL, KT, SE, CT
    CH, NL, KT, SE, CT = FAMILIES[model]


BF, F4 = 2, 4


def round_ch(c: int) -> int:
    return 16 if c <= 16 else 32 if c <= 32 else (c + 63) // 64 * 64


def teacher_layer(b: int, l: int) -> Tuple[int, int, int, int, int]:
    """(t, k, cin, cout, stride), stored widths."""
    return teacher_layer_t(b, l)[:5]


def teacher_layer_t(b: int, l: int) -> Tuple[int, int, int, int, int, int, int]:
    """(t, k, cin, cout, stride, cin_true, cout_true)."""
    if b == 0:
        return ((1, 3, 32, 16, 1, 32, 16), (6, 3, 16, 32, 2, 16, 24), (6, 3, 32, 32, 1, 24, 24))[l]
    cin, cout = CH[b], CH[b + 1]
    s = DIV[b + 1] // DIV[b]
    k = KT[b]
    return (6, k, cin, cout, s, CT[b], CT[b + 1]) if l == 0 else (6, k, cout, cout, 1, CT[b + 1], CT[b + 1])


def teacher_true_macs(S: int = 224) -> float:
    """Multiply-accumulates of the teacher body (stem + every MBConv) at its true widths."""
    macs = (S // 2) ** 2 * 32 * 27.0
    for b in range(6):
        hw = S // DIV[b] if b else S // 2
        for l in range(NL[b]):
            t, k, _, _, st, ci, co = teacher_layer_t(b, l)
            E = ci * t
            ho = (hw - 1) // st + 1
            if t != 1:
                macs += hw * hw * ci * E
            macs += ho * ho * E * k * k + ho * ho * E * co
            if SE:
                macs += 2 * E * max(1, ci // 4)
            hw = ho
    return macs


def _mb(acc, n, hin, cin, E, k, stride, cout, res, expand, train, last):
    """Accumulate flops/bytes of one MBConv layer (teacher: train=False)."""
    ho = (hin - 1) // stride + 1
    mi, mo = n * hin * hin, n * ho * ho
    f = b = 0.0
    if expand:
        f += 2.0 * mi * cin * E
        b += (mi * cin + mi * E) * BF
    f += 2.0 * mo * E * k * k
    b += (mi * E + mo * E) * BF
    f += 2.0 * mo * E * cout
    b += (mo * E + mo * cout + (mo * cout if res and not train else 0)) * BF
    if train:
        # BN stats (read) + apply (read, write) on y1, y2; stats on y3; apply3 (or loss: + target read)
        if expand:
            b += 3 * mi * E * BF
        b += 3 * mo * E * BF
        b += mo * cout * BF
        b += (2 * mo * cout + (mo * cout if res else 0) + (mo * cout if last else 0)) * BF
        # backward: BN3 bwd (g, y3 -> dy3), 1x1 wgrad + dgrad (masked by a2), BN2 bwd, dw wgrad + dgrad,
        # BN1 bwd, expand wgrad [+ dgrad (+ residual)]
        f += 2 * 2.0 * mo * E * cout
        f += 2 * 2.0 * mo * E * k * k
        b += 3 * mo * cout * BF
        b += (mo * cout + mo * E) * BF + (mo * cout + 2 * mo * E) * BF
        b += 3 * mo * E * BF
        b += (mi * E + mo * E) * BF + (mo * E + 2 * mi * E) * BF
        if expand:
            f += 2.0 * mi * cin * E * 2
            b += 3 * mi * E * BF
            b += (mi * cin + mi * E) * BF + (mi * E + mi * cin + (mi * cin if res else 0)) * BF
    acc[0] += f
    acc[1] += b
    return ho


def block_work(b: int, n: int, S: int, path: Sequence[int]) -> Tuple[float, float, float, float, int]:
    """(teacher flops, teacher bytes, student flops, student bytes, student params of the path)."""
    t = [0.0, 0.0]
    s = [0.0, 0.0]
    hw = S // DIV[b]
    params = 0
    if b == 0:
        P = S // 2
        t[0] += 2.0 * n * P * P * 32 * 27
        t[1] += (n * S * S * 3 + n * P * P * 32) * BF
        s[0] += 2 * 2.0 * n * P * P * 32 * 27
        s[1] += (n * S * S * 3 + n * P * P * 32) * BF * 2 + 5 * n * P * P * 32 * BF
        params += 32 * 27 + 64
        hw = P
    hs = hw
    for l in range(NL[b]):
        tt, k, cin, cout, st, cin_t, cout_t = teacher_layer_t(b, l)
        E = cin if tt == 1 else round_ch(cin * tt)
        res = st == 1 and cin_t == cout_t  # residual by the true widths
        hw = _mb(t, n, hw, cin, E, k, st, cout, res, tt != 1, False, False)
        sl = l + 1 if b == 0 else l
        if b == 0 and l == 0:
            sk, se = 3, 1
        else:
            c = int(path[sl])
            sk, se = KS[c % 3], ES[c // 3]
        if SE:  # teacher squeeze-excite: pool (read), two tiny FCs, scale (read + write)
            ho = (hw - 1) // 1 + 1
            t[0] += 2.0 * n * 2 * E * max(1, cin // 4)
            t[1] += 3 * n * ho * ho * E * BF
        Es = cin if se == 1 else round_ch(cin * se)
        hs = _mb(s, n, hs, cin, Es, sk, st, cout, res, se != 1, True, l == NL[b] - 1)
        params += (Es * cin if se != 1 else 0) + Es * sk * sk + cout * Es + 4 * Es + 2 * cout
    # SGD over the active path: read w, v, g, write w, v, bf16 shadow
    s[1] += params * (5 * F4 + BF)
    return t[0], t[1], s[0], s[1], params


def step_work(n: int, S: int, paths: Dict[int, Sequence[int]], blocks: Sequence[int] = range(6)):
    """(flops, bytes) of one step over `blocks` (teacher fwd + student fwd/bwd + update)."""
    f = b = 0.0
    for k in blocks:
        tf, tb, sf, sb, _ = block_work(k, n, S, paths[k])
        f += tf + sf
        b += tb + sb
    return f, b


def act_bytes_per_sample(boundary: int, S: int) -> int:
    hw = S // DIV[boundary]
    return hw * hw * CH[boundary] * BF


def teacher_param_bytes(b: int) -> int:
    n = 32 * 9 * 16 + 32 if b == 0 else 0
    for l in range(NL[b]):
        tt, k, cin, cout, st = teacher_layer(b, l)
        E = cin if tt == 1 else round_ch(cin * tt)
        n += (E * cin + E if tt != 1 else 0) + E * k * k + E + cout * E + cout
        if SE:
            cs = max(1, cin // 4)
            n += 2 * cs * E + cs + E
    return n * BF


def path_param_bytes(b: int, path: Sequence[int]) -> int:
    return block_work(b, 1, 32, path)[4] * F4


def paths_for(draw: int, blocks: Sequence[int] = range(6), seed: int = 7) -> Dict[int, List[int]]:
    """The seeded single-path sampler (Philox, mb_oracle.c mbo_sample_path) restated host-side so the
    product does not depend on the oracle library."""
    out = {}
    for b in blocks:
        layers = NL[b] + (1 if b == 0 else 0)
        p = []
        for l in range(layers):
            if b == 0 and l < 2:
                p.append(0)
                continue
            o = _philox((draw & 0xFFFFFFFF, (draw >> 32) & 0xFFFFFFFF, l, b), (seed, 0x5EA4C400))
            p.append(o % 6)
        out[b] = p
    return out


def _philox(c, k):
    c0, c1, c2, c3 = c
    k0, k1 = k
    M = 0xFFFFFFFF
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B9) & M
            k1 = (k1 + 0xBB67AE85) & M
        p0 = 0xD2511F53 * c0
        p1 = 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & M, p1 & M, ((p0 >> 32) ^ c3 ^ k1) & M, p0 & M
    return c0
