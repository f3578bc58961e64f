"""GPU kernel-level checks through the C-ABI (include/pbdk.h).

Convolutions are floating point: checked against torch fp32 on the same
bf16-valued operands with tolerance |err| <= 2e-2 * max|ref| (fprop: one bf16
rounding of the output) and 1e-3 * max|ref| (wgrad, fp32 output).
"""
import ctypes

import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2301_12443_b200 import _lib
    return _lib


def desc(L, n, h, c, k, r, stride):
    pad = r // 2
    p = (h + 2 * pad - r) // stride + 1
    return L.ConvDesc(n, h, h, c, k, r, r, stride, pad, p, p)


CASES = [(2, 32, 64, 64, 3, 1), (2, 32, 16, 64, 3, 1), (2, 32, 16, 32, 3, 1), (2, 32, 32, 64, 3, 1),
         (3, 32, 64, 128, 3, 2), (3, 32, 64, 128, 1, 2), (4, 16, 128, 128, 3, 1), (4, 8, 256, 512, 3, 2),
         (5, 4, 512, 512, 3, 1), (2, 16, 128, 256, 3, 2), (3, 16, 32, 64, 3, 2), (9, 4, 64, 32, 3, 1),
         # few output tiles -> split-K clusters (DSMEM reduction)
         (16, 4, 512, 512, 3, 1), (32, 8, 256, 256, 3, 2), (8, 4, 512, 256, 3, 1), (4, 8, 256, 128, 3, 1)]


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("epi", [0, 1, 2, 3, 4])
def test_conv_fprop_epilogues(L, case, epi):
    n, h, c, k, r, st = case
    d = desc(L, n, h, c, k, r, st)
    torch.manual_seed(hash(case) % 1000 + epi)
    x = (torch.rand(n, h, h, c, device="cuda") * 2 - 1).bfloat16()
    w = ((torch.rand(k, r, r, c, device="cuda") * 2 - 1) / (r * r * c) ** 0.5).bfloat16()
    bias = torch.rand(k, device="cuda") - 0.5
    aux = (torch.rand(n, d.p, d.q, k, device="cuda") * 2 - 1).bfloat16()
    y = torch.empty(n, d.p, d.q, k, device="cuda", dtype=torch.bfloat16)
    rc = L.lib().pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), bias.data_ptr(),
                                 aux.data_ptr(), epi, stream())
    assert rc == 0
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), stride=st,
                   padding=r // 2).permute(0, 2, 3, 1)
    if epi in (1, 2, 3):
        ref = ref + bias
    if epi == 3:
        ref = ref + aux.float()
    if epi in (2, 3):
        ref = ref.clamp_min(0)
    if epi == 4:
        ref = torch.where(aux.float() > 0, ref, torch.zeros_like(ref))
    torch.cuda.synchronize()
    err = (y.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-3


WGRAD_EXTRA = [  # narrow inputs -> the multi-tap kernel (every tap in one CTA), k = 16 .. 128
    (4, 32, 16, 16, 3, 1), (4, 32, 32, 32, 3, 1), (2, 32, 16, 128, 3, 1), (2, 32, 32, 128, 3, 1),
    (96, 32, 16, 32, 3, 1), (96, 32, 32, 64, 3, 1), (96, 32, 16, 16, 3, 1), (96, 32, 32, 32, 3, 1),
    (96, 32, 16, 128, 3, 1), (384, 16, 32, 64, 3, 1), (64, 32, 16, 32, 3, 1),
    # c = 64: one filter row per CTA (co tiles, stride 2); wider inputs stay on the per-tap kernel
    (128, 16, 64, 64, 3, 1), (128, 32, 64, 128, 3, 2), (64, 16, 64, 256, 3, 1), (32, 16, 128, 256, 3, 1)]


@pytest.mark.parametrize("case", CASES + WGRAD_EXTRA)
def test_conv_wgrad(L, case):
    n, h, c, k, r, st = case
    d = desc(L, n, h, c, k, r, st)
    torch.manual_seed(hash(case) % 997)
    x = (torch.rand(n, h, h, c, device="cuda") * 2 - 1).bfloat16()
    dy = (torch.rand(n, d.p, d.q, k, device="cuda") * 2 - 1).bfloat16()
    dw = torch.empty(k, r, r, c, device="cuda")
    wsb = L.lib().pbdk_conv_wgrad_workspace_bytes(ctypes.byref(d))
    ws = torch.empty(max(wsb, 16), device="cuda", dtype=torch.uint8)
    rc = L.lib().pbdk_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb,
                                 stream())
    assert rc == 0
    ref = torch.nn.grad.conv2d_weight(x.float().permute(0, 3, 1, 2), (k, c, r, r), dy.float().permute(0, 3, 1, 2),
                                      stride=st, padding=r // 2).permute(0, 2, 3, 1)
    torch.cuda.synchronize()
    assert (dw - ref).abs().max().item() <= 1e-3 * ref.abs().max().item() + 1e-4


@pytest.mark.parametrize("case", [(16, 4, 512, 512, 3, 1), (32, 8, 256, 256, 3, 2), (64, 16, 128, 128, 3, 1)])
def test_conv_fprop_deterministic(L, case):
    """Split-K partials are reduced in a fixed order: two runs are bit-identical."""
    n, h, c, k, r, st = case
    d = desc(L, n, h, c, k, r, st)
    torch.manual_seed(7)
    x = (torch.rand(n, h, h, c, device="cuda") * 2 - 1).bfloat16()
    w = ((torch.rand(k, r, r, c, device="cuda") * 2 - 1) / (r * r * c) ** 0.5).bfloat16()
    outs = []
    for _ in range(2):
        y = torch.empty(n, d.p, d.q, k, device="cuda", dtype=torch.bfloat16)
        assert L.lib().pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), None, None, 0,
                                       stream()) == 0
        outs.append(y)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


def test_weight_flip(L):
    w = torch.randn(64, 3, 3, 32, device="cuda").bfloat16()
    wt = torch.empty(32, 3, 3, 64, device="cuda", dtype=torch.bfloat16)
    assert L.lib().pbdk_weight_flip(w.data_ptr(), wt.data_ptr(), 64, 3, 3, 32, stream()) == 0
    torch.cuda.synchronize()
    assert torch.equal(wt, w.flip(1, 2).permute(3, 1, 2, 0).contiguous())


@pytest.mark.parametrize("regs", [
    # ResNet conv2 filter (32x32-tiled transpose) + MBConv transposes / depthwise flip (scattered)
    [(12, 64, 3, 3, 32), (12 + 64 * 9 * 32 + 8, 96, 1, 1, 24), (40000, 48, 5, 5, 1), (52000, 20, 1, 1, 96)],
    # tiled only: the four student conv2 shapes of the CIFAR step at their executor offsets' alignment
    [(4, 64, 3, 3, 32), (20000, 128, 3, 3, 64), (96000, 256, 3, 3, 128), (400000, 64, 1, 1, 96)],
    # unaligned offset: a k, c multiple of 32 that must still take the scatter path
    [(6, 64, 3, 3, 32)],
], ids=["mixed", "tiled", "unaligned"])
def test_sgd_momentum_flip_equals_sgd_then_flip(L, regs):
    """The update with fused flips == pbdk_sgd_momentum followed by pbdk_weight_flip of the shadow
    (bitwise: same fp32 update, same bf16 rounding), for the ResNet conv2 filters (tiled transpose)
    and the MBConv transposes / depthwise flip (scattered), regions at unaligned offsets too."""
    import ctypes as C

    torch.manual_seed(5)
    n = 420000
    w0 = torch.randn(n, device="cuda")
    v0 = torch.randn(n, device="cuda")
    g = torch.randn(n, device="cuda")
    ref_w, ref_v = w0.clone(), v0.clone()
    ref_sh = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    assert L.lib().pbdk_sgd_momentum(ref_w.data_ptr(), ref_v.data_ptr(), g.data_ptr(), ref_sh.data_ptr(), n,
                                     C.c_float(0.05), C.c_float(0.9), None, stream()) == 0
    want = []
    for off, k, r, s, c in regs:
        wt = torch.empty(k * r * s * c, device="cuda", dtype=torch.bfloat16)
        assert L.lib().pbdk_weight_flip(ref_sh[off:].data_ptr(), wt.data_ptr(), k, r, s, c, stream()) == 0
        want.append(wt)
    got = [torch.full_like(t, float("nan")) for t in want]
    arr = (L.FlipRegion * len(regs))(*[L.FlipRegion(off, k, r, s, c, t.data_ptr())
                                       for (off, k, r, s, c), t in zip(regs, got)])
    w, v = w0.clone(), v0.clone()
    sh = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    cnt = torch.zeros(1, device="cuda", dtype=torch.int64)
    assert L.lib().pbdk_sgd_momentum_flip(w.data_ptr(), v.data_ptr(), g.data_ptr(), sh.data_ptr(), n,
                                          C.c_float(0.05), C.c_float(0.9), cnt.data_ptr(), arr, len(regs),
                                          stream()) == 0
    torch.cuda.synchronize()
    assert torch.equal(w, ref_w) and torch.equal(v, ref_v) and torch.equal(sh, ref_sh)
    assert int(cnt.item()) == 1
    for a, b in zip(got, want):
        assert torch.equal(a, b)
    # ResNet conv2 region == the torch restatement of the flip
    off, k, r, s, c = regs[0]
    ref0 = ref_sh[off:off + k * r * s * c].view(k, r, s, c).flip(1, 2).permute(3, 1, 2, 0).reshape(-1)
    assert torch.equal(got[0], ref0)


def test_unsupported_shapes_fail_loudly(L):
    d = L.ConvDesc(2, 30, 30, 64, 64, 3, 3, 1, 1, 30, 30)  # 30x30 output does not tile 128 rows
    x = torch.zeros(2, 30, 30, 64, device="cuda", dtype=torch.bfloat16)
    assert L.lib().pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), x.data_ptr(), x.data_ptr(), None, None, 0,
                                   stream()) == 1


@pytest.mark.parametrize("case", [(96, 32, 16, 32, 3, 1), (96, 32, 32, 64, 3, 1), (32, 16, 128, 128, 3, 1),
                                  (128, 16, 64, 64, 3, 1)])
def test_conv_wgrad_deterministic(L, case):
    """Split partials are summed in split order: two runs are bit-identical."""
    n, h, c, k, r, st = case
    d = desc(L, n, h, c, k, r, st)
    torch.manual_seed(11)
    x = (torch.rand(n, h, h, c, device="cuda") * 2 - 1).bfloat16()
    dy = (torch.rand(n, d.p, d.q, k, device="cuda") * 2 - 1).bfloat16()
    wsb = L.lib().pbdk_conv_wgrad_workspace_bytes(ctypes.byref(d))
    ws = torch.empty(max(wsb, 16), device="cuda", dtype=torch.uint8)
    outs = []
    for _ in range(2):
        dw = torch.empty(k, r, r, c, device="cuda")
        assert L.lib().pbdk_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(),
                                       wsb, stream()) == 0
        outs.append(dw)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
