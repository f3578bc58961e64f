"""Depthwise forward kernels (K8, include/pbdk.h pbdk_dw_fwd): the shared-memory staged-tile kernel is
bit-identical to the per-strip register kernel (same fmaf order; that one is bit-exact against the
oracle through tests/test_gpu_mb.py) on every MBConv shape class, and both match torch fp32."""
import ctypes

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


class DwDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("n", "h", "w", "c", "k", "stride", "p", "q")]


@pytest.fixture(scope="module")
def L():
    from paper_2301_12443_b200 import _lib
    lib = _lib.lib()
    lib.pbdk_dw_fwd.argtypes = [ctypes.POINTER(DwDesc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("n,h,c,k,st", [(2, 112, 32, 3, 1), (3, 112, 96, 3, 2), (2, 56, 192, 5, 1),
                                        (2, 56, 192, 7, 2), (4, 28, 384, 3, 1), (3, 14, 576, 5, 1),
                                        (5, 14, 768, 7, 2), (6, 7, 1152, 3, 1), (2, 30, 64, 5, 1)])
@pytest.mark.parametrize("act", [0, 1])
def test_staged_tiles_bitwise_equal_per_strip(L, n, h, c, k, st, act):
    torch.manual_seed(n * h + c + k)
    p = (h + 2 * (k // 2) - k) // st + 1
    d = DwDesc(n, h, h, c, k, st, p, p)
    x = torch.randn(n, h, h, c, device="cuda").bfloat16()
    w = (torch.randn(c, k, k, device="cuda") * 0.3).bfloat16()
    wt = w.permute(1, 2, 0).flip(0, 1).contiguous()  # [k][k][c] flipped tap-major
    bias = torch.randn(c, device="cuda") * 0.1
    ys = []
    for variant in (0, 1):
        y = torch.full((n, p, p, c), 7.0, device="cuda").bfloat16()
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        assert L.pbdk_dw_fwd(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), bias.data_ptr(), y.data_ptr(), act,
                             variant, s) == 0
        ys.append(y)
    torch.cuda.synchronize()
    assert torch.equal(ys[0].view(torch.int16), ys[1].view(torch.int16))
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.float()[:, None], bias, stride=st, padding=k // 2, groups=c)
    ref = ref.permute(0, 2, 3, 1)
    if act == 1:
        ref = ref.clamp(0.0, 6.0)
    assert (ys[1].float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


@pytest.mark.parametrize("n,h,c,k", [(2, 112, 32, 3), (2, 56, 192, 5), (3, 28, 384, 7), (3, 14, 576, 3),
                                     (4, 7, 1152, 5), (2, 30, 64, 3)])
@pytest.mark.parametrize("masked", [False, True])
def test_dgrad_staged_tiles_bitwise_equal_per_pixel(L, n, h, c, k, masked):
    L.pbdk_dw_dgrad.argtypes = [ctypes.POINTER(DwDesc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    torch.manual_seed(n + h + c + k)
    d = DwDesc(n, h, h, c, k, 1, h, h)
    dy = torch.randn(n, h, h, c, device="cuda").bfloat16()
    w = (torch.randn(c, k, k, device="cuda") * 0.3).bfloat16()
    wt = w.permute(1, 2, 0).flip(0, 1).contiguous()
    act = (torch.rand(n, h, h, c, device="cuda") * 9.0 - 1.5).bfloat16() if masked else None
    outs = []
    for variant in (0, 1):
        dx = torch.full((n, h, h, c), 7.0, device="cuda").bfloat16()
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        assert L.pbdk_dw_dgrad(ctypes.byref(d), dy.data_ptr(), wt.data_ptr(),
                               act.data_ptr() if masked else None, dx.data_ptr(), variant, s) == 0
        outs.append(dx)
    torch.cuda.synchronize()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    # dx = correlation of dy with the spatially flipped filter (stride 1, pad k // 2)
    ref = F.conv2d(dy.float().permute(0, 3, 1, 2), w.float().flip(1, 2)[:, None], padding=k // 2, groups=c)
    ref = ref.permute(0, 2, 3, 1)
    if masked:
        a = act.float()
        ref = torch.where((a > 0) & (a < 6), ref, torch.zeros_like(ref))
    assert (outs[1].float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()
