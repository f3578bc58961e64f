"""fp32 convolutions on the tensor cores (3xTF32, tcgen05 kind::tf32; conv_tf32.cu) through the C-ABI.

Checked against float64 torch convolutions of the same fp32 operands.  Tolerance, per output
element: the split keeps hi + lo == x exactly and drops only a_lo*b_lo plus the tf32 reading of the
lo parts (<= ~3*2^-21 relative per product), and the fp32 accumulation adds a random-walk error, so
  |y - ref| <= 2^-16 * sum |a*b|        (the same convolution over |x|, |w|, in float64)
which plain TF32 (one product per term, ~2^-11) or a dropped correction term would fail by orders
of magnitude.
"""
import ctypes

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

TOL = 2.0 ** -16


@pytest.fixture(scope="module")
def L():
    from paper_2301_12443_b200 import _lib
    return _lib


def desc(L, n, h, c, k, r, stride):
    pad = r // 2
    p = (h + 2 * pad - r) // stride + 1
    return L.ConvDesc(n, h, h, c, k, r, r, stride, pad, p, p)


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def split(L, x):
    """plain [..., c] -> split [..., 2c] through the library's own splitter"""
    c = x.shape[-1]
    out = torch.empty(*x.shape[:-1], 2 * c, device=x.device, dtype=torch.float32)
    assert L.lib().pbdk_split_tf32(x.data_ptr(), out.data_ptr(), x.numel() // c, c, stream()) == 0
    return out


def unsplit(y, k):
    return y[..., :k] + y[..., k:]


# (n, h, c, k, r, stride): the fp32 ResNet workload's convs (teacher, student, dgrad) + odd batches
CASES = [(3, 32, 16, 64, 3, 1), (2, 32, 64, 64, 3, 1), (3, 32, 64, 128, 3, 2), (3, 32, 64, 128, 1, 2),
         (2, 16, 128, 128, 3, 1), (3, 16, 128, 256, 3, 2), (2, 8, 256, 256, 3, 1), (5, 8, 256, 512, 3, 2),
         (3, 4, 512, 512, 3, 1), (2, 32, 16, 32, 3, 1), (2, 32, 32, 64, 3, 1), (2, 32, 64, 32, 3, 1),
         (3, 16, 64, 64, 3, 1), (3, 8, 256, 128, 3, 1), (5, 4, 256, 512, 1, 2)]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("epi,y_split", [(0, 0), (1, 1), (2, 1), (3, 1), (4, 0)])
def test_conv3x_fprop(L, case, epi, y_split):
    n, h, c, k, r, st = case
    d = desc(L, n, h, c, k, r, st)
    g = torch.Generator(device="cuda").manual_seed(hash(case) % 1000 + epi)
    x = torch.rand(n, h, h, c, device="cuda", generator=g) * 2 - 1
    w = (torch.rand(k, r, r, c, device="cuda", generator=g) * 2 - 1) / (r * r * c) ** 0.5
    bias = torch.rand(k, device="cuda", generator=g) - 0.5
    aux = torch.rand(n, d.p, d.q, k, device="cuda", generator=g) * 2 - 1
    y = torch.full((n, d.p, d.q, 2 * k if y_split else k), float("nan"), device="cuda")
    xs, ws, auxs = split(L, x), split(L, w), split(L, aux)  # keep the operands alive across the launch
    rc = L.lib().pbdk_conv3x_fprop(ctypes.byref(d), xs.data_ptr(), ws.data_ptr(), y.data_ptr(), y_split,
                                   bias.data_ptr(), auxs.data_ptr(), epi, stream())
    assert rc == 0
    ref = F.conv2d(x.double().permute(0, 3, 1, 2), w.double().permute(0, 3, 1, 2), stride=st,
                   padding=r // 2).permute(0, 2, 3, 1)
    absref = F.conv2d(x.double().abs().permute(0, 3, 1, 2), w.double().abs().permute(0, 3, 1, 2), stride=st,
                      padding=r // 2).permute(0, 2, 3, 1)
    if epi in (1, 2, 3):
        ref = ref + bias.double()
    if epi == 3:
        ref = ref + aux.double()
    if epi in (2, 3):
        ref = ref.clamp_min(0)
    if epi == 4:
        ref = torch.where(aux > 0, ref, torch.zeros_like(ref))
    torch.cuda.synchronize()
    got = unsplit(y, k) if y_split else y
    if y_split:  # the stored hi part is a tf32 value and hi + lo is the fp32 result
        assert torch.equal(y[..., :k].view(torch.int32) & 0x1FFF, torch.zeros_like(y[..., :k], dtype=torch.int32))
    err = (got.double() - ref).abs()
    assert bool((err <= TOL * absref + 1e-12).all()), (err / absref.clamp_min(1e-30)).max().item()


WGRAD = [(4, 32, 32, 32, 3, 1), (4, 32, 32, 64, 1, 1), (3, 32, 32, 64, 3, 1), (4, 32, 64, 32, 3, 1),
         (3, 32, 64, 64, 3, 2), (3, 32, 64, 128, 1, 2), (5, 16, 64, 128, 3, 1), (3, 16, 128, 256, 3, 2),
         (4, 8, 128, 256, 3, 1), (6, 8, 256, 512, 3, 2), (7, 4, 256, 512, 3, 1), (64, 32, 32, 32, 3, 1),
         (64, 4, 256, 512, 3, 1)]


@pytest.mark.parametrize("case", WGRAD)
def test_conv3x_wgrad(L, case):
    n, h, c, k, r, st = case
    d = desc(L, n, h, c, k, r, st)
    g = torch.Generator(device="cuda").manual_seed(hash(case) % 977)
    x = torch.rand(n, h, h, c, device="cuda", generator=g) * 2 - 1
    dy = torch.rand(n, d.p, d.q, k, device="cuda", generator=g) * 2 - 1
    dw = torch.full((k, r, r, c), float("nan"), device="cuda")
    wsb = L.lib().pbdk_conv3x_wgrad_workspace_bytes(ctypes.byref(d))
    ws = torch.empty(max(wsb, 4), dtype=torch.uint8, device="cuda")
    xs, dys = split(L, x), split(L, dy)
    rc = L.lib().pbdk_conv3x_wgrad(ctypes.byref(d), xs.data_ptr(), dys.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb,
                                   stream())
    assert rc == 0
    xd = x.double().permute(0, 3, 1, 2).requires_grad_(False)
    ref = torch.nn.grad.conv2d_weight(xd, (k, c, r, r), dy.double().permute(0, 3, 1, 2), stride=st,
                                      padding=r // 2).permute(0, 2, 3, 1)
    absref = torch.nn.grad.conv2d_weight(xd.abs(), (k, c, r, r), dy.double().abs().permute(0, 3, 1, 2), stride=st,
                                         padding=r // 2).permute(0, 2, 3, 1)
    torch.cuda.synchronize()
    err = (dw.double() - ref).abs()
    assert bool((err <= TOL * absref + 1e-12).all()), (err / absref.clamp_min(1e-30)).max().item()
    # deterministic: a second call is bitwise equal
    dw2 = torch.empty_like(dw)
    assert L.lib().pbdk_conv3x_wgrad(ctypes.byref(d), xs.data_ptr(), dys.data_ptr(), dw2.data_ptr(), ws.data_ptr(),
                                     wsb, stream()) == 0
    torch.cuda.synchronize()
    assert torch.equal(dw, dw2)


def test_flip_split(L):
    k, r, c = 64, 3, 32
    w = torch.randn(k, r, r, c, device="cuda")
    wt = torch.empty(c, r, r, 2 * k, device="cuda")
    assert L.lib().pbdk_weight_flip_split(w.data_ptr(), wt.data_ptr(), k, r, r, c, stream()) == 0
    torch.cuda.synchronize()
    want = w.flip(1, 2).permute(3, 1, 2, 0)
    assert torch.equal(unsplit(wt, k), want)
