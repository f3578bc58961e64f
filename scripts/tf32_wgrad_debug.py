"""Debug: 3xTF32 wgrad vs fp64 reference; prints error structure."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_12443_b200 import _lib as L  # noqa: E402


def st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def split(x):
    c = x.shape[-1]
    out = torch.empty(*x.shape[:-1], 2 * c, device="cuda")
    assert L.lib().pbdk_split_tf32(x.data_ptr(), out.data_ptr(), x.numel() // c, c, st()) == 0
    return out


for (n, h, c, k, r) in [(1, 32, 32, 32, 1), (1, 32, 32, 128, 1), (1, 32, 64, 32, 1), (4, 32, 32, 64, 3)]:
    pad = r // 2
    d = L.ConvDesc(n, h, h, c, k, r, r, 1, pad, h, h)
    x = torch.rand(n, h, h, c, device="cuda") * 2 - 1
    dy = torch.rand(n, h, h, k, device="cuda") * 2 - 1
    dw = torch.full((k, r, r, c), float("nan"), device="cuda")
    wsb = L.lib().pbdk_conv3x_wgrad_workspace_bytes(ctypes.byref(d))
    ws = torch.full((max(wsb, 4) // 4,), float("nan"), device="cuda")
    xs, dys = split(x), split(dy)
    rc = L.lib().pbdk_conv3x_wgrad(ctypes.byref(d), xs.data_ptr(), dys.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb,
                                   st())
    torch.cuda.synchronize()
    ref = torch.nn.grad.conv2d_weight(x.double().permute(0, 3, 1, 2), (k, c, r, r), dy.double().permute(0, 3, 1, 2),
                                      padding=pad).permute(0, 2, 3, 1)
    e = (dw.double() - ref).abs()
    print((n, h, c, k, r), "rc", rc, "ws", wsb, "rel", (e.max() / ref.abs().max()).item(), "nan",
          torch.isnan(dw).sum().item(), "zero", (dw == 0).sum().item(), "of", dw.numel())
    print(" got", dw.flatten()[:6].tolist())
    print(" ref", ref.flatten()[:6].tolist())
    # which rows/cols are right?
    ok = e < 1e-3 * ref.abs().max()
    print(" ok rows(k)", ok.all(-1).all(-1).all(-1).sum().item(), "ok cols(c)", ok.all(0).all(0).all(0).sum().item(),
          "ok elems", ok.sum().item())
    # is it a transposed / permuted result?  compare to ref sums
    print(" sum got", dw.double().sum().item(), "sum ref", ref.sum().item())
