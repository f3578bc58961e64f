"""Debug: 3xTF32 fprop error per shape (isolates chunking / swizzle / taps)."""
import ctypes
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2301_12443_b200 import _lib as L  # noqa: E402


def st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def split(x):
    c = x.shape[-1]
    out = torch.empty(*x.shape[:-1], 2 * c, device="cuda")
    assert L.lib().pbdk_split_tf32(x.data_ptr(), out.data_ptr(), x.numel() // c, c, st()) == 0
    return out


for (n, h, c, k, r) in [(2, 32, 16, 64, 1), (2, 32, 32, 64, 1), (2, 32, 64, 64, 1), (2, 32, 32, 64, 3),
                        (2, 32, 16, 64, 3), (2, 32, 32, 32, 1), (2, 32, 32, 16, 1), (1, 32, 32, 128, 1)]:
    pad = r // 2
    d = L.ConvDesc(n, h, h, c, k, r, r, 1, pad, h, h)
    x = torch.rand(n, h, h, c, device="cuda") * 2 - 1
    w = (torch.rand(k, r, r, c, device="cuda") * 2 - 1) / (r * r * c) ** 0.5
    y = torch.full((n, h, h, k), float("nan"), device="cuda")
    xs, wsp = split(x), split(w)
    rc = L.lib().pbdk_conv3x_fprop(ctypes.byref(d), xs.data_ptr(), wsp.data_ptr(), y.data_ptr(), 0, None,
                                   None, 0, st())
    torch.cuda.synchronize()
    ref = F.conv2d(x.double().permute(0, 3, 1, 2), w.double().permute(0, 3, 1, 2), padding=pad).permute(0, 2, 3, 1)
    e = (y.double() - ref).abs()
    print((n, h, c, k, r), "rc", rc, "rel", (e.max() / ref.abs().max()).item(), "nan", torch.isnan(y).sum().item(),
          "bad rows", (e.amax(-1) > 1e-3).sum().item(), "of", n * h * h, "bad cols", (e.amax((0, 1, 2)) > 1e-3).sum().item())
