"""Per-CTA cycle counters of the halo fprop kernel (PBDK_CONV_DEBUG=4, buffer passed as aux)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PBDK_CONV_DEBUG", "4")
import torch
from paper_2301_12443_b200 import _lib
L = _lib.lib()
n, h, c, k = 256, 32, 64, 64
d = _lib.ConvDesc(n, h, h, c, k, 3, 3, 1, 1, h, h)
x = torch.randn(n, h, h, c, device="cuda").bfloat16()
w = (torch.randn(k, 3, 3, c, device="cuda") * 0.05).bfloat16()
y = torch.empty(n, h, h, k, device="cuda", dtype=torch.bfloat16)
buf = torch.zeros(148 * 8 + 64, dtype=torch.int64, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    assert L.pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), None, buf.data_ptr(), 0, s) == 0
torch.cuda.synchronize()
b = buf[:148 * 8].view(148, 8).cpu().double()
tl = buf[148 * 8:].view(16, 4).cpu().tolist()
names = ["total", "mma_wait_tempty", "mma_wait_full", "mma_issue", "epi_wait_tfull", "epi_work", "prologue", "ns_total"]
for i, nme in enumerate(names):
    if nme != "-":
        print(f"{nme:16s} mean {b[:, i].mean():10.0f}  min {b[:, i].min():10.0f}  max {b[:, i].max():10.0f}")
for i, r in enumerate(tl):
    print("tile", i, r)
