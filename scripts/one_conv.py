"""Launch one conv shape a few times (for ncu captures)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_12443_b200 import _lib
n, h, c, k, r, st = (int(v) for v in (sys.argv[1:7] if len(sys.argv) > 6 else (256, 32, 64, 64, 3, 1)))
mode = sys.argv[7] if len(sys.argv) > 7 else "fprop"
L = _lib.lib()
p = (h + 2 * (r // 2) - r) // st + 1
d = _lib.ConvDesc(n, h, h, c, k, r, r, st, r // 2, p, p)
x = torch.randn(n, h, h, c, device="cuda").bfloat16()
w = (torch.randn(k, r, r, c, device="cuda") * 0.05).bfloat16()
y = torch.empty(n, p, p, k, device="cuda", dtype=torch.bfloat16)
dw = torch.empty(k, r, r, c, device="cuda")
wsb = L.pbdk_conv_wgrad_workspace_bytes(ctypes.byref(d))
ws = torch.empty(max(16, wsb), device="cuda", dtype=torch.uint8)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(4):
    if mode == "fprop":
        assert L.pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), None, None, 0, s) == 0
    else:
        assert L.pbdk_conv_wgrad(ctypes.byref(d), x.data_ptr(), y.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb, s) == 0
torch.cuda.synchronize()
print("ok")
