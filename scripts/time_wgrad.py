"""Time one conv wgrad (kernel + split reduction) in a CUDA graph: n h c k r stride."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_12443_b200 import _lib
n, h, c, k, r, st = (int(v) for v in sys.argv[1:7])
L = _lib.lib()
p = (h + 2 * (r // 2) - r) // st + 1
d = _lib.ConvDesc(n, h, h, c, k, r, r, st, r // 2, p, p)
x = torch.randn(n, h, h, c, device="cuda").bfloat16()
dy = torch.randn(n, p, p, k, device="cuda").bfloat16()
dw = torch.empty(k, r, r, c, device="cuda")
wsb = L.pbdk_conv_wgrad_workspace_bytes(ctypes.byref(d))
ws = torch.empty(max(wsb, 16), device="cuda", dtype=torch.uint8)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
f = lambda: L.pbdk_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb, s)
for _ in range(5): assert f() == 0
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(50): assert f() == 0
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
ref = torch.nn.grad.conv2d_weight(x.float().permute(0, 3, 1, 2), (k, c, r, r), dy.float().permute(0, 3, 1, 2),
                                  stride=st, padding=r // 2).permute(0, 2, 3, 1)
err = ((dw - ref).abs().max() / ref.abs().max()).item()
print(f"wgrad n{n} h{h} c{c} k{k} r{r} s{st}: {ms*1e3:.1f} us {2.0*n*p*p*k*r*r*c/ms/1e9:.0f} TFLOP/s ws {wsb/1e6:.1f} MB relerr {err:.1e}")
