import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_12443_b200 import _lib
n, h, c, k, r, st = (int(v) for v in sys.argv[1:7])
epi = int(sys.argv[7]) if len(sys.argv) > 7 else 0
L = _lib.lib()
if os.environ.get("STEP_SCOPE"):  # the ResNet executor's plan settings (two epilogue warps per lane quarter)
    L.pbdk_conv_scope.argtypes = [ctypes.c_int, ctypes.c_int]
    L.pbdk_conv_scope.restype = None
    L.pbdk_conv_scope(0, 2)
p = (h + 2 * (r // 2) - r) // st + 1
d = _lib.ConvDesc(n, h, h, c, k, r, r, st, r // 2, p, p)
x = torch.randn(n, h, h, c, device="cuda").bfloat16()
w = (torch.randn(k, r, r, c, device="cuda") * 0.05).bfloat16()
y = torch.empty(n, p, p, k, device="cuda", dtype=torch.bfloat16)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
bias = torch.zeros(k, device="cuda")
aux = torch.randn(n, p, p, k, device="cuda").bfloat16()
f = lambda: L.pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), bias.data_ptr(), aux.data_ptr(), epi, s)
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
print(f"{ms*1e3:.1f} us {2.0*n*p*p*k*r*r*c/ms/1e9:.0f} TFLOP/s")
