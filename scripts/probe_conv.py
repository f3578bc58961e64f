"""GPU probe: tcgen05 conv fprop / wgrad vs torch fp32 on the same bf16 inputs."""
import ctypes, sys, time
import torch
import torch.nn.functional as F

lib = ctypes.CDLL("paper_2301_12443_b200/lib/libpbd.so")

class Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("n", "h", "w", "c", "k", "r", "s", "stride", "pad", "p", "q")]

lib.pbdk_conv_fprop.argtypes = [ctypes.POINTER(Desc)] + [ctypes.c_void_p] * 5 + [ctypes.c_int, ctypes.c_void_p]
lib.pbdk_conv_wgrad.argtypes = [ctypes.POINTER(Desc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
lib.pbdk_conv_wgrad_workspace_bytes.argtypes = [ctypes.POINTER(Desc)]
lib.pbdk_conv_wgrad_workspace_bytes.restype = ctypes.c_size_t

def mk(n, h, w, c, k, r, stride):
    pad = r // 2
    p = (h + 2 * pad - r) // stride + 1
    q = (w + 2 * pad - r) // stride + 1
    return Desc(n, h, w, c, k, r, r, stride, pad, p, q)

torch.manual_seed(0)
dev = "cuda"
ok = True
cases = [
    (2, 32, 32, 64, 64, 3, 1), (2, 32, 32, 16, 64, 3, 1), (2, 32, 32, 16, 32, 3, 1), (2, 32, 32, 32, 64, 3, 1),
    (3, 32, 32, 64, 128, 3, 2), (3, 32, 32, 64, 128, 1, 2), (4, 16, 16, 128, 128, 3, 1), (4, 8, 8, 256, 512, 3, 2),
    (5, 4, 4, 512, 512, 3, 1), (2, 16, 16, 128, 256, 3, 2), (16, 8, 8, 256, 256, 3, 1), (8, 32, 32, 16, 64, 1, 1),
]
for (n, h, w, c, k, r, st) in cases:
    d = mk(n, h, w, c, k, r, st)
    x = (torch.rand(n, h, w, c, device=dev) * 2 - 1).bfloat16()
    wt = ((torch.rand(k, r, r, c, device=dev) * 2 - 1) * (1.0 / (r * r * c) ** 0.5)).bfloat16()
    y = torch.empty(n, d.p, d.q, k, device=dev, dtype=torch.bfloat16)
    rc = lib.pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(), None, None, 0, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = F.conv2d(x.float().permute(0, 3, 1, 2), wt.float().permute(0, 3, 1, 2), stride=st, padding=r // 2).permute(0, 2, 3, 1)
    err = (y.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    good = rc == 0 and err <= 0.02 * scale + 1e-3
    ok &= good
    print(f"fprop n{n} {h}x{w} c{c}->k{k} r{r} s{st}: rc={rc} maxerr={err:.4g} scale={scale:.3g} {'OK' if good else 'FAIL'}", flush=True)
    # wgrad
    dy = (torch.rand(n, d.p, d.q, k, device=dev) * 2 - 1).bfloat16()
    dw = torch.empty(k, r, r, c, device=dev, dtype=torch.float32)
    wsb = lib.pbdk_conv_wgrad_workspace_bytes(ctypes.byref(d))
    ws = torch.empty(max(wsb, 16), device=dev, dtype=torch.uint8)
    rc = lib.pbdk_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    refw = torch.nn.grad.conv2d_weight(x.float().permute(0, 3, 1, 2), (k, c, r, r), dy.float().permute(0, 3, 1, 2), stride=st, padding=r // 2).permute(0, 2, 3, 1)
    err = (dw - refw).abs().max().item()
    scale = refw.abs().max().item()
    good = rc == 0 and err <= 1e-3 * scale + 1e-3
    ok &= good
    print(f"wgrad n{n} {h}x{w} c{c}->k{k} r{r} s{st}: rc={rc} ws={wsb} maxerr={err:.4g} scale={scale:.3g} {'OK' if good else 'FAIL'}", flush=True)

# quick throughput: teacher layer1 conv at b=256
for (n, h, w, c, k, r, st) in [(256, 32, 32, 64, 64, 3, 1), (256, 16, 16, 128, 128, 3, 1), (256, 8, 8, 256, 256, 3, 1), (256, 4, 4, 512, 512, 3, 1)]:
    d = mk(n, h, w, c, k, r, st)
    x = (torch.rand(n, h, w, c, device=dev) * 2 - 1).bfloat16()
    wt = ((torch.rand(k, r, r, c, device=dev) * 2 - 1) * 0.05).bfloat16()
    y = torch.empty(n, d.p, d.q, k, device=dev, dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lib.pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(), None, None, 0, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); iters = 20
    for _ in range(iters):
        lib.pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(), None, None, 0, s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 2.0 * n * d.p * d.q * k * r * r * c
    print(f"perf fprop n{n} {h}x{w} c{c}->k{k}: {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s", flush=True)
    dy = (torch.rand(n, d.p, d.q, k, device=dev) * 2 - 1).bfloat16()
    dw = torch.empty(k, r, r, c, device=dev, dtype=torch.float32)
    wsb = lib.pbdk_conv_wgrad_workspace_bytes(ctypes.byref(d))
    ws = torch.empty(max(wsb, 16), device=dev, dtype=torch.uint8)
    for _ in range(3):
        lib.pbdk_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb, s)
    e0.record()
    for _ in range(iters):
        lib.pbdk_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb, s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"perf wgrad n{n} {h}x{w} c{c}->k{k}: {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s", flush=True)
print("ALL OK" if ok else "SOME FAILED")
