"""Per-shape time of every convolution in the CIFAR step (b=256), each timed alone with the step's
plan settings (two epilogue warps per lane quarter), CUDA events over 50 graph-replayed launches.
Prints launches/step x us -> per-step us, share of the summed conv time and TFLOP/s, so the
bench's "dominant kernel" is the single shape with the largest per-step time.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_12443_b200 import _lib, models  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
L = _lib.lib()
L.pbdk_conv_scope.argtypes = [ctypes.c_int, ctypes.c_int]
L.pbdk_conv_scope.restype = None
L.pbdk_conv_scope(0, 2)

shapes = {}  # (cin, cout, r, stride, hin) -> [launches per step, role]


def add(c, role):
    key = (c[0], c[1], c[2], c[3], c[4])
    ent = shapes.setdefault(key, [0, set()])
    ent[0] += 1
    ent[1].add(role)


for k in range(models.BLOCKS):
    for c, _ in models.teacher_convs(k):
        add(c, f"T{k}")
    g = models.student_geom(k)
    add((g["cin"], g["mid"], 3, g["stride"], g["hin"]), f"S{k}.c1")
    add((g["mid"], g["cout"], 3, 1, g["hout"]), f"S{k}.c2")
    add((g["cin"], g["cout"], 1, g["stride"], g["hin"]), f"S{k}.sc")
    add((g["cout"], g["mid"], 3, 1, g["hout"]), f"S{k}.dgrad")

rows = []
for (c, k, r, st, h), (cnt, roles) in shapes.items():
    if c == 3:
        c = 16  # the stem reads the 16-channel padded image
    p = (h + 2 * (r // 2) - r) // st + 1
    d = _lib.ConvDesc(N, h, h, c, k, r, r, st, r // 2, p, p)
    x = torch.randn(N, h, h, c, device="cuda").bfloat16()
    w = (torch.randn(k, r, r, c, device="cuda") * 0.05).bfloat16()
    y = torch.empty(N, p, p, k, device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(k, device="cuda")
    aux = torch.randn(N, p, p, k, device="cuda").bfloat16()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f = lambda: L.pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), bias.data_ptr(),  # noqa
                                  aux.data_ptr(), 2, s)
    for _ in range(5):
        assert f() == 0
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(50):
            assert f() == 0
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    tf = 2.0 * N * p * p * k * r * r * c / (us * 1e-6) / 1e12
    rows.append((cnt * us, cnt, us, tf, f"{c}->{k} {r}x{r} s{st} @{h}", ",".join(sorted(roles))))
    del gr

tot = sum(r[0] for r in rows)
print(f"# b={N}: summed conv time {tot:.1f} us per step (each shape alone, whole GPU)")
for per_step, cnt, us, tf, name, roles in sorted(rows, reverse=True):
    print(f"{per_step:8.1f} us {100 * per_step / tot:5.1f}%  {cnt}x {us:6.1f} us {tf:6.0f} TF/s  {name:22s} {roles}")
