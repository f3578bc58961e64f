"""Graph-replay time of each phase alone (teacher / students / update) vs the fused step, b=256."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_12443_b200 import executor as ex
b = 256
p = ex.Partition(0, 3, b, b)
p.init_params()
for _ in range(2):
    p.step()
torch.cuda.synchronize()


def timeit(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


p.capture_phases(False)
names = ["teacher", "students", "update"]
for ph in range(3):
    try:
        print(f"{names[ph]:9s} {timeit(lambda: p.replay_phase(ph)):.4f} ms")
    except Exception as e:  # noqa: BLE001
        print(names[ph], "n/a", e)
p.capture()
print(f"step      {timeit(p.replay):.4f} ms")
