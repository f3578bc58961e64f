import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch
from paper_2301_12443_b200 import executor as ex
b = 256
p = ex.Partition(0, 3, b, b)
p.init_params()
p.set_timing(True)
for _ in range(3):
    p.step()
torch.cuda.synchronize()
t, s = p.block_times()
print("block teacher ms", [round(x, 4) for x in t], "student ms", [round(x, 4) for x in s])
p.set_timing(False)
p.capture()
for _ in range(3):
    p.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    p.replay()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"graph step {ms:.3f} ms  -> {b/ms*1e3:.0f} samples/s; launches/step {p.launches_per_step()}")
print("losses", p.losses())
