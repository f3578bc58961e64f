"""Time the MobileNetV2 -> ProxylessNAS step (configs[2] shape) on one GPU: graph replay and
per-block CUDA-event times.  python scripts/mb_step.py [batch] [image] [draw]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_12443_b200 import executor as ex  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
S = int(sys.argv[2]) if len(sys.argv) > 2 else 224
draw = int(sys.argv[3]) if len(sys.argv) > 3 else 0
steps = int(os.environ.get("STEPS", "20"))
from oracle import mb  # noqa: E402  (path sampler only)
if os.environ.get("MODEL") == "effb0":
    mb.set_family(1)

p = ex.Partition(0, 5, b, b, model=os.environ.get("MODEL", "mbv2"), image=S)
p.init_params()
for k in range(6):
    p.set_path(k, mb.sample_path(k, draw))
print("paths", {k: p.paths[k] for k in range(6)})
print("mem GiB", torch.cuda.memory_allocated() / 2**30, "reserved by driver:", torch.cuda.mem_get_info())
if os.environ.get("PROFILE"):
    for _ in range(2):
        p.step()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("step")
    p.step()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    sys.exit(0)
p.set_timing(True)
for _ in range(3):
    p.step()
torch.cuda.synchronize()
t, s = p.block_times()
print("teacher ms", [round(x, 3) for x in t], "sum", round(sum(t), 3))
print("student ms", [round(x, 3) for x in s], "sum", round(sum(s), 3))
p.set_timing(False)
p.capture()
for _ in range(3):
    p.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    p.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"step {ms:.3f} ms  -> {b / ms * 1e3:.0f} samples/s ; launches/step {p.launches_per_step()}")
print("losses", p.losses())
