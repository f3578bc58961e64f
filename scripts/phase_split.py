"""Teacher-only / student-only / update-only graph times vs the whole step (b=256, one GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_12443_b200 import executor as ex
b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = ex.Partition(0, 3, b, b)
p.init_params()
p.capture_phases(False)


def t(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


tt = t(lambda: p.replay_phase(0))
ts = t(lambda: p.replay_phase(1))
tu = t(lambda: p.replay_phase(2))
tall = t(lambda: (p.replay_phase(0), p.replay_phase(1), p.replay_phase(2)))
print(f"teacher {tt*1e3:.1f} us  student {ts*1e3:.1f} us  update {tu*1e3:.1f} us  sequential-phases step {tall*1e3:.1f} us")
q = ex.Partition(0, 3, b, b)
q.init_params()
q.capture()
print(f"one-graph step {t(q.replay)*1e3:.1f} us")
