"""Per-block timeline of one eager CIFAR step at b=256 (CUDA events of the executor, ms from the step start):
teacher and student spans of every block — which chain ends the step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_12443_b200 import executor as ex  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = ex.Partition(0, 3, b, b)
p.init_params()
p.set_timing(True)
for i in range(6):
    p.trace_mark()
    p.step()
    torch.cuda.synchronize()
ts, te, ss, se = p.block_trace()
for k in range(4):
    print(f"block {k}: teacher {ts[k]:.3f}-{te[k]:.3f} ms  student {ss[k]:.3f}-{se[k]:.3f} ms "
          f"(student {se[k] - ss[k]:.3f})")
print("step end", max(se + te))
