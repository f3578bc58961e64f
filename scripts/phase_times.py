"""Per-block teacher / student phase times (CUDA events inside the executor, warm, b=256)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_12443_b200 import executor as ex
b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = ex.Partition(0, 3, b, b)
p.init_params()
p.set_timing(True)
ts, ss = [], []
for i in range(12):
    p.step()
    torch.cuda.synchronize()
    t, s = p.block_times()
    if i >= 2:
        ts.append(t); ss.append(s)
import statistics as st
tm = [st.median(x[k] for x in ts) for k in range(4)]
sm = [st.median(x[k] for x in ss) for k in range(4)]
print("teacher ms", [round(v, 4) for v in tm], "sum", round(sum(tm), 4))
print("student ms", [round(v, 4) for v in sm], "sum", round(sum(sm), 4))
