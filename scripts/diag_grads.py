"""Per-tensor gradient agreement GPU vs oracle after one step (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import bd
from paper_2301_12443_b200 import executor as ex
from tests.gpu_helpers import to_oracle_layout
for b in (4, 32):
    p = ex.Partition(0, 3, b, b); p.init_params()
    p.teacher_forward(); p.student_step(); torch.cuda.synchronize()
    x = bd.make_input(b, 0, 1); act = x
    tp = {k: bd.teacher_params(k, 1) for k in range(4)}
    for k in range(4):
        t = bd.teacher_fwd(k, tp[k], act, 1)
        loss, g = bd.student_fwd_bwd(k, bd.student_params(k), act, t, b, 1)
        base, lay, total = p.layouts[k]
        gg = to_oracle_layout(k, p.grads()[base:base+total].cpu().numpy())
        olay = bd.student_layout(k)
        msg = []
        for name, (o, n) in olay.items():
            a, w = gg[o:o+n], g[o:o+n]
            msg.append(f"{name}:{np.linalg.norm(a-w)/max(np.linalg.norm(w),1e-30):.2e}")
        print(f"b={b} block {k} loss gpu={p.losses()[k]:.6f} oracle={loss:.6f} | " + " ".join(msg), flush=True)
        act = t
