"""Probe: fp32 (3xTF32) executor vs the oracle's fp32 mode at b=64 (configs[0]); prints error stats."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import bd  # noqa: E402
from paper_2301_12443_b200 import executor as ex  # noqa: E402
from tests.gpu_helpers import to_oracle_layout  # noqa: E402

b = 64
p = ex.Partition(0, 3, b, b, model="resnet_fp32")
p.init_params()
p.teacher_forward()
p.student_step()
torch.cuda.synchronize()
x = p.value(p.input_act())[:b].cpu().numpy()
print("input exact:", np.array_equal(x[..., :3], bd.make_input(b, 0, 0)), "pad zero:", not x[..., 3:].any())
for k in range(4):
    prev = bd.make_input(b, 0, 0) if k == 0 else p.value(p.teacher_act(k - 1))[:b].cpu().numpy()
    got = p.value(p.teacher_act(k))[:b].cpu().numpy()
    want = bd.teacher_fwd(k, bd.teacher_params(k, 0), prev, 0)
    d = np.abs(got.astype(np.float64) - want)
    print(f"teacher {k}: max {d.max() / np.abs(want).max():.3e} mean {d.mean() / np.abs(want).max():.3e}")
for k in range(4):
    prev = bd.make_input(b, 0, 0) if k == 0 else p.value(p.teacher_act(k - 1))[:b].cpu().numpy()
    tk = p.value(p.teacher_act(k))[:b].cpu().numpy()
    loss, g = bd.student_fwd_bwd(k, bd.student_params(k), prev, tk, b, 0)
    base, _, total = p.layouts[k]
    gg = to_oracle_layout(k, p.grads()[base:base + total].cpu().numpy(), "resnet_fp32")
    out = [f"student {k}: loss {abs(p.losses()[k] - loss) / abs(loss):.3e}"]
    for name, (o, n) in bd.student_layout(k).items():
        out.append(f"{name} {np.linalg.norm(gg[o:o+n] - g[o:o+n]) / (np.linalg.norm(g[o:o+n]) + 1e-30):.2e}")
    print(" ".join(out))
# 3 steps end to end vs the oracle trainer (fp32)
q = ex.Partition(0, 3, b, b, model="resnet_fp32")
q.init_params()
tr = bd.Trainer(b, bf16_mode=0)
for s in range(3):
    q.step()
    torch.cuda.synchronize()
    want = tr.step(s)
    print("step", s, "losses rel", [f"{abs(q.losses()[k] - want[k]) / abs(want[k]):.2e}" for k in range(4)])
for k in range(4):
    base, _, total = q.layouts[k]
    w = to_oracle_layout(k, q.params()[base:base + total].cpu().numpy(), "resnet_fp32")
    w0 = bd.student_params(k)
    print("block", k, "weights delta rel L2", np.linalg.norm((w - w0) - (tr.sp[k] - w0)) / np.linalg.norm(tr.sp[k] - w0))
