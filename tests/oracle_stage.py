"""TEST ONLY: a CPU stage with the executor.Partition interface, computed by the oracle.

Lets tests/test_runtime_gloo.py drive the real multi-rank host logic of
paper_2301_12443_b200/runtime.py (placement, relay resharding, group
allreduce, DPU/barrier, epoch sync) with the gloo backend on CPU.
"""
import numpy as np
import torch

from oracle import bd


class OracleStage:
    device = torch.device("cpu")

    def __init__(self, lo, hi, n, first, global_batch):
        self.lo, self.hi, self.n, self.first, self.b = lo, hi, n, first, global_batch
        self.blocks = list(range(lo, hi + 1))
        self.tp = {k: bd.teacher_params(k, 1) for k in self.blocks}
        self.sp = {k: bd.student_params(k) for k in self.blocks}
        self.mom = {k: np.zeros_like(self.sp[k]) for k in self.blocks}
        self.sizes = [self.sp[k].size for k in self.blocks]
        g = bd.geom(lo)
        self.in_buf = torch.zeros(n, g["hin"], g["hin"], g["cin"])
        g = bd.geom(hi)
        self.out_buf = torch.zeros(n, g["hout"], g["hout"], g["cout"])
        self.grad_buf = torch.zeros(sum(self.sizes))
        self.step_idx = 0
        self._losses = [0.0] * len(self.blocks)
        self.acts = None

    def input_act(self):
        return self.in_buf

    def teacher_out(self):
        return self.out_buf

    def grads(self):
        return self.grad_buf

    def teacher_forward(self):
        if self.lo == 0:
            x = bd.make_input(self.n, self.step_idx * self.b + self.first, 1)
        else:
            x = self.in_buf.numpy().copy()
        acts = [x]
        for k in self.blocks:
            acts.append(bd.teacher_fwd(k, self.tp[k], acts[-1], 1))
        self.acts = acts
        self.out_buf.copy_(torch.from_numpy(acts[-1]))

    def student_step(self):
        parts = []
        for i, k in enumerate(self.blocks):
            loss, g = bd.student_fwd_bwd(k, self.sp[k], self.acts[i], self.acts[i + 1], self.b, 1)
            self._losses[i] = loss
            parts.append(g)
        self.grad_buf.copy_(torch.from_numpy(np.concatenate(parts)))

    def apply_update(self):
        off = 0
        g = self.grad_buf.numpy()
        for k, sz in zip(self.blocks, self.sizes):
            bd.sgd(self.sp[k], self.mom[k], g[off:off + sz].copy())
            off += sz
        self.step_idx += 1

    def losses(self):
        return list(self._losses)

    # state migration (runtime.PipeBD.migrate)
    def block_state(self, k):
        return [torch.from_numpy(self.sp[k]), torch.from_numpy(self.mom[k])]

    def block_state_like(self, k):  # any block, owned or not
        n = int(bd.lib().bdo_student_param_count(k))
        return [torch.empty(n), torch.empty(n)]

    def set_block_state(self, k, w, v):
        self.sp[k][:] = w.numpy()
        self.mom[k][:] = v.numpy()

    def step_index(self):
        return self.step_idx

    def set_step_index(self, step):
        self.step_idx = int(step)
