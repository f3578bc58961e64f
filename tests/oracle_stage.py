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
        self.mask = (1 << len(self.blocks)) - 1
        offs = np.cumsum([0] + self.sizes)
        self.layouts = {k: (int(offs[i]), None, self.sizes[i]) for i, k in enumerate(self.blocks)}

    def set_train_mask(self, mask):
        """Bit i = student block lo + i trains (the executor's pbdx_set_train_mask)."""
        self.mask = mask

    def _trains(self, i):
        return (self.mask >> i) & 1

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
            if not self._trains(i):
                parts.append(np.zeros_like(self.sp[k]))
                continue
            loss, g = bd.student_fwd_bwd(k, self.sp[k], self.acts[i], self.acts[i + 1], self.b, 1)
            self._losses[i] = loss
            parts.append(g)
        self.grad_buf.copy_(torch.from_numpy(np.concatenate(parts)))

    def apply_update(self):
        off = 0
        g = self.grad_buf.numpy()
        for i, (k, sz) in enumerate(zip(self.blocks, self.sizes)):
            if self._trains(i):
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


class MbOracleStage(OracleStage):
    """The MobileNetV2 -> ProxylessNAS workload (oracle/mb_oracle.c) behind the same interface:
    image side S, a fixed single path per block."""

    def __init__(self, lo, hi, n, first, global_batch, S, paths):
        from oracle import mb
        self.mb = mb
        self.lo, self.hi, self.n, self.first, self.b, self.S = lo, hi, n, first, global_batch, S
        self.paths = paths
        self.blocks = list(range(lo, hi + 1))
        self.tp = {k: mb.teacher_params(k) for k in self.blocks}
        self.sp = {k: mb.student_params(k) for k in self.blocks}
        self.mom = {k: np.zeros_like(self.sp[k]) for k in self.blocks}
        self.sizes = [self.sp[k].size for k in self.blocks]
        self.in_buf = torch.zeros(mb.act_shape(lo, n, S) if lo > 0 else (n, S, S, 3))
        self.out_buf = torch.zeros(mb.act_shape(hi + 1, n, S))
        self.grad_buf = torch.zeros(sum(self.sizes))
        self.step_idx = 0
        self._losses = [0.0] * len(self.blocks)
        self.acts = None

    def teacher_forward(self):
        mb = self.mb
        if self.lo == 0:
            x = mb.image(self.n, self.step_idx * self.b + self.first, self.S)
        else:
            x = self.in_buf.numpy().copy()
        acts = [x]
        for k in self.blocks:
            acts.append(mb.teacher_fwd(k, self.tp[k], acts[-1], self.S))
        self.acts = acts
        self.out_buf.copy_(torch.from_numpy(acts[-1]))

    def student_step(self):
        mb = self.mb
        parts = []
        for i, k in enumerate(self.blocks):
            norm = float(self.b) * mb.true_channels(k + 1) * mb.hw(k + 1, self.S) ** 2
            g, loss = mb.student_fwd_bwd(k, self.sp[k], self.paths[k], self.acts[i], self.acts[i + 1], self.S, norm)
            self._losses[i] = loss
            parts.append(g)
        self.grad_buf.copy_(torch.from_numpy(np.concatenate(parts)))

    def apply_update(self):
        off = 0
        g = self.grad_buf.numpy()
        for k, sz in zip(self.blocks, self.sizes):
            self.mb.sgd_path(k, self.paths[k], self.sp[k], self.mom[k], g[off:off + sz].copy())
            off += sz
        self.step_idx += 1

    def block_state_like(self, k):
        n = self.mb.student_param_count(k)
        return [torch.empty(n), torch.empty(n)]
