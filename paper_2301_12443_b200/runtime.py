"""Multi-GPU Pipe-BD driver: one process per GPU over torch.distributed.

Each rank owns one device slot of a schedule document (best_schedule output,
schedule.cpp:361-373): partition j = contiguous blocks [lo, hi] replicated over
the device group G_j, every member running its shard of the global batch
(remainder rule SPEC.md:231).  Per step, rank r in partition j runs the
per-device body of Algorithm 1:

    j == 0 : load_data()                       (synthetic on device, or host upload)
    j  > 0 : receive(t_{lo-1} shard)           relay from the ranks of G_{j-1}     [TR]
    T.forward                                   pbdx_teacher_forward
    j < P-1: send(t_hi shards)                  relay to the ranks of G_{j+1}       [TR]
    S.forward / S.backward(L(s,t))              pbdx_student_step
    |G_j| > 1: share_gradient()                 all_reduce(SUM) inside G_j          [AHD]
    (dpu=False: wait_all_devices())             barrier                             [DPU]
    S.update_weight()                           pbdx_apply_update

The relay reshards when |G_{j-1}| != |G_j|: every (sender, receiver) pair whose
sample ranges overlap exchanges exactly the overlapping rows (NHWC rows are
sample-major, so a shard slice is contiguous).  All P2P ops of one boundary
are issued as one batch_isend_irecv group (NCCL group semantics, no deadlock).

The stage object is pluggable: ``executor.Partition`` on B200s (the product
path), and an oracle-backed stage in tests/ to exercise this host logic with
the gloo backend on CPU (world size 2+).
"""
from __future__ import annotations

import json
import time
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Tuple

import torch
import torch.distributed as dist

from . import core


def shard(global_batch: int, group: int, index: int) -> Tuple[int, int]:
    """(first, count) of member `index` of a group of `group` devices."""
    base, extra = divmod(global_batch, group)
    count = base + (1 if index < extra else 0)
    return index * base + min(index, extra), count


@dataclass
class Placement:
    partition: int
    block_lo: int
    block_hi: int
    group: List[int]
    index: int
    first: int
    count: int
    per_device_batch: int


def placements(schedule: dict, global_batch: int) -> Dict[int, Placement]:
    out = {}
    for j, p in enumerate(schedule["partitions"]):
        lo, hi = p["blocks"]
        devs = list(p["devices"])
        for i, d in enumerate(devs):
            f, c = shard(global_batch, len(devs), i)
            out[d] = Placement(j, lo, hi, devs, i, f, c, p["per_device_batch"])
    return out


def relay_plan(schedule: dict, global_batch: int, boundary: int) -> List[Tuple[int, int, int, int, int]]:
    """Messages across boundary (partition boundary-1 -> boundary):
    (sender rank, receiver rank, sender row offset, receiver row offset, rows)."""
    up = schedule["partitions"][boundary - 1]["devices"]
    down = schedule["partitions"][boundary]["devices"]
    msgs = []
    for a, ra in enumerate(up):
        fa, ca = shard(global_batch, len(up), a)
        for c, rc in enumerate(down):
            fc, cc = shard(global_batch, len(down), c)
            lo, hi = max(fa, fc), min(fa + ca, fc + cc)
            if hi > lo:
                msgs.append((ra, rc, lo - fa, lo - fc, hi - lo))
    return msgs


def peer_wiring(schedule: dict, global_batch: int, rank: int, endpoints: Dict[int, dict]):
    """K11 peer relay wiring of `rank` (include/pbdx.h): endpoints[r] = {"input", "mailbox", "row"} are
    rank r's input buffer, relay mailbox (device pointers valid in THIS process) and relay row bytes.
    Returns (remote consumed-flag pointers, one per sender; send messages (src_row, rows, dst, flag)).
    Slot rule: a receiver's ready slot for a sender = the sender's index in its sender list; a sender's
    consumed slot for a receiver = the receiver's index in its receiver list (both ascending ranks)."""
    place = placements(schedule, global_batch)
    me = place[rank]
    nparts = len(schedule["partitions"])

    def senders_of(r):
        return [m for m in relay_plan(schedule, global_batch, place[r].partition) if m[1] == r]

    def receivers_of(r):
        return [m for m in relay_plan(schedule, global_batch, place[r].partition + 1) if m[0] == r]

    recv = []
    if me.partition > 0:
        for src, _, _, _, _ in senders_of(rank):
            slot = [m[1] for m in receivers_of(src)].index(rank)
            recv.append(endpoints[src]["mailbox"] + 8 * (16 + slot))
    send = []
    if me.partition + 1 < nparts:
        for _, dst, src_off, dst_off, rows in receivers_of(rank):
            slot = [m[0] for m in senders_of(dst)].index(rank)
            send.append((src_off, rows, endpoints[dst]["input"] + dst_off * endpoints[dst]["row"],
                         endpoints[dst]["mailbox"] + 8 * slot))
    return recv, send


class PipeBD:
    """This rank's share of a Pipe-BD schedule.

    make_stage(block_lo, block_hi, n, first) -> stage with the executor.Partition interface:
      input_act(), teacher_out(), grads(), teacher_forward(), student_step(), apply_update(), losses().
    """

    def __init__(self, schedule: dict, global_batch: int, make_stage: Callable, dpu: bool = True,
                 groups: Optional[Dict[int, object]] = None, relay: str = "nccl", grad_share: Optional[str] = None):
        """relay: "nccl" (batch_isend_irecv of the overlapping row slices) or "peer" (K11: the
        sender's SMs store straight into the receiver's input through NVLink/IPC peer memory,
        device-side flags, no host handshake; stages must be executor.Partition on CUDA)."""
        if relay not in ("nccl", "peer"):
            raise ValueError(f"unknown relay {relay!r}")
        self.relay = relay
        # with the peer relay the DP groups also share gradients over peer memory (no NCCL allreduce)
        self.grad_share = grad_share if grad_share is not None else ("peer" if relay == "peer" else "nccl")
        self._ipc_mapped: List[int] = []
        self.schedule = schedule
        self.b = global_batch
        self.dpu = dpu
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.place = placements(schedule, global_batch)
        if self.rank not in self.place:
            raise ValueError(f"rank {self.rank} has no device slot in the schedule")
        me = self.place[self.rank]
        self.me = me
        self.nparts = len(schedule["partitions"])
        # one communicator per multi-device group (every rank must take part in new_group)
        self.groups = groups if groups is not None else {}
        if groups is None:
            for j, p in enumerate(schedule["partitions"]):
                devs = list(p["devices"])
                g = dist.new_group(devs) if len(devs) > 1 else None
                self.groups[j] = g
        self.stage = make_stage(me.block_lo, me.block_hi, me.count, me.first)
        self.recv_msgs = [m for m in relay_plan(schedule, global_batch, me.partition) if m[1] == self.rank] \
            if me.partition > 0 else []
        self.send_msgs = [m for m in relay_plan(schedule, global_batch, me.partition + 1) if m[0] == self.rank] \
            if me.partition + 1 < self.nparts else []
        self._pending_sends: List = []
        if relay == "peer":
            self._wire_peer()

    def _wire_peer(self):
        """Exchange the relay endpoints (CUDA IPC handles) and configure this rank's stage."""
        import os
        from . import executor
        for p in self._ipc_mapped:
            executor.ipc_close(p)
        self._ipc_mapped = []
        st = self.stage
        mine = {"pid": os.getpid(), "input": st.input_ptr(), "mailbox": st.mailbox_ptr(), "row": st.row_bytes_in(),
                "grads": st.grads_ptr(), "params": st.params_ptr(),
                "h_input": executor.ipc_export(st.input_ptr()), "h_mailbox": executor.ipc_export(st.mailbox_ptr()),
                "h_grads": executor.ipc_export(st.grads_ptr()), "h_params": executor.ipc_export(st.params_ptr())}
        allp = [None] * self.world
        dist.all_gather_object(allp, mine)
        endpoints = {}
        group = list(self.me.group)
        peers = {m[1] for m in self.send_msgs} | {m[0] for m in self.recv_msgs} | set(group)
        for r, e in enumerate(allp):
            if e["pid"] == mine["pid"]:
                endpoints[r] = {"input": e["input"], "mailbox": e["mailbox"], "row": e["row"], "grads": e["grads"],
                                "params": e["params"]}
            elif r in peers:
                ip, mb, gr = (executor.ipc_open(e["h_input"]), executor.ipc_open(e["h_mailbox"]),
                              executor.ipc_open(e["h_grads"]))
                pa = executor.ipc_open(e["h_params"]) if r in group else None
                self._ipc_mapped += [ip, mb, gr] + ([pa] if pa is not None else [])
                endpoints[r] = {"input": ip, "mailbox": mb, "row": e["row"], "grads": gr, "params": pa}
        recv, send = peer_wiring(self.schedule, self.b, self.rank, endpoints)
        st.relay_set_recv(recv)
        st.relay_set_send(send)
        # share_gradient over peer memory inside the DP group (fused into the update kernel)
        if len(group) > 1 and self.grad_share == "peer":
            st.dp_set_group(group.index(self.rank), [endpoints[r]["grads"] for r in group],
                            [endpoints[r]["mailbox"] for r in group], [endpoints[r]["params"] for r in group])
        torch.cuda.synchronize(st.device)
        dist.barrier()

    # -- relay
    def _recv_input(self):
        if not self.recv_msgs or self.relay == "peer":
            return
        buf = self.stage.input_act()
        ops = [dist.P2POp(dist.irecv, buf[dst_off:dst_off + rows], src) for src, _, _, dst_off, rows in self.recv_msgs]
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    def _send_output(self):
        if not self.send_msgs or self.relay == "peer":
            return
        out = self.stage.teacher_out()
        ops = [dist.P2POp(dist.isend, out[src_off:src_off + rows], dst) for _, dst, src_off, _, rows in self.send_msgs]
        self._pending_sends = dist.batch_isend_irecv(ops)

    def _finish_sends(self):
        for w in self._pending_sends:
            w.wait()
        self._pending_sends = []

    # -- Algorithm 1, one step
    def use_graphs(self):
        """Replay each phase as a CUDA graph (stages that support capture_phases)."""
        if hasattr(self.stage, "capture_phases"):
            # a rank that relays nothing downstream keeps the teacher->student overlap in one graph
            # (the peer relay is issued inside the teacher phase on a side stream, so it never splits it)
            self.stage.capture_phases(fuse_teacher_student=not self.send_msgs or self.relay == "peer")
            self._graphs = True

    def _phase(self, i, fn):
        if getattr(self, "_graphs", False):
            self.stage.replay_phase(i)
        else:
            fn()

    def step(self, trace: Optional[Callable[[str], None]] = None):
        """One step of Algorithm 1 on this rank.  trace(name) is called at the phase boundaries
        ("start", "teacher", "student", "share", "barrier", "update") for measured timelines."""
        tr = trace or (lambda name: None)
        tr("start")
        self._recv_input()
        self._finish_sends()  # the previous step's send must drain before t_hi is overwritten
        self._phase(0, self.stage.teacher_forward)
        tr("teacher")
        self._send_output()
        self._phase(1, self.stage.student_step)
        tr("student")
        g = self.groups.get(self.me.partition)
        if g is not None and self.grad_share == "nccl":
            dist.all_reduce(self.stage.grads(), op=dist.ReduceOp.SUM, group=g)
        tr("share")
        if not self.dpu:
            dist.barrier()
        tr("barrier")
        self._phase(2, self.stage.apply_update)
        tr("update")

    def end_epoch(self):
        """Full synchronisation at the epoch boundary (simulate.cpp:263)."""
        self._finish_sends()
        dist.barrier()

    # -- reconfiguration (schedule.cpp:347-359): at an epoch boundary
    def measured_block_times(self) -> Dict[int, Tuple[int, float, float]]:
        """{block: (per-device batch, teacher ms, student ms)} of this rank's blocks (needs timing on)."""
        if not hasattr(self.stage, "block_times"):
            return {}
        t, s = self.stage.block_times()
        return {k: (self.me.per_device_batch, t[i], s[i]) for i, k in enumerate(range(self.me.block_lo,
                                                                                     self.me.block_hi + 1))}

    def maybe_reconfigure(self, profile: dict, threshold: float, make_stage: Callable,
                          measured: Optional[Dict[int, Tuple[int, float, float]]] = None) -> Optional[dict]:
        """Gather the monitored block times, re-plan on rank 0 with reconfigure(), broadcast the
        decision and migrate if the schedule changed.  Returns the new schedule or None."""
        mine = measured if measured is not None else self.measured_block_times()
        gathered = [None] * self.world
        dist.all_gather_object(gathered, mine)
        obj = [None]
        if self.rank == 0:
            merged = {}
            for d in gathered:
                for k, v in (d or {}).items():
                    merged.setdefault(int(k), v)
            observed = observed_profile(profile, merged)
            obj = [core.reconfigure(profile, self.schedule, observed, threshold)]
        dist.broadcast_object_list(obj, src=0)
        new = obj[0]
        if new is not None and new["partitions"] != self.schedule["partitions"]:
            self.migrate(new, make_stage)
            return new
        return None

    def migrate(self, new_schedule: dict, make_stage: Callable):
        """Move every student block's weights and momentum from its old owners to its new owners
        (P2P from the first member of the old group), rebuild the stage, communicators and relay
        plan, and keep the data stream's step index."""
        self._finish_sends()
        old_place, new_place = self.place, placements(new_schedule, self.b)
        step_index = self.stage.step_index()
        B = len({k for p in self.schedule["partitions"] for k in range(p["blocks"][0], p["blocks"][1] + 1)})
        # current state of the blocks this rank owns (identical across its DP group after sync)
        # Owned copies: block_state() returns zero-copy views of the executor's device arena, which
        # is freed when the old stage is dropped below (make_stage) — the views must not outlive it.
        state = {k: [t.clone() for t in self.stage.block_state(k)]
                 for k in range(self.me.block_lo, self.me.block_hi + 1)}
        nme = new_place[self.rank]
        incoming = {}
        ops = []
        for k in range(B):
            src = next(r for r, pl in sorted(old_place.items()) if pl.block_lo <= k <= pl.block_hi)
            owners = [r for r, pl in sorted(new_place.items()) if pl.block_lo <= k <= pl.block_hi]
            if self.rank == src:
                for dst in owners:
                    if dst != src:
                        ops += [dist.P2POp(dist.isend, t, dst) for t in state[k]]
            if self.rank in owners and self.rank != src:
                bufs = self.stage.block_state_like(k)
                incoming[k] = bufs
                ops += [dist.P2POp(dist.irecv, b_, src) for b_ in bufs]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for k in range(nme.block_lo, nme.block_hi + 1):
            if k not in incoming:
                incoming[k] = state[k]
        # rebuild this rank's share of the new schedule
        self.schedule = new_schedule
        self.place = new_place
        self.me = nme
        self.nparts = len(new_schedule["partitions"])
        self.groups = {}
        for j, p in enumerate(new_schedule["partitions"]):
            devs = list(p["devices"])
            self.groups[j] = dist.new_group(devs) if len(devs) > 1 else None
        self.stage = None  # release the old executor (its arena) before allocating the new one
        self.stage = make_stage(nme.block_lo, nme.block_hi, nme.count, nme.first)
        for k, (w, v) in incoming.items():
            self.stage.set_block_state(k, w, v)
        self.stage.set_step_index(step_index)
        self.recv_msgs = [m for m in relay_plan(new_schedule, self.b, nme.partition) if m[1] == self.rank] \
            if nme.partition > 0 else []
        self.send_msgs = [m for m in relay_plan(new_schedule, self.b, nme.partition + 1) if m[0] == self.rank] \
            if nme.partition + 1 < self.nparts else []
        self._pending_sends = []
        if self.relay == "peer":
            self._wire_peer()
        if getattr(self, "_graphs", False):
            self.use_graphs()

    # -- checkpoint / resume (the reference persists only profile/schedule/report JSON)
    def save_checkpoint(self, path: str):
        """Write every student block's fp32 weights + momentum and the data stream's step index
        under directory `path` (collective: call on every rank at a step boundary).

        One file per block, written by the first member of the block's DP group (members hold
        identical state after the group's gradient share), so a checkpoint is independent of the
        schedule that wrote it: load_checkpoint() under any other schedule / world size resumes
        bit-identically.  Layout: meta.json + block_KK.bin = weights then momentum, little-endian
        fp32 in the executor's padded student layout (executor.Partition.block_state)."""
        import os
        self._finish_sends()
        os.makedirs(path, exist_ok=True)
        dist.barrier()
        if self.me.index == 0:
            for k in range(self.me.block_lo, self.me.block_hi + 1):
                w, v = (t.detach().to("cpu", torch.float32).contiguous() for t in self.stage.block_state(k))
                tmp = os.path.join(path, f".block_{k:02d}.bin.{self.rank}")
                with open(tmp, "wb") as f:
                    f.write(w.numpy().tobytes())
                    f.write(v.numpy().tobytes())
                os.replace(tmp, os.path.join(path, f"block_{k:02d}.bin"))
        sizes = {k: int(self.stage.block_state(k)[0].numel()) for k in range(self.me.block_lo, self.me.block_hi + 1)}
        gathered = [None] * self.world
        dist.all_gather_object(gathered, (sizes, int(self.stage.step_index())))
        if self.rank == 0:
            steps = {s for _, s in gathered}
            if len(steps) != 1:
                raise RuntimeError(f"ranks disagree on the step index: {sorted(steps)}")
            meta = {"format": "pbd-b200-checkpoint/1", "global_batch": self.b, "step": steps.pop(),
                    "block_numel": {str(k): n for d, _ in gathered for k, n in sorted(d.items())},
                    "schedule": self.schedule}
            tmp = os.path.join(path, ".meta.json.tmp")
            with open(tmp, "w") as f:
                json.dump(meta, f, indent=1, sort_keys=True)
            os.replace(tmp, os.path.join(path, "meta.json"))
        dist.barrier()

    def load_checkpoint(self, path: str) -> dict:
        """Restore this rank's blocks and the step index from a save_checkpoint() directory (written
        under any schedule).  Raises ValueError on a global-batch or block-size mismatch, OSError on
        missing files.  Returns the checkpoint's meta document."""
        import os
        import numpy as np
        with open(os.path.join(path, "meta.json")) as f:
            meta = json.load(f)
        if meta.get("format") != "pbd-b200-checkpoint/1":
            raise ValueError(f"not a pbd-b200 checkpoint: {meta.get('format')!r}")
        if meta["global_batch"] != self.b:
            raise ValueError(f"checkpoint global batch {meta['global_batch']} != {self.b} (the data stream "
                             "index is per global batch)")
        self._finish_sends()
        for k in range(self.me.block_lo, self.me.block_hi + 1):
            n = int(self.stage.block_state(k)[0].numel())
            if meta["block_numel"].get(str(k)) != n:
                raise ValueError(f"block {k}: checkpoint holds {meta['block_numel'].get(str(k))} parameters, "
                                 f"this model {n}")
            raw = np.fromfile(os.path.join(path, f"block_{k:02d}.bin"), dtype="<f4")
            if raw.size != 2 * n:
                raise ValueError(f"block {k}: truncated state file ({raw.size} of {2 * n} floats)")
            dev = _dev_of(self.stage)
            w = torch.from_numpy(raw[:n].copy()).to(dev)
            v = torch.from_numpy(raw[n:].copy()).to(dev)
            self.stage.set_block_state(k, w, v)
        self.stage.set_step_index(int(meta["step"]))
        if _dev_of(self.stage).type == "cuda":
            torch.cuda.synchronize(_dev_of(self.stage))
        dist.barrier()
        return meta

    def block_losses(self) -> Dict[int, float]:
        """Per-block loss of the last step summed over each DP group (the global-batch MSE)."""
        local = self.stage.losses()
        g = self.groups.get(self.me.partition)
        t = torch.tensor(local, dtype=torch.float64, device=_dev_of(self.stage))
        if g is not None:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=g)
        return {k: float(v) for k, v in zip(range(self.me.block_lo, self.me.block_hi + 1), t.tolist())}


def measured_report(pipe: "PipeBD", steps: int) -> Optional[dict]:
    """Measured timelines of `steps` eager steps in the reference's report format (save_report,
    simulate.cpp:431-465; categories simulate.hpp:32-42), one lane per rank on a common timebase
    (each rank's zero is a CUDA event recorded right after a barrier).  Per step: data_load
    (partition 0) or recv_wait (relay), teacher_fwd / student_fwd_bwd per block from the executor's
    CUDA events (student blocks run on their own streams; the part overlapping the teacher lane is
    flagged `overlapped` and kept out of the category totals, as the reference does for overlapped
    sends), grad_share (NCCL allreduce), barrier_wait, weight_update.  Returns the document on rank 0
    (None elsewhere); feed it to core.report_steady_state / core.validate_prediction / core.gantt_svg."""
    stage = pipe.stage
    dev = stage.device
    stream = torch.cuda.current_stream(dev)
    stage.set_timing(True)
    torch.cuda.synchronize(dev)
    dist.barrier()
    zero = torch.cuda.Event(enable_timing=True)
    zero.record(stream)
    lane = []
    lo = pipe.me.block_lo
    for s in range(steps):
        marks = {}

        def tr(name, marks=marks):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            marks[name] = e
            if name == "start":
                stage.trace_mark(stream)

        pipe.step(trace=tr)
        torch.cuda.synchronize(dev)
        base = zero.elapsed_time(marks["start"])
        t = {k: zero.elapsed_time(e) for k, e in marks.items()}
        t0, t1, s0, s1 = stage.block_trace()
        first_teacher = base + t0[0]
        lane.append(("data_load" if lo == 0 else "recv_wait", None, t["start"], first_teacher, s, False))
        for i, k in enumerate(stage.blocks):
            lane.append(("teacher_fwd", k, base + t0[i], base + t1[i], s, False))
        teacher_end = base + t1[-1]
        for i, k in enumerate(stage.blocks):
            a, b = base + s0[i], base + s1[i]
            if a < teacher_end:  # concurrent with the teacher lane: its own stream
                lane.append(("student_fwd_bwd", k, a, b, s, True))
            else:
                lane.append(("student_fwd_bwd", k, a, b, s, False))
        lane.append(("grad_share", None, t["student"], t["share"], s, False))
        lane.append(("barrier_wait", None, t["share"], t["barrier"], s, False))
        lane.append(("weight_update", None, t["barrier"], t["update"], s, False))
    stage.set_timing(False)
    # serialise the lane: non-overlapped events tile it (student tails past the teacher extend it),
    # gaps become idle
    events = []
    busy_end = 0.0
    seq = sorted([e for e in lane if not e[5] and e[3] > e[2]], key=lambda e: (e[2], e[3]))
    for cat, blk, a, b, st, _ in seq:
        a = max(a, busy_end)
        if b <= a:
            continue
        if a > busy_end + 1e-6:
            events.append({"category": "idle", "block": None, "start_ms": busy_end, "end_ms": a, "step": st,
                           "epoch": 0, "overlapped": False})
        events.append({"category": cat, "block": blk, "start_ms": a, "end_ms": b, "step": st, "epoch": 0,
                       "overlapped": False})
        busy_end = b
    for cat, blk, a, b, st, ov in lane:
        if ov:
            events.append({"category": cat, "block": blk, "start_ms": a, "end_ms": b, "step": st, "epoch": 0,
                           "overlapped": True})
    events.sort(key=lambda e: (e["start_ms"], e["overlapped"]))
    gathered = [None] * pipe.world
    dist.all_gather_object(gathered, events)
    if pipe.rank != 0:
        return None
    makespan = max((e["end_ms"] for ev in gathered for e in ev), default=0.0)
    totals = {c: 0.0 for c in ("data_load", "teacher_fwd", "student_fwd_bwd", "send", "recv_wait", "grad_share",
                               "weight_update", "barrier_wait", "idle")}
    overlapped = 0.0
    for ev in gathered:
        for e in ev:
            d = e["end_ms"] - e["start_ms"]
            if e["overlapped"]:
                overlapped += d
            else:
                totals[e["category"]] += d
    # pad every lane with idle to the makespan (the reference's timelines are idle-filled)
    for ev in gathered:
        end = max((e["end_ms"] for e in ev if not e["overlapped"]), default=0.0)
        if makespan > end + 1e-6:
            ev.append({"category": "idle", "block": None, "start_ms": end, "end_ms": makespan, "step": steps - 1,
                       "epoch": 0, "overlapped": False})
            totals["idle"] += makespan - end
    n = len(gathered)
    bubble = (totals["idle"] + totals["recv_wait"] + totals["barrier_wait"]) / (makespan * n) if makespan else 0.0
    rep = {"num_devices": n, "makespan_ms": makespan, "steady_state_step_ms": 0.0, "bubble_ratio": bubble,
           "category_totals_ms": totals, "overlapped_send_ms": 0.0, "overlapped_compute_ms": overlapped,
           "peak_mem_bytes": [0.0] * n,
           "sim": {"steps_per_epoch": steps, "epochs": 1, "dpu": pipe.dpu, "overlap_send": True, "overlap_load": True,
                   "epoch_sync_ms": 0.0, "weight_update_ms": 0.0},
           "timelines": gathered, "measured": True}
    if steps >= 4:
        rep["steady_state_step_ms"] = core.report_steady_state(rep)
    return rep


def _dev_of(stage):
    return getattr(stage, "device", torch.device("cpu"))


# ---------------------------------------------------------------- device profiler + AHD on B200

def profile_blocks(global_batch: int, world: int, keys: Optional[List[int]] = None, reps: int = 5,
                   device: Optional[torch.device] = None, model: str = "resnet", image: Optional[int] = None,
                   paths: Optional[Dict[int, List[int]]] = None) -> dict:
    """Measure T_k(b), S_k(b) of every block on this GPU with CUDA events ("runs steps
    of each block with feasible batch sizes") and emit a profile document (profile.hpp:30-86).
    model "mbv2": the active single path `paths[k]` of the supernet is what is timed."""
    from . import executor, models, mb_models
    keys = keys or sorted({max(1, global_batch // d) for d in (16, 8, 4, 2, 1)})
    nblocks = models.BLOCKS if model == "resnet" else 6
    if model != "resnet":
        mb_models.set_family(model)
        image = image or 224
        paths = paths or mb_models.paths_for(0)
    blocks = []
    for k in range(nblocks):
        tms, sms = {}, {}
        for n in keys:
            p = executor.Partition(k, k, n, max(n, global_batch), device=device, model=model, image=image)
            p.init_params()
            if model != "resnet":
                p.set_path(k, paths[k])
            p.set_timing(True)
            t_samples, s_samples = [], []
            for r in range(reps + 2):
                p.step()
                tt, ss = p.block_times()
                if r >= 2:
                    t_samples.append(tt[0])
                    s_samples.append(ss[0])
            tms[n] = sorted(t_samples)[len(t_samples) // 2]
            sms[n] = sorted(s_samples)[len(s_samples) // 2]
            del p
        # the profile format requires non-decreasing times in batch (profile.cpp:37-55)
        run_t = run_s = 0.0
        for n in keys:
            run_t = max(run_t, tms[n])
            run_s = max(run_s, sms[n])
            tms[n], sms[n] = run_t, run_s
        if model == "resnet":
            act = models.T_HW[k + 1] ** 2 * models.T_CH[k + 1] * 2
            tparams = sum(c[1] * c[2] * c[2] * (16 if c[0] == 3 else c[0]) * 2 for c, _ in models.teacher_convs(k))
            pbytes = models.student_param_count(k) * 4
        else:
            act = mb_models.act_bytes_per_sample(k + 1, image)
            tparams = mb_models.teacher_param_bytes(k)
            pbytes = mb_models.path_param_bytes(k, paths[k])
        blocks.append({"id": k, "teacher_ms": {str(n): tms[n] for n in keys},
                       "student_ms": {str(n): sms[n] for n in keys}, "act_bytes_per_sample": float(act),
                       "param_bytes": float(pbytes), "teacher_param_bytes": float(tparams)})
    return {"blocks": blocks, "global_batch": global_batch, "hardware": hardware_spec(world, device)}


# NVLink 5 fallback bandwidths (bytes per ms) when fewer than two GPUs are visible: 900 GB/s per
# direction nominal, derated to what peer copies typically sustain (~85 %); the DP exchange
# (PartitionBase::dp_update) moves the ring-allreduce volume with peer loads at ~the same rate (~80 %).
FALLBACK_LINK_BYTES_PER_MS = 7.7e8
FALLBACK_ALLREDUCE_BYTES_PER_MS = 7.25e8


def measure_peer_bandwidth(src: int = 0, dst: int = 1, nbytes: int = 256 << 20, reps: int = 5) -> Optional[float]:
    """Peer copy bandwidth GPU src -> dst in bytes/ms (CUDA events around device-to-device copies over
    NVLink), or None when fewer than two GPUs are visible / peer access is unavailable."""
    if torch.cuda.device_count() < 2 or not torch.cuda.can_device_access_peer(src, dst):
        return None
    a = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", src))
    b = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", dst))
    with torch.cuda.device(dst):
        b.copy_(a)  # warm (peer mapping)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            b.copy_(a, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    return nbytes / ms


def hardware_spec(world: int, device: Optional[torch.device] = None) -> dict:
    """HardwareSpec (profile.hpp:66-77) of this node: link and exchange bandwidth from a peer-copy
    microbenchmark when >= 2 GPUs are visible (both C_i and DPC_j move bytes GPU-to-GPU over NVLink:
    the relay with SM peer stores, the DP exchange with peer loads of exactly the ring-allreduce
    volume), the documented fallbacks otherwise; device memory from the device properties."""
    bw = measure_peer_bandwidth()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    mem = float(torch.cuda.get_device_properties(dev).total_memory) if torch.cuda.is_available() else 1.8e11
    return {"num_devices": world,
            "link_bytes_per_ms": bw if bw is not None else FALLBACK_LINK_BYTES_PER_MS,
            "allreduce_bytes_per_ms": bw if bw is not None else FALLBACK_ALLREDUCE_BYTES_PER_MS,
            "mem_bytes_per_device": mem, "data_load_ms_per_batch": 0.0, "min_utilization_floor": 1.0}


def observed_profile(reference: dict, measured: Dict[int, Tuple[int, float, float]]) -> dict:
    """Monitoring (schedule.cpp:319-359): a running partition only observes its
    blocks at its own per-device batch b_j.  The observed document rescales every key of block k
    by observed/predicted at b_j, preserving the key structure profile_drift() requires."""
    obs = json.loads(json.dumps(reference))
    for k, (bj, t_ms, s_ms) in measured.items():
        bt = core.exec_time(reference, k, "teacher", bj)
        bs = core.exec_time(reference, k, "student", bj)
        blk = obs["blocks"][k]
        blk["teacher_ms"] = {key: v * (t_ms / bt) for key, v in blk["teacher_ms"].items()}
        blk["student_ms"] = {key: v * (s_ms / bs) for key, v in blk["student_ms"].items()}
    return obs


# ---------------------------------------------------------------- the paper's baselines on devices

class _StepTimer:
    """Per-step device time of this rank (CUDA events on the stage's device; wall clock on CPU)."""

    def __init__(self, device):
        self.cuda = device.type == "cuda"
        self.device = device

    def __enter__(self):
        if self.cuda:
            torch.cuda.synchronize(self.device)
            self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            self.e0.record()
        else:
            import time as _t
            self.t0 = _t.perf_counter()
        return self

    def __exit__(self, *exc):
        if self.cuda:
            self.e1.record()
            torch.cuda.synchronize(self.device)
            self.ms = self.e0.elapsed_time(self.e1)
        else:
            import time as _t
            self.ms = (_t.perf_counter() - self.t0) * 1e3


def _max_over_ranks(x: float, device) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device if device.type == "cuda" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def run_baseline(kind: str, plan: dict, global_batch: int, make_stage: Callable, steps: int, warmup: int = 1,
                 rank: int = 0, world: int = 1) -> dict:
    """Execute one of the paper's baselines for real (plans from core.baseline_plan,
    schedule.cpp:246-303; their simulated timelines simulate.cpp:269-386):

      dp: every block in turn, on all `world` ranks data-parallel: phase k runs the teacher prefix
          T_0..T_k (recomputed, no relay) and student k on this rank's shard, all-reduces block k's
          gradients (torch.distributed, the DDP allreduce of PAPER.md:395) and updates it;
      ls: LPT block assignment (plan["device_blocks"]): this rank runs T_0..T_{last assigned} and its
          assigned students on the full batch, no communication.

    make_stage(lo, hi, n, first) -> a stage with set_train_mask / layouts / grads (executor.Partition or
    the oracle stage of the CPU tests).  Returns per-phase step ms (max over ranks) and the time to
    train every block for one step of data ("all_blocks_ms": the sum of the phases for dp, the slowest
    rank for ls), plus the final stages' block weights for the caller's checks."""
    out = {"kind": kind, "plan": plan, "states": {}}
    if kind == "dp":
        first, n = shard(global_batch, world, rank)
        phase_ms = []
        for k in range(len(plan["phase_step_ms"])):
            st = make_stage(0, k, n, first)
            st.set_train_mask(1 << k)
            base, _, total = st.layouts[k]
            dev = _dev_of(st)
            times = []
            for s in range(warmup + steps):
                with _StepTimer(dev) as t:
                    st.teacher_forward()
                    st.student_step()
                    if world > 1:
                        g = st.grads()[base:base + total]
                        dist.all_reduce(g)
                    st.apply_update()
                if s >= warmup:
                    times.append(t.ms)
            phase_ms.append(_max_over_ranks(sorted(times)[len(times) // 2], dev))
            out["states"][k] = [x.detach().cpu().clone() for x in st.block_state(k)]
            del st
        out["phase_ms"] = phase_ms
        out["all_blocks_ms"] = sum(phase_ms)
        return out
    if kind == "ls":
        mine = plan["device_blocks"][rank] if rank < len(plan["device_blocks"]) else []
        ms = 0.0
        dev = torch.device("cpu")
        if mine:
            st = make_stage(0, max(mine), global_batch, 0)
            st.set_train_mask(sum(1 << k for k in mine))
            dev = _dev_of(st)
            times = []
            for s in range(warmup + steps):
                with _StepTimer(dev) as t:
                    st.teacher_forward()
                    st.student_step()
                    st.apply_update()
                if s >= warmup:
                    times.append(t.ms)
            ms = sorted(times)[len(times) // 2]
            out["states"] = {k: [x.detach().cpu().clone() for x in st.block_state(k)] for k in mine}
        out["device_ms"] = ms
        out["all_blocks_ms"] = _max_over_ranks(ms, dev)
        return out
    raise ValueError("baseline kind must be dp or ls")


# ---------------------------------------------------------------- bench entry (torchrun, N > 1)

def bench_pipeline(args, rank: int, world: int, local_rank: int) -> dict:
    """torchrun entry of bench.py for N GPUs (also usable at N=1 with --pipeline): measure the block
    profile on the GPU, pick the schedule with best_schedule, run Algorithm 1 across the ranks."""
    import os
    import time as _time
    from . import executor
    dev = torch.device("cuda", local_rank)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        # NCCL (one process per GPU).  PBD_DIST_BACKEND=gloo lets several ranks share one GPU (the CI /
        # single-GPU exercise of this exact path: the relay is the K11 peer relay either way)
        backend = os.environ.get("PBD_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    gb = args.batch * world
    wl = getattr(args, "workload", "cifar")
    model = wl if wl in ("mbv2", "effb0") else "resnet"
    image = getattr(args, "image", 224) if model != "resnet" else None
    from . import mb_models
    if model != "resnet":
        mb_models.set_family(model)
    paths = mb_models.paths_for(0) if model != "resnet" else None
    # profile on rank 0's GPU, schedule on rank 0, broadcast the documents
    obj = [None, None]
    if rank == 0:
        prof = profile_blocks(gb, world, device=dev, model=model, image=image, paths=paths)
        # --no-ahd: contiguous_only (TR / pure pipeline, schedule.cpp:172-185; configs[1] at B = N = 4)
        sched, meta = core.best_schedule(prof, contiguous_only=getattr(args, "no_ahd", False))
        obj = [sched, {"profile": prof, "meta": meta}]
    dist.broadcast_object_list(obj, src=0)
    sched, info = obj

    def make_stage(lo, hi, n, first):
        p = executor.Partition(lo, hi, n, gb, device=dev, model=model, image=image)
        p.init_params()
        p.set_shard(n, first)
        for k in range(lo, hi + 1):
            if paths is not None:
                p.set_path(k, paths[k])
        return p

    def timed(pipe, steps, e2e_hook=None):
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = _time.perf_counter()
        e0.record()
        for _ in range(steps):
            if e2e_hook is not None:
                e2e_hook(pipe, "pre")
            pipe.step()
            if e2e_hook is not None:
                e2e_hook(pipe, "post")
        pipe._finish_sends()
        e1.record()
        torch.cuda.synchronize(dev)
        wall = (_time.perf_counter() - t0) / steps * 1e3
        t = torch.tensor([e0.elapsed_time(e1) / steps, wall], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0]), float(t[1])

    pipe = PipeBD(sched, gb, make_stage, relay=getattr(args, "relay", "peer"))
    if not getattr(args, "no_graph", False):
        pipe.use_graphs()
    for _ in range(max(3, args.warmup)):
        pipe.step()
    ms, _ = timed(pipe, args.steps)
    losses = pipe.block_losses()

    # e2e: partition-0 ranks copy every step's images from pinned host memory (CIFAR: staged double
    # buffer on a copy stream, overlapped with the previous step; MBConv: upload per step); the last
    # partition reads every step's losses back (on the host one step later).
    me = pipe.me
    host = None
    stream = torch.cuda.current_stream(dev)
    staged = True  # both models pack staged slots inside the step (input mode 2)
    if me.partition == 0:
        pipe.stage.set_external_input(2 if staged else 1)
        side = image or 32
        host = torch.empty(me.count, side, side, 3, dtype=torch.float32).pin_memory().uniform_(-1, 1)
        if getattr(pipe, "_graphs", False):
            pipe.use_graphs()  # re-capture without the on-device data generation
    loss_host = [torch.empty(len(pipe.stage.blocks), dtype=torch.float64).pin_memory() for _ in range(2)]
    copy_stream = torch.cuda.Stream(dev)
    ev_copy = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    state = {"s": 0, "p0": int(pipe.stage.step_counter().item()) & 1 if staged and host is not None else 0}

    def hook(p, when):
        s_ = state["s"]
        cur, nxt = (state["p0"] + s_) & 1, (state["p0"] + s_ + 1) & 1
        if when == "pre" and host is not None:
            if not staged:
                p.stage.upload_images(host)
                return
            if s_ == 0:
                p.stage.stage_images(host, cur, stream)
                ev_copy[cur].record(stream)
            if s_ >= 1:
                copy_stream.wait_event(ev_done[nxt])
            p.stage.stage_images(host, nxt, copy_stream)  # the next step's images, overlapped
            ev_copy[nxt].record(copy_stream)
            stream.wait_event(ev_copy[cur])
        elif when == "post":
            ev_done[cur].record(stream)
            if me.partition == pipe.nparts - 1:
                loss_host[cur].copy_(p.stage.losses_tensor(), non_blocking=True)
                if s_ >= 1:
                    ev_done[nxt].synchronize()  # the previous step's losses are on the host
            state["s"] = s_ + 1

    _, e2e_ms = timed(pipe, args.steps, hook)
    all_losses = [None] * world
    dist.all_gather_object(all_losses, losses)
    pred = core.predicted_step_time(info["profile"], sched)
    h2d = (me.count * (image or 32) ** 2 * 3 * 4) if host is not None else 0
    relay_mode, launches, nblk = pipe.relay, pipe.stage.launches_per_step(), len(pipe.stage.blocks)
    baselines = None
    if not getattr(args, "no_baselines", False) and model == "resnet":
        # the paper's DP and LS baselines on the same ranks, bounded step counts
        del pipe
        torch.cuda.synchronize(dev)

        def plain_stage(lo, hi, n, first):
            p = executor.Partition(lo, hi, n, gb, device=dev, model=model, image=image)
            p.init_params()
            p.set_shard(n, first)
            return p

        nb = min(args.steps, 20)
        baselines = {}
        for kind in ("dp", "ls"):
            plan = core.baseline_plan(info["profile"], kind)
            res = run_baseline(kind, plan, gb, plain_stage, steps=nb, warmup=3, rank=rank, world=world)
            baselines[kind] = {"all_blocks_ms": res["all_blocks_ms"], "predicted_ms": plan["step_ms"],
                               "pipebd_step_ms": ms, "speedup": res["all_blocks_ms"] / ms, "steps": nb}
            if kind == "dp":
                baselines[kind]["phase_ms"] = res["phase_ms"]
            else:
                baselines[kind]["device_blocks"] = plan["device_blocks"]
        baselines["note"] = ("time to train every block for one step of data on the same ranks: DP (blocks in "
                             "turn, teacher prefix recomputed, NCCL allreduce) / LS (LPT blocks per rank, full "
                             "batch) vs Pipe-BD's step; dp_schedule / ls_schedule plans (schedule.cpp:246-303)")
    dist.barrier()
    dist.destroy_process_group()
    return {"metric": "blockwise-distill samples/sec", "value": gb / ms * 1e3, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (Philox4x32-10 on device)",
            "config": {"workload": ("cifar-resnet18-teacher/slim-student 4 blocks (configs[1])" if model == "resnet"
                                    else f"{model}-teacher/proxyless-supernet 6 blocks {image}x{image} "
                                         f"({'configs[2]' if model == 'mbv2' else 'configs[3]'})"),
                       "global_batch": gb,
                       "parallelism": "ahd " + ";".join(f"{p['blocks']}x{len(p['devices'])}"
                                                        for p in sched["partitions"]),
                       "relay": relay_mode,
                       "l2": "no flush: per-step working set > 126 MB L2"},
            "e2e": {"value": gb / e2e_ms * 1e3, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8 * nblk, "ms_per_step": e2e_ms},
            "schedule": sched, "predicted_step_ms": pred["step_ms"], "profile": info["profile"],
            "block_losses": {k: v for d in all_losses for k, v in d.items()},
            "gpu_launches": launches * args.steps, "baselines_measured": baselines,
            "roofline": _step_roofline(model, image, paths, gb, ms, world)}


def _step_roofline(model, image, paths, gb, ms, world) -> dict:
    """Whole-job step roofline of a multi-rank run: algorithmic work of the global step (models.py /
    mb_models.py accounting) over the measured step time and the peaks of `world` GPUs."""
    import json as _json
    import os as _os
    from . import mb_models, models
    root = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
    peaks = {"hbm_gbs": 6650.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    path = _os.path.join(root, "MEASURED_PEAKS.json")
    if _os.path.exists(path):
        with open(path) as f:
            d = _json.load(f)
        peaks = {"hbm_gbs": d["hbm_gbs"], "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                 "source": "measured"}
    if model == "resnet":
        flops, nbytes = models.step_flops(gb), models.step_bytes(gb)
    else:
        flops, nbytes = mb_models.step_work(gb, image, paths)
    t_tensor = flops / (peaks["bf16_tflops_sustained"] * 1e12 * world)
    t_hbm = nbytes / (peaks["hbm_gbs"] * 1e9 * world)
    bound = "tensor" if t_tensor >= t_hbm else "hbm"
    achieved = flops / (ms * 1e-3) / 1e12 / world if bound == "tensor" else nbytes / (ms * 1e-3) / 1e9 / world
    peak = peaks["bf16_tflops_sustained"] if bound == "tensor" else peaks["hbm_gbs"]
    return {"bound": bound, "kernel": "whole step, per GPU (all ranks)", "achieved": achieved, "peak": peak,
            "unit": "TFLOP/s" if bound == "tensor" else "GB/s", "frac": achieved / peak, "traffic": None,
            "peak_source": peaks["source"] + " sustained"}
