"""K11 peer relay (include/pbdx.h, relay.cu): teacher activations stored by the sender's SMs straight
into the receiver's input buffer, device-side sequence flags, no host handshake.

On one GPU the "peers" are several executors sharing the device (in-process: raw pointers; across
processes: CUDA IPC mappings of the same device memory), which exercises exactly the kernels, the
flag protocol, the slot wiring and the graph capture used across NVLink.  The relayed pipeline
must be BITWISE identical to (a) one partition holding all blocks (pure pipeline: same kernels,
same shard) and (b) the same schedule driven with host-side copies (resharded DP groups).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2301_12443_b200 import runtime

pytestmark = pytest.mark.gpu


def sched(parts, b):
    return {"flags": {"tr": True, "dpu": True, "ahd": True},
            "partitions": [{"blocks": [lo, hi], "devices": devs, "per_device_batch": -(-b // len(devs))}
                           for lo, hi, devs in parts],
            "predicted": {"partition_ms": [0.0] * len(parts), "step_ms": 0.0}}


def _state(stages):
    out = {}
    for r, p in stages.items():
        out[r] = (p.params().cpu().clone(), p.momentum().cpu().clone(), p.losses(), p.teacher_out()[:p.n].float().cpu())
    return out


def _dp_sum(schedule, stages):
    for p in schedule["partitions"]:
        devs = p["devices"]
        if len(devs) > 1:
            tot = stages[devs[0]].grads().clone()
            for r in devs[1:]:
                tot += stages[r].grads()
            for r in devs:
                stages[r].grads().copy_(tot)


def run_inprocess(ex, schedule, b, steps, mode):
    place = runtime.placements(schedule, b)
    stages = {}
    for r, pl in sorted(place.items()):
        p = ex.Partition(pl.block_lo, pl.block_hi, pl.per_device_batch, b)
        p.init_params()
        p.set_shard(pl.count, pl.first)
        stages[r] = p
    streams = {r: torch.cuda.Stream() for r in stages}
    if mode in ("peer", "peer-eager", "peer-dp"):
        eps = {r: {"input": p.input_ptr(), "mailbox": p.mailbox_ptr(), "row": p.row_bytes_in()}
               for r, p in stages.items()}
        for r, p in stages.items():
            recv, send = runtime.peer_wiring(schedule, b, r, eps)
            p.relay_set_recv(recv)
            p.relay_set_send(send)
        if mode == "peer-dp":  # gradients shared over peer memory, fused into the update
            for part in schedule["partitions"]:
                devs = part["devices"]
                if len(devs) > 1:
                    for r in devs:
                        stages[r].dp_set_group(devs.index(r), [stages[q].grads_ptr() for q in devs],
                                               [stages[q].mailbox_ptr() for q in devs],
                                               [stages[q].params_ptr() for q in devs])
        if mode in ("peer", "peer-dp"):
            for r, p in stages.items():
                p.capture_phases(fuse_teacher_student=True, stream=streams[r])
    torch.cuda.synchronize()
    nparts = len(schedule["partitions"])
    for _ in range(steps):
        if mode == "peer-dp":  # the whole step of every rank is device-side: one graph each
            for r, p in stages.items():
                p.replay_phase(0, streams[r])
            for r, p in stages.items():
                p.replay_phase(2, streams[r])
            torch.cuda.synchronize()
            continue
        if mode == "peer":
            for r, p in stages.items():  # every rank's whole forward/backward, device-side relay
                p.replay_phase(0, streams[r])
        elif mode == "peer-eager":
            for r, p in stages.items():
                p.teacher_forward(streams[r])
                p.student_step(streams[r])
        else:  # host copies of the overlapping row ranges (the NCCL path's data movement)
            for j in range(nparts):
                for r in schedule["partitions"][j]["devices"]:
                    if j > 0:
                        for src, dst, so, do, rows in runtime.relay_plan(schedule, b, j):
                            if dst == r:
                                stages[r].input_act()[do:do + rows].copy_(stages[src].teacher_out()[so:so + rows])
                    stages[r].teacher_forward()
            for p in stages.values():
                p.student_step()
        torch.cuda.synchronize()
        _dp_sum(schedule, stages)
        torch.cuda.synchronize()
        for r, p in stages.items():
            if mode == "peer":
                p.replay_phase(2, streams[r])
            else:
                p.apply_update(streams[r] if mode == "peer-eager" else None)
        torch.cuda.synchronize()
    return _state(stages)


@pytest.fixture(scope="module")
def ex():
    from paper_2301_12443_b200 import executor
    return executor


def _single(ex, b, steps):
    p = ex.Partition(0, 3, b, b)
    p.init_params()
    for _ in range(steps):
        p.step()
    torch.cuda.synchronize()
    return p


@pytest.mark.parametrize("mode", ["peer", "peer-eager"])
def test_pure_pipeline_peer_relay_bitwise(ex, mode):
    b, steps = 8, 3
    s = sched([(0, 1, [0]), (2, 3, [1])], b)
    got = run_inprocess(ex, s, b, steps, mode)
    ref = _single(ex, b, steps)
    want_params = ref.params().cpu()
    n0 = got[0][0].numel()
    assert torch.equal(torch.cat([got[0][0], got[1][0]]), want_params)
    assert got[0][2] + got[1][2] == ref.losses()
    assert torch.equal(got[1][3], ref.teacher_out().float().cpu())


def test_resharded_hybrid_peer_relay_bitwise(ex):
    """[0]x1 -> [1-2]x2 -> [3]x1: 1->2 and 2->1 resharding, DP group in the middle."""
    b, steps = 10, 3  # odd shard split exercises the remainder rule
    s = sched([(0, 0, [0]), (1, 2, [1, 2]), (3, 3, [3])], b)
    got = run_inprocess(ex, s, b, steps, "peer")
    want = run_inprocess(ex, s, b, steps, "copy")
    for r in got:
        assert torch.equal(got[r][0], want[r][0]), r
        assert torch.equal(got[r][1], want[r][1]), r
        assert got[r][2] == want[r][2], r
        assert torch.equal(got[r][3], want[r][3]), r


@pytest.mark.parametrize("parts,b", [([(0, 3, [0, 1])], 8), ([(0, 0, [0]), (1, 2, [1, 2]), (3, 3, [3])], 10),
                                     ([(0, 1, [0, 1, 2]), (2, 3, [3, 4])], 7)])
def test_dp_gradients_over_peer_memory_bitwise(ex, parts, b):
    """share_gradient + update over peer memory (pbdx_dp_set_group / pbdx_dp_set_params): each member sums
    its slice of the group's gradient slabs in member order and updates it, then gathers the other slices
    (reduce-scatter + all-gather) — identical to the host-side sum, every member identical (momentum
    completed from the slice owners by dp_sync_state when read)."""
    s = sched(parts, b)
    got = run_inprocess(ex, s, b, 3, "peer-dp")
    want = run_inprocess(ex, s, b, 3, "copy")
    for r in got:
        assert torch.equal(got[r][0], want[r][0]), r
        assert torch.equal(got[r][1], want[r][1]), r
        assert got[r][2] == want[r][2], r
    for _, _, devs in parts:
        for r in devs[1:]:
            assert torch.equal(got[r][0], got[devs[0]][0])  # DP members hold identical weights


def test_peer_relay_many_steps_no_drift(ex):
    """Sequence flags keep advancing across many graph replays (the slot protocol never stalls)."""
    b = 4
    s = sched([(0, 0, [0]), (1, 1, [1]), (2, 3, [2])], b)
    got = run_inprocess(ex, s, b, 40, "peer")
    want = run_inprocess(ex, s, b, 40, "copy")
    for r in got:
        assert torch.equal(got[r][0], want[r][0])


# ---------------------------------------------------------------- two processes, CUDA IPC mappings

def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _ipc_worker(rank, world, port, schedule, b, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2301_12443_b200 import executor
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def make(lo, hi, n, first):
            p = executor.Partition(lo, hi, n, b)
            p.init_params()
            p.set_shard(n, first)
            return p
        pipe = runtime.PipeBD(schedule, b, make, relay="peer")
        pipe.use_graphs()
        for _ in range(steps):
            pipe.step()
        torch.cuda.synchronize()
        dist.barrier()
        q.put((rank, pipe.stage.params().cpu().numpy(), pipe.stage.losses()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_dp_group_across_processes_ipc(ex):
    """[0-3]x2 in two processes: gradients shared through CUDA IPC mappings of each other's buffers."""
    b, steps = 8, 3
    s = sched([(0, 3, [0, 1])], b)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, s, b, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, params, losses = q.get(timeout=300)
        res[r] = (params, losses)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = run_inprocess(ex, s, b, steps, "copy")
    for r in (0, 1):
        assert np.array_equal(res[r][0], want[r][0].numpy())


def test_peer_relay_across_processes_ipc(ex):
    b, steps = 8, 3
    s = sched([(0, 1, [0]), (2, 3, [1])], b)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, s, b, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, params, losses = q.get(timeout=300)
        res[r] = (params, losses)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = _single(ex, b, steps)
    assert np.array_equal(np.concatenate([res[0][0], res[1][0]]), ref.params().cpu().numpy())
    assert res[0][1] + res[1][1] == ref.losses()


def _ckpt_worker(rank, world, port, schedule, b, steps, path, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2301_12443_b200 import executor
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def make(lo, hi, n, first):
            p = executor.Partition(lo, hi, n, b)
            p.init_params()
            p.set_shard(n, first)
            return p
        pipe = runtime.PipeBD(schedule, b, make, relay="peer")
        if mode == "resume":
            pipe.load_checkpoint(path)
        pipe.use_graphs()
        for _ in range(steps):
            pipe.step()
        torch.cuda.synchronize()
        if mode == "save":
            pipe.save_checkpoint(path)
        dist.barrier()
        q.put((rank, pipe.stage.params().cpu().numpy(), pipe.stage.losses()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_checkpoint_resume_bitwise_across_schedules(ex, tmp_path):
    """Save after 3 steps of a 2-process peer-relayed pipeline, resume in ONE process holding every
    block: 3 more steps are bit-identical to 6 uninterrupted steps."""
    b, steps = 8, 3
    ck = str(tmp_path / "ckpt")
    for world, parts, mode in ((2, [(0, 1, [0]), (2, 3, [1])], "save"), (1, [(0, 3, [0])], "resume")):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_ckpt_worker, args=(r, world, port, sched(parts, b), b, steps, ck, mode, q))
                 for r in range(world)]
        for p in procs:
            p.start()
        res = dict((r, (pr, lo)) for r, pr, lo in (q.get(timeout=300) for _ in range(world)))
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
    ref = _single(ex, b, 2 * steps)
    assert np.array_equal(res[0][0], ref.params().cpu().numpy())
    assert res[0][1] == ref.losses()


def _migrate_worker(rank, world, port, sched_a, sched_b, b, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2301_12443_b200 import executor
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def make(lo, hi, n, first):
            p = executor.Partition(lo, hi, n, b)
            p.init_params()
            p.set_shard(n, first)
            return p
        pipe = runtime.PipeBD(sched_a, b, make, relay="peer")
        for _ in range(steps):
            pipe.step()
        pipe.end_epoch()
        torch.cuda.synchronize()
        # rebuild the stage: the old executor's arena is freed while its state is handed over
        pipe.migrate(sched_b, make)
        for _ in range(steps):
            pipe.step()
        torch.cuda.synchronize()
        q.put((rank, pipe.stage.params().cpu().numpy(), pipe.stage.momentum().cpu().numpy(), pipe.stage.losses()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_migrate_with_device_executor_bitwise(ex):
    """runtime.PipeBD.migrate on real executors (the handed-over state must not be views of the
    old executor's freed arena): 3 steps, migrate (stage rebuilt), 3 more steps == 6 uninterrupted steps."""
    b, steps = 8, 3
    s = sched([(0, 3, [0])], b)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    proc = ctx.Process(target=_migrate_worker, args=(0, 1, port, s, s, b, steps, q))
    proc.start()
    _, params, mom, losses = q.get(timeout=300)
    proc.join(timeout=120)
    assert proc.exitcode == 0
    ref = _single(ex, b, 2 * steps)
    assert np.array_equal(params, ref.params().cpu().numpy())
    assert np.array_equal(mom, ref.momentum().cpu().numpy())
    assert losses == ref.losses()
