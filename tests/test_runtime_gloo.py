"""Multi-rank host logic of runtime.py on CPU (gloo, world size 2 and 3).

The stages are oracle-backed (tests/oracle_stage.py); the placement, the
relay resharding between groups of different sizes, the group allreduce and
the DPU / barrier paths are the product's.  The distributed run must equal a
single-process run of the same schedule (the oracle Trainer with the same DP
shards): identical per-block losses and student weights.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2301_12443_b200 import runtime


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def sched(parts, b):
    return {"flags": {"tr": True, "dpu": True, "ahd": True},
            "partitions": [{"blocks": [lo, hi], "devices": devs, "per_device_batch": -(-b // len(devs))}
                           for lo, hi, devs in parts],
            "predicted": {"partition_ms": [0.0] * len(parts), "step_ms": 0.0}}


def _worker(rank, world, port, schedule, b, steps, dpu, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.set_num_threads(2)
    os.environ["OMP_NUM_THREADS"] = "2"
    from tests.oracle_stage import OracleStage
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pipe = runtime.PipeBD(schedule, b, lambda lo, hi, n, first: OracleStage(lo, hi, n, first, b), dpu=dpu)
        for _ in range(steps):
            pipe.step()
        pipe.end_epoch()
        losses = pipe.block_losses()
        q.put((rank, losses, {k: pipe.stage.sp[k] for k in pipe.stage.blocks}, pipe.me.index))
    finally:
        dist.destroy_process_group()


def run_dist(schedule, world, b, steps, dpu=True):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, schedule, b, steps, dpu, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("parts,world,dpu", [
    ([(0, 1, [0]), (2, 3, [1])], 2, True),          # pure pipeline (teacher relaying)
    ([(0, 3, [0, 1])], 2, True),                     # internal relaying: one DP group of 2
    ([(0, 0, [0, 1]), (1, 3, [2])], 3, False),       # hybrid: resharding 2 -> 1, TR without DPU
    ([(0, 1, [0]), (2, 3, [1, 2])], 3, True),        # hybrid: resharding 1 -> 2
])
def test_distributed_equals_single_process(parts, world, dpu):
    from oracle import bd
    b, steps = 5, 2   # odd batch: uneven shards (remainder rule)
    s = sched(parts, b)
    out = run_dist(s, world, b, steps, dpu)
    groups = {}
    for lo, hi, devs in parts:
        for k in range(lo, hi + 1):
            groups[k] = len(devs)
    tr = bd.Trainer(b, bf16_mode=1)
    for st in range(steps):
        want = tr.step(st, groups)
    for rank, losses, params, index in out:
        for k, v in losses.items():
            assert v == pytest.approx(want[k], rel=1e-12, abs=1e-15), (rank, k)
        for k, p in params.items():
            np.testing.assert_allclose(p, tr.sp[k], rtol=1e-6, atol=1e-9)


def test_relay_plan_covers_every_row_once():
    for b in (5, 7, 64, 255):
        for g_up in range(1, 5):
            for g_dn in range(1, 5):
                ups = list(range(g_up))
                dns = list(range(g_up, g_up + g_dn))
                s = sched([(0, 0, ups), (1, 3, dns)], b)
                msgs = runtime.relay_plan(s, b, 1)
                got = np.zeros(b, int)
                for src, dst, so, do, rows in msgs:
                    fs, cs = runtime.shard(b, g_up, ups.index(src))
                    fd, cd = runtime.shard(b, g_dn, dns.index(dst))
                    assert 0 <= so and so + rows <= cs and 0 <= do and do + rows <= cd
                    assert fs + so == fd + do
                    got[fd + do: fd + do + rows] += 1
                assert (got == 1).all()


def _migrate_worker(rank, world, port, sched_a, sched_b, b, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.set_num_threads(2)
    from tests.oracle_stage import OracleStage
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        make = lambda lo, hi, n, first: OracleStage(lo, hi, n, first, b)  # noqa: E731
        pipe = runtime.PipeBD(sched_a, b, make)
        for _ in range(steps):
            pipe.step()
        pipe.end_epoch()
        pipe.migrate(sched_b, make)
        for _ in range(steps):
            pipe.step()
        pipe.end_epoch()
        losses = pipe.block_losses()
        q.put((rank, losses, {k: pipe.stage.sp[k] for k in pipe.stage.blocks}))
    finally:
        dist.destroy_process_group()


def test_reconfiguration_migrates_state_exactly():
    """Epoch-boundary re-plan (schedule.cpp:347-359): 2 steps on schedule A, migrate
    weights + momentum to schedule B, 2 more steps == single process with A's then B's DP shards."""
    from oracle import bd
    b, steps, world = 5, 2, 3
    parts_a = [(0, 0, [0, 1]), (1, 3, [2])]
    parts_b = [(0, 1, [0]), (2, 3, [1, 2])]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_migrate_worker, args=(r, world, port, sched(parts_a, b), sched(parts_b, b), b, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    def groups(parts):
        return {k: len(devs) for lo, hi, devs in parts for k in range(lo, hi + 1)}

    tr = bd.Trainer(b, bf16_mode=1)
    for st in range(steps):
        tr.step(st, groups(parts_a))
    for st in range(steps, 2 * steps):
        want = tr.step(st, groups(parts_b))
    for rank, losses, params in out:
        for k, v in losses.items():
            assert v == pytest.approx(want[k], rel=1e-12, abs=1e-15), (rank, k)
        for k, p in params.items():
            np.testing.assert_allclose(p, tr.sp[k], rtol=1e-6, atol=1e-9)


def test_peer_wiring_slots_are_consistent():
    """K11 wiring (runtime.peer_wiring): every sender writes exactly the flag slot its receiver waits
    on, every receiver releases exactly the slot its sender waits on, and the peer stores cover each
    receiver's input rows once."""
    for b in (5, 8, 255):
        for parts in ([(0, 0, [0]), (1, 2, [1, 2]), (3, 3, [3])], [(0, 1, [0, 1, 2]), (2, 3, [3, 4])],
                      [(0, 0, [0, 1]), (1, 1, [2]), (2, 3, [3, 4, 5])]):
            s = sched(parts, b)
            place = runtime.placements(s, b)
            eps = {r: {"input": 10 ** 9 * (r + 1), "mailbox": 10 ** 12 * (r + 1), "row": 1000} for r in place}
            wiring = {r: runtime.peer_wiring(s, b, r, eps) for r in place}
            for r, (recv, send) in wiring.items():
                pl = place[r]
                senders = [m[0] for m in runtime.relay_plan(s, b, pl.partition) if m[1] == r] if pl.partition else []
                # receiver r waits on mailbox[i] for sender i; sender i must write exactly that address
                for i, src in enumerate(senders):
                    flags = [f for _, _, dst, f in wiring[src][1] if eps[r]["input"] <= dst < eps[r]["input"] + 10 ** 9]
                    assert flags == [eps[r]["mailbox"] + 8 * i]
                    # r releases into sender's consumed slot = r's index among src's receivers
                    recvs = [m[1] for m in runtime.relay_plan(s, b, place[src].partition + 1) if m[0] == src]
                    assert recv[i] == eps[src]["mailbox"] + 8 * (16 + recvs.index(r))
                if senders:
                    rows = np.zeros(pl.count, int)
                    for src in senders:
                        for _, nrows, dst, _ in wiring[src][1]:
                            off = dst - eps[r]["input"]
                            if 0 <= off < 10 ** 9:
                                rows[off // 1000: off // 1000 + nrows] += 1
                    assert (rows == 1).all()


def _mb_worker(rank, world, port, schedule, b, S, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.set_num_threads(2)
    os.environ["OMP_NUM_THREADS"] = "2"
    from oracle import mb
    from tests.oracle_stage import MbOracleStage
    paths = {k: mb.sample_path(k, 2) for k in range(6)}
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pipe = runtime.PipeBD(schedule, b, lambda lo, hi, n, first: MbOracleStage(lo, hi, n, first, b, S, paths))
        for _ in range(steps):
            pipe.step()
        pipe.end_epoch()
        q.put((rank, pipe.block_losses(), {k: pipe.stage.sp[k] for k in pipe.stage.blocks}))
    finally:
        dist.destroy_process_group()


def test_mbv2_hybrid_distributed_equals_single_process():
    """configs[2] workload through the multi-rank runtime: [0-1]x1 -> [2-4]x2 -> [5]x1 (1->2 and 2->1
    resharding, a DP group over the supernet's path-sparse gradients) == one process, same shards."""
    from oracle import mb
    b, S, steps, world = 3, 32, 2, 4
    parts = [(0, 1, [0]), (2, 4, [1, 2]), (5, 5, [3])]
    s = sched(parts, b)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_mb_worker, args=(r, world, port, s, b, S, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    paths = {k: mb.sample_path(k, 2) for k in range(6)}
    groups = {k: len(devs) for lo, hi, devs in parts for k in range(lo, hi + 1)}
    tr = mb.Trainer(b, S)
    for st in range(steps):
        want = tr.step(st, paths, groups)
    for rank, losses, params in out:
        for k, v in losses.items():
            assert v == pytest.approx(want[k], rel=1e-12, abs=1e-15), (rank, k)
        for k, p in params.items():
            np.testing.assert_allclose(p, tr.sp[k], rtol=1e-6, atol=1e-9)


def _ckpt_worker(rank, world, port, schedule, b, steps, path, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.set_num_threads(2)
    from tests.oracle_stage import OracleStage
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pipe = runtime.PipeBD(schedule, b, lambda lo, hi, n, first: OracleStage(lo, hi, n, first, b))
        if mode == "resume":
            try:
                meta = pipe.load_checkpoint(path)
            except ValueError as e:
                q.put((rank, "error", str(e)))
                return
            assert meta["step"] == steps
        for _ in range(steps):
            pipe.step()
        pipe.end_epoch()
        if mode == "save":
            pipe.save_checkpoint(path)
        q.put((rank, pipe.block_losses(), {k: pipe.stage.sp[k].copy() for k in pipe.stage.blocks}))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_checkpoint_resume_under_another_schedule(tmp_path):
    """save_checkpoint on 3 ranks ([0]x2 -> [1-3]x1), resume on 2 ranks ([0-1] -> [2-3]): the resumed
    run equals one uninterrupted single-process run with A's then B's DP shards."""
    from oracle import bd
    b, steps = 5, 2
    parts_a = [(0, 0, [0, 1]), (1, 3, [2])]
    parts_b = [(0, 1, [0]), (2, 3, [1])]
    ck = str(tmp_path / "ckpt")
    _spawn(_ckpt_worker, 3, sched(parts_a, b), b, steps, ck, "save")
    assert sorted(os.listdir(ck)) == ["block_00.bin", "block_01.bin", "block_02.bin", "block_03.bin", "meta.json"]
    out = _spawn(_ckpt_worker, 2, sched(parts_b, b), b, steps, ck, "resume")

    def groups(parts):
        return {k: len(devs) for lo, hi, devs in parts for k in range(lo, hi + 1)}

    tr = bd.Trainer(b, bf16_mode=1)
    for st in range(steps):
        tr.step(st, groups(parts_a))
    for st in range(steps, 2 * steps):
        want = tr.step(st, groups(parts_b))
    for rank, losses, params in out:
        for k, v in losses.items():
            assert v == pytest.approx(want[k], rel=1e-12, abs=1e-15), (rank, k)
        for k, p in params.items():
            np.testing.assert_allclose(p, tr.sp[k], rtol=1e-6, atol=1e-9)


def test_checkpoint_rejects_mismatch(tmp_path):
    import json
    ck = str(tmp_path / "ckpt")
    b = 5
    _spawn(_ckpt_worker, 1, sched([(0, 3, [0])], b), b, 1, ck, "save")
    meta = json.load(open(os.path.join(ck, "meta.json")))
    assert meta["step"] == 1 and meta["global_batch"] == b and set(meta["block_numel"]) == {"0", "1", "2", "3"}
    (rank, tag, msg), = _spawn(_ckpt_worker, 1, sched([(0, 3, [0])], 7), 7, 1, ck, "resume")
    assert tag == "error" and "global batch" in msg


def _baseline_worker(rank, world, port, kind, plan, b, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.set_num_threads(2)
    from tests.oracle_stage import OracleStage
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = runtime.run_baseline(kind, plan, b, lambda lo, hi, n, first: OracleStage(lo, hi, n, first, b),
                                   steps=1, warmup=0, rank=rank, world=world)
        q.put((rank, {k: v[0].numpy().copy() for k, v in res["states"].items()}, res["all_blocks_ms"]))
    finally:
        dist.destroy_process_group()


def test_dp_baseline_on_ranks_equals_ddp_oracle():
    """The paper's DP baseline executed on 2 ranks (runtime.run_baseline, plan = core.baseline_plan 'dp'):
    each block in turn, teacher prefix recomputed, gradients all-reduced over the shards — one step of
    block k equals the oracle's DDP step of block k on the same 2 shards (remainder rule, odd batch)."""
    from oracle import bd
    from paper_2301_12443_b200 import core
    from tests.profiles import proportional_doc
    b = 5
    plan = core.baseline_plan(proportional_doc([1, 1, 1, 1], [1, 1, 1, 1], 2, b), "dp")
    assert len(plan["phase_step_ms"]) == 4 and plan["per_device_batch"] == 3
    out = _spawn(_baseline_worker, 2, "dp", plan, b)
    tr = bd.Trainer(b, bf16_mode=1)
    tr.step(0, {k: 2 for k in range(4)})
    for rank, states, ms in out:
        assert ms > 0
        for k, w in states.items():
            np.testing.assert_allclose(w, tr.sp[k], rtol=1e-6, atol=1e-9)


def test_ls_baseline_on_ranks_equals_oracle():
    """LS baseline on 2 ranks: the LPT assignment of core.baseline_plan 'ls' (schedule.cpp:261-303), each
    rank trains its blocks on the full batch with its own teacher prefix, no communication."""
    from oracle import bd
    from paper_2301_12443_b200 import core
    from tests.profiles import proportional_doc
    b = 4
    plan = core.baseline_plan(proportional_doc([1, 2, 3, 4], [1, 2, 3, 4], 2, b), "ls")
    assert sorted(k for d in plan["device_blocks"] for k in d) == [0, 1, 2, 3]
    out = _spawn(_baseline_worker, 2, "ls", plan, b)
    tr = bd.Trainer(b, bf16_mode=1)
    tr.step(0)
    seen = set()
    for rank, states, ms in out:
        assert sorted(states) == sorted(plan["device_blocks"][rank])
        for k, w in states.items():
            np.testing.assert_allclose(w, tr.sp[k], rtol=1e-6, atol=1e-9)
            seen.add(k)
    assert seen == {0, 1, 2, 3}
