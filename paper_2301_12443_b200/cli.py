"""GPU-side commands of the `pbd` command line (the host-only ones — schedule, simulate, compare,
profile-gen, report — are the C++ binary lib/pbd, csrc/tools/pbd_cli.cpp).

  python -m paper_2301_12443_b200.cli profile --model resnet|mbv2|effb0 [--global-batch B]
         [--devices N] [--image S] [--out profile.json]
      measure T_k(b), S_k(b) of every block on this GPU with CUDA events and write the reference's
      profile document (profile.hpp:30-86; the paper's profiling step)
  [torchrun ...] python -m paper_2301_12443_b200.cli run --schedule schedule.json [--model ...]
         [--global-batch B] [--steps K] [--trace report.json] [--gantt timeline.svg]
         [--resume DIR] [--save DIR]
      run a schedule with one process per GPU (K11 peer relay, gradients over peer memory) and
      optionally write the measured-timeline report + Gantt chart; --resume / --save restore / write
      a per-block checkpoint (runtime.PipeBD.save_checkpoint, schedule-independent)

Exit codes follow the reference CLI (pbd_cli.cpp:29-32): 0 ok, 1 validation, 2 infeasible, 3 I/O.
"""
from __future__ import annotations

import argparse
import json
import os
import sys


def _profile(a) -> int:
    import torch
    from . import runtime
    model = a.model
    prof = runtime.profile_blocks(a.global_batch, a.devices, device=torch.device("cuda", 0), model=model,
                                  image=a.image if model != "resnet" else None)
    text = json.dumps(prof, indent=2, sort_keys=True) + "\n"
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


def _run(a) -> int:
    import torch
    import torch.distributed as dist
    from . import core, executor, mb_models, runtime
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl" if world > 1 else "gloo", rank=rank, world_size=world)
    try:
        with open(a.schedule) as f:
            sched = json.load(f)
        ndev = sum(len(p["devices"]) for p in sched["partitions"])
        if ndev != world:
            print(f"error: schedule uses {ndev} devices, {world} ranks running", file=sys.stderr)
            return 1
        paths = None
        if a.model != "resnet":
            mb_models.set_family(a.model)
            paths = mb_models.paths_for(0)

        def make(lo, hi, n, first):
            p = executor.Partition(lo, hi, n, a.global_batch, device=dev, model=a.model,
                                   image=a.image if a.model != "resnet" else None)
            p.init_params()
            p.set_shard(n, first)
            if paths is not None:
                for k in range(lo, hi + 1):
                    p.set_path(k, paths[k])
            return p

        pipe = runtime.PipeBD(sched, a.global_batch, make, relay="peer")
        if a.resume:
            meta = pipe.load_checkpoint(a.resume)
            if rank == 0:
                print(f"resumed at step {meta['step']} from {a.resume}", file=sys.stderr)
        for _ in range(a.steps):
            pipe.step()
        losses = pipe.block_losses()
        if a.save:
            pipe.save_checkpoint(a.save)
        rep = runtime.measured_report(pipe, max(4, a.trace_steps)) if (a.trace or a.gantt) else None
        gathered = [None] * world
        dist.all_gather_object(gathered, losses)
        if rank == 0:
            merged = {k: v for d in gathered for k, v in d.items()}
            print(json.dumps({"block_losses": merged}))
            if rep is not None:
                if a.trace:
                    with open(a.trace, "w") as f:
                        json.dump(rep, f)
                if a.gantt:
                    with open(a.gantt, "w") as f:
                        f.write(core.gantt_svg(rep, "measured"))
                print(f"measured steady-state step: {rep['steady_state_step_ms']:.4f} ms")
        dist.barrier()
    finally:
        dist.destroy_process_group()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="pbd-gpu")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("profile")
    p.add_argument("--model", choices=["resnet", "mbv2", "effb0"], default="resnet")
    p.add_argument("--global-batch", type=int, default=256)
    p.add_argument("--devices", type=int, default=8)
    p.add_argument("--image", type=int, default=224)
    p.add_argument("--out")
    r = sub.add_parser("run")
    r.add_argument("--schedule", required=True)
    r.add_argument("--model", choices=["resnet", "mbv2", "effb0"], default="resnet")
    r.add_argument("--global-batch", type=int, default=256)
    r.add_argument("--image", type=int, default=224)
    r.add_argument("--steps", type=int, default=10)
    r.add_argument("--trace")
    r.add_argument("--trace-steps", type=int, default=8)
    r.add_argument("--gantt")
    r.add_argument("--resume")
    r.add_argument("--save")
    a = ap.parse_args(argv)
    try:
        return _profile(a) if a.cmd == "profile" else _run(a)
    except (OSError, IOError) as e:
        print(f"io error: {e}", file=sys.stderr)
        return 3
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
