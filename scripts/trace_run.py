"""Measured timelines of real runs: run the Pipe-BD runtime for a few steps
with CUDA-event tracing, build the reference-format report (runtime.measured_report), check the
measured steady-state step against the partitioner's prediction (core.validate_prediction) and
render the Gantt chart.  One process per rank (torchrun, or spawned here: WORLD ranks sharing the
visible GPUs round-robin, gloo for the control plane, K11 peer relay for the activations).

  python scripts/trace_run.py [world] [global_batch] [out_prefix]
"""
import json
import os
import socket
import sys

import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, gb, prefix):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2301_12443_b200 import core, executor, runtime
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        obj = [None, None]
        if rank == 0:
            prof = runtime.profile_blocks(gb, world, device=dev)
            if world > 1:  # a pure pipeline across the ranks (contiguous_only: one block range per rank)
                sched, _ = core.best_schedule(prof, contiguous_only=True)
            else:
                sched, _ = core.best_schedule(prof)
            obj = [sched, prof]
        dist.broadcast_object_list(obj, src=0)
        sched, prof = obj

        def make(lo, hi, n, first):
            p = executor.Partition(lo, hi, n, gb, device=dev)
            p.init_params()
            p.set_shard(n, first)
            return p

        pipe = runtime.PipeBD(sched, gb, make, relay="peer")
        for _ in range(3):
            pipe.step()
        rep = runtime.measured_report(pipe, 12)
        if rank == 0:
            pred = core.predicted_step_time(prof, sched)
            err = core.validate_prediction(rep, prof, sched)
            summary = {"schedule": sched["partitions"], "predicted_step_ms": pred["step_ms"],
                       "measured_steady_step_ms": rep["steady_state_step_ms"], "relative_error": err,
                       "bubble_ratio": rep["bubble_ratio"], "category_totals_ms": rep["category_totals_ms"],
                       "overlapped_compute_ms": rep["overlapped_compute_ms"], "world": world, "global_batch": gb,
                       "gpus_visible": torch.cuda.device_count()}
            with open(prefix + "_report.json", "w") as f:
                json.dump(rep, f)
            with open(prefix + "_summary.json", "w") as f:
                json.dump(summary, f, indent=1)
            with open(prefix + "_gantt.svg", "w") as f:
                f.write(core.gantt_svg(rep, f"measured: {world} rank(s), b={gb}, schedule "
                                            + " ".join(f"{p['blocks']}x{len(p['devices'])}" for p in sched["partitions"])))
            print(json.dumps(summary))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    gb = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    prefix = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/trace"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(worker, args=(world, port, gb, prefix), nprocs=world, join=True)


if __name__ == "__main__":
    main()
