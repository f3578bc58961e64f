"""configs[4]: an imbalanced block-time workload exercising the partitioner's
reconfiguration on DEVICE-MEASURED times.  Epoch 0 runs the MobileNetV2 -> ProxylessNAS supernet
with the sampled path; at the epoch boundary the late blocks switch to their heaviest candidates
(k7, e6: the "drift injected by switching a block's active candidate at epoch E").  The monitor
re-times every block at the per-device batch the CURRENT schedule gives it (what a running
partition observes), runtime.observed_profile rescales the profile, and reconfigure()
(schedule.cpp:347-359) re-plans for N GPUs.  Writes one JSON document (stdout).

  python scripts/reconfig_mbv2.py [global_batch] [image] [num_devices]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_12443_b200 import core, executor, mb_models, runtime  # noqa: E402


def measure(k, n, gb, image, path, reps=5):
    p = executor.Partition(k, k, n, gb, model="mbv2", image=image)
    p.init_params()
    p.set_path(k, path)
    p.set_timing(True)
    ts, ss = [], []
    for r in range(reps + 2):
        p.step()
        t, s = p.block_times()
        if r >= 2:
            ts.append(t[0])
            ss.append(s[0])
    return sorted(ts)[len(ts) // 2], sorted(ss)[len(ss) // 2]


def main():
    gb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    image = int(sys.argv[2]) if len(sys.argv) > 2 else 224
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    threshold = 0.10
    paths0 = mb_models.paths_for(0)
    prof = runtime.profile_blocks(gb, N, model="mbv2", image=image, paths=paths0)
    sched0, meta0 = core.best_schedule(prof)
    # epoch boundary: the late blocks switch to their heaviest candidate
    paths1 = {k: list(v) for k, v in paths0.items()}
    for k in (4, 5):
        paths1[k] = [5] * len(paths1[k])
    place = runtime.placements(sched0, gb)
    measured = {}
    for j, part in enumerate(sched0["partitions"]):
        lo, hi = part["blocks"]
        bj = part["per_device_batch"]
        for k in range(lo, hi + 1):
            t, s = measure(k, bj, gb, image, paths1[k])
            measured[k] = (bj, t, s)
    observed = runtime.observed_profile(prof, measured)
    drift = core.profile_drift(prof, observed)
    new = core.reconfigure(prof, sched0, observed, threshold)
    pred_old_on_new = core.predicted_step_time(observed, sched0)["step_ms"]
    out = {"global_batch": gb, "image": image, "num_devices": N, "threshold": threshold,
           "paths_epoch0": paths0, "paths_epoch1": paths1,
           "schedule_epoch0": sched0["partitions"], "predicted_step_ms_epoch0": meta0.get("step_ms", None)
           or core.predicted_step_time(prof, sched0)["step_ms"],
           "measured_at_current_shards": {str(k): v for k, v in measured.items()}, "drift": drift,
           "replanned": new is not None,
           "schedule_epoch1": new["partitions"] if new else None,
           "predicted_step_ms_epoch1_old_schedule": pred_old_on_new,
           "predicted_step_ms_epoch1_new_schedule": core.predicted_step_time(observed, new)["step_ms"] if new
           else None,
           "profile_epoch0": prof, "profile_observed": observed}
    print(json.dumps(out))


if __name__ == "__main__":
    torch.cuda.init()
    main()
