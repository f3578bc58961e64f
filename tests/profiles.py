"""Profile-document fixtures restated from the reference tests (test data, not code):
proportional_doc (proj/tests/testutil.hpp:51-83) and random_doc (testutil.hpp:87-129)."""
import random


def proportional_doc(teacher_full, student_full, devices, global_batch, param_bytes=0.0,
                     allreduce_bytes_per_ms=1.0e6, act_bytes_per_sample=0.0, data_load_ms=0.0):
    blocks = []
    for i, (t, s) in enumerate(zip(teacher_full, student_full)):
        tm, sm = {}, {}
        for denom in (4, 2, 1):
            b = global_batch // denom
            tm[str(b)] = t / denom
            sm[str(b)] = s / denom
        blocks.append({"id": i, "teacher_ms": tm, "student_ms": sm, "act_bytes_per_sample": act_bytes_per_sample,
                       "param_bytes": param_bytes, "teacher_param_bytes": param_bytes})
    return {"blocks": blocks,
            "hardware": {"num_devices": devices, "link_bytes_per_ms": 1.0e9,
                         "allreduce_bytes_per_ms": allreduce_bytes_per_ms, "mem_bytes_per_device": 1.0e18,
                         "data_load_ms_per_batch": data_load_ms, "min_utilization_floor": 1.0e-6},
            "global_batch": global_batch}


def random_doc(rng: random.Random, max_blocks=6, max_devices=6, mem=1.0e18, overrides=False):
    B = rng.randint(1, max_blocks)
    N = rng.randint(1, max_devices)
    blocks = []
    for i in range(B):
        keys = rng.randint(1, 3)
        batch = 8 + int(rng.random() * 56.0)
        t = 0.2 + 4.0 * rng.random()
        s = 0.2 + 4.0 * rng.random()
        tm, sm = {}, {}
        for _ in range(keys):
            tm[str(batch)] = t
            sm[str(batch)] = s
            batch += 8 + int(rng.random() * 120.0)
            t += 3.0 * rng.random()
            s += 3.0 * rng.random()
        blk = {"id": i, "teacher_ms": tm, "student_ms": sm, "act_bytes_per_sample": 1024.0 * rng.random(),
               "param_bytes": 1.0e5 + 1.0e6 * rng.random(), "teacher_param_bytes": 1.0e5 + 1.0e6 * rng.random()}
        if overrides and rng.random() < 0.3:
            blk["dpc_ms_override"] = rng.random()
        blocks.append(blk)
    return {"blocks": blocks,
            "hardware": {"num_devices": N, "link_bytes_per_ms": 1.0e6 + 1.0e8 * rng.random(),
                         "allreduce_bytes_per_ms": 1.0e6 + 1.0e8 * rng.random(), "mem_bytes_per_device": mem,
                         "data_load_ms_per_batch": 0.2 * rng.random(),
                         "min_utilization_floor": 0.05 + 0.9 * rng.random()},
            "global_batch": max(N, 32 + int(rng.random() * 480.0))}
