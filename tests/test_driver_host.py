"""Host-only wiring of the C++ driver (include/pbdr.h) against runtime.py's (CPU)."""
import json
import random

import pytest

from paper_2301_12443_b200 import driver, runtime


def _sched(rng):
    nb = rng.randint(1, 6)
    cuts = sorted(rng.sample(range(1, nb), rng.randint(0, nb - 1))) if nb > 1 else []
    bounds = [0] + cuts + [nb]
    parts, dev = [], 0
    for i in range(len(bounds) - 1):
        g = rng.randint(1, 3)
        parts.append({"blocks": [bounds[i], bounds[i + 1] - 1], "devices": list(range(dev, dev + g)),
                      "per_device_batch": 1})
        dev += g
    return {"flags": {"tr": True, "dpu": True, "ahd": True}, "partitions": parts,
            "predicted": {"partition_ms": [0.0] * len(parts), "step_ms": 0.0}}


def test_relay_plan_matches_runtime():
    rng = random.Random(7)
    for _ in range(300):
        s = _sched(rng)
        b = rng.randint(8, 64)
        for p in s["partitions"]:
            p["per_device_batch"] = -(-b // len(p["devices"]))
        for k in range(1, len(s["partitions"])):
            assert driver.relay_plan(s, b, k) == runtime.relay_plan(s, b, k), (json.dumps(s), b, k)


def test_relay_plan_rejects_bad_boundary():
    s = _sched(random.Random(1))
    with pytest.raises(ValueError):
        driver.relay_plan(s, 16, 0)
