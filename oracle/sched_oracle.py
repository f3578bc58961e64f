"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the reference partitioner.

Restates, operation for operation (Python floats are IEEE doubles, so the same
evaluation order gives the same bits):
  exec_time            proj/core/src/cost_model.cpp:38-66
  allreduce/dpc        cost_model.cpp:79-96
  memory_estimate      cost_model.cpp:98-112
  compositions         schedule.cpp:37-50
  enumerate_configs    schedule.cpp:115-134 (+ build_config :52-69)
  partition_cost       schedule.cpp:136-146
  predicted_step_time  schedule.cpp:148-165
  best_schedule        schedule.cpp:167-244 (strict <, lowest index wins)
Pinned by tests/test_oracle_sched.py against the reference tests' golden
values and against oracle/_ref (the reference compiled unmodified).
Documents are the reference JSON profile format (proj/README.md:141-162).
"""
from __future__ import annotations

from typing import Dict, List, Tuple


def _tmap(m: Dict) -> List[Tuple[int, float]]:
    return sorted((int(k), float(v)) for k, v in m.items())


class Model:
    def __init__(self, doc: dict, act_mem_multiplier: float = 3.0):
        self.blocks = doc["blocks"]
        self.hw = doc["hardware"]
        self.global_batch = int(doc["global_batch"])
        self.mult = act_mem_multiplier
        self.t = [_tmap(b["teacher_ms"]) for b in self.blocks]
        self.s = [_tmap(b["student_ms"]) for b in self.blocks]

    @property
    def num_blocks(self):
        return len(self.blocks)

    @property
    def num_devices(self):
        return int(self.hw["num_devices"])

    # cost_model.cpp:38-66
    def exec_time(self, block: int, role: str, batch: int) -> float:
        m = self.t[block] if role == "teacher" else self.s[block]
        x = float(batch)
        min_b, min_ms = m[0]
        if batch <= min_b:
            if batch == min_b:
                return min_ms
            a = min_ms * x / min_b
            b = min_ms * float(self.hw["min_utilization_floor"])
            return b if a < b else a  # std::max(a, b)
        max_b, max_ms = m[-1]
        if batch >= max_b:
            if batch == max_b:
                return max_ms
            if len(m) == 1:
                return max_ms * x / max_b
            b1, t1 = m[-2]
            slope = (max_ms - t1) / float(max_b - b1)
            return max_ms + slope * (x - max_b)
        for i, (kb, kt) in enumerate(m):
            if kb >= batch:
                if kb == batch:
                    return kt
                lb, lt = m[i - 1]
                frac = (x - lb) / float(kb - lb)
                return lt + frac * (kt - lt)
        raise AssertionError("unreachable")

    # cost_model.cpp:79-86
    def allreduce_time(self, param_bytes: float, g: int) -> float:
        if g == 1:
            return 0.0
        gf = float(g)
        return 2.0 * (gf - 1.0) / gf * param_bytes / float(self.hw["allreduce_bytes_per_ms"])

    # cost_model.cpp:88-96
    def dpc_time(self, lo: int, hi: int, g: int) -> float:
        if g == 1:
            return 0.0
        total = 0.0
        for k in range(lo, hi + 1):
            b = self.blocks[k]
            total += float(b["dpc_ms_override"]) if "dpc_ms_override" in b else self.allreduce_time(
                float(b["param_bytes"]), g)
        return total

    # cost_model.cpp:98-112
    def memory_estimate(self, lo: int, hi: int, pdb: int) -> float:
        total = 0.0
        for k in range(lo, hi + 1):
            b = self.blocks[k]
            total += float(b["param_bytes"]) + float(b["teacher_param_bytes"]) + \
                float(b["act_bytes_per_sample"]) * pdb * self.mult
        return total

    # schedule.cpp:136-146
    def partition_cost(self, lo: int, hi: int, g: int, pdb: int) -> float:
        total = 0.0
        for k in range(lo, hi + 1):
            total += self.exec_time(k, "teacher", pdb)
            total += self.exec_time(k, "student", pdb)
        return total + self.dpc_time(lo, hi, g)


def compositions(total: int, parts: int) -> List[List[int]]:
    """schedule.cpp:37-50 — ordered compositions, lexicographic."""
    if parts == 1:
        return [[total]]
    out = []
    for first in range(1, total - (parts - 1) + 1):
        for rest in compositions(total - first, parts - 1):
            out.append([first] + rest)
    return out


def enumerate_configs(B: int, N: int, gb: int = 0) -> List[List[Tuple[int, int, int, int]]]:
    """schedule.cpp:115-134 — list of configs, each a list of (lo, hi, g, pdb)."""
    out = []
    for parts in range(1, min(B, N) + 1):
        for bc in compositions(B, parts):
            for gc in compositions(N, parts):
                cfg, lo = [], 0
                for nb, g in zip(bc, gc):
                    cfg.append((lo, lo + nb - 1, g, (gb + g - 1) // g if gb > 0 else 0))
                    lo += nb
                out.append(cfg)
    return out


def predicted_step_time(m: Model, cfg) -> Tuple[List[float], float, bool]:
    """schedule.cpp:148-165."""
    pms, feasible = [], True
    for (lo, hi, g, pdb) in cfg:
        pms.append(m.partition_cost(lo, hi, g, pdb))
        if feasible and m.memory_estimate(lo, hi, pdb) > float(m.hw["mem_bytes_per_device"]):
            feasible = False
    return pms, max(pms), feasible


def best_schedule(doc: dict, contiguous_only: bool = False):
    """schedule.cpp:167-244. Returns (config, partition_ms, step_ms, configs_evaluated)."""
    m = Model(doc)
    configs = enumerate_configs(m.num_blocks, m.num_devices, m.global_batch)
    if contiguous_only:
        configs = [c for c in configs if len(c) == m.num_devices and all(p[2] == 1 for p in c)]
        if not configs:
            raise ValueError("infeasible: contiguous-only search needs at least as many blocks as devices")
    best = None
    for i, cfg in enumerate(configs):
        pms, step, ok = predicted_step_time(m, cfg)
        if not ok:
            continue
        if best is None or step < best[2]:
            best = (cfg, pms, step, i)
    if best is None:
        raise ValueError("infeasible: no feasible configuration")
    return best[0], best[1], best[2], len(configs)
