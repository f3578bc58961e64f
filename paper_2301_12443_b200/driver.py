"""ctypes face of the single-process multi-GPU driver (include/pbdr.h, csrc/exec/driver.cpp).

The driver is C++: it builds one pbdx executor per schedule device, wires the K11 peer relay and the
peer-memory DP exchange, and enqueues one CUDA graph per rank per step.  This module only binds it
(the torch.distributed flavour, one process per GPU, is runtime.PipeBD).
"""
from __future__ import annotations

import ctypes
import json
from typing import Dict, List, Optional

import torch

from . import executor
from ._lib import lib as _raw_lib

MODELS = {"resnet": 0, "mbv2": 1, "effb0": 2, "resnet_fp32": 3}


class PbdrDesc(ctypes.Structure):
    _fields_ = [("global_batch", ctypes.c_int), ("model", ctypes.c_int), ("image", ctypes.c_int),
                ("seed_data", ctypes.c_uint32), ("seed_teacher", ctypes.c_uint32), ("seed_student", ctypes.c_uint32),
                ("lr", ctypes.c_float), ("momentum", ctypes.c_float), ("graphs", ctypes.c_int)]


def lib() -> ctypes.CDLL:
    L = _raw_lib()
    if getattr(L, "_pbdr_bound", False):
        return L
    V, I, P = ctypes.c_void_p, ctypes.c_int, ctypes.POINTER
    L.pbdr_create.argtypes = [ctypes.c_char_p, P(PbdrDesc), P(I), I, P(V)]
    L.pbdr_destroy.argtypes = [V]
    L.pbdr_destroy.restype = None
    for name in ("pbdr_step", "pbdr_sync", "pbdr_num_blocks"):
        getattr(L, name).argtypes = [V]
    L.pbdr_block_losses.argtypes = [V, P(ctypes.c_double)]
    L.pbdr_rank.argtypes = [V, I, P(V), P(I)]
    L.pbdr_device_count.argtypes = []
    L.pbdr_relay_plan.argtypes = [ctypes.c_char_p, I, I, P(ctypes.c_longlong), I]
    L._pbdr_bound = True
    return L


def relay_plan(schedule: dict, global_batch: int, boundary: int) -> List[tuple]:
    """The C++ driver's relay messages (runtime.relay_plan's contract), host-only."""
    buf = (ctypes.c_longlong * (5 * 256))()
    n = lib().pbdr_relay_plan(json.dumps(schedule).encode(), global_batch, boundary, buf, 256)
    if n < 0:
        raise ValueError(f"pbdr_relay_plan failed ({-n})")
    return [tuple(int(buf[5 * i + j]) for j in range(5)) for i in range(n)]


class Driver:
    def __init__(self, schedule: dict, global_batch: int, devices: Optional[List[int]] = None, model: str = "resnet",
                 image: int = 0, graphs: bool = True, seeds=(1234, 1, 2), lr: float = 0.1, momentum: float = 0.9):
        nranks = sum(len(p["devices"]) for p in schedule["partitions"])
        devices = devices if devices is not None else [0] * nranks
        self.model = model
        self.nranks = nranks
        d = PbdrDesc(global_batch, MODELS[model], image or (32 if model.startswith("resnet") else 224), seeds[0],
                     seeds[1], seeds[2], lr, momentum, int(graphs))
        h = ctypes.c_void_p()
        rc = lib().pbdr_create(json.dumps(schedule).encode(), ctypes.byref(d), (ctypes.c_int * nranks)(*devices),
                               nranks, ctypes.byref(h))
        if rc != 0:
            raise RuntimeError(f"pbdr_create failed ({rc})")
        self.handle = h
        self.schedule = schedule

    def __del__(self):
        if getattr(self, "handle", None):
            lib().pbdr_destroy(self.handle)
            self.handle = None

    def step(self):
        if lib().pbdr_step(self.handle) != 0:
            raise RuntimeError("pbdr_step failed")

    def sync(self):
        if lib().pbdr_sync(self.handle) != 0:
            raise RuntimeError("pbdr_sync failed")

    def block_losses(self) -> List[float]:
        n = lib().pbdr_num_blocks(self.handle)
        out = (ctypes.c_double * n)()
        if lib().pbdr_block_losses(self.handle, out) != 0:
            raise RuntimeError("pbdr_block_losses failed")
        return list(out)

    def rank_state(self, r: int) -> Dict[str, torch.Tensor]:
        """params / momentum (DP momentum completed from the slice owners) / teacher output of rank r."""
        ex, dev = ctypes.c_void_p(), ctypes.c_int()
        if lib().pbdr_rank(self.handle, r, ctypes.byref(ex), ctypes.byref(dev)) != 0:
            raise RuntimeError("pbdr_rank failed")
        L = executor.lib()
        group = next(p["devices"] for p in self.schedule["partitions"] if r in p["devices"])
        with torch.cuda.device(dev.value):
            if len(group) > 1:
                L.pbdx_dp_sync_state(ex, None)
            torch.cuda.synchronize()

            def buf(which, dtype):
                p, n = ctypes.c_void_p(), ctypes.c_size_t()
                L.pbdx_buffer(ex, which, ctypes.byref(p), ctypes.byref(n))
                el = torch.tensor([], dtype=dtype).element_size()
                ts = {torch.float32: "<f4", torch.float64: "<f8"}[dtype]
                return torch.as_tensor(executor._CudaArray(p.value, (n.value // el,), ts), device=f"cuda:{dev.value}")

            return {"params": buf(executor.BUF_PARAMS, torch.float32).clone().cpu(),
                    "momentum": buf(executor.BUF_MOMENTUM, torch.float32).clone().cpu(),
                    "losses": buf(executor.BUF_LOSSES, torch.float64).clone().cpu()}
