"""Python face of the per-GPU partition executor (include/pbdx.h).

``Partition`` owns one device's share of a Pipe-BD schedule: blocks
[block_lo, block_hi] of the CIFAR ResNet-18 teacher / slim student chain at a
shard of the global batch.  It exposes the three phases of Algorithm 1's
per-device body so that the multi-GPU driver (runtime.py)
can put the activation relay and the gradient allreduce between them, and
wraps the executor's device buffers as torch tensors (zero copy, through
``__cuda_array_interface__``) so torch.distributed/NCCL can move them.
"""
from __future__ import annotations

import ctypes
from typing import Dict, List, Optional, Tuple

import torch

from . import _lib

(BUF_INPUT, BUF_TEACHER_OUT, BUF_GRADS, BUF_PARAMS, BUF_MOMENTUM, BUF_LOSSES, BUF_STEP, BUF_TEACHER_PARAMS,
 BUF_MAILBOX) = range(9)
RELAY_MAX_PEERS = 16  # relay.hpp kRelayMaxPeers: mailbox = [ready x16 | consumed x16] uint64
BLOCKS = 4
T_CH = (3, 64, 128, 256, 512)
T_HW = (32, 32, 16, 8, 4)
STUDENT_TENSORS = ("w1", "w2", "wsc", "g1", "b1", "g2", "b2", "gsc", "bsc")


MODEL_RESNET_CIFAR, MODEL_MBV2_PROXYLESS, MODEL_EFFB0_PROXYLESS, MODEL_RESNET_CIFAR_FP32 = 0, 1, 2, 3
MODELS = {"resnet": MODEL_RESNET_CIFAR, "mbv2": MODEL_MBV2_PROXYLESS, "effb0": MODEL_EFFB0_PROXYLESS,
          "resnet_fp32": MODEL_RESNET_CIFAR_FP32}
RESNETS = ("resnet", "resnet_fp32")


class PbdxDesc(ctypes.Structure):
    _fields_ = [("block_lo", ctypes.c_int), ("block_hi", ctypes.c_int), ("n_max", ctypes.c_int),
                ("global_batch", ctypes.c_int), ("seed_data", ctypes.c_uint32), ("seed_teacher", ctypes.c_uint32),
                ("seed_student", ctypes.c_uint32), ("lr", ctypes.c_float), ("momentum", ctypes.c_float),
                ("model", ctypes.c_int), ("image", ctypes.c_int)]


class RelayMsg(ctypes.Structure):
    """pbdx_relay_msg (include/pbdx.h)."""
    _fields_ = [("src_row", ctypes.c_longlong), ("rows", ctypes.c_longlong), ("dst", ctypes.c_void_p),
                ("remote_flag", ctypes.c_void_p)]


def _bind(L):
    if getattr(L, "_pbdx_bound", False):
        return L
    V, I, P = ctypes.c_void_p, ctypes.c_int, ctypes.POINTER
    L.pbdx_create.argtypes = [P(PbdxDesc), P(V)]
    L.pbdx_destroy.argtypes = [V]
    L.pbdx_destroy.restype = None
    for name in ("pbdx_init_params", "pbdx_teacher_forward", "pbdx_student_step", "pbdx_apply_update", "pbdx_step",
                 "pbdx_capture", "pbdx_replay"):
        getattr(L, name).argtypes = [V, V]
    L.pbdx_capture_phases.argtypes = [V, I, V]
    L.pbdx_replay_phase.argtypes = [V, I, V]
    L.pbdx_set_shard.argtypes = [V, I, I]
    L.pbdx_set_input_mode.argtypes = [V, I]
    L.pbdx_upload_images.argtypes = [V, V, I, V]
    L.pbdx_stage_images.argtypes = [V, V, I, I, V]
    L.pbdx_buffer.argtypes = [V, I, P(V), P(ctypes.c_size_t)]
    L.pbdx_num_blocks.argtypes = [V]
    L.pbdx_teacher_act.argtypes = [V, I, P(V), P(ctypes.c_size_t)]
    L.pbdx_set_timing.argtypes = [V, I]
    L.pbdx_block_times.argtypes = [V, P(ctypes.c_float), P(ctypes.c_float)]
    L.pbdx_student_layout.argtypes = [I, P(ctypes.c_long)]
    L.pbdx_student_layout.restype = ctypes.c_long
    L.pbdx_student_layout_fp32.argtypes = [I, P(ctypes.c_long)]
    L.pbdx_student_layout_fp32.restype = ctypes.c_long
    L.pbdx_launches_per_step.argtypes = [V]
    L.pbdx_refresh_shadows.argtypes = [V, V]
    L.pbdx_relay_set_recv.argtypes = [V, I, P(V)]
    L.pbdx_relay_set_send.argtypes = [V, I, P(RelayMsg)]
    L.pbdx_ipc_export.argtypes = [V, ctypes.c_char_p]
    L.pbdx_ipc_open.argtypes = [ctypes.c_char_p, P(V)]
    L.pbdx_ipc_close.argtypes = [V]
    L.pbdx_set_path.argtypes = [V, I, P(I), I]
    L.pbdx_trace_mark.argtypes = [V, V]
    L.pbdx_set_train_mask.argtypes = [V, ctypes.c_uint]
    L.pbdx_dp_set_group.argtypes = [V, I, I, P(V), P(V)]
    L.pbdx_dp_set_params.argtypes = [V, I, P(V)]
    L.pbdx_dp_sync_state.argtypes = [V, V]
    L.pbdx_dp_peer_bytes.argtypes = [ctypes.c_longlong, I, I]
    L.pbdx_dp_peer_bytes.restype = ctypes.c_longlong
    L.pbdx_block_trace.argtypes = [V] + [P(ctypes.c_float)] * 4
    L.pbdx_mb_layers.argtypes = [I, I]
    L.pbdx_mb_candidates.argtypes = [I, I, I]
    L.pbdx_mb_candidate_offset.argtypes = [I, I, I, I, P(ctypes.c_long)]
    L.pbdx_mb_candidate_offset.restype = ctypes.c_long
    L.pbdx_mb_block_params.argtypes = [I, I]
    L.pbdx_mb_block_params.restype = ctypes.c_long
    L._pbdx_bound = True
    return L


def lib():
    return _bind(_lib.lib())


class DeviceError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc == 1:
        raise ValueError(f"{what}: invalid argument / unsupported shape")
    if rc != 0:
        raise DeviceError(f"{what}: CUDA error (rc={rc})")


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def student_layout(block: int, model: str = "resnet") -> Tuple[Dict[str, Tuple[int, int]], int]:
    """{tensor: (offset, count)} of a block's flat (padded) student parameters."""
    offs = (ctypes.c_long * 9)()
    total = (lib().pbdx_student_layout_fp32 if model == "resnet_fp32" else lib().pbdx_student_layout)(block, offs)
    if total < 0:
        raise ValueError("bad block")
    bounds = list(offs) + [total]
    return {name: (bounds[i], bounds[i + 1] - bounds[i]) for i, name in enumerate(STUDENT_TENSORS)}, total


def stored_channels(c: int, model: str = "resnet") -> int:
    """Stored channels of a ResNet activation (bf16: the image padded to 16; fp32: padded to 32 and
    kept split, [hi | lo], so the buffer holds twice this many fp32 values per pixel)."""
    if model == "resnet_fp32":
        return 32 if c == 3 else c
    return 16 if c == 3 else c


# ---------------------------------------------------------------- MobileNetV2 -> ProxylessNAS geometry
MB_CH = {"mbv2": (3, 32, 32, 64, 128, 192, 320), "effb0": (3, 32, 64, 128, 128, 192, 320)}
MB_DIV = (1, 4, 8, 16, 16, 32, 32)
MB_BLOCKS = 6


def mb_layers(block: int, model: str = "mbv2") -> int:
    return int(lib().pbdx_mb_layers(MODELS[model], block))


def mb_candidates(block: int, layer: int, model: str = "mbv2") -> int:
    return int(lib().pbdx_mb_candidates(MODELS[model], block, layer))


def mb_candidate_span(block: int, layer: int, cand: int, model: str = "mbv2") -> Tuple[int, int]:
    """(offset inside the block's flat supernet parameters, count) of one candidate."""
    n = ctypes.c_long()
    off = lib().pbdx_mb_candidate_offset(MODELS[model], block, layer, cand, ctypes.byref(n))
    if off < 0:
        raise ValueError("bad (block, layer, candidate)")
    return int(off), int(n.value)


def mb_block_params(block: int, model: str = "mbv2") -> int:
    return int(lib().pbdx_mb_block_params(MODELS[model], block))


class Partition:
    """One device's share of a Pipe-BD schedule.  model: "resnet" (CIFAR ResNet-18 -> slim residual
    student, 4 blocks, 32x32, bf16), "resnet_fp32" (the same in fp32: 3xTF32 tensor-core convolutions,
    configs[0]) or "mbv2" / "effb0" (MobileNetV2 / EfficientNet-B0 -> ProxylessNAS supernet, 6 blocks)."""

    def __init__(self, block_lo: int, block_hi: int, n_max: int, global_batch: int, seed_data: int = 1234,
                 seed_teacher: int = 1, seed_student: int = 2, lr: float = 0.1, momentum: float = 0.9,
                 device: Optional[torch.device] = None, model: str = "resnet", image: Optional[int] = None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.block_lo, self.block_hi, self.n_max, self.global_batch = block_lo, block_hi, n_max, global_batch
        self.model = model
        self.image = image if image is not None else (32 if model in RESNETS else 224)
        self.act_dtype = torch.float32 if model == "resnet_fp32" else torch.bfloat16
        self.n = n_max
        self.first = 0
        d = PbdxDesc(block_lo, block_hi, n_max, global_batch, seed_data, seed_teacher, seed_student, lr, momentum,
                     MODELS[model], self.image)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib().pbdx_create(ctypes.byref(d), ctypes.byref(h)), "pbdx_create")
        self.handle = h
        self.blocks = list(range(block_lo, block_hi + 1))
        self.layouts = {}
        off = 0
        for k in self.blocks:
            if model in RESNETS:
                lay, total = student_layout(k, model)
            else:
                lay, total = {}, mb_block_params(k, model)
            self.layouts[k] = (off, lay, total)
            off += total

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().pbdx_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.handle = None

    # -- plumbing
    def _stream(self, stream=None) -> ctypes.c_void_p:
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def buffer_ptr(self, which: int) -> Tuple[int, int]:
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().pbdx_buffer(self.handle, which, ctypes.byref(p), ctypes.byref(n)), "pbdx_buffer")
        return p.value, n.value

    def tensor(self, which: int, shape=None, dtype=torch.float32) -> torch.Tensor:
        ptr, nbytes = self.buffer_ptr(which)
        typestr = {torch.float32: "<f4", torch.bfloat16: "<V2", torch.float64: "<f8", torch.int64: "<i8"}[dtype]
        itemsize = torch.empty((), dtype=dtype).element_size()
        shape = shape or (nbytes // itemsize,)
        if dtype == torch.bfloat16:
            raw = torch.as_tensor(_CudaArray(ptr, tuple(shape), "<i2"), device=self.device)
            return raw.view(torch.bfloat16)
        return torch.as_tensor(_CudaArray(ptr, tuple(shape), typestr), device=self.device)

    # -- views the driver moves with NCCL
    def input_act(self) -> torch.Tensor:
        return self.tensor(BUF_INPUT, (self.n_max,) + self.act_hwc(self.block_lo), self.act_dtype)

    def teacher_out(self) -> torch.Tensor:
        return self.tensor(BUF_TEACHER_OUT, (self.n_max,) + self.act_hwc(self.block_hi + 1), self.act_dtype)

    def teacher_act(self, k: int) -> torch.Tensor:
        """Teacher output t_k of a block inside the partition (NHWC, n_max rows; bf16, or split fp32
        [..., hi | lo] for resnet_fp32 — see value())."""
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().pbdx_teacher_act(self.handle, k, ctypes.byref(p), ctypes.byref(n)), "pbdx_teacher_act")
        shape = (self.n_max,) + self.act_hwc(k + 1)
        if self.act_dtype == torch.float32:
            return torch.as_tensor(_CudaArray(p.value, shape, "<f4"), device=self.device)
        return torch.as_tensor(_CudaArray(p.value, shape, "<i2"), device=self.device).view(torch.bfloat16)

    def value(self, act: torch.Tensor) -> torch.Tensor:
        """fp32 values of an activation view: bf16 widened, split fp32 [..., hi | lo] summed (exact)."""
        if self.act_dtype == torch.float32:
            c = act.shape[-1] // 2
            return act[..., :c] + act[..., c:]
        return act.float()

    def set_path(self, block: int, path):
        """Active candidate per student layer of `block` (mbv2 supernet)."""
        arr = (ctypes.c_int * len(path))(*[int(c) for c in path])
        _check(lib().pbdx_set_path(self.handle, block, arr, len(path)), "set_path")
        self.paths = getattr(self, "paths", {})
        self.paths[block] = [int(c) for c in path]

    def grads(self) -> torch.Tensor:
        return self.tensor(BUF_GRADS)

    def params(self) -> torch.Tensor:
        return self.tensor(BUF_PARAMS)

    def momentum(self) -> torch.Tensor:
        """fp32 momentum.  In a DP group it is sharded by the exchange: completed from the peers first."""
        if getattr(self, "_dp", False):
            self.dp_sync_state()
            torch.cuda.synchronize(self.device)
        return self.tensor(BUF_MOMENTUM)

    def losses_tensor(self) -> torch.Tensor:
        return self.tensor(BUF_LOSSES, (len(self.blocks),), torch.float64)

    def step_counter(self) -> torch.Tensor:
        return self.tensor(BUF_STEP, (1,), torch.int64)

    def block_params(self, k: int, which: str = "params") -> Dict[str, torch.Tensor]:
        base, lay, _ = self.layouts[k]
        flat = {"params": self.params, "grads": self.grads, "momentum": self.momentum}[which]()
        return {name: flat[base + o: base + o + n] for name, (o, n) in lay.items()}

    # -- geometry of block boundaries (boundary 0 = the stored 16-channel image)
    def act_hwc(self, boundary: int) -> Tuple[int, int, int]:
        if self.model in RESNETS:
            split = 2 if self.model == "resnet_fp32" else 1
            return T_HW[boundary], T_HW[boundary], split * stored_channels(T_CH[boundary], self.model)
        hw = self.image // MB_DIV[boundary]
        return hw, hw, 16 if boundary == 0 else MB_CH[self.model][boundary]

    # -- K11 peer relay (include/pbdx.h): device pointers of this rank's relay endpoints
    def row_bytes_in(self) -> int:
        h, w, c = self.act_hwc(self.block_lo)
        return h * w * c * self.act_dtype.itemsize

    def row_bytes_out(self) -> int:
        h, w, c = self.act_hwc(self.block_hi + 1)
        return h * w * c * self.act_dtype.itemsize

    def mailbox_ptr(self) -> int:
        return self.buffer_ptr(BUF_MAILBOX)[0]

    def input_ptr(self) -> int:
        return self.buffer_ptr(BUF_INPUT)[0]

    def relay_set_recv(self, remote_consumed_flags: List[int]):
        arr = (ctypes.c_void_p * max(1, len(remote_consumed_flags)))(*remote_consumed_flags)
        _check(lib().pbdx_relay_set_recv(self.handle, len(remote_consumed_flags), arr), "relay_set_recv")

    def relay_set_send(self, msgs: List[Tuple[int, int, int, int]]):
        """msgs: (src_row, rows, dst device pointer, remote ready-flag pointer)."""
        arr = (RelayMsg * max(1, len(msgs)))(*[RelayMsg(a, b, c, d) for a, b, c, d in msgs])
        _check(lib().pbdx_relay_set_send(self.handle, len(msgs), arr), "relay_set_send")

    # -- phases of Algorithm 1
    def init_params(self, stream=None):
        _check(lib().pbdx_init_params(self.handle, self._stream(stream)), "init_params")

    def set_shard(self, n: int, first: int):
        _check(lib().pbdx_set_shard(self.handle, n, first), "set_shard")
        self.n, self.first = n, first

    def set_external_input(self, external):
        """False/0 synthetic (Philox on device), True/1 upload_images, 2 staged double buffer (stage_images)."""
        _check(lib().pbdx_set_input_mode(self.handle, int(external)), "set_input_mode")

    def stage_images(self, host: torch.Tensor, slot: int, stream=None):
        """Input mode 2: copy a step's host images (pinned fp32 NHWC) into staging slot 0/1 on `stream`;
        the step packs slot (step counter & 1)."""
        assert host.dtype == torch.float32 and not host.is_cuda and host.is_contiguous()
        _check(lib().pbdx_stage_images(self.handle, ctypes.c_void_p(host.data_ptr()), host.shape[0], int(slot),
                                       self._stream(stream)), "stage_images")

    def upload_images(self, host: torch.Tensor, stream=None):
        """host: fp32 NHWC [n, S, S, 3] (pinned for an async copy)."""
        assert host.dtype == torch.float32 and not host.is_cuda and host.is_contiguous()
        _check(lib().pbdx_upload_images(self.handle, ctypes.c_void_p(host.data_ptr()), host.shape[0],
                                        self._stream(stream)), "upload_images")

    def teacher_forward(self, stream=None):
        _check(lib().pbdx_teacher_forward(self.handle, self._stream(stream)), "teacher_forward")

    def student_step(self, stream=None):
        _check(lib().pbdx_student_step(self.handle, self._stream(stream)), "student_step")

    def apply_update(self, stream=None):
        _check(lib().pbdx_apply_update(self.handle, self._stream(stream)), "apply_update")

    def step(self, stream=None):
        _check(lib().pbdx_step(self.handle, self._stream(stream)), "step")

    def capture(self, stream=None):
        _check(lib().pbdx_capture(self.handle, self._stream(stream)), "capture")

    def replay(self, stream=None):
        _check(lib().pbdx_replay(self.handle, self._stream(stream)), "replay")

    def capture_phases(self, fuse_teacher_student: bool = False, stream=None):
        """Capture teacher_forward / student_step / apply_update as three CUDA graphs (phase 0 holds
        both forward phases when fuse_teacher_student)."""
        _check(lib().pbdx_capture_phases(self.handle, int(fuse_teacher_student), self._stream(stream)),
               "capture_phases")
        self._phased = True

    def replay_phase(self, phase: int, stream=None):
        _check(lib().pbdx_replay_phase(self.handle, phase, self._stream(stream)), "replay_phase")

    def set_timing(self, on: bool):
        _check(lib().pbdx_set_timing(self.handle, int(on)), "set_timing")

    def block_times(self) -> Tuple[List[float], List[float]]:
        nb = len(self.blocks)
        t, s = (ctypes.c_float * nb)(), (ctypes.c_float * nb)()
        _check(lib().pbdx_block_times(self.handle, t, s), "block_times")
        return list(t), list(s)

    def dp_set_group(self, me: int, peer_grads: List[int], peer_mailboxes: List[int],
                     peer_params: Optional[List[int]] = None):
        """DP group over peer memory (include/pbdx.h pbdx_dp_set_group / pbdx_dp_set_params): member pointers
        in member order.  The exchange is a reduce-scatter + all-gather, so groups of size > 1 also need
        every member's master-weight buffer (peer_params)."""
        n = len(peer_grads)
        g = (ctypes.c_void_p * n)(*[p or 0 for p in peer_grads])
        m = (ctypes.c_void_p * n)(*[p or 0 for p in peer_mailboxes])
        _check(lib().pbdx_dp_set_group(self.handle, n, me, g, m), "dp_set_group")
        if n > 1:
            if peer_params is None:
                raise ValueError("dp group of size > 1 needs peer_params")
            pp = (ctypes.c_void_p * n)(*[p or 0 for p in peer_params])
            _check(lib().pbdx_dp_set_params(self.handle, n, pp), "dp_set_params")
        self._dp = n > 1

    def params_ptr(self) -> int:
        return self.buffer_ptr(BUF_PARAMS)[0]

    def dp_sync_state(self, stream=None):
        """Complete the DP-sharded momentum (and weights) from the slice owners (before reading state)."""
        _check(lib().pbdx_dp_sync_state(self.handle, self._stream(stream)), "dp_sync_state")

    def grads_ptr(self) -> int:
        return self.buffer_ptr(BUF_GRADS)[0]

    def set_train_mask(self, mask: int):
        """Bit i = student block block_lo + i trains (DP-baseline mode trains one block of [0, k])."""
        _check(lib().pbdx_set_train_mask(self.handle, int(mask)), "set_train_mask")

    def trace_mark(self, stream=None):
        """Reference event for block_trace (measured timelines)."""
        _check(lib().pbdx_trace_mark(self.handle, self._stream(stream)), "trace_mark")

    def block_trace(self):
        """(teacher start, teacher end, student start, student end) per block of the last timed step,
        ms relative to the last trace_mark."""
        nb = len(self.blocks)
        arrs = [(ctypes.c_float * nb)() for _ in range(4)]
        _check(lib().pbdx_block_trace(self.handle, *arrs), "block_trace")
        return tuple(list(a) for a in arrs)

    def launches_per_step(self) -> int:
        return int(lib().pbdx_launches_per_step(self.handle))

    def losses(self) -> List[float]:
        return self.losses_tensor().cpu().tolist()

    # -- state migration (runtime.PipeBD.migrate)
    def block_state(self, k: int) -> List[torch.Tensor]:
        """[weights, momentum] of student block k (fp32, padded layout) — views into device memory (momentum()
        completes a DP-sharded momentum first)."""
        base, _, total = self.layouts[k]
        return [self.params()[base:base + total], self.momentum()[base:base + total]]

    def block_state_like(self, k: int) -> List[torch.Tensor]:
        """Receive buffers for any block's state (owned by this partition or not)."""
        total = student_layout(k, self.model)[1] if self.model in RESNETS else mb_block_params(k, self.model)
        return [torch.empty(total, dtype=torch.float32, device=self.device) for _ in range(2)]

    def set_block_state(self, k: int, weights: torch.Tensor, momentum: torch.Tensor):
        """Overwrite block k's master weights and momentum, then refresh the bf16 shadows (an SGD
        launch with zero gradient and lr 0 is an exact cast)."""
        w, v = self.block_state(k)
        w.copy_(weights)
        v.copy_(momentum)
        self.grads().zero_()
        self._refresh_shadows()

    def _refresh_shadows(self):
        _check(lib().pbdx_refresh_shadows(self.handle, self._stream(None)), "refresh_shadows")

    def step_index(self) -> int:
        return int(self.step_counter().item())

    def set_step_index(self, step: int):
        self.step_counter().fill_(int(step))


# ---------------------------------------------------------------- CUDA IPC of relay endpoints
def ipc_export(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(lib().pbdx_ipc_export(ctypes.c_void_p(ptr), buf), "ipc_export")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check(lib().pbdx_ipc_open(ctypes.c_char_p(handle), ctypes.byref(p)), "ipc_open")
    return p.value


def ipc_close(ptr: int):
    _check(lib().pbdx_ipc_close(ctypes.c_void_p(ptr)), "ipc_close")
