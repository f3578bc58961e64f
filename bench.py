#!/usr/bin/env python
"""Blockwise-distillation throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W]          # our sm_100a path
  python bench.py --impl reference [...]                    # CPU reference arm

Workload (BASELINE.json configs[1]): CIFAR-shaped 32x32 synthetic data,
ResNet-18-CIFAR 4-block teacher -> slim residual student, bf16 operands / fp32
accumulation and master weights, global batch 256 per GPU.  At N=1 the whole
chain runs on one GPU (the IR point of the AHD space, schedule.cpp:305-317).
Under torchrun (N>1) every rank runs the schedule best_schedule() picks on a
device-measured profile (weak scaling: global batch 256*N), with K11 peer-memory
relays between pipeline stages (--relay nccl: NCCL send/recv) and the DP exchange
as a reduce-scatter + all-gather over peer memory fused into the update (runtime.py).

One JSON line on rank 0; see DESIGN.md §5 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "blockwise-distill samples/sec"
TF32_PEAK_TFLOPS = 1100.0  # nominal dense tf32 (B200_PROFILING.md); not in MEASURED_PEAKS.json
UNIT = "samples/s"
PER_GPU_BATCH = 256


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 1000 for the ~1 ms CIFAR step so the clock sampler sees the "
                         "timed region, 300 for the MBConv workloads, 20 for --impl reference)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=None, help="global batch per GPU (default 256; cifar_fp32: 64)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=["cifar", "cifar_fp32", "mbv2", "effb0"], default="cifar",
                    help="cifar: configs[1] (headline, bf16); cifar_fp32: configs[0] (the same chain in fp32, batch "
                         "64, 3xTF32 tensor-core convolutions); mbv2: configs[2] MobileNetV2 -> ProxylessNAS at "
                         "224x224; effb0: configs[3] EfficientNet-B0 -> ProxylessNAS")
    ap.add_argument("--image", type=int, default=224, help="mbv2 image side")
    ap.add_argument("--relay", choices=["peer", "nccl"], default="peer",
                    help="N>1 teacher-activation relay: K11 peer stores over NVLink (default) or NCCL send/recv")
    ap.add_argument("--no-ahd", action="store_true",
                    help="N>1: search only contiguous one-group-per-partition schedules (pure pipeline)")
    ap.add_argument("--no-baselines", action="store_true",
                    help="N>1: skip the measured DP / LS baselines (runtime.run_baseline)")
    ap.add_argument("--pipeline", action="store_true",
                    help="use the multi-GPU runtime (profile -> best_schedule -> PipeBD) even at N=1")
    args = ap.parse_args()
    if args.batch is None:
        args.batch = 64 if args.workload == "cifar_fp32" else PER_GPU_BATCH
    if args.steps is None:
        args.steps = 20 if args.impl == "reference" else (1000 if args.workload.startswith("cifar") else 300)
    return args


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- roofline helpers
def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def ncu_traffic(kernel_key):
    """DRAM bytes per launch for the dominant kernel from the committed ncu capture (or None)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return d.get("kernels", {}).get(kernel_key, {}).get("dram_bytes")


def time_dominant_kernel(torch, batch):
    """CUDA-event timing of the dominant kernel (teacher block-0 3x3 conv, 64->64 @32x32 with the
    bias+ReLU epilogue, tcgen05 — the single conv shape with the largest time per step, 4 launches)
    launched alone with the step's own plan settings (two epilogue warps per TMEM lane quarter, the
    ResNet executor's ConvGridScope): 50 back-to-back launches replayed from a CUDA graph on the
    current stream (so host-side plan building and ctypes overhead stay out of the device timing);
    algorithmic FLOPs = 2*M*N*K."""
    import ctypes
    from paper_2301_12443_b200 import _lib
    L = _lib.lib()
    L.pbdk_conv_scope.argtypes = [ctypes.c_int, ctypes.c_int]
    L.pbdk_conv_scope.restype = None
    L.pbdk_conv_scope(0, 2)
    d = _lib.ConvDesc(batch, 32, 32, 64, 64, 3, 3, 1, 1, 32, 32)
    x = torch.randn(batch, 32, 32, 64, device="cuda").bfloat16()
    w = (torch.randn(64, 3, 3, 64, device="cuda") * 0.05).bfloat16()
    bias = torch.zeros(64, device="cuda")
    y = torch.empty(batch, 32, 32, 64, device="cuda", dtype=torch.bfloat16)
    reps = 50

    def launch():
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        rc = L.pbdk_conv_fprop(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), bias.data_ptr(), None, 2, s)
        assert rc == 0

    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            launch()
    g.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    L.pbdk_conv_scope(0, 0)
    flops = 2.0 * batch * 32 * 32 * 64 * 9 * 64
    return "conv_fprop_bn64_bkc64", flops, ms


def time_dominant_kernel_fp32(torch, batch):
    """configs[0]: the same dominant conv (teacher block-0 3x3, 64->64 @32x32, bias+ReLU) in fp32 as
    3xTF32 on the tensor cores (split operands, split output), 50 launches from a CUDA graph.
    Algorithmic FLOPs = 2*M*N*K; the tensor cores execute 3x that (three tf32 MMAs per product)."""
    import ctypes
    from paper_2301_12443_b200 import _lib
    L = _lib.lib()
    d = _lib.ConvDesc(batch, 32, 32, 64, 64, 3, 3, 1, 1, 32, 32)
    x = torch.randn(batch, 32, 32, 128, device="cuda")
    w = torch.randn(64, 3, 3, 128, device="cuda") * 0.05
    bias = torch.zeros(64, device="cuda")
    y = torch.empty(batch, 32, 32, 128, device="cuda")
    reps = 50

    def launch():
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        rc = L.pbdk_conv3x_fprop(ctypes.byref(d), x.data_ptr(), w.data_ptr(), y.data_ptr(), 1, bias.data_ptr(), None,
                                 2, s)
        assert rc == 0

    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            launch()
    g.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 2.0 * batch * 32 * 32 * 64 * 9 * 64
    return "conv3x_fprop_bn64_ck32", flops, ms


# ---------------------------------------------------------------- CPU legs
def cpu_oracle_rate(samples_per_step=256, budget_s=15.0, max_steps=16, bf16_mode=1):
    """The oracle (C restatement, OpenMP) on the host cores: samples/s over as many whole steps as fit
    in about `budget_s` seconds of CPU work (bounded sample of the same workload)."""
    from oracle import bd
    tr = bd.Trainer(samples_per_step, bf16_mode=bf16_mode)
    tr.step(0)  # warm (allocation, page faults)
    t0 = time.perf_counter()
    steps = 0
    while steps < max_steps and (steps < 2 or time.perf_counter() - t0 < budget_s):
        tr.step(1 + steps)
        steps += 1
    dt = time.perf_counter() - t0
    return samples_per_step * steps / dt, bd.lib().bdo_threads(), dt, steps


def run_reference(args, rank, world):
    """--impl reference: the CPU implementation of the path on the host cores, same metric, config and
    global batch as our arm.  The reference itself has no executable distillation step, so
    this is the oracle port (oracle/bd_oracle.c, OpenMP over every host core): each step is one whole
    global batch (256 samples per GPU, all 4 blocks, teacher fwd + student fwd/bwd + SGD).  The run is
    bounded: after one warm-up step, steps are timed until `--steps` are done or ~150 s of CPU time
    elapsed (min 2), and the line says how many ran.  Only oracle/ libraries are loaded here (no repo
    product .so); the reference's own partitioner (oracle/_ref, compiled unmodified) is timed beside it."""
    if rank != 0:
        return
    from oracle import bd
    gb = args.batch * max(1, args.gpus)
    fp32 = args.workload == "cifar_fp32"
    tr = bd.Trainer(gb, bf16_mode=0 if fp32 else 1)
    warm = min(args.warmup, 1)
    for w in range(warm):
        tr.step(w)
    budget_s = float(os.environ.get("PBD_REF_BUDGET_S", "150"))
    t0 = time.perf_counter()
    done = 0
    while done < args.steps and (done < 2 or time.perf_counter() - t0 < budget_s):
        tr.step(warm + done)
        done += 1
    dt = time.perf_counter() - t0
    rate = gb * done / dt
    threads = bd.lib().bdo_threads()
    sample = f"{done} whole steps of the {gb}-sample global batch (all 4 blocks, fwd+bwd+SGD), {dt:.1f} s"
    line = {"metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": done, "warmup": warm, "ms_per_step": dt / done * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp32" if fp32 else "bf16-emulated fp32",
            "data": "synthetic (Philox4x32-10, DESIGN.md §3)",
            "config": {"workload": "cifar-resnet18-teacher/slim-student 4 blocks (%s)" % (
                           "configs[0], fp32" if fp32 else "configs[1]"),
                       "global_batch": gb, "image": "32x32x3", "blocks": 4, "parallelism": "cpu",
                       "steps_requested": args.steps, "warmup_requested": args.warmup,
                       "same_config": True},
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    try:
        from oracle import ref
        if ref.available():
            prof = ref.synth_profile(shape="front-heavy", blocks=10, front_weight=4.0, curvature=0.4,
                                     num_devices=8)
            line["partitioner"] = {"reference_best_schedule_ms": ref.time_best_schedule(prof, threads=1, reps=20),
                                   "case": "B=10 N=8 (11440 configs), reference core compiled unmodified"}
    except Exception as e:  # pragma: no cover - informational only
        line["partitioner"] = {"error": str(e)}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2301_12443_b200 import executor, models
    ngpu = max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank % ngpu)  # % ngpu: ranks may share a GPU (PBD_DIST_BACKEND=gloo runs)
    dev = torch.device("cuda", local_rank % ngpu)
    if world > 1 or args.pipeline:
        from paper_2301_12443_b200 import runtime
        with ClockSampler(local_rank) as clocks:
            res = runtime.bench_pipeline(args, rank, world, local_rank % ngpu)
        if rank == 0:
            res["clocks"] = clocks.summary()
            res["cpu_baseline"] = None
            print(json.dumps(res), flush=True)
        return

    if args.workload in ("mbv2", "effb0"):
        return run_ours_mbv2(args, dev, local_rank)

    b = args.batch
    fp32 = args.workload == "cifar_fp32"
    model = "resnet_fp32" if fp32 else "resnet"
    part = executor.Partition(0, 3, b, b, device=dev, model=model)
    part.init_params()
    stream = torch.cuda.current_stream(dev)
    use_graph = not args.no_graph
    if use_graph:
        part.capture()

    def one():
        (part.replay if use_graph else part.step)()

    for _ in range(max(3, args.warmup)):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            one()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    value = b / ms * 1e3
    losses = part.losses()

    # ---- e2e through the public API with host buffers: every step H2D of its images from pinned memory
    # (on a copy stream, into the staging slot the previous step is not reading — overlapped with the
    # previous step's compute), the step, and a D2H read of its losses (read on the host one step later)
    e2e_part = executor.Partition(0, 3, b, b, device=dev, model=model)
    e2e_part.init_params()
    e2e_part.set_external_input(2)
    host = torch.empty(b, 32, 32, 3, dtype=torch.float32).pin_memory()
    host.uniform_(-1.0, 1.0)
    copy_stream = torch.cuda.Stream(dev)
    parity0 = int(e2e_part.step_counter().item()) & 1
    if use_graph:
        e2e_part.capture()
    loss_host = [torch.empty(4, dtype=torch.float64).pin_memory() for _ in range(2)]
    lt = e2e_part.losses_tensor()
    ev_copy = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    seen = []

    def run_e2e(nsteps):
        e2e_part.stage_images(host, parity0, stream)  # the first step's images
        ev_copy[parity0].record(stream)
        for s_ in range(nsteps):
            cur, nxt = (parity0 + s_) & 1, (parity0 + s_ + 1) & 1
            if s_ + 1 < nsteps:  # next step's images into the other slot, once step s-1 released it
                if s_ >= 1:
                    copy_stream.wait_event(ev_done[nxt])
                e2e_part.stage_images(host, nxt, copy_stream)
                ev_copy[nxt].record(copy_stream)
            stream.wait_event(ev_copy[cur])
            (e2e_part.replay if use_graph else e2e_part.step)(stream)
            loss_host[cur].copy_(lt, non_blocking=True)
            ev_done[cur].record(stream)
            if s_ >= 1:  # the host reads the previous step's losses
                ev_done[1 - cur].synchronize()
                seen.append(float(loss_host[1 - cur].sum()))
        ev_done[(parity0 + nsteps - 1) & 1].synchronize()
        seen.append(float(loss_host[(parity0 + nsteps - 1) & 1].sum()))

    run_e2e(3)
    torch.cuda.synchronize()
    parity0 = int(e2e_part.step_counter().item()) & 1
    t0 = time.perf_counter()
    run_e2e(args.steps)
    e2e_ms = (time.perf_counter() - t0) / args.steps * 1e3
    e2e = {"value": b / e2e_ms * 1e3, "unit": UNIT, "h2d_bytes_per_step": b * 32 * 32 * 3 * 4,
           "d2h_bytes_per_step": 32, "ms_per_step": e2e_ms,
           "note": "host wall clock; per step: pinned H2D of the step's images on a copy stream (double-buffered "
                   "staging, overlapped with the previous step), the step graph, D2H of the 4 block losses"}
    assert all(math.isfinite(x) for x in seen), seen
    del e2e_part

    # ---- roofline of the dominant kernel + step-level accounting
    peaks = measured_peaks()
    key, kflops, kms = (time_dominant_kernel_fp32 if fp32 else time_dominant_kernel)(torch, b)
    achieved = kflops / (kms * 1e-3) / 1e12
    traffic = ncu_traffic(key)
    if fp32:  # no measured tf32 figure: the nominal dense tf32 peak (B200_PROFILING.md), 3 MMAs per product
        roof = {"bound": "tensor", "kernel": key, "achieved": 3 * achieved, "peak": TF32_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": 3 * achieved / TF32_PEAK_TFLOPS, "traffic": traffic,
                "launch_us": kms * 1e3, "algorithmic_tflops": achieved,
                "peak_source": "nominal dense tf32 (B200_PROFILING.md; MEASURED_PEAKS.json has no tf32 figure); "
                               "achieved counts the 3 tf32 MMAs per product of the 3xTF32 split"}
    else:
        roof = {"bound": "tensor", "kernel": key, "achieved": achieved, "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["bf16_tflops"], "traffic": traffic,
                "launch_us": kms * 1e3, "peak_source": peaks["source"] + " burst (kernel timed alone)"}
    from paper_2301_12443_b200 import models as _m
    sflops, sbytes = _m.step_flops(b), _m.step_bytes(b, act_bytes=4 if fp32 else 2)
    peak_t = (TF32_PEAK_TFLOPS / 3.0) if fp32 else peaks["bf16_tflops_sustained"]
    t_roof = max(sflops / (peak_t * 1e12), sbytes / (peaks["hbm_gbs"] * 1e9))
    step_roof = {"step_flops": sflops, "step_bytes": sbytes, "t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms,
                 "achieved_tflops": sflops / (ms * 1e-3) / 1e12,
                 "note": "algorithmic work (each tensor written + read once, weights once) / measured step; peak = " +
                         ("nominal tf32 / 3 (3xTF32)" if fp32 else "sustained bf16") + ", measured HBM"}

    # ---- the paper's DP baseline measured on the same GPU:
    # blocks trained one after another, every step recomputing the teacher prefix T_0..T_k
    dp_ms = []
    for k in range(4):
        dp = executor.Partition(0, k, b, b, device=dev, model=model)
        dp.init_params()
        dp.set_train_mask(1 << k)
        dp.capture()
        for _ in range(3):
            dp.replay()
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(10, args.steps // 4)
        d0.record(stream)
        for _ in range(reps):
            dp.replay()
        d1.record(stream)
        torch.cuda.synchronize()
        dp_ms.append(d0.elapsed_time(d1) / reps)
        del dp
    dp_line = {"per_block_step_ms": dp_ms, "all_blocks_ms": sum(dp_ms), "pipebd_step_ms": ms,
               "speedup": sum(dp_ms) / ms,
               "note": "time to train every block for one step of data: DP baseline (sequential blocks, teacher "
                       "prefix recomputed) vs Pipe-BD's single pass (teacher relayed once) on 1 GPU"}

    cpu = None
    if not args.no_cpu_baseline:
        rate, cores, dt, nsteps = cpu_oracle_rate(b, bf16_mode=0 if fp32 else 1)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{nsteps} whole steps of the same {b}-sample batch (oracle/bd_oracle.c, {dt:.1f} s)"}

    working_set = models.step_working_set_bytes(b) * (3 if fp32 else 1)  # fp32: ~2x bytes, split operands 2x again
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp32" if fp32 else "bf16",
            "data": "synthetic (Philox4x32-10 inputs generated on device each step; random-init weights)",
            "config": {"workload": "cifar-resnet18-teacher/slim-student 4 blocks, IR point on 1 GPU (%s)" % (
                           "configs[0]: fp32, 3xTF32 tensor-core convolutions" if fp32 else "configs[1]"),
                       "global_batch": b, "image": "32x32x3", "blocks": 4, "parallelism": "ir1 (blocks 0-3 on 1 GPU)",
                       "cuda_graph": use_graph,
                       "l2": f"no flush: per-step working set {working_set / 2**30:.2f} GiB > 126 MB L2"},
            "e2e": e2e, "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu,
            "dp_baseline_measured": dp_line,
            "gpu_launches": part.launches_per_step() * args.steps, "clocks": clocks.summary(),
            "losses_last_step": losses}
    print(json.dumps(line), flush=True)


def run_ours_mbv2(args, dev, local_rank):
    """configs[2]: MobileNetV2 teacher -> ProxylessNAS supernet student, 6 blocks, 224x224, all blocks on
    one GPU (the IR point); the seeded single path of epoch 0 (draw 0) is active, graph replay."""
    import torch
    from paper_2301_12443_b200 import executor, mb_models
    b, S, model = args.batch, args.image, args.workload
    mb_models.set_family(model)
    paths = mb_models.paths_for(0)
    part = executor.Partition(0, 5, b, b, device=dev, model=model, image=S)
    part.init_params()
    for k in range(6):
        part.set_path(k, paths[k])
    stream = torch.cuda.current_stream(dev)
    part.capture()
    for _ in range(max(3, args.warmup)):
        part.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            part.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    losses = part.losses()
    # e2e: every step's fp32 images H2D from pinned memory on a copy stream into the staging slot the
    # running step is not reading (overlapped), the step graph, D2H of the 6 block losses (host clock)
    part.set_external_input(2)
    host = torch.empty(b, S, S, 3, dtype=torch.float32).pin_memory().uniform_(-1.0, 1.0)
    part.capture()
    lt = part.losses_tensor()
    loss_host = [torch.empty(6, dtype=torch.float64).pin_memory() for _ in range(2)]
    copy_stream = torch.cuda.Stream(dev)
    ev_copy = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]

    def run_e2e(nsteps):
        p0 = int(part.step_counter().item()) & 1
        part.stage_images(host, p0, stream)
        ev_copy[p0].record(stream)
        for s_ in range(nsteps):
            cur, nxt = (p0 + s_) & 1, (p0 + s_ + 1) & 1
            if s_ + 1 < nsteps:
                if s_ >= 1:
                    copy_stream.wait_event(ev_done[nxt])
                part.stage_images(host, nxt, copy_stream)
                ev_copy[nxt].record(copy_stream)
            stream.wait_event(ev_copy[cur])
            part.replay(stream)
            loss_host[cur].copy_(lt, non_blocking=True)
            ev_done[cur].record(stream)
            if s_ >= 1:
                ev_done[1 - cur].synchronize()
        torch.cuda.synchronize()

    run_e2e(2)
    n_e2e = max(3, args.steps // 4)
    t0 = time.perf_counter()
    run_e2e(n_e2e)
    e2e_ms = (time.perf_counter() - t0) / n_e2e * 1e3
    # ProxylessNAS step (nas.py): architecture round + weight round, paths resampled from softmax(alpha)
    # every round (eager launches: a new path invalidates the captured graphs), host alpha update
    from paper_2301_12443_b200 import nas
    part.set_external_input(0)
    arch = nas.ArchParams(range(6))
    for s_ in range(2):
        nas.nas_step(part, arch, s_)
    torch.cuda.synchronize()
    n_nas = 10
    t0 = time.perf_counter()
    for s_ in range(n_nas):
        nas.nas_step(part, arch, 2 + s_)
    torch.cuda.synchronize()
    nas_ms = (time.perf_counter() - t0) / n_nas * 1e3
    nas_line = {"ms_per_step": nas_ms, "samples_per_s": b / nas_ms * 1e3, "rounds": 2, "steps": n_nas,
                "alpha_entropy": [round(arch.entropy(k), 4) for k in range(6)],
                "note": "host wall clock; one NAS step = teacher fwd + architecture round (student fwd/bwd, "
                        "REINFORCE alpha update from the block losses) + weight round (student fwd/bwd + SGD), "
                        "paths ~ softmax(alpha) each round, eager launches"}
    peaks = measured_peaks()
    flops, nbytes = mb_models.step_work(b, S, paths)
    t_roof = max(flops / (peaks["bf16_tflops_sustained"] * 1e12), nbytes / (peaks["hbm_gbs"] * 1e9))
    achieved = nbytes / (ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": "whole step (HBM-bound: arithmetic intensity %.1f flop/B)" % (flops / nbytes),
            "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
            "traffic": None, "step_bytes": nbytes, "step_flops": flops, "t_roof_ms": t_roof * 1e3,
            "peak_source": peaks["source"]}
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import mb
        mb.set_family(1 if model == "effb0" else 0)
        tr = mb.Trainer(1, S)
        tr.step(0, paths)
        t0 = time.perf_counter()
        nsteps = 0
        while nsteps < 200 and (nsteps < 2 or time.perf_counter() - t0 < 10.0):  # ~10 s bounded sample
            tr.step(1 + nsteps, paths)
            nsteps += 1
        dt = time.perf_counter() - t0
        cpu = {"value": nsteps / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"1 sample x {nsteps} steps, all 6 blocks (oracle/mb_oracle.c, {dt:.1f} s)"}
    line = {"metric": METRIC, "value": b / ms * 1e3, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (Philox4x32-10 images on device each step; random-init weights)",
            "config": {"workload": ("MobileNetV2-1.0 teacher (true widths 24/32/64/96/160/320, stored zero-padded "
                                    "to tile multiples) / ProxylessNAS supernet, 6 blocks, IR point on 1 GPU "
                                    "(configs[2])"
                                    if model == "mbv2" else
                                    "EfficientNet-B0 teacher (swish, SE; true widths 24/40/80/112/192/320, stored "
                                    "zero-padded) / ProxylessNAS supernet, 6 blocks, IR point on 1 GPU (configs[3])"),
                       "global_batch": b, "image": f"{S}x{S}x3", "blocks": 6, "paths": paths,
                       "parallelism": "ir1 (blocks 0-5 on 1 GPU)", "cuda_graph": True,
                       "l2": "no flush: per-step working set > 20 GiB >> 126 MB L2"},
            "e2e": {"value": b / e2e_ms * 1e3, "unit": UNIT, "h2d_bytes_per_step": b * S * S * 3 * 4,
                    "d2h_bytes_per_step": 48, "ms_per_step": e2e_ms},
            "roofline": roof, "cpu_baseline": cpu, "gpu_launches": part.launches_per_step() * args.steps,
            "clocks": clocks.summary(), "losses_last_step": losses, "nas_step": nas_line}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
