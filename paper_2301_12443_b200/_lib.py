"""ctypes binding of the in-tree product library ``lib/libpbd.so``.

There is deliberately no fallback: if the library is missing or was not built
for sm_100a the import fails loudly (the round-end driver checks which ``.so``
files the tests and the bench actually loaded).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PBD_LIB_VARIANT=exp loads the experiments build (make EXPERIMENTS=1 -> lib-exp/, A/B scripts only)
LIB_PATH = os.path.join(_HERE, "lib-exp" if os.environ.get("PBD_LIB_VARIANT") == "exp" else "lib", "libpbd.so")

c_int, c_long, c_double, c_size_t, c_void_p, c_char_p = (
    ctypes.c_int, ctypes.c_long, ctypes.c_double, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_char_p)
c_char_pp = ctypes.POINTER(ctypes.c_char_p)


class ConvDesc(ctypes.Structure):
    """pbdk_conv_desc (include/pbdk.h)."""
    _fields_ = [(n, c_int) for n in ("n", "h", "w", "c", "k", "r", "s", "stride", "pad", "p", "q")]


class FlipRegion(ctypes.Structure):
    """pbdk_flip_region (include/pbdk.h)."""
    _fields_ = [("off", c_size_t), ("k", c_int), ("r", c_int), ("s", c_int), ("c", c_int), ("dst", c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2301_12443_b200). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    # host core (include/pbd_capi.h)
    L.pbd_free.argtypes = [c_void_p]
    L.pbd_free.restype = None
    L.pbd_enumerate_count.argtypes = [c_int, c_int]
    L.pbd_enumerate_count.restype = c_long
    L.pbd_best_schedule.argtypes = [c_char_p, c_int, c_int, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p),
                                    ctypes.POINTER(c_void_p)]
    for name in ("pbd_predicted_step_time",):
        getattr(L, name).argtypes = [c_char_p, c_char_p, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p)]
    L.pbd_simulate.argtypes = [c_char_p, c_char_p, c_char_p, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p)]
    L.pbd_reconfigure.argtypes = [c_char_p, c_char_p, c_char_p, c_double, ctypes.POINTER(c_void_p),
                                  ctypes.POINTER(c_void_p)]
    L.pbd_profile_drift.argtypes = [c_char_p, c_char_p, ctypes.POINTER(c_double), ctypes.POINTER(c_void_p)]
    L.pbd_exec_time.argtypes = [c_char_p, c_int, c_int, c_int, ctypes.POINTER(c_double), ctypes.POINTER(c_void_p)]
    L.pbd_load_save_profile.argtypes = [c_char_p, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p)]
    L.pbd_synth_profile.argtypes = [c_char_p, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p)]
    L.pbd_shard_range.argtypes = [c_int, c_int, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]
    L.pbd_time_best_schedule.argtypes = [c_char_p, c_int, ctypes.POINTER(c_double), ctypes.POINTER(c_void_p)]
    L.pbd_baseline_plan.argtypes = [c_char_p, c_int, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p)]
    L.pbd_baseline_plan.restype = c_int
    for name in ("pbd_best_schedule", "pbd_predicted_step_time", "pbd_simulate", "pbd_reconfigure",
                 "pbd_profile_drift", "pbd_exec_time", "pbd_load_save_profile", "pbd_synth_profile",
                 "pbd_shard_range", "pbd_time_best_schedule"):
        getattr(L, name).restype = c_int
    # kernels (include/pbdk.h)
    L.pbdk_build_info.restype = c_char_p
    L.pbdk_conv_fprop.argtypes = [ctypes.POINTER(ConvDesc), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                  c_void_p]
    L.pbdk_conv_wgrad_workspace_bytes.argtypes = [ctypes.POINTER(ConvDesc)]
    L.pbdk_conv_wgrad_workspace_bytes.restype = c_size_t
    L.pbdk_conv_wgrad.argtypes = [ctypes.POINTER(ConvDesc), c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                  c_void_p]
    L.pbdk_weight_flip.argtypes = [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p]
    L.pbdk_conv3x_fprop.argtypes = [ctypes.POINTER(ConvDesc), c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                    c_int, c_void_p]
    L.pbdk_conv3x_wgrad_workspace_bytes.argtypes = [ctypes.POINTER(ConvDesc)]
    L.pbdk_conv3x_wgrad_workspace_bytes.restype = c_size_t
    L.pbdk_conv3x_wgrad.argtypes = [ctypes.POINTER(ConvDesc), c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                    c_void_p]
    L.pbdk_sgd_momentum.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, ctypes.c_float,
                                    ctypes.c_float, c_void_p, c_void_p]
    L.pbdk_sgd_momentum.restype = c_int
    L.pbdk_sgd_momentum_flip.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, ctypes.c_float,
                                         ctypes.c_float, c_void_p, ctypes.POINTER(FlipRegion), c_int, c_void_p]
    L.pbdk_sgd_momentum_flip.restype = c_int
    L.pbdk_split_tf32.argtypes = [c_void_p, c_void_p, c_size_t, c_int, c_void_p]
    L.pbdk_weight_flip_split.argtypes = [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p]
    for name in ("pbdk_conv_fprop", "pbdk_conv_wgrad", "pbdk_weight_flip", "pbdk_conv3x_fprop", "pbdk_conv3x_wgrad",
                 "pbdk_split_tf32", "pbdk_weight_flip_split"):
        getattr(L, name).restype = c_int
    _lib = L
    return L


def take_string(ptr: c_void_p) -> str:
    """Copy a malloc'ed C string returned by libpbd and free it."""
    if not ptr:
        return ""
    s = ctypes.cast(ptr, c_char_p).value.decode()
    lib().pbd_free(ptr)
    return s
