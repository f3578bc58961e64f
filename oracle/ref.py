"""TEST INFRASTRUCTURE ONLY — ctypes face of oracle/_ref/libpbd_ref.so.

That library is the reference's own core (proj/core/src/*.cpp, unmodified)
compiled by oracle/Makefile plus ref_shim.cpp.  Only tests/, smoke() and
bench.py's cpu_baseline / --impl reference legs may use it, as the checker.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libpbd_ref.so")

_L = None
V = ctypes.c_void_p


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _L
    if _L is None:
        L = ctypes.CDLL(REF_LIB)
        P = ctypes.POINTER
        L.ref_free.argtypes = [V]
        L.ref_enumerate_count.argtypes = [ctypes.c_int, ctypes.c_int]
        L.ref_enumerate_count.restype = ctypes.c_long
        L.ref_enumerate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P(V), P(V)]
        L.ref_exec_time.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, P(ctypes.c_double), P(V)]
        L.ref_best_schedule.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, P(V), P(V), P(V)]
        L.ref_time_best_schedule.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, P(ctypes.c_double), P(V)]
        L.ref_predicted_step_time.argtypes = [ctypes.c_char_p, ctypes.c_char_p, P(V), P(V)]
        L.ref_simulate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, P(V), P(V)]
        L.ref_reconfigure.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_double, P(V), P(V)]
        L.ref_profile_drift.argtypes = [ctypes.c_char_p, ctypes.c_char_p, P(ctypes.c_double), P(V)]
        L.ref_load_save_profile.argtypes = [ctypes.c_char_p, P(V), P(V)]
        L.ref_synth_profile.argtypes = [ctypes.c_char_p, P(V), P(V)]
        L.ref_report_render.argtypes = [ctypes.c_char_p, ctypes.c_char_p, P(V), P(V)]
        _L = L
    return _L


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _take(p):
    if not p:
        return ""
    s = ctypes.cast(p, ctypes.c_char_p).value.decode()
    lib().ref_free(p)
    return s


def _t(doc):
    return (doc if isinstance(doc, str) else json.dumps(doc)).encode()


def _chk(rc, err):
    if rc:
        raise RefError(rc, _take(err))


def enumerate_count(b, n):
    return lib().ref_enumerate_count(b, n)


def enumerate_configs(b, n, gb=0):
    out, err = V(), V()
    _chk(lib().ref_enumerate(b, n, gb, ctypes.byref(out), ctypes.byref(err)), err)
    return [l for l in _take(out).split("\n") if l]


def exec_time(profile, block, role, batch):
    d, err = ctypes.c_double(), V()
    _chk(lib().ref_exec_time(_t(profile), block, 0 if role == "teacher" else 1, batch, ctypes.byref(d),
                             ctypes.byref(err)), err)
    return d.value


def best_schedule(profile, contiguous_only=False, threads=0):
    out, meta, err = V(), V(), V()
    _chk(lib().ref_best_schedule(_t(profile), int(contiguous_only), threads, ctypes.byref(out), ctypes.byref(meta),
                                 ctypes.byref(err)), err)
    return json.loads(_take(out)), json.loads(_take(meta))


def time_best_schedule(profile, threads=1, reps=10):
    d, err = ctypes.c_double(), V()
    _chk(lib().ref_time_best_schedule(_t(profile), threads, reps, ctypes.byref(d), ctypes.byref(err)), err)
    return d.value


def predicted_step_time(profile, schedule):
    out, err = V(), V()
    _chk(lib().ref_predicted_step_time(_t(profile), _t(schedule), ctypes.byref(out), ctypes.byref(err)), err)
    return json.loads(_take(out))


def simulate(profile, schedule, sim=None):
    out, err = V(), V()
    _chk(lib().ref_simulate(_t(profile), _t(schedule), json.dumps(sim or {}).encode(), ctypes.byref(out),
                            ctypes.byref(err)), err)
    return json.loads(_take(out))


def reconfigure(profile, schedule, observed, threshold) -> Optional[dict]:
    out, err = V(), V()
    _chk(lib().ref_reconfigure(_t(profile), _t(schedule), _t(observed), float(threshold), ctypes.byref(out),
                               ctypes.byref(err)), err)
    s = _take(out)
    return json.loads(s) if s else None


def profile_drift(a, b):
    d, err = ctypes.c_double(), V()
    _chk(lib().ref_profile_drift(_t(a), _t(b), ctypes.byref(d), ctypes.byref(err)), err)
    return d.value


def load_save_profile(profile):
    out, err = V(), V()
    _chk(lib().ref_load_save_profile(_t(profile), ctypes.byref(out), ctypes.byref(err)), err)
    return _take(out)


def synth_profile(**spec):
    out, err = V(), V()
    _chk(lib().ref_synth_profile(json.dumps(spec).encode(), ctypes.byref(out), ctypes.byref(err)), err)
    return json.loads(_take(out))


def report_render(profile, sim=None):
    """speedup/breakdown tables (text, csv, json) + two gantt_svg renderings, "\n@@\n"-separated."""
    out, err = V(), V()
    _chk(lib().ref_report_render(_t(profile), json.dumps(sim or {}).encode(), ctypes.byref(out), ctypes.byref(err)),
         err)
    return _take(out)
