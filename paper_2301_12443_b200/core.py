"""Python face of the host-side Pipe-BD core (libpbd.so, include/pbd_capi.h).

Mirrors the reference C++ API of ``pbd::core`` (proj/core/include/pbd/*.hpp)
with the same operation names, argument meanings and error classes; documents
are the reference's JSON formats (profile: proj/README.md:141-162, schedule:
schedule.cpp:361-373, report: simulate.cpp:431-465).
"""
from __future__ import annotations

import ctypes
import json
from typing import Optional, Tuple, Union

from . import _lib

Doc = Union[str, dict]


class PbdError(RuntimeError):
    pass


class ValidationError(PbdError):
    """errors.hpp:23-26 — CLI exit code 1."""


class InfeasibleError(PbdError):
    """errors.hpp:29-32 — CLI exit code 2."""


class IoError(PbdError):
    """errors.hpp:35-38 — CLI exit code 3."""


_ERRORS = {1: ValidationError, 2: InfeasibleError, 3: IoError, 4: PbdError}


def _text(doc: Doc) -> bytes:
    return (doc if isinstance(doc, str) else json.dumps(doc)).encode()


def _check(rc: int, err: ctypes.c_void_p) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, PbdError)(_lib.take_string(err) or f"pbd error {rc}")


def enumerate_count(blocks: int, devices: int) -> int:
    """|enumerate_configs(B, N)| (schedule.cpp:115-134); -1 on invalid input."""
    return int(_lib.lib().pbd_enumerate_count(blocks, devices))


def best_schedule(profile: Doc, contiguous_only: bool = False, threads: int = 0) -> Tuple[dict, dict]:
    """AHD search (schedule.cpp:167-244). Returns (schedule document, provenance)."""
    out, meta, err = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    rc = _lib.lib().pbd_best_schedule(_text(profile), int(contiguous_only), threads, ctypes.byref(out),
                                      ctypes.byref(meta), ctypes.byref(err))
    _check(rc, err)
    return json.loads(_lib.take_string(out)), json.loads(_lib.take_string(meta))


def best_schedule_text(profile: Doc, contiguous_only: bool = False) -> str:
    out, meta, err = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    rc = _lib.lib().pbd_best_schedule(_text(profile), int(contiguous_only), 0, ctypes.byref(out), ctypes.byref(meta),
                                      ctypes.byref(err))
    _check(rc, err)
    _lib.take_string(meta)
    return _lib.take_string(out)


def baseline_plan(profile: Doc, kind: str) -> dict:
    """dp_schedule / ls_schedule (schedule.cpp:246-303) of a profile: the paper's DP and LS baselines."""
    out, err = ctypes.c_void_p(), ctypes.c_void_p()
    rc = _lib.lib().pbd_baseline_plan(_text(profile), {"dp": 0, "ls": 1}[kind], ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return json.loads(_lib.take_string(out))


def predicted_step_time(profile: Doc, schedule: Doc) -> dict:
    out, err = ctypes.c_void_p(), ctypes.c_void_p()
    rc = _lib.lib().pbd_predicted_step_time(_text(profile), _text(schedule), ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return json.loads(_lib.take_string(out))


def simulate(profile: Doc, schedule: Doc, sim: Optional[dict] = None) -> dict:
    out, err = ctypes.c_void_p(), ctypes.c_void_p()
    rc = _lib.lib().pbd_simulate(_text(profile), _text(schedule), json.dumps(sim or {}).encode(), ctypes.byref(out),
                                 ctypes.byref(err))
    _check(rc, err)
    return json.loads(_lib.take_string(out))


def reconfigure(profile: Doc, schedule: Doc, observed: Doc, threshold: float) -> Optional[dict]:
    """schedule.cpp:347-359: a new schedule when drift > threshold, else None."""
    out, err = ctypes.c_void_p(), ctypes.c_void_p()
    rc = _lib.lib().pbd_reconfigure(_text(profile), _text(schedule), _text(observed), float(threshold),
                                    ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    s = _lib.take_string(out)
    return json.loads(s) if s else None


def profile_drift(reference: Doc, observed: Doc) -> float:
    d, err = ctypes.c_double(), ctypes.c_void_p()
    rc = _lib.lib().pbd_profile_drift(_text(reference), _text(observed), ctypes.byref(d), ctypes.byref(err))
    _check(rc, err)
    return d.value


def exec_time(profile: Doc, block: int, role: str, batch: int) -> float:
    d, err = ctypes.c_double(), ctypes.c_void_p()
    rc = _lib.lib().pbd_exec_time(_text(profile), block, 0 if role == "teacher" else 1, batch, ctypes.byref(d),
                                  ctypes.byref(err))
    _check(rc, err)
    return d.value


def load_save_profile(profile: Doc) -> str:
    out, err = ctypes.c_void_p(), ctypes.c_void_p()
    rc = _lib.lib().pbd_load_save_profile(_text(profile), ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return _lib.take_string(out)


def synth_profile(**spec) -> dict:
    out, err = ctypes.c_void_p(), ctypes.c_void_p()
    rc = _lib.lib().pbd_synth_profile(json.dumps(spec).encode(), ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return json.loads(_lib.take_string(out))


def shard_range(global_batch: int, group_size: int, rank: int) -> Tuple[int, int]:
    """(first sample, count) of `rank` in its group — remainder rule of SPEC.md:231."""
    f, c = ctypes.c_int(), ctypes.c_int()
    rc = _lib.lib().pbd_shard_range(global_batch, group_size, rank, ctypes.byref(f), ctypes.byref(c))
    if rc != 0:
        raise ValidationError("bad shard rank")
    return f.value, c.value


def time_best_schedule(profile: Doc, reps: int = 20) -> float:
    ms, err = ctypes.c_double(), ctypes.c_void_p()
    rc = _lib.lib().pbd_time_best_schedule(_text(profile), reps, ctypes.byref(ms), ctypes.byref(err))
    _check(rc, err)
    return ms.value


# ---------------------------------------------------------------- reports of real runs
def report_steady_state(report: Doc) -> float:
    """steady_state_step_time (simulate.cpp:388-424) of any report document, simulated or measured."""
    d, err = ctypes.c_double(), ctypes.c_void_p()
    L = _lib.lib()
    L.pbd_report_steady_state.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_void_p)]
    rc = L.pbd_report_steady_state(_text(report), ctypes.byref(d), ctypes.byref(err))
    _check(rc, err)
    return d.value


def validate_prediction(report: Doc, profile: Doc, schedule: Doc) -> float:
    """|steady(report) - predicted step_ms| / predicted (simulate.cpp:426-429): how far a measured run is
    from the plan the partitioner made on `profile`."""
    d, err = ctypes.c_double(), ctypes.c_void_p()
    L = _lib.lib()
    L.pbd_validate_prediction.argtypes = [ctypes.c_char_p] * 3 + [ctypes.POINTER(ctypes.c_double),
                                                                   ctypes.POINTER(ctypes.c_void_p)]
    rc = L.pbd_validate_prediction(_text(report), _text(profile), _text(schedule), ctypes.byref(d), ctypes.byref(err))
    _check(rc, err)
    return d.value


def gantt_svg(report: Doc, title: str = "") -> str:
    out, err = ctypes.c_void_p(), ctypes.c_void_p()
    L = _lib.lib()
    L.pbd_gantt_svg.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                ctypes.POINTER(ctypes.c_void_p)]
    rc = L.pbd_gantt_svg(_text(report), title.encode(), ctypes.byref(out), ctypes.byref(err))
    _check(rc, err)
    return _lib.take_string(out)
