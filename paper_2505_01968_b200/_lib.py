"""ctypes binding of librapp_b200.so (include/rapp_b200.h).

The product path has no CPU fallback: if the library cannot be loaded, or no CUDA
device is visible, every call raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (DeviceError, FilterDegenerateError, InvariantViolation, PlacementError,
                     TableFormatError)

LIB_PATH = os.environ.get(
    "RAPP_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "librapp_b200.so"))

RAPP_OK = 0
RAPP_E_VALUE = 1
RAPP_E_TABLE = 2
RAPP_E_ARG = 3
RAPP_E_CUDA = 4
RAPP_E_PLACEMENT = 5
RAPP_E_INVARIANT = 6
RAPP_E_DEGENERATE = 7

c_dp = ctypes.POINTER(ctypes.c_double)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_vp = ctypes.c_void_p

_lib = None
_lock = threading.Lock()

# (name, restype, argtypes) for every symbol include/rapp_b200.h declares.
SIGNATURES = [
    ("rapp_last_error", ctypes.c_char_p, []),
    ("rapp_version", ctypes.c_char_p, []),
    ("rapp_locate", ctypes.c_int, [c_dp, ctypes.c_int64, ctypes.c_double, c_i64p, c_i64p, c_dp]),
    ("rapp_interp3", ctypes.c_int, [c_dp, ctypes.c_int64, c_dp, ctypes.c_int64, c_dp,
                                    ctypes.c_int64, c_dp, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, c_dp]),
    ("rapp_interp3_many", ctypes.c_int, [c_dp, ctypes.c_int64, c_dp, ctypes.c_int64, c_dp,
                                         ctypes.c_int64, c_dp, c_dp, ctypes.c_int64, c_dp]),
    ("rapp_ctx_create", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("rapp_ctx_destroy", ctypes.c_int, [c_vp]),
    ("rapp_shutdown", ctypes.c_int, []),
    ("rapp_ctx_info", ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int)]),
    ("rapp_table_create", ctypes.c_int, [c_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         c_dp, c_dp, c_dp, c_dp, c_i32p]),
    ("rapp_table_count", ctypes.c_int, [c_vp, c_i32p]),
    ("rapp_interp3_many_dev", ctypes.c_int, [c_vp, ctypes.c_int32, c_vp, ctypes.c_int64, c_vp,
                                             c_vp, c_vp]),
    ("rapp_interp3_many_host", ctypes.c_int, [c_vp, ctypes.c_int32, c_dp, ctypes.c_int64,
                                              c_dp]),
    ("rapp_table_points", ctypes.c_int, [c_vp, ctypes.c_int32, ctypes.c_int64, c_dp, c_dp,
                                         c_dp]),
    ("rapp_csv_parse", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int64, c_i64p,
                                      c_i64p, c_i64p, c_dp, c_i64p, ctypes.c_char_p,
                                      ctypes.c_int64, c_i32p]),
    ("rapp_ingest_create", ctypes.c_int, [c_vp, ctypes.c_int64, c_i64p, c_i64p, c_i64p, c_dp,
                                          ctypes.POINTER(c_vp)]),
    ("rapp_ingest_shape", ctypes.c_int, [c_vp, c_i64p, c_i64p, c_i64p, c_i32p, c_i32p,
                                         c_i32p]),
    ("rapp_ingest_read", ctypes.c_int, [c_vp, c_i64p, c_i64p, c_i64p, c_dp, c_vp, c_vp]),
    ("rapp_ingest_destroy", ctypes.c_int, [c_vp]),
    ("rapp_mec_batch", ctypes.c_int, [c_vp, ctypes.c_int64, c_i32p, c_dp, ctypes.c_int32,
                                      c_i64p, c_i64p, c_i64p]),
    ("rapp_mec_plan_create", ctypes.c_int, [c_vp, ctypes.c_int64, c_i32p, ctypes.c_int32,
                                            c_i64p, c_i64p, ctypes.POINTER(c_vp)]),
    ("rapp_mec_plan_destroy", ctypes.c_int, [c_vp]),
    ("rapp_mec_plan_points", ctypes.c_int, [c_vp, c_i64p]),
    ("rapp_mec_plan_run_dev", ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, c_vp,
                                             c_vp, c_vp]),
    ("rapp_mec_plan_run", ctypes.c_int, [c_vp, c_dp, ctypes.c_int64, ctypes.c_int64, c_i64p]),
    ("rapp_mec_plan_set_slo", ctypes.c_int, [c_vp, c_vp]),
    ("rapp_mec_plan_timing", ctypes.c_int, [c_vp, ctypes.c_int]),
    ("rapp_mec_plan_kernel_time", ctypes.c_int, [c_vp, c_dp, c_i64p]),
    ("rapp_metrics_finalize", ctypes.c_int, [c_vp, ctypes.c_int64, c_dp, c_i64p, c_i64p, c_dp,
                                             c_i64p, c_dp, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_int32, c_dp, ctypes.c_int32, c_i32p, c_dp,
                                             c_dp, c_dp, c_dp]),
    ("rapp_mlp_create", ctypes.c_int, [c_vp, ctypes.c_int32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       ctypes.c_float, ctypes.POINTER(c_vp)]),
    ("rapp_mlp_destroy", ctypes.c_int, [c_vp]),
    ("rapp_mlp_predict_dev", ctypes.c_int, [c_vp, ctypes.c_int32, c_vp, ctypes.c_int64, c_vp,
                                            c_vp]),
    ("rapp_mlp_predict_host", ctypes.c_int, [c_vp, ctypes.c_int32, c_dp, ctypes.c_int64,
                                             c_dp]),
    ("rapp_mlp_search_dev", ctypes.c_int, [c_vp, ctypes.c_int64, c_vp, c_vp, ctypes.c_int32,
                                           c_vp, ctypes.c_int32, c_vp, ctypes.c_int32, c_vp,
                                           c_vp, c_vp]),
    ("rapp_mlp_debug_dev", ctypes.c_int, [c_vp, ctypes.c_int32, c_vp, ctypes.c_int64, c_vp,
                                          c_vp, c_vp]),
    ("rapp_probe_fp64", ctypes.c_int, [ctypes.c_int, c_dp, c_dp]),
    ("rapp_tick_create", ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, c_vp, c_i64p,
                                        ctypes.c_int64, c_i64p, c_i32p, c_i32p, ctypes.c_int64,
                                        c_vp, ctypes.c_int64, ctypes.POINTER(c_vp)]),
    ("rapp_tick_destroy", ctypes.c_int, [c_vp]),
    ("rapp_tick_run", ctypes.c_int, [c_vp, ctypes.c_double, c_vp, c_vp, c_vp, c_vp,
                                     ctypes.c_int64, c_i64p, c_vp, c_vp]),
    ("rapp_tick_submit", ctypes.c_int, [c_vp, ctypes.c_double, c_vp, c_vp, c_vp,
                                        ctypes.c_int64]),
    ("rapp_tick_collect", ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, c_i64p, c_vp, c_vp]),
    ("rapp_tick_release", ctypes.c_int, [c_vp, c_i64p, ctypes.c_int64]),
    ("rapp_tick_run_dev", ctypes.c_int, [c_vp, ctypes.c_double, c_vp, c_vp, c_vp]),
    ("rapp_tick_outputs_dev", ctypes.c_int, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                                             ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    ("rapp_tick_pod_count", ctypes.c_int, [c_vp, c_i64p]),
    ("rapp_tick_read_pods", ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, c_i64p]),
    ("rapp_tick_set_slo", ctypes.c_int, [c_vp, c_vp]),
    ("rapp_tick_read_fns", ctypes.c_int, [c_vp, c_vp]),
    ("rapp_tick_read_parts", ctypes.c_int, [c_vp, c_i64p, c_i32p, c_i32p, c_i32p,
                                            ctypes.c_int64]),
    ("rapp_tick_counter", ctypes.c_int, [c_vp, c_i64p]),
    ("rapp_launch_count", ctypes.c_int64, []),
]


def load(path: str = LIB_PATH):
    """Loads the library and declares every exported signature (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceError(
                    f"{path} is missing: build it with `python -m paper_2505_01968_b200._build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    return load().rapp_last_error().decode("utf-8", "replace")


def check(rc: int, what: str = "") -> None:
    """Maps a C-ABI status onto the reference's exception types."""
    if rc == RAPP_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == RAPP_E_VALUE:
        raise ValueError(msg)
    if rc == RAPP_E_TABLE:
        raise TableFormatError(msg)
    if rc == RAPP_E_PLACEMENT:
        raise PlacementError(msg)
    if rc == RAPP_E_INVARIANT:
        raise InvariantViolation(msg)
    if rc == RAPP_E_DEGENERATE:
        raise FilterDegenerateError(msg)
    raise DeviceError(msg)


def dptr(a) -> ctypes.POINTER(ctypes.c_double):
    return a.ctypes.data_as(c_dp)


def i64ptr(a):
    return a.ctypes.data_as(c_i64p)


def i32ptr(a):
    return a.ctypes.data_as(c_i32p)


class Context:
    """One library context (device table pool + host pipeline) per CUDA device."""

    _by_device: dict[int, "Context"] = {}

    def __init__(self, device: int):
        lib = load()
        h = c_vp()
        check(lib.rapp_ctx_create(int(device), ctypes.byref(h)), "rapp_ctx_create")
        self.handle = h
        self.device = int(device)
        sm = ctypes.c_int()
        check(lib.rapp_ctx_info(h, None, ctypes.byref(sm)))
        self.sm_count = sm.value

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        if device is None:
            device = int(os.environ.get("RAPP_DEVICE", "0"))
        ctx = cls._by_device.get(device)
        if ctx is None:
            ctx = cls._by_device[device] = Context(device)
        return ctx


    @classmethod
    def close_all(cls) -> None:
        """Destroys every context (table pools, staging).  Only for a clean shutdown once
        no table, plan, tick world or model of the process is alive any more (leak checks)."""
        lib = load()
        for dev, ctx in list(cls._by_device.items()):
            lib.rapp_ctx_destroy(ctx.handle)
            del cls._by_device[dev]
        lib.rapp_shutdown()


def launch_count() -> int:
    return int(load().rapp_launch_count())
