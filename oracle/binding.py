"""ctypes binding for oracle/liboracle.so and loader for oracle/_ref (test-only)."""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build_oracle() -> None:
    """Builds liboracle.so (and oracle/_ref when the reference tree exists)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def load_oracle():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build_oracle()
        lib = ctypes.CDLL(path)
        lib.or_locate.argtypes = [_dp, ctypes.c_int64, ctypes.c_double, _i64p, _i64p, _dp]
        lib.or_locate.restype = None
        lib.or_interp3.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp,
                                   ctypes.c_int64, _dp, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double]
        lib.or_interp3.restype = ctypes.c_double
        lib.or_interp3_many.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp,
                                        ctypes.c_int64, _dp, _dp, ctypes.c_int64, _dp]
        lib.or_interp3_many.restype = None
        lib.or_throughput_from_latency.argtypes = [ctypes.c_double, ctypes.c_double]
        lib.or_throughput_from_latency.restype = ctypes.c_double
        lib.or_most_efficient_config.argtypes = [
            _dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp,
            ctypes.c_double, ctypes.c_int64, _i64p, ctypes.c_int64, _i64p]
        lib.or_most_efficient_config.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _d(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def or_locate(axis, x):
    lib = load_oracle()
    axis = _f64(axis)
    lo, hi, t = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    lib.or_locate(_d(axis), len(axis), float(x), ctypes.byref(lo), ctypes.byref(hi),
                  ctypes.byref(t))
    return lo.value, hi.value, t.value


def or_interp3(b_axis, s_axis, q_axis, values, b, s, q):
    lib = load_oracle()
    b_axis, s_axis, q_axis, values = map(_f64, (b_axis, s_axis, q_axis, values))
    return lib.or_interp3(_d(b_axis), len(b_axis), _d(s_axis), len(s_axis), _d(q_axis),
                          len(q_axis), _d(values), float(b), float(s), float(q))


def or_interp3_many(b_axis, s_axis, q_axis, values, coords, out=None):
    lib = load_oracle()
    b_axis, s_axis, q_axis, values, coords = map(_f64, (b_axis, s_axis, q_axis, values,
                                                        coords))
    n = coords.shape[0]
    if out is None:
        out = np.empty(n, dtype=np.float64)
    lib.or_interp3_many(_d(b_axis), len(b_axis), _d(s_axis), len(s_axis), _d(q_axis),
                        len(q_axis), _d(values), _d(coords), n, _d(out))
    return out


def or_throughput(batch, latency_ms):
    return load_oracle().or_throughput_from_latency(float(batch), float(latency_ms))


def or_most_efficient_config(b_axis, s_axis, q_axis, values, target, quota_step=10,
                             batches=None):
    """Returns (b, s, q); raises ValueError like hs/perf.py:114-117."""
    lib = load_oracle()
    b_axis, s_axis, q_axis, values = map(_f64, (b_axis, s_axis, q_axis, values))
    out = np.zeros(3, dtype=np.int64)
    if batches is None:
        allowed_p, nallowed = None, -1
    else:
        allowed = np.ascontiguousarray([int(b) for b in batches], dtype=np.int64)
        allowed_p, nallowed = allowed.ctypes.data_as(_i64p), len(allowed)
    rc = lib.or_most_efficient_config(_d(b_axis), len(b_axis), _d(s_axis), len(s_axis),
                                      _d(q_axis), len(q_axis), _d(values), float(target),
                                      int(quota_step), allowed_p, nallowed,
                                      out.ctypes.data_as(_i64p))
    if rc:
        raise ValueError("target_rps must be positive and quota_step in [1, 100]")
    return int(out[0]), int(out[1]), int(out[2])


def load_reference_kernel():
    """The reference's own compiled kernel (oracle/_ref), or None if not built."""
    global _REF
    if _REF is None:
        hits = glob.glob(os.path.join(_HERE, "_ref", "_grid_cy*.so"))
        if not hits:
            return None
        spec = importlib.util.spec_from_file_location("_grid_cy", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF
