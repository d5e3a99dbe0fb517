"""Device-backed twin of the reference kernel module `hybridscale._kernels`.

Same three entry points and argument meaning as hs/_kernels/_grid_cy.pyx:54-74, but
every evaluation runs on the B200 through librapp_b200.so (include/rapp_b200.h).  The
reference module's BACKEND stays "cython"/"python" (its tests pin that set,
pkg/tests/test_kernels.py:90-91); this module reports BACKEND = "b200".
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

BACKEND = "b200"


def _axis(a) -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError("Buffer has wrong number of dimensions (expected 1, got %d)" % arr.ndim)
    return arr


def _grid(values, nb, ns, nq) -> np.ndarray:
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim != 3:
        raise ValueError("Buffer has wrong number of dimensions (expected 3, got %d)" % v.ndim)
    if v.shape[0] < nb or v.shape[1] < ns or v.shape[2] < nq:
        # the Cython kernel would read out of bounds; refuse instead
        raise ValueError(f"values shape {v.shape} smaller than axes ({nb}, {ns}, {nq})")
    if v.shape != (nb, ns, nq):
        v = np.ascontiguousarray(v[:nb, :ns, :nq])
    return v


def locate(axis, x: float) -> tuple[int, int, float]:
    """Bracketing indices and offset of x on an ascending axis (_grid_cy.pyx:9-33, 54-58)."""
    a = _axis(axis)
    lo, hi, t = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    if len(a) == 0:
        raise IndexError("Out of bounds on buffer access (axis 0)")
    _lib.check(_lib.load().rapp_locate(_lib.dptr(a), len(a), float(x), ctypes.byref(lo),
                                       ctypes.byref(hi), ctypes.byref(t)), "locate")
    return lo.value, hi.value, t.value


def interp3(b_axis, s_axis, q_axis, values, b: float, s: float, q: float) -> float:
    """Trilinear interpolation of values[batch, sm, quota] (_grid_cy.pyx:36-51, 61-64)."""
    ba, sa, qa = _axis(b_axis), _axis(s_axis), _axis(q_axis)
    v = _grid(values, len(ba), len(sa), len(qa))
    out = ctypes.c_double()
    _lib.check(_lib.load().rapp_interp3(_lib.dptr(ba), len(ba), _lib.dptr(sa), len(sa),
                                        _lib.dptr(qa), len(qa), _lib.dptr(v), float(b),
                                        float(s), float(q), ctypes.byref(out)), "interp3")
    return out.value


def interp3_many(b_axis, s_axis, q_axis, values, coords, out) -> None:
    """Batched interp3 over coords[n, 3] into out[n] in place (_grid_cy.pyx:67-74)."""
    ba, sa, qa = _axis(b_axis), _axis(s_axis), _axis(q_axis)
    v = _grid(values, len(ba), len(sa), len(qa))
    c = np.ascontiguousarray(coords, dtype=np.float64)
    if c.ndim != 2 or (c.shape[0] and c.shape[1] < 3):
        raise ValueError("coords must be shaped (n, 3)")
    if c.shape[1] != 3:
        c = np.ascontiguousarray(c[:, :3])
    if not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.ndim != 1 or \
            not out.flags.c_contiguous or not out.flags.writeable:
        raise ValueError("out must be a writable contiguous float64 vector")
    n = out.shape[0]
    if n > c.shape[0]:
        raise IndexError("Out of bounds on buffer access (axis 0)")
    _lib.check(_lib.load().rapp_interp3_many(_lib.dptr(ba), len(ba), _lib.dptr(sa), len(sa),
                                             _lib.dptr(qa), len(qa), _lib.dptr(v),
                                             _lib.dptr(c), n, _lib.dptr(out)),
               "interp3_many")


__all__ = ["interp3", "interp3_many", "locate", "BACKEND"]
