"""ctypes wrapper of oracle/local_update.c -- TEST INFRASTRUCTURE ONLY.

A compiled OpenMP restatement of the two operator passes of the oracle's
Woodbury local update (oracle/admm_ref.py LocalSolve.solve): what bench.py's
CPU-baseline legs time next to the NumPy oracle.  The
product package never imports this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "local_update.c")
LIB = os.path.join(_HERE, "liblocal_update.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(SRC) > os.path.getmtime(LIB):
        subprocess.run(["gcc", "-O3", "-fopenmp", "-ffast-math", "-fPIC", "-shared",
                        "-o", LIB + ".tmp", SRC, "-lm"], check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        h = C.CDLL(LIB)
        fp, dp, ip = C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_int)
        h.lu_forward.argtypes = [fp, C.c_long, C.c_int, C.c_int, ip, dp, dp]
        h.lu_adjoint.argtypes = [fp, C.c_long, C.c_int, C.c_int, ip, dp, dp]
        h.lu_forward.restype = h.lu_adjoint.restype = None
        h.lu_chol_solve.argtypes = [dp, C.c_long, C.c_int, dp]
        h.lu_chol_solve.restype = None
        h.lu_threads.restype = C.c_int
        h.lu_set_threads.argtypes = [C.c_int]
        _lib = h
    return _lib


def threads() -> int:
    return int(_load().lu_threads())


def set_threads(n: int) -> None:
    _load().lu_set_threads(int(n))


def _check(a: np.ndarray):
    assert a.dtype == np.complex64 and a.ndim == 2 and a.flags.f_contiguous, "complex64 column-major operator"


def _cols(cols):
    if cols is None:
        return None, None
    c = np.ascontiguousarray(cols, dtype=np.int32)
    return c, c.ctypes.data_as(C.POINTER(C.c_int))


def forward(a: np.ndarray, x: np.ndarray, cols=None) -> np.ndarray:
    """A[:, cols] @ x with fp64 accumulation (x: complex128, one entry per listed column)."""
    _check(a)
    keep, cp = _cols(cols)
    n = a.shape[1] if keep is None else keep.size
    x = np.ascontiguousarray(x, dtype=np.complex128)
    assert x.size == n
    v = np.empty(a.shape[0], dtype=np.complex128)
    _load().lu_forward(a.ctypes.data_as(C.POINTER(C.c_float)), a.strides[1] // 8, a.shape[0], n, cp,
                       x.ctypes.data_as(C.POINTER(C.c_double)), v.ctypes.data_as(C.POINTER(C.c_double)))
    return v


def adjoint(a: np.ndarray, w: np.ndarray, cols=None) -> np.ndarray:
    """A[:, cols]^H @ w with fp64 accumulation."""
    _check(a)
    keep, cp = _cols(cols)
    n = a.shape[1] if keep is None else keep.size
    w = np.ascontiguousarray(w, dtype=np.complex128)
    assert w.size == a.shape[0]
    z = np.empty(n, dtype=np.complex128)
    _load().lu_adjoint(a.ctypes.data_as(C.POINTER(C.c_float)), a.strides[1] // 8, a.shape[0], n, cp,
                       w.ctypes.data_as(C.POINTER(C.c_double)), z.ctypes.data_as(C.POINTER(C.c_double)))
    return z


def chol_solve(fac_lower: np.ndarray, b: np.ndarray) -> np.ndarray:
    """(L L^H)^{-1} b for a lower Cholesky factor (complex128, column-major)."""
    assert fac_lower.dtype == np.complex128 and fac_lower.flags.f_contiguous
    x = np.array(b, dtype=np.complex128, copy=True)
    _load().lu_chol_solve(fac_lower.ctypes.data_as(C.POINTER(C.c_double)), fac_lower.strides[1] // 16,
                          fac_lower.shape[0], x.ctypes.data_as(C.POINTER(C.c_double)))
    return x


def local_update(sensor, a64: np.ndarray, gap: np.ndarray, sigma: np.ndarray) -> None:
    """SensorRef.local_update (admm.hpp:111-126) of a dual-form sensor with the
    two operator passes (on the complex64 operator `a64`, the same matrix the
    sensor holds promoted to complex128) and the Cholesky solve between them
    through the compiled kernels."""
    from . import admm_ref
    h, cache = sensor.h, sensor.cache
    assert cache.form == "dual"
    j = sensor.active
    cols = None if j.size == a64.shape[1] else j
    rhs = sensor.data + h.beta * gap[j] + h.beta * sensor.x_hat - sigma[j]
    v = forward(a64, rhs, cols)
    fac = getattr(cache, "_fac_f", None)
    if fac is None:  # the lower factor, column-major, once per factorization
        assert cache.fac[1], "lower Cholesky factor expected"
        fac = cache._fac_f = np.asfortranarray(cache.fac[0])
    w = chol_solve(fac, v)
    sensor.x_hat = admm_ref.cdiv(rhs - cache.mu * adjoint(a64, w, cols), cache.beta)
    sensor.x_full[j] = sensor.x_hat
    sensor.history.append(sensor.x_full.copy())
    if len(sensor.history) > h.screening_window + 1:
        sensor.history.popleft()
