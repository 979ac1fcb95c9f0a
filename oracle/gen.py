"""ctypes wrapper of oracle/baseline_gen.c -- TEST INFRASTRUCTURE ONLY.

Host-side BASELINE operators for bench.py's CPU-baseline / reference legs
(config 3 sensors take minutes in NumPy); bitwise equal to
paper_2307_08606_b200.scenario.baseline_operator (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "baseline_gen.c")
LIB = os.path.join(_HERE, "libbaseline_gen.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(SRC) > os.path.getmtime(LIB):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                        "-o", LIB + ".tmp", SRC, "-lm"], check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        h = C.CDLL(LIB)
        dp = C.POINTER(C.c_double)
        h.baseline_operator_c64.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp, dp, dp, C.c_double, C.c_double,
                                            C.c_double, C.c_double, C.POINTER(C.c_float)]
        h.baseline_operator_c64.restype = None
        _lib = h
    return _lib


def baseline_operator(cfg, q: int, out: np.ndarray | None = None) -> np.ndarray:
    """A_q of a BaselineConfig as a column-major (KM x N) complex64 array."""
    from paper_2307_08606_b200 import scenario
    pix, tx, rx = scenario.baseline_geometry(cfg)
    u = np.ascontiguousarray(scenario.baseline_phases(cfg, q))
    pix = np.ascontiguousarray(pix)
    txq = np.ascontiguousarray(tx[q])
    rxq = np.ascontiguousarray(rx[q])
    if out is None:
        out = np.empty((cfg.KM, cfg.N), dtype=np.complex64, order="F")
    assert out.flags.f_contiguous and out.dtype == np.complex64 and out.shape == (cfg.KM, cfg.N)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    _load().baseline_operator_c64(cfg.M, cfg.K, cfg.N, dp(pix), dp(txq), dp(rxq), dp(u), cfg.bw / cfg.pulse,
                                  cfg.fc, cfg.pulse / cfg.K, scenario.SPEED_OF_LIGHT,
                                  out.ctypes.data_as(C.POINTER(C.c_float)))
    return out
