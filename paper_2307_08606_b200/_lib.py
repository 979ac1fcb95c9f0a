"""ctypes binding of libradmm_b200.so (include/radmm_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: if the library is missing, importing the
solver API raises, and every compute entry point needs a Blackwell GPU.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RADMM_LIB_PATH") or os.path.join(_HERE, "libradmm_b200.so")  # override: A/B of builds

OK, INVALID_ARGUMENT, NUMERICAL, TRANSPORT, CUDA, OUT_OF_MEMORY = range(6)
PTR_HOST, PTR_DEVICE = 0, 1
VEC_X_GLOBAL, VEC_S, VEC_SIGMA, VEC_SIGMA_PRE_GLOBAL, VEC_GAP = range(5)


class RadmmError(RuntimeError):
    """Base class; ``code`` is the radmm_status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(RadmmError, ValueError):
    """std::invalid_argument of the reference (admm.hpp:41-57,69-80)."""


class NumericalError(RadmmError):
    """std::runtime_error("factorize: Cholesky failed") (solver_core.hpp:42-43)."""


class TransportError(RadmmError):
    """TransportError of the reference runtime (runtime.hpp:27-35); NCCL here."""


class CudaError(RadmmError):
    pass


_EXC = {INVALID_ARGUMENT: InvalidArgument, NUMERICAL: NumericalError, TRANSPORT: TransportError,
        CUDA: CudaError, OUT_OF_MEMORY: CudaError}


class Hyper(C.Structure):
    _fields_ = [("mu", C.c_double), ("lambda_", C.c_double), ("beta", C.c_double),
                ("eps_abs", C.c_double), ("eps_rel", C.c_double), ("screening_window", C.c_int32),
                ("screening_tol", C.c_double), ("max_iter", C.c_int32)]


class Record(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("pri_res", C.c_double), ("dual_res", C.c_double),
                ("eps_pri", C.c_double), ("eps_dual", C.c_double), ("active_fraction", C.c_double),
                ("ms_elapsed", C.c_double), ("bytes_sent", C.c_uint64)]


class View(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("x_global", C.POINTER(C.c_double)),
                ("s", C.POINTER(C.c_double)), ("sigma", C.POINTER(C.c_double)),
                ("active_sizes", C.POINTER(C.c_int32)), ("converged", C.c_int32),
                ("screening_trigger", C.c_int32)]


OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(View))


class Options(C.Structure):
    _fields_ = [("mode", C.c_int), ("disable_screening", C.c_int32), ("fixed_iterations", C.c_int32),
                ("observer", OBSERVER), ("observer_user", C.c_void_p), ("skip_refinement", C.c_int32)]


class Summary(C.Structure):
    _fields_ = [("converged", C.c_int32), ("screening_stalled", C.c_int32), ("iterations", C.c_int32),
                ("total_active_solves", C.c_uint64), ("total_bytes", C.c_uint64),
                ("setup_ms", C.c_double), ("solve_ms", C.c_double), ("kernel_launches", C.c_int64),
                ("rebuilds", C.c_int64), ("downdates", C.c_int64), ("refine_skipped", C.c_int64)]


class PhaseStat(C.Structure):
    _fields_ = [("calls", C.c_int64), ("launches", C.c_int64), ("total_ms", C.c_double), ("bytes", C.c_double)]


PHASES = ["forward", "gapply", "adjoint", "primal", "exchange", "fusion", "screen", "refactor", "sweep"]


# Every symbol include/radmm_b200.h declares, with its argument types.
_VP = C.c_void_p
_DP = C.POINTER(C.c_double)
_FP = C.POINTER(C.c_float)
_IP = C.POINTER(C.c_int32)
SIGNATURES = {
    "radmm_last_error": (C.c_char_p, []),
    "radmm_version": (C.c_int, []),
    "radmm_build_features": (C.c_int, []),
    "radmm_set_tuning": (C.c_int, [C.c_char_p, C.c_int, C.c_int]),
    "radmm_hyperparams_default": (C.c_int, [C.POINTER(Hyper)]),
    "radmm_hyperparams_validate": (C.c_int, [C.POINTER(Hyper)]),
    "radmm_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(_VP)]),
    "radmm_ctx_destroy": (C.c_int, [_VP]),
    "radmm_set_operator_c64": (C.c_int, [_VP, C.c_int, C.c_int, _VP, C.c_int64, C.c_int]),
    "radmm_set_operator_c128": (C.c_int, [_VP, C.c_int, C.c_int, _VP, C.c_int64, C.c_int]),
    "radmm_set_measurement": (C.c_int, [_VP, C.c_int, _VP, C.c_int]),
    "radmm_generate_dechirp_operator": (C.c_int, [_VP, C.c_int, C.c_int, C.c_int, _DP, _DP, _DP, _DP,
                                                  C.c_double, C.c_double, C.c_double]),
    "radmm_generate_echo_operator": (C.c_int, [_VP, C.c_int, C.c_int, C.c_int, _DP, _DP, _DP, C.c_double,
                                               C.c_double, C.c_double, C.c_double]),
    "radmm_get_operator_c64": (C.c_int, [_VP, C.c_int, _VP]),
    "radmm_run": (C.c_int, [_VP, C.POINTER(Hyper), C.POINTER(Options), C.POINTER(Summary)]),
    "radmm_set_frame_measurement": (C.c_int, [_VP, C.c_int, C.c_int, _VP, C.c_int]),
    "radmm_run_frames": (C.c_int, [_VP, C.c_int, C.POINTER(Hyper), C.POINTER(Options), C.POINTER(Summary)]),
    "radmm_frame": (C.c_int, [_VP, C.c_int, C.POINTER(_VP)]),
    "radmm_get_image": (C.c_int, [_VP, _DP]),
    "radmm_get_vector": (C.c_int, [_VP, C.c_int, _DP]),
    "radmm_get_sensor_image": (C.c_int, [_VP, C.c_int, _DP]),
    "radmm_get_record_count": (C.c_int, [_VP, C.POINTER(C.c_int)]),
    "radmm_get_records": (C.c_int, [_VP, C.POINTER(Record), C.c_int]),
    "radmm_get_active_sizes": (C.c_int, [_VP, _IP, C.c_int]),
    "radmm_get_active_set": (C.c_int, [_VP, C.c_int, _IP, C.POINTER(C.c_int)]),
    "radmm_get_removal_log_size": (C.c_int, [_VP, C.POINTER(C.c_int)]),
    "radmm_get_removal_log": (C.c_int, [_VP, _IP, C.c_int]),
    "radmm_factorize": (C.c_int, [C.c_int, C.c_int, C.c_int, _DP, C.c_double, C.c_double, C.POINTER(_VP)]),
    "radmm_solve_local": (C.c_int, [_VP, _DP, _DP]),
    "radmm_solve_cache_destroy": (C.c_int, [_VP]),
    "radmm_soft_threshold": (C.c_int, [C.c_int, _DP, C.c_int64, C.c_double, _DP]),
    "radmm_apply_operator": (C.c_int, [_VP, C.c_int, _DP, _DP]),
    "radmm_apply_adjoint": (C.c_int, [_VP, C.c_int, _DP, _DP]),
    "radmm_back_projection": (C.c_int, [_VP, _DP]),
    "radmm_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_VP)]),
    "radmm_host_free": (C.c_int, [_VP]),
    "radmm_pool_trim": (C.c_int, [C.c_int]),
    "radmm_set_profiling": (C.c_int, [_VP, C.c_int]),
    "radmm_get_phase_stats": (C.c_int, [_VP, C.POINTER(PhaseStat)]),
    "radmm_get_iteration_stats": (C.c_int, [_VP, _DP, C.POINTER(C.c_int64), C.c_int]),
    "radmm_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "radmm_set_transport_timeout": (C.c_int, [_VP, C.c_int]),
    "radmm_ctx_create_sharded": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(C.c_uint8), C.POINTER(_VP)]),
}

_lib = None


def lib():
    """Load the CUDA library (raises loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                              "there is no CPU fallback")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status: int) -> None:
    if status != OK:
        msg = lib().radmm_last_error().decode(errors="replace")
        raise _EXC.get(status, RadmmError)(status, msg)
