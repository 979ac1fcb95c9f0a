"""Python mirror of the reference solver API, backed by the CUDA library.

Same names, argument meanings and error behaviour as the reference
(``/root/reference/proj/include/radmm``):

=========================  ==============================================
this module                reference
=========================  ==============================================
``Mode``                   ``enum class Mode``            admm.hpp:25
``Hyperparams``            ``struct Hyperparams``         admm.hpp:31-58
``ForwardOperator``        ``ForwardOperator::from_matrix`` forward_model.hpp:126-133
``Problem``                ``struct Problem``             admm.hpp:60-81
``IterationRecord``        ``struct IterationRecord``     admm.hpp:284-295
``ConvergenceReport``      ``struct ConvergenceReport``   admm.hpp:297-322
``RunResult``              ``struct RunResult``           admm.hpp:324-335
``IterationView``          ``struct IterationView``       admm.hpp:339-347
``run``                    ``run(...)``                   admm.hpp:357-445
``soft_threshold``         solver_core.hpp:14-23
``factorize``/``solve_local``/``LocalSolveCache``  solver_core.hpp:30-66
``objective_value``/``nmse_db``/``relative_l2_diff``  admm.hpp:450-483
=========================  ==============================================

Every compute call runs on the GPU through ``libradmm_b200.so``; there is no
CPU path.  ``Solver`` keeps one device context alive across runs (operators
stay resident in HBM), which is what a serving deployment uses.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import InvalidArgument, NumericalError, TransportError, CudaError  # noqa: F401


class Mode(enum.IntEnum):
    SADMM = 0
    ASADMM = 1

    # reference spelling
    kSadmm = 0
    kAsadmm = 1


def mode_name(m: Mode) -> str:
    return "sadmm" if Mode(m) == Mode.SADMM else "asadmm"


@dataclass
class Hyperparams:
    """admm.hpp:31-58.  ``lambda_`` is the reference's ``lambda``."""
    mu: float = 3.0
    lambda_: float = 20.0
    beta: float = 100.0
    eps_abs: float = 1e-4
    eps_rel: float = 1e-2
    screening_window: int = 5
    screening_tol: float = 1e-5
    max_iter: int = 1000

    def _c(self) -> _lib.Hyper:
        return _lib.Hyper(self.mu, self.lambda_, self.beta, self.eps_abs, self.eps_rel,
                          int(self.screening_window), self.screening_tol, int(self.max_iter))

    def validate(self) -> None:
        _lib.check(_lib.lib().radmm_hyperparams_validate(C.byref(self._c())))


class ForwardOperator:
    """Dense operator container (ForwardOperator::from_matrix).

    ``matrix`` is rows x N (row r = m*K + k, column n = pixel).  complex64
    matrices are used as is; complex128 ones are rounded to complex64 on the
    device (the operator is stored and streamed as complex64).
    """

    def __init__(self, matrix: np.ndarray):
        if matrix.ndim != 2:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "ForwardOperator: matrix must be 2-D")
        self._m = matrix

    @staticmethod
    def from_matrix(a: np.ndarray) -> "ForwardOperator":
        return ForwardOperator(np.asarray(a))

    def rows(self) -> int:
        return self._m.shape[0]

    def cols(self) -> int:
        return self._m.shape[1]

    def is_dense(self) -> bool:
        return True

    def matrix(self) -> np.ndarray:
        return self._m


@dataclass
class Problem:
    operators: list = field(default_factory=list)
    measurements: list = field(default_factory=list)

    def sensor_count(self) -> int:
        return len(self.operators)

    def pixel_count(self) -> int:
        return self.operators[0].cols() if self.operators else 0

    def validate(self) -> None:  # admm.hpp:69-80
        if not self.operators:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "Problem: needs at least one sensor")
        if len(self.operators) != len(self.measurements):
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "Problem: one measurement per operator")
        for op, y in zip(self.operators, self.measurements):
            if op.cols() != self.operators[0].cols():
                raise InvalidArgument(_lib.INVALID_ARGUMENT, "Problem: operators disagree on pixel count")
            if np.asarray(y).shape[0] != op.rows():
                raise InvalidArgument(_lib.INVALID_ARGUMENT, "Problem: measurement length mismatch")


@dataclass
class IterationRecord:
    iteration: int = 0
    pri_res: float = 0.0
    dual_res: float = 0.0
    eps_pri: float = 0.0
    eps_dual: float = 0.0
    active_fraction: float = 0.0
    ms_elapsed: float = 0.0
    bytes_sent: int = 0
    active_sizes: list = field(default_factory=list)
    sensor_bytes: list = field(default_factory=list)


def contribution_size(n: int) -> int:  # wire.hpp:54-56
    return 1 + 4 + 8 + 4 + n * (4 + 16)


@dataclass
class ConvergenceReport:
    iterations: list = field(default_factory=list)
    total_active_solves: int = 0
    total_bytes: int = 0

    def csv(self) -> str:
        """ConvergenceReport::write_csv (admm.hpp:302-314)."""
        out = ["iter,pri_res,dual_res,eps_pri,eps_dual,active_frac,ms_elapsed,bytes_sent\n"]
        for r in self.iterations:
            out.append("%d,%.12g,%.12g,%.12g,%.12g,%.12g,%.3f,%d\n" % (
                r.iteration, r.pri_res, r.dual_res, r.eps_pri, r.eps_dual, r.active_fraction,
                r.ms_elapsed, r.bytes_sent))
        return "".join(out)

    def write_csv(self, out) -> None:
        if isinstance(out, str):
            try:
                with open(out, "w") as f:
                    f.write(self.csv())
            except OSError as e:
                raise RuntimeError("ConvergenceReport: cannot open " + out) from e
        else:
            out.write(self.csv())


@dataclass
class RunResult:
    image: np.ndarray = None
    x_global: np.ndarray = None
    s: np.ndarray = None
    sigma: np.ndarray = None
    sigma_pre_global: np.ndarray = None
    sensor_images: list = field(default_factory=list)
    converged: bool = False
    screening_stalled: bool = False
    iterations: int = 0
    report: ConvergenceReport = field(default_factory=ConvergenceReport)
    # build-side diagnostics
    setup_ms: float = 0.0
    solve_ms: float = 0.0
    kernel_launches: int = 0
    rebuilds: int = 0
    downdates: int = 0
    active_sets: list = field(default_factory=list)
    removal_log: np.ndarray = None
    refine_skipped: int = 0   # dual sensors solved without KM-space refinement (memory)


@dataclass
class IterationView:
    iteration: int
    x_global: np.ndarray
    s: np.ndarray
    sigma: np.ndarray
    active_sizes: list
    converged: bool
    screening_trigger: bool


def _c128(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.complex128))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Solver:
    """One device context holding a Problem resident in HBM (C ABI ctx)."""

    def __init__(self, n_pixels: int, n_sensors: int, device: int = 0, _ctx=None, q_total=None, q_begin=0):
        self.N = int(n_pixels)
        self.Q = int(n_sensors)
        self.Q_total = int(q_total if q_total is not None else n_sensors)
        self.q_begin = int(q_begin)
        self.device = device
        L = _lib.lib()
        if _ctx is None:
            h = C.c_void_p()
            _lib.check(L.radmm_ctx_create(device, self.N, self.Q, C.byref(h)))
            self._h = h
        else:
            self._h = _ctx
        self.rows = [0] * self.Q

    @classmethod
    def from_problem(cls, problem: Problem, device: int = 0) -> "Solver":
        problem.validate()
        s = cls(problem.pixel_count(), problem.sensor_count(), device)
        for q, (op, y) in enumerate(zip(problem.operators, problem.measurements)):
            s.set_operator(q, op.matrix())
            s.set_measurement(q, y)
        return s

    def close(self) -> None:
        if getattr(self, "_borrowed", False):  # a frame handle: owned by its parent
            self._h = None
            return
        if getattr(self, "_h", None):
            _lib.lib().radmm_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- problem -------------------------------------------------------
    def set_operator(self, q: int, a: np.ndarray) -> None:
        a = np.asarray(a)
        if a.ndim != 2 or a.shape[1] != self.N:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "Problem: operators disagree on pixel count")
        rows = a.shape[0]
        L = _lib.lib()
        if a.dtype == np.complex64:
            f = np.asfortranarray(a)
            _lib.check(L.radmm_set_operator_c64(self._h, q, rows, f.ctypes.data_as(C.c_void_p), rows,
                                                _lib.PTR_HOST))
        else:
            f = np.asfortranarray(a, dtype=np.complex128)
            _lib.check(L.radmm_set_operator_c128(self._h, q, rows, f.ctypes.data_as(C.c_void_p), rows,
                                                 _lib.PTR_HOST))
        self.rows[q] = rows

    def set_operator_ptr(self, q: int, rows: int, ptr: int, lda: int, device_ptr: bool) -> None:
        """Column-major complex64 operator at a raw host or device pointer."""
        _lib.check(_lib.lib().radmm_set_operator_c64(self._h, q, rows, C.c_void_p(ptr), lda,
                                                     _lib.PTR_DEVICE if device_ptr else _lib.PTR_HOST))
        self.rows[q] = rows

    def set_measurement(self, q: int, y) -> None:
        y = _c128(y)
        if self.rows[q] and y.shape[0] != self.rows[q]:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "Problem: measurement length mismatch")
        _lib.check(_lib.lib().radmm_set_measurement(self._h, q, y.ctypes.data_as(C.c_void_p), _lib.PTR_HOST))

    def set_measurement_ptr(self, q: int, ptr: int, device_ptr: bool) -> None:
        _lib.check(_lib.lib().radmm_set_measurement(self._h, q, C.c_void_p(ptr),
                                                    _lib.PTR_DEVICE if device_ptr else _lib.PTR_HOST))

    def generate_dechirp_operator(self, q, M, K, pix, tx, rx, phi, fc, bw, pulse) -> None:
        pix = np.ascontiguousarray(pix, dtype=np.float64)
        tx = np.ascontiguousarray(tx, dtype=np.float64)
        rx = np.ascontiguousarray(rx, dtype=np.float64)
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        _lib.check(_lib.lib().radmm_generate_dechirp_operator(self._h, q, M, K, _dptr(pix), _dptr(tx),
                                                              _dptr(rx), _dptr(phi), fc, bw, pulse))
        self.rows[q] = M * K

    def generate_echo_operator(self, q: int, grid, sensor, waveform, k_samples: int | None = None) -> None:
        """ForwardOperator::dense(EchoKernel(grid, sensor, waveform))
        (forward_model.hpp:32-114) assembled on the device (complex64).
        ``grid``/``sensor``/``waveform``: scenario.SceneGrid / SensorArray /
        Waveform; K defaults to the reference's derive_sample_count."""
        from . import scenario as _sc
        k = int(k_samples) if k_samples is not None else _sc.derive_sample_count(grid, sensor, waveform)
        pix = np.ascontiguousarray(grid.centers(), dtype=np.float64)
        tx = np.ascontiguousarray(sensor.tx_position, dtype=np.float64)
        rx = np.ascontiguousarray(np.asarray(sensor.rx_positions, dtype=np.float64).reshape(-1, 3))
        M = rx.shape[0]
        _lib.check(_lib.lib().radmm_generate_echo_operator(self._h, q, M, k, _dptr(pix), _dptr(tx), _dptr(rx),
                                                           waveform.fc, waveform.sample_rate, waveform.chirp_rate,
                                                           waveform.pulse_duration))
        self.rows[q] = M * k

    def get_operator(self, q: int) -> np.ndarray:
        rows = self.rows[q]
        out = np.empty((self.N, rows), dtype=np.complex64)  # column-major rows x N
        return self.get_operator_into(q, out).T

    def get_operator_into(self, q: int, out: np.ndarray) -> np.ndarray:
        """Copy sensor q's device operator into ``out`` (N x rows C-contiguous
        complex64, i.e. the rows x N column-major matrix), e.g. a PinnedBuffer."""
        if out.shape != (self.N, self.rows[q]) or out.dtype != np.complex64 or not out.flags.c_contiguous:
            raise ValueError("get_operator_into: need an (N, rows) C-contiguous complex64 buffer")
        _lib.check(_lib.lib().radmm_get_operator_c64(self._h, q, out.ctypes.data_as(C.c_void_p)))
        return out

    def apply(self, q: int, x) -> np.ndarray:
        """ForwardOperator::apply (forward_model.hpp:147-160) on the GPU."""
        x = _c128(x)
        if x.shape[0] != self.N:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "ForwardOperator::apply: size mismatch")
        y = np.empty(self.rows[q], dtype=np.complex128)
        _lib.check(_lib.lib().radmm_apply_operator(self._h, q, _dptr(x), _dptr(y)))
        return y

    def apply_adjoint(self, q: int, y) -> np.ndarray:
        """ForwardOperator::apply_adjoint (forward_model.hpp:162-177) on the GPU."""
        y = _c128(y)
        if y.shape[0] != self.rows[q]:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "ForwardOperator::apply_adjoint: size mismatch")
        x = np.empty(self.N, dtype=np.complex128)
        _lib.check(_lib.lib().radmm_apply_adjoint(self._h, q, _dptr(y), _dptr(x)))
        return x

    # ---- multi-frame batches (BASELINE config 5) -------------------------
    def set_frame_measurement(self, frame: int, q: int, y) -> None:
        """Measurement of sensor q in frame `frame` (frames share this
        solver's operators; see radmm_set_frame_measurement)."""
        y = _c128(y)
        if self.rows[q] and y.shape[0] != self.rows[q]:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "Problem: measurement length mismatch")
        _lib.check(_lib.lib().radmm_set_frame_measurement(self._h, int(frame), q, y.ctypes.data_as(C.c_void_p),
                                                          _lib.PTR_HOST))

    def frame(self, f: int) -> "Solver":
        """Borrowed Solver view of frame f (result getters); owned by self."""
        h = C.c_void_p()
        _lib.check(_lib.lib().radmm_frame(self._h, int(f), C.byref(h)))
        v = Solver(self.N, self.Q, self.device, _ctx=h)
        v.rows = list(self.rows)
        v._borrowed = True
        return v

    def run_frames(self, hypers, mode: Mode = Mode.ASADMM, disable_screening: bool = False,
                   fixed_iterations: bool = False, fetch: bool = True, skip_refinement: bool = False) -> list:
        """Solve frames 0..F-1 (F = len(hypers)) in lockstep on the resident
        operators; frame f follows run(problem_f, hypers[f]) (admm.hpp:357-445)
        with its own stopping rule.  Frames that still share the full active
        set go through frame-batched fp64 tensor-core contractions with a
        different summation order (3M complex products) than the per-frame
        kernels; with the KM-space refinement of every solve the batched
        frames stop at exactly the sequential runs' iterations and sit within
        ~1e-9 of them and 2.5e-8 of the fp64 oracle after 100 iterations at
        config 5 (tests/test_gpu_fixtures.py::test_c5_batched_frames_match_oracle,
        profiles/r02_frames_c5.json).  Returns one RunResult per frame."""
        hypers = list(hypers)
        F = len(hypers)
        arr = (_lib.Hyper * F)(*[h._c() for h in hypers])
        summ = (_lib.Summary * F)()
        opts = _lib.Options(int(mode), int(bool(disable_screening)), int(bool(fixed_iterations)),
                            _lib.OBSERVER(), None, int(bool(skip_refinement)))
        _lib.check(_lib.lib().radmm_run_frames(self._h, F, arr, C.byref(opts), summ))
        out = []
        for f in range(F):
            sm = summ[f]
            res = RunResult(converged=bool(sm.converged), screening_stalled=bool(sm.screening_stalled),
                            iterations=int(sm.iterations), setup_ms=sm.setup_ms, solve_ms=sm.solve_ms,
                            kernel_launches=int(sm.kernel_launches), rebuilds=int(sm.rebuilds),
                            downdates=int(sm.downdates), refine_skipped=int(sm.refine_skipped))
            res.report.total_active_solves = int(sm.total_active_solves)
            res.report.total_bytes = int(sm.total_bytes)
            if fetch:
                self.frame(f)._fetch(res)
            out.append(res)
        return out

    def back_projection(self) -> np.ndarray:
        """back_projection (forward_model.hpp:201-220) on the resident operators
        and measurements: |sum_q A_q^H y_q| normalised to unit peak."""
        img = np.empty(self.N)
        _lib.check(_lib.lib().radmm_back_projection(self._h, _dptr(img)))
        return img

    def set_profiling(self, enabled: bool) -> None:
        _lib.check(_lib.lib().radmm_set_profiling(self._h, int(bool(enabled))))

    def phase_stats(self) -> dict:
        arr = (_lib.PhaseStat * len(_lib.PHASES))()
        _lib.check(_lib.lib().radmm_get_phase_stats(self._h, arr))
        return {name: dict(calls=int(a.calls), launches=int(a.launches), ms=float(a.total_ms),
                           bytes=float(a.bytes)) for name, a in zip(_lib.PHASES, arr)}

    def iteration_stats(self, iterations: int):
        ms = np.empty(max(1, iterations))
        ln = np.empty(max(1, iterations), dtype=np.int64)
        _lib.check(_lib.lib().radmm_get_iteration_stats(self._h, _dptr(ms), ln.ctypes.data_as(C.POINTER(C.c_int64)),
                                                        ms.size))
        return ms[:iterations], ln[:iterations]

    # ---- run -----------------------------------------------------------
    def run(self, hyper: Hyperparams, mode: Mode = Mode.ASADMM, observer=None,
            disable_screening: bool = False, fixed_iterations: bool = False,
            fetch: bool = True, skip_refinement: bool = False) -> RunResult:
        L = _lib.lib()
        hc = hyper._c()
        cb = OBSERVER_NONE = _lib.OBSERVER()
        if observer is not None:
            N, Qt = self.N, self.Q

            def _obs(_user, vp):
                v = vp.contents
                cv = lambda p: np.ctypeslib.as_array(p, shape=(2 * N,)).view(np.complex128).copy()  # noqa: E731
                sizes = list(np.ctypeslib.as_array(v.active_sizes, shape=(self.Q_total,)))
                observer(IterationView(int(v.iteration), cv(v.x_global), cv(v.s), cv(v.sigma), sizes,
                                       bool(v.converged), bool(v.screening_trigger)))

            cb = _lib.OBSERVER(_obs)
            del Qt
        opts = _lib.Options(int(mode), int(bool(disable_screening)), int(bool(fixed_iterations)), cb, None,
                            int(bool(skip_refinement)))
        summ = _lib.Summary()
        _lib.check(L.radmm_run(self._h, C.byref(hc), C.byref(opts), C.byref(summ)))
        del OBSERVER_NONE
        res = RunResult(converged=bool(summ.converged), screening_stalled=bool(summ.screening_stalled),
                        iterations=int(summ.iterations), setup_ms=summ.setup_ms, solve_ms=summ.solve_ms,
                        kernel_launches=int(summ.kernel_launches), rebuilds=int(summ.rebuilds),
                        downdates=int(summ.downdates), refine_skipped=int(summ.refine_skipped))
        res.report.total_active_solves = int(summ.total_active_solves)
        res.report.total_bytes = int(summ.total_bytes)
        if fetch:
            self._fetch(res)
        return res

    def _fetch(self, res: RunResult) -> None:
        L = _lib.lib()
        N = self.N
        img = np.empty(N)
        _lib.check(L.radmm_get_image(self._h, _dptr(img)))
        res.image = img

        def vec(which):
            out = np.empty(N, dtype=np.complex128)
            _lib.check(L.radmm_get_vector(self._h, which, out.ctypes.data_as(C.POINTER(C.c_double))))
            return out

        res.x_global = vec(_lib.VEC_X_GLOBAL)
        res.s = vec(_lib.VEC_S)
        res.sigma = vec(_lib.VEC_SIGMA)
        res.sigma_pre_global = vec(_lib.VEC_SIGMA_PRE_GLOBAL)
        res.sensor_images = []
        res.active_sets = []
        for q in range(self.Q):
            out = np.empty(N, dtype=np.complex128)
            _lib.check(L.radmm_get_sensor_image(self._h, q, out.ctypes.data_as(C.POINTER(C.c_double))))
            res.sensor_images.append(out)
            cnt = C.c_int()
            _lib.check(L.radmm_get_active_set(self._h, q, None, C.byref(cnt)))
            js = np.empty(cnt.value, dtype=np.int32)
            _lib.check(L.radmm_get_active_set(self._h, q, js.ctypes.data_as(C.POINTER(C.c_int32)),
                                              C.byref(cnt)))
            res.active_sets.append(js)
        n = C.c_int()
        _lib.check(L.radmm_get_record_count(self._h, C.byref(n)))
        recs = (_lib.Record * max(1, n.value))()
        _lib.check(L.radmm_get_records(self._h, recs, n.value))
        sizes = np.empty(max(1, n.value * self.Q_total), dtype=np.int32)
        _lib.check(L.radmm_get_active_sizes(self._h, sizes.ctypes.data_as(C.POINTER(C.c_int32)), sizes.size))
        res.report.iterations = []
        for k in range(n.value):
            r = recs[k]
            sz = [int(x) for x in sizes[k * self.Q_total:(k + 1) * self.Q_total]]
            res.report.iterations.append(IterationRecord(
                int(r.iteration), r.pri_res, r.dual_res, r.eps_pri, r.eps_dual, r.active_fraction,
                r.ms_elapsed, int(r.bytes_sent), sz, [contribution_size(s) for s in sz]))
        m = C.c_int()
        _lib.check(L.radmm_get_removal_log_size(self._h, C.byref(m)))
        log = np.empty(max(1, 3 * m.value), dtype=np.int32)
        _lib.check(L.radmm_get_removal_log(self._h, log.ctypes.data_as(C.POINTER(C.c_int32)), m.value))
        res.removal_log = log[:3 * m.value].reshape(m.value, 3)


def set_tuning(name: str, value: int | None) -> None:
    """Override a RADMM_* tuning switch for this
    process; ``None`` removes the override (the environment applies again)."""
    _lib.check(_lib.lib().radmm_set_tuning(name.encode(), int(value or 0), int(value is None)))


def pool_trim(device: int = 0) -> None:
    """Give the device memory of closed solvers back to the driver now
    (radmm_pool_trim): ``Solver.close()`` returns as soon as the memory is back
    in the library's pool and lets a background thread do this."""
    _lib.check(_lib.lib().radmm_pool_trim(int(device)))


class PinnedBuffer:
    """Page-locked host memory (radmm_host_alloc) viewed as a NumPy array --
    where callers stage large operators so uploads run at full host-link
    speed.  ``free()`` (or garbage collection) releases it."""

    def __init__(self, shape, dtype=np.complex64):
        dtype = np.dtype(dtype)
        n = int(np.prod(shape)) * dtype.itemsize
        p = C.c_void_p()
        _lib.check(_lib.lib().radmm_host_alloc(n, C.byref(p)))
        self._p = p
        buf = (C.c_char * n).from_address(p.value) if n else bytearray()
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def free(self) -> None:
        if getattr(self, "_p", None) is not None and self._p.value:
            self.array = None
            _lib.check(_lib.lib().radmm_host_free(self._p))
        self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def run(problem: Problem, hyper: Hyperparams, mode: Mode = Mode.ASADMM, observer=None,
        disable_screening: bool = False, *, fixed_iterations: bool = False, device: int = 0) -> RunResult:
    """run(problem, hyper, mode, observer, disable_screening) (admm.hpp:357-445)."""
    problem.validate()
    hyper.validate()
    solver = Solver.from_problem(problem, device)
    try:
        return solver.run(hyper, mode, observer, disable_screening, fixed_iterations)
    finally:
        solver.close()


def back_projection(operators, measurements, device: int = 0) -> np.ndarray:
    """back_projection(operators, measurements) (forward_model.hpp:201-220):
    the matched-filter image |sum_q A_q^H y_q| / peak, computed on the GPU."""
    ops = [op if isinstance(op, ForwardOperator) else ForwardOperator.from_matrix(op) for op in operators]
    if not ops or len(ops) != len(measurements):
        raise InvalidArgument(_lib.INVALID_ARGUMENT, "back_projection: need one measurement per operator")
    if any(op.cols() != ops[0].cols() for op in ops):
        raise InvalidArgument(_lib.INVALID_ARGUMENT, "back_projection: operators disagree on pixel count")
    solver = Solver.from_problem(Problem(ops, list(measurements)), device)
    try:
        return solver.back_projection()
    finally:
        solver.close()


# ---- solver_core.hpp --------------------------------------------------------
def soft_threshold(v, kappa: float, device: int = 0) -> np.ndarray:
    """solver_core.hpp:14-23, on the GPU."""
    v = _c128(v)
    out = np.empty_like(v)
    _lib.check(_lib.lib().radmm_soft_threshold(device, v.ctypes.data_as(C.POINTER(C.c_double)), v.shape[0],
                                               float(kappa), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


class LocalSolveCache:
    """Cached inverse of mu A^H A + beta I (solver_core.hpp:30-58)."""

    def __init__(self, a_hat, mu: float, beta: float, device: int = 0):
        a = np.asfortranarray(np.asarray(a_hat, dtype=np.complex128))
        if a.ndim != 2:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "factorize: matrix must be 2-D")
        h = C.c_void_p()
        _lib.check(_lib.lib().radmm_factorize(device, a.shape[0], a.shape[1], _dptr(a), float(mu), float(beta),
                                              C.byref(h)))
        self._h = h
        self._size = a.shape[1]

    def size(self) -> int:
        return self._size

    def solve(self, rhs) -> np.ndarray:
        rhs = _c128(rhs)
        if rhs.shape[0] != self._size:
            raise InvalidArgument(_lib.INVALID_ARGUMENT, "solve_local: rhs size does not match active set")
        out = np.empty_like(rhs)
        _lib.check(_lib.lib().radmm_solve_local(self._h, _dptr(rhs), _dptr(out)))
        return out

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.lib().radmm_solve_cache_destroy(self._h)
                self._h = None
        except Exception:
            pass


def factorize(a_hat, mu: float, beta: float) -> LocalSolveCache:
    return LocalSolveCache(a_hat, mu, beta)


def solve_local(cache: LocalSolveCache, rhs) -> np.ndarray:
    return cache.solve(rhs)


# ---- evaluation helpers (admm.hpp:450-483), host-side ------------------------
def objective_value(problem: Problem, sensor_images, mu: float, lam: float) -> float:
    if len(sensor_images) != len(problem.operators):
        raise InvalidArgument(_lib.INVALID_ARGUMENT, "objective_value: one image per sensor")
    f = 0.0
    total = np.zeros(problem.pixel_count(), dtype=np.complex128)
    for op, y, x in zip(problem.operators, problem.measurements, sensor_images):
        r = _c128(y) - op.matrix().astype(np.complex128) @ x
        f += 0.5 * mu * float(np.vdot(r, r).real)
        total = total + x
    return f + lam * float(np.abs(total).sum())


def nmse_db(estimate, truth) -> float:
    estimate, truth = np.asarray(estimate, float), np.asarray(truth, float)
    den = float(truth @ truth)
    if den == 0.0:
        raise InvalidArgument(_lib.INVALID_ARGUMENT, "nmse_db: reference image is all zero")
    e2 = float(estimate @ estimate)
    alpha = float(estimate @ truth) / e2 if e2 > 0 else 0.0
    d = alpha * estimate - truth
    return 10.0 * math.log10(float(d @ d) / den)


def relative_l2_diff(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    den = max(float(np.linalg.norm(a)), float(np.linalg.norm(b)))
    return 0.0 if den == 0.0 else float(np.linalg.norm(a - b)) / den
