"""CPU oracle: fp64 NumPy/SciPy restatement of the reference ASADMM engine.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2307_08606_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, as the checker and as
the timed CPU baseline -- never as the product path.

It restates, statement by statement, the reference engine
(``/root/reference/proj/include/radmm``):

* ``soft_threshold``        -- solver_core.hpp:14-23
* ``LocalSolve``            -- LocalSolveCache, solver_core.hpp:30-58.  The
  reference factors the N_q x N_q matrix mu*A^H A + beta*I with LLT.  For
  wide active sets (N_q > rows) the identical linear system is solved through
  the rows x rows capacitance beta*I + mu*A A^H (Woodbury identity); both
  forms use LAPACK Cholesky (zpotrf/zpotrs).  The form is selected per
  rebuild, like the CUDA path.
* ``SensorRef``             -- SensorCore, admm.hpp:88-192
* ``FusionRef``             -- FusionCore, admm.hpp:197-282
* ``run``                   -- run(), admm.hpp:357-445
* ``objective_value``/``nmse_db``/``relative_l2_diff`` -- admm.hpp:450-483
* wire sizes                -- wire.hpp:54-63

Build-only additions (off by default, never change the reference semantics
when off): ``fixed_iterations`` (do not stop on convergence) and
``forced_masks`` (mask replay: adopt externally supplied active sets at each
screening step and report where the oracle's own decision differs and by how
much |zeta - tol|).

Parity pins: tests/test_oracle_pins.py checks this module against every
published number of the reference for this path (proj/test_output.txt:21-27,
tests/test_screening_scenario.cpp:14-35, tests/test_admm.cpp, ...).
"""
from __future__ import annotations

import math
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla


@dataclass
class Hyper:
    """Hyperparams, admm.hpp:31-58 (defaults :32-39)."""
    mu: float = 3.0
    lambda_: float = 20.0
    beta: float = 100.0
    eps_abs: float = 1e-4
    eps_rel: float = 1e-2
    screening_window: int = 5
    screening_tol: float = 1e-5
    max_iter: int = 1000

    def validate(self) -> None:  # admm.hpp:41-57
        if not self.mu > 0.0:
            raise ValueError("Hyperparams: mu must be > 0")
        if not self.lambda_ >= 0.0:
            raise ValueError("Hyperparams: lambda must be >= 0")
        if not self.beta > 0.0:
            raise ValueError("Hyperparams: beta must be > 0")
        if not self.eps_abs > 0.0:
            raise ValueError("Hyperparams: eps_abs must be > 0")
        if not self.eps_rel > 0.0:
            raise ValueError("Hyperparams: eps_rel must be > 0")
        if self.screening_window < 2:
            raise ValueError("Hyperparams: screening_window needs at least one successive pair")
        if not self.screening_tol >= 0.0:
            raise ValueError("Hyperparams: screening_tol must be >= 0")
        if self.max_iter < 1:
            raise ValueError("Hyperparams: max_iter must be >= 1")


def contribution_size(n: int) -> int:  # wire.hpp:54-56
    return 1 + 4 + 8 + 4 + n * (4 + 16)


def notice_size(n: int) -> int:  # wire.hpp:60-62
    return 1 + 4 + 8 + 4 + n * (4 + 16)


def cdiv(v: np.ndarray, d: float) -> np.ndarray:
    """complex / real the way std::complex<double> / double does it: each
    component divided by d.  (NumPy's complex division multiplies by the
    reciprocal, which is not the reference's rounding.)"""
    v = np.ascontiguousarray(v, dtype=np.complex128)
    return (v.view(np.float64) / d).view(np.complex128)


def soft_threshold(v: np.ndarray, kappa: float) -> np.ndarray:
    """out_i = mag > kappa ? v_i (1 - kappa/mag) : 0  (solver_core.hpp:14-23)."""
    if not kappa >= 0.0:
        raise ValueError("soft_threshold: kappa must be >= 0")
    mag = np.abs(v)
    out = np.zeros_like(v)
    m = mag > kappa
    out[m] = v[m] * (1.0 - kappa / mag[m])
    return out


class LocalSolve:
    """LocalSolveCache (solver_core.hpp:30-58), primal or Woodbury form."""

    def __init__(self, a_hat: np.ndarray, mu: float, beta: float, form: str = "auto"):
        if not mu > 0.0:
            raise ValueError("factorize: mu must be > 0")
        if not beta > 0.0:
            raise ValueError("factorize: beta must be > 0")
        if not np.all(np.isfinite(a_hat)):
            raise ValueError("factorize: matrix has non-finite entries")
        rows, nq = a_hat.shape
        if form == "auto":
            form = "primal" if nq <= rows else "dual"
        self.form, self.size, self.mu, self.beta = form, nq, mu, beta
        self.a_hat = a_hat
        # A_hat^H kept contiguous once (speed only: NumPy would otherwise
        # materialise the conjugate transpose on every solve)
        self.a_hat_h = np.ascontiguousarray(a_hat.conj().T) if form == "dual" else None
        if form == "primal":
            gram = mu * (a_hat.conj().T @ a_hat)       # solver_core.hpp:39
            gram[np.diag_indices(nq)] += beta           # :40
            self.fac = sla.cho_factor(gram, lower=True, check_finite=False)
        else:
            cap = mu * (a_hat @ a_hat.conj().T)
            cap[np.diag_indices(rows)] += beta
            self.fac = sla.cho_factor(cap, lower=True, check_finite=False)

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        if rhs.shape[0] != self.size:
            raise ValueError("solve_local: rhs size does not match active set")
        if self.form == "primal":
            return sla.cho_solve(self.fac, rhs, check_finite=False)
        v = self.a_hat @ rhs
        w = sla.cho_solve(self.fac, v, check_finite=False)
        return cdiv(rhs - self.mu * (self.a_hat_h @ w), self.beta)


class SensorRef:
    """SensorCore (admm.hpp:88-192)."""

    def __init__(self, a: np.ndarray, y: np.ndarray, hyper: Hyper, form: str = "auto"):
        self.a = a
        self.y = y
        self.h = hyper
        self.form = form
        n = a.shape[1]
        self.n = n
        self.active = np.arange(n)                         # :99-100
        self.x_full = np.zeros(n, dtype=np.complex128)     # :101
        self.x_hat = np.zeros(n, dtype=np.complex128)      # :102
        self.history = deque([self.x_full.copy()])         # :103-104
        self.stalled = False
        self.last_zeta = None
        self.rebuild()                                     # :106

    def local_update(self, gap: np.ndarray, sigma: np.ndarray) -> None:
        """admm.hpp:111-126."""
        beta = self.h.beta
        j = self.active
        rhs = self.data + beta * gap[j] + beta * self.x_hat - sigma[j]
        self.x_hat = self.cache.solve(rhs)
        self.x_full[j] = self.x_hat
        self.history.append(self.x_full.copy())
        if len(self.history) > self.h.screening_window + 1:
            self.history.popleft()

    def zeta(self) -> np.ndarray | None:
        """Mean |change| over the last W steps for active pixels (admm.hpp:140-144)."""
        w = self.h.screening_window
        if len(self.history) < w + 1:
            return None
        j = self.active
        z = np.zeros(j.size)
        hist = self.history
        for h in range(len(hist) - w, len(hist)):
            z += np.abs(hist[h][j] - hist[h - 1][j])
        return z / float(w)

    def screen(self, forced_keep: np.ndarray | None = None):
        """admm.hpp:134-159.  ``forced_keep`` (mask replay) overrides the keep set."""
        z = self.zeta()
        self.last_zeta = z
        if z is None:
            return np.empty(0, dtype=np.int64)
        keep_mask = z >= self.h.screening_tol
        if forced_keep is not None:
            keep_mask = np.isin(self.active, forced_keep)
        removed = self.active[~keep_mask]
        if removed.size == 0:
            return removed
        if not keep_mask.any():
            self.stalled = True
            return np.empty(0, dtype=np.int64)
        self.active = self.active[keep_mask]
        self.x_hat = self.x_full[self.active].copy()
        self.rebuild()
        return removed

    def rebuild(self) -> None:
        """admm.hpp:171-179."""
        j = self.active
        a_hat = self.a if j.size == self.n else self.a[:, j]   # (no copy while every pixel is active)
        frozen = self.x_full.copy()
        frozen[j] = 0.0
        y_eff = self.y - self.a @ frozen
        self.data = self.h.mu * (a_hat.conj().T @ y_eff)
        self.cache = LocalSolve(a_hat, self.h.mu, self.h.beta, self.form)


class FusionRef:
    """FusionCore (admm.hpp:197-282)."""

    def __init__(self, n: int, q_count: int, hyper: Hyper):
        self.h = hyper
        self.n = n
        self.contrib = [np.zeros(n, dtype=np.complex128) for _ in range(q_count)]
        z = lambda: np.zeros(n, dtype=np.complex128)  # noqa: E731
        self.s, self.x_g, self.x_g_prev = z(), z(), z()
        self.sigma, self.sigma_pre, self.gap = z(), z(), z()
        self.iteration = 0
        self.has_prev = False
        self.pri = self.dual = self.eps_pri = self.eps_dual = 0.0
        self.converged = self.trigger = False

    def set_contribution(self, sensor_id: int, idx: np.ndarray, values: np.ndarray) -> None:
        if sensor_id < 1 or sensor_id > len(self.contrib):
            raise ValueError("FusionCore: sensor id out of range")
        self.contrib[sensor_id - 1][idx] = values

    def round(self) -> None:
        """admm.hpp:236-258."""
        h = self.h
        self.iteration += 1
        s = np.zeros(self.n, dtype=np.complex128)
        for c in self.contrib:            # fixed sensor order
            s = s + c
        s = cdiv(s, float(len(self.contrib)))
        self.s = s
        self.x_g_prev = self.x_g
        self.sigma_pre = self.sigma
        self.x_g = soft_threshold(s + cdiv(self.sigma, h.beta), h.lambda_ / h.beta)
        eta = s - self.x_g
        self.pri = float(np.linalg.norm(eta))
        self.dual = h.beta * float(np.linalg.norm(self.x_g - self.x_g_prev))
        self.sigma = self.sigma + h.beta * eta
        root_n = math.sqrt(float(self.n))
        self.eps_pri = root_n * h.eps_abs + h.eps_rel * max(float(np.linalg.norm(s)),
                                                             float(np.linalg.norm(self.x_g)))
        self.eps_dual = root_n * h.eps_abs + h.eps_rel * float(np.linalg.norm(self.sigma))
        self.trigger = self.pri <= self.eps_pri
        self.converged = self.has_prev and self.trigger and self.dual <= self.eps_dual
        self.has_prev = True
        self.gap = self.x_g - s


@dataclass
class Record:
    """IterationRecord (admm.hpp:284-295)."""
    iteration: int
    pri_res: float
    dual_res: float
    eps_pri: float
    eps_dual: float
    active_fraction: float
    ms_elapsed: float
    bytes_sent: int
    active_sizes: list
    sensor_bytes: list


@dataclass
class ScreenEvent:
    """Oracle-side log of one screening step (for mask parity)."""
    iteration: int
    sensor: int
    active_before: np.ndarray
    zeta: np.ndarray | None
    removed: np.ndarray
    own_removed: np.ndarray


@dataclass
class Result:
    """RunResult (admm.hpp:324-335) plus oracle-side screening logs."""
    image: np.ndarray
    x_global: np.ndarray
    s: np.ndarray
    sigma: np.ndarray
    sigma_pre_global: np.ndarray
    sensor_images: list
    converged: bool
    screening_stalled: bool
    iterations: int
    records: list
    total_active_solves: int
    total_bytes: int
    events: list = field(default_factory=list)
    masks: list = field(default_factory=list)   # masks[k-1][q] = active set after screening at k


def run(ops, ys, hyper: Hyper, asadmm: bool = True, observer=None,
        disable_screening: bool = False, fixed_iterations: bool = False,
        forced_masks=None, form: str = "auto", keep_masks: bool = False) -> Result:
    """run() (admm.hpp:357-445).

    ops: per-sensor (rows_q x N) complex arrays (promoted to complex128);
    ys: per-sensor complex measurements.  ``forced_masks(k, q)`` may return the
    active set to adopt when screening runs at iteration k (mask replay).
    """
    if not ops or len(ops) != len(ys):
        raise ValueError("Problem: one measurement per operator")
    n = ops[0].shape[1]
    for a, y in zip(ops, ys):
        if a.shape[1] != n:
            raise ValueError("Problem: operators disagree on pixel count")
        if y.shape[0] != a.shape[0]:
            raise ValueError("Problem: measurement length mismatch")
    hyper.validate()
    q_count = len(ops)
    sensors = [SensorRef(np.asarray(a, dtype=np.complex128), np.asarray(y, dtype=np.complex128),
                         hyper, form) for a, y in zip(ops, ys)]
    fusion = FusionRef(n, q_count, hyper)
    records, events, masks = [], [], []
    total_solves = total_bytes = 0
    t0 = time.perf_counter()
    staged_trigger = False
    iterations = 0
    converged = False
    for k in range(1, hyper.max_iter + 1):
        notice_bytes = 0
        if asadmm and not disable_screening and staged_trigger:      # :380-386
            for q, sensor in enumerate(sensors):
                before = sensor.active.copy()
                forced = forced_masks(k, q) if forced_masks is not None else None
                removed = sensor.screen(forced)
                own = np.empty(0, dtype=np.int64)
                if sensor.last_zeta is not None:
                    own = before[sensor.last_zeta < hyper.screening_tol]
                events.append(ScreenEvent(k, q, before, sensor.last_zeta, removed, own))
                if removed.size:
                    notice_bytes += notice_size(removed.size)
        for sensor in sensors:                                        # :389-390
            sensor.local_update(fusion.gap, fusion.sigma)
        for q, sensor in enumerate(sensors):                          # :391-394
            fusion.set_contribution(q + 1, sensor.active, sensor.x_hat)
        fusion.round()                                                # :395
        sizes = [int(s.active.size) for s in sensors]
        sbytes = [contribution_size(sz) for sz in sizes]
        rec = Record(k, fusion.pri, fusion.dual, fusion.eps_pri, fusion.eps_dual,
                     max(sizes) / n, (time.perf_counter() - t0) * 1e3,
                     notice_bytes + sum(sbytes), sizes, sbytes)
        total_solves += sum(sizes)
        total_bytes += rec.bytes_sent
        records.append(rec)
        if keep_masks:
            masks.append([s.active.copy() for s in sensors])
        if observer is not None:
            observer(k, fusion, sensors)
        iterations = k
        if fusion.converged and not fixed_iterations:
            converged = True
            break
        staged_trigger = fusion.trigger
    if fixed_iterations:
        converged = fusion.converged
    return Result(np.abs(fusion.x_g), fusion.x_g.copy(), fusion.s.copy(), fusion.sigma.copy(),
                  fusion.sigma_pre.copy(), [s.x_full.copy() for s in sensors], converged,
                  any(s.stalled for s in sensors), iterations, records, total_solves,
                  total_bytes, events, masks)


# ---------------------------------------------------------------------------
# Evaluation helpers (admm.hpp:450-483) and the reference test oracles
# (tests/oracles.hpp:18-125).
# ---------------------------------------------------------------------------
def objective_value(ops, ys, sensor_images, mu: float, lam: float) -> float:
    f = 0.0
    total = np.zeros(ops[0].shape[1], dtype=np.complex128)
    for a, y, x in zip(ops, ys, sensor_images):
        r = y - a @ x
        f += 0.5 * mu * float(np.vdot(r, r).real)
        total = total + x
    return f + lam * float(np.abs(total).sum())


def nmse_db(estimate: np.ndarray, truth: np.ndarray) -> float:
    den = float(truth @ truth)
    if den == 0.0:
        raise ValueError("nmse_db: reference image is all zero")
    e2 = float(estimate @ estimate)
    alpha = float(estimate @ truth) / e2 if e2 > 0 else 0.0
    d = alpha * estimate - truth
    return 10.0 * math.log10(float(d @ d) / den)


def relative_l2_diff(a: np.ndarray, b: np.ndarray) -> float:
    den = max(float(np.linalg.norm(a)), float(np.linalg.norm(b)))
    return 0.0 if den == 0.0 else float(np.linalg.norm(a - b)) / den


def straight_line_sadmm(ops, ys, mu, lam, beta, eps_abs, eps_rel, max_iter):
    """reference_sharing_solver (tests/oracles.hpp:37-81): LU solves, no cache."""
    q_count = len(ops)
    n = ops[0].shape[1]
    x = [np.zeros(n, dtype=np.complex128) for _ in range(q_count)]
    x_g = np.zeros(n, dtype=np.complex128)
    sigma = np.zeros(n, dtype=np.complex128)
    has_prev = False
    it, conv = 0, False
    for k in range(1, max_iter + 1):
        s_prev = sum(x) / q_count
        nxt = []
        for a, y, xq in zip(ops, ys, x):
            sys = mu * (a.conj().T @ a) + beta * np.eye(n)
            rhs = mu * (a.conj().T @ y) + beta * (x_g - s_prev) + beta * xq - sigma
            nxt.append(sla.lu_solve(sla.lu_factor(sys), rhs))
        x = nxt
        s = sum(x) / q_count
        x_prev = x_g
        x_g = soft_threshold(s + cdiv(sigma, beta), lam / beta)
        pri = np.linalg.norm(s - x_g)
        dual = beta * np.linalg.norm(x_g - x_prev)
        sigma = sigma + beta * (s - x_g)
        rn = math.sqrt(n)
        ep = rn * eps_abs + eps_rel * max(np.linalg.norm(s), np.linalg.norm(x_g))
        ed = rn * eps_abs + eps_rel * np.linalg.norm(sigma)
        it = k
        if has_prev and pri <= ep and dual <= ed:
            conv = True
            break
        has_prev = True
    return it, conv, x_g


def prox_gradient_objective(ops, ys, mu, lam, iterations):
    """Long-run proximal gradient on the block objective (tests/oracles.hpp:102-125)."""
    q_count = len(ops)
    n = ops[0].shape[1]
    lip = max(mu * float(np.linalg.eigvalsh(a.conj().T @ a).max()) for a in ops)
    gamma = 1.0 / lip
    x = [np.zeros(n, dtype=np.complex128) for _ in range(q_count)]
    for _ in range(iterations):
        v = [xq - gamma * (mu * (a.conj().T @ (a @ xq - y))) for a, y, xq in zip(ops, ys, x)]
        u = sum(v)
        w = soft_threshold(u, gamma * q_count * lam)
        x = [vq + (w - u) / q_count for vq in v]
    return objective_value(ops, ys, x, mu, lam)
