"""Input generation: geometry, operators, scenes and noisy echoes.

Host-side setup for the solver (not the hot path).  Two families:

1. The reference's own scenarios, restated so their published numbers can pin
   the oracle and the CUDA path:
   * ``SceneGrid``/``SensorArray``/``Waveform``      -- geometry.hpp:19-92
   * ``echo_operator`` (EchoKernel + ForwardOperator::dense)
                                                     -- forward_model.hpp:32-114
   * ``generate_scene``                              -- scene.hpp:60-90
   * ``simulate_measurement(s)``                     -- scene.hpp:128-181
   * ``desk_scenario``/``full_scenario``             -- scenario.hpp:286-363
   * ``build_simulation``                            -- scenario.hpp:373-385
   * ``tiny_scenario``                               -- tests/fixtures.hpp:13-93
   * ``gaussian_instance``                           -- tests/acceptance.cpp:70-84

2. The BASELINE.json dechirped-LFM workloads (configs 1-5), whose geometry
   choices BASELINE leaves open are pinned here:
   ``baseline_config``/``baseline_problem`` build them on the host (numpy,
   small sizes) and the CUDA library has a bit-compatible device generator for
   the large ones.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .rng import MT19937_64, ComplexGaussian, StdNormal, mix_seed, uniform01

SPEED_OF_LIGHT = 299792458.0  # geometry.hpp:11
PI = 3.141592653589793238462643383279502884


# --------------------------------------------------------------------------
# Geometry (geometry.hpp:19-92)
# --------------------------------------------------------------------------
@dataclass
class SceneGrid:
    nx: int
    ny: int
    cell_size: float
    origin: tuple = (0.0, 0.0)

    @property
    def pixel_count(self) -> int:
        return self.nx * self.ny

    def index_of(self, ix: int, iy: int) -> int:
        return iy * self.nx + ix

    def centers(self) -> np.ndarray:
        n = np.arange(self.pixel_count)
        ix, iy = n % self.nx, n // self.nx
        return np.stack([self.origin[0] + ix * self.cell_size,
                         self.origin[1] + iy * self.cell_size,
                         np.zeros(self.pixel_count)], axis=1)

    def validate(self) -> None:
        if self.nx < 1 or self.ny < 1:
            raise ValueError("SceneGrid: nx and ny must be >= 1")
        if not self.cell_size > 0.0:
            raise ValueError("SceneGrid: cell_size must be > 0")


@dataclass
class SensorArray:
    id: int
    tx_position: tuple
    rx_positions: list

    @property
    def receiver_count(self) -> int:
        return len(self.rx_positions)

    def validate(self) -> None:
        if self.id < 1:
            raise ValueError("SensorArray: id must be >= 1")
        if not self.rx_positions:
            raise ValueError("SensorArray: needs at least one receiver")
        if len({tuple(r) for r in self.rx_positions}) != len(self.rx_positions):
            raise ValueError("SensorArray: receiver positions must be pairwise distinct")


@dataclass
class Waveform:
    fc: float
    bw: float
    pulse_duration: float
    sample_rate: float
    fast_time_samples: int = 0

    @property
    def chirp_rate(self) -> float:
        return self.bw / self.pulse_duration

    def validate(self) -> None:
        if not (self.fc > 0 and self.bw > 0 and self.pulse_duration > 0 and self.sample_rate > 0):
            raise ValueError("Waveform: parameters must be > 0")
        if self.sample_rate < self.bw:
            raise ValueError("Waveform: sample_rate must be >= bw")
        if self.fast_time_samples < 0:
            raise ValueError("Waveform: fast_time_samples must be >= 0")


def _dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    d = a - b
    return np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])


# --------------------------------------------------------------------------
# EchoKernel operator (forward_model.hpp:32-114)
# --------------------------------------------------------------------------
DENSE_BUDGET = 1 << 25  # forward_model.hpp:89


def echo_delays(grid: SceneGrid, sensor: SensorArray) -> np.ndarray:
    """tau[m, n] = (|tx - p_n| + |rx_m - p_n|) / c  (forward_model.hpp:42-47)."""
    p = grid.centers()
    tx = np.asarray(sensor.tx_position, dtype=np.float64)
    d_tx = _dist(tx[None, :], p)
    out = np.empty((sensor.receiver_count, grid.pixel_count))
    for m, rx in enumerate(sensor.rx_positions):
        d_rx = _dist(np.asarray(rx, dtype=np.float64)[None, :], p)
        out[m] = (d_tx + d_rx) / SPEED_OF_LIGHT
    return out


def derive_sample_count(grid, sensor, wf) -> int:
    """K = ceil((T + tau_max) * fs)  (forward_model.hpp:57-62)."""
    if wf.fast_time_samples > 0:
        return wf.fast_time_samples
    tau_max = float(echo_delays(grid, sensor).max())
    return int(math.ceil((wf.pulse_duration + tau_max) * wf.sample_rate))


def echo_operator(grid: SceneGrid, sensor: SensorArray, wf: Waveform,
                  entry_budget: int = DENSE_BUDGET) -> np.ndarray:
    """Dense (M*K) x N complex128 operator, row r = m*K + k.

    a(m,k,n) = exp(-j 2 pi fc tau) * exp(j pi alpha t^2) for 0 <= t <= T,
    t = k/fs - tau  (forward_model.hpp:64-71, 91-114).
    """
    grid.validate(); sensor.validate(); wf.validate()
    k_samples = derive_sample_count(grid, sensor, wf)
    rows = sensor.receiver_count * k_samples
    cols = grid.pixel_count
    if rows * cols > entry_budget:
        raise OverflowError(f"dense operator: {rows * cols} entries exceed the budget of "
                            f"{entry_budget}; use a matrix-free operator instead")
    tau = echo_delays(grid, sensor)
    a = np.zeros((rows, cols), dtype=np.complex128)
    k = np.arange(k_samples, dtype=np.float64)
    alpha = wf.chirp_rate
    for m in range(sensor.receiver_count):
        t = k[:, None] / wf.sample_rate - tau[m][None, :]
        inside = (t >= 0.0) & (t <= wf.pulse_duration)
        phase = -2.0 * PI * wf.fc * tau[m][None, :] + PI * alpha * t * t
        blk = np.where(inside, np.cos(phase) + 1j * np.sin(phase), 0.0)
        a[m * k_samples:(m + 1) * k_samples] = blk
    return a


def back_projection(ops, ys) -> np.ndarray:
    """|sum_q A_q^H y_q| normalised to unit peak (forward_model.hpp:203-220)."""
    acc = sum(np.conj(a).T @ y for a, y in zip(ops, ys))
    img = np.abs(acc)
    peak = img.max()
    return img / peak if peak > 0 else img


# --------------------------------------------------------------------------
# Scene + noise (scene.hpp:21-181)
# --------------------------------------------------------------------------
@dataclass
class TargetSpec:
    shape: list
    base_amplitude: float
    aspect_profile: dict = field(default_factory=dict)  # 1-based sensor id -> scale

    def scale_for(self, q: int) -> float:
        return self.aspect_profile.get(q, 0.0)


def generate_scene(grid: SceneGrid, targets, sensor_count: int):
    """Per-sensor reflectivities with sorted per-pixel sums (scene.hpp:60-90)."""
    n = grid.pixel_count
    per_sensor = []
    for q in range(1, sensor_count + 1):
        contrib = [[] for _ in range(n)]
        for t in targets:
            v = t.base_amplitude * t.scale_for(q)
            if v == 0.0:
                continue
            for p in t.shape:
                contrib[p].append(v)
        img = np.zeros(n)
        for p in range(n):
            acc = 0.0
            for v in sorted(contrib[p]):
                acc += v
            img[p] = acc
        per_sensor.append(img)
    composite = np.zeros(n)
    for img in per_sensor:
        composite = composite + img
    return per_sensor, composite


def simulate_measurement(a: np.ndarray, x_gt: np.ndarray, snr_db: float, seed: int):
    """y = A x + w with |Ax|^2 / E|w|^2 = 10^(snr/10)  (scene.hpp:128-157)."""
    y = a.astype(np.complex128, copy=False) @ x_gt.astype(np.complex128)
    if math.isinf(snr_db):
        return y, 0.0
    power = float(np.vdot(y, y).real)
    if power == 0.0:
        raise ValueError("simulate_measurement: zero scene has no defined SNR")
    sigma = math.sqrt(power / (a.shape[0] * 10.0 ** (snr_db / 10.0)))
    return y + sigma * ComplexGaussian(seed).draw(a.shape[0]), sigma


def simulate_measurements(ops, per_sensor, snr_db: float, base_seed: int):
    """Per-sensor seeds mix_seed(base, q), q 1-based (scene.hpp:166-181)."""
    return [simulate_measurement(a, x, snr_db, mix_seed(base_seed, q + 1))[0]
            for q, (a, x) in enumerate(zip(ops, per_sensor))]


# --------------------------------------------------------------------------
# Reference scenarios (scenario.hpp:252-385, tests/fixtures.hpp)
# --------------------------------------------------------------------------
@dataclass
class Scenario:
    name: str
    grid: SceneGrid
    waveform: Waveform
    sensors: list
    targets: list
    snr_db: float = 3.0
    seed: int = 1
    hyper: dict = field(default_factory=dict)  # overrides of Hyperparams defaults


def _rect(grid, ix0, ix1, iy0, iy1):
    return [grid.index_of(ix, iy) for iy in range(iy0, iy1 + 1) for ix in range(ix0, ix1 + 1)]


def _linear_array(sid, tx_x, half_span, receivers):
    rx = []
    for m in range(receivers):
        frac = 0.0 if receivers == 1 else 2.0 * m / float(receivers - 1) - 1.0
        rx.append((tx_x + frac * half_span, 0.0, 0.0))
    return SensorArray(sid, (tx_x, -0.05, 0.0), rx)


def desk_scenario() -> Scenario:
    """16x16 grid, Q=4, M=4, 3 GHz sweep (scenario.hpp:286-320)."""
    g = SceneGrid(16, 16, 0.20, (-1.5, 1.0))
    wf = Waveform(10e9, 3e9, 2.0e-6, 3e9, 0)
    sensors = [_linear_array(q + 1, x, 0.6, 4) for q, x in enumerate([-4.0, -1.5, 1.5, 4.0])]
    targets = [
        TargetSpec(_rect(g, 3, 5, 10, 12), 2.7, {1: 1.0, 2: 0.7, 3: 0.4}),
        TargetSpec(_rect(g, 6, 10, 5, 5), 0.54, {1: 0.6, 2: 1.0, 3: 0.5, 4: 1.0}),
        TargetSpec([g.index_of(12, 3), g.index_of(14, 3)], 1.5, {2: 0.8, 4: 0.9}),
        TargetSpec([g.index_of(13, 13)], 1.8, {1: 0.5, 3: 1.0, 4: 0.6}),
    ]
    return Scenario("desk", g, wf, sensors, targets, 3.0, 1)


def full_scenario() -> Scenario:
    """64x64 grid, Q=4, M=8, 4 GHz sweep (scenario.hpp:328-363)."""
    g = SceneGrid(64, 64, 0.05, (-1.575, 1.0))
    wf = Waveform(10e9, 4e9, 40e-9, 4e9, 0)
    sensors = [_linear_array(q + 1, x, 1.05, 8) for q, x in enumerate([-4.0, -1.5, 1.5, 4.0])]
    ell = _rect(g, 42, 43, 36, 43) + _rect(g, 44, 49, 42, 43)
    targets = [
        TargetSpec(_rect(g, 12, 16, 40, 44), 4.0, {1: 1.0, 2: 0.7, 3: 0.4}),
        TargetSpec(ell, 3.5, {2: 0.9, 3: 1.0}),
        TargetSpec(_rect(g, 24, 40, 20, 21), 3.0, {1: 0.6, 3: 0.5, 4: 1.0}),
        TargetSpec(_rect(g, 52, 53, 10, 11), 4.5, {2: 0.8, 4: 0.9}),
    ]
    return Scenario("full", g, wf, sensors, targets, 3.0, 1)


@dataclass
class Simulation:
    ops: list          # per-sensor complex128 operators (rows_q x N)
    ys: list           # per-sensor complex128 measurements
    per_sensor: list   # ground-truth real images x_q
    composite: np.ndarray


def build_simulation(sc: Scenario) -> Simulation:
    """generate_scene + build_operator + simulate_measurements (scenario.hpp:373-385)."""
    per_sensor, composite = generate_scene(sc.grid, sc.targets, len(sc.sensors))
    ops = [echo_operator(sc.grid, s, sc.waveform) for s in sc.sensors]
    ys = simulate_measurements(ops, per_sensor, sc.snr_db, sc.seed)
    return Simulation(ops, ys, per_sensor, composite)


def tiny_scenario(snr_db: float, seed: int) -> Simulation:
    """Two 2-receiver sensors over an 8x8 grid (tests/fixtures.hpp:13-93)."""
    g = SceneGrid(8, 8, 0.05, (-0.175, 1.2))
    wf = Waveform(5e9, 3e9, 30e-9, 3e9, 0)

    def sensor(sid, off):
        return SensorArray(sid, (off, -0.3, 0.0), [(off - 0.3, -0.3, 0.0), (off + 0.3, -0.3, 0.0)])

    targets = [TargetSpec([9, 10, 17, 18], 4.0, {1: 1.0, 2: 0.6}),
               TargetSpec([44, 45, 46], 3.2, {2: 1.0}),
               TargetSpec([29], 4.8, {1: 0.9, 2: 0.9})]
    sc = Scenario("tiny", g, wf, [sensor(1, -0.4), sensor(2, 0.4)], targets, snr_db, seed)
    return build_simulation(sc)


def gaussian_instance(rows: int, cols: int, q_count: int, seed: int):
    """Complex Gaussian operators and data (tests/acceptance.cpp:70-84).

    A(r,c) = (N(0,1) + jN(0,1)) / sqrt(2 rows) filled row by row from one
    persistent libstdc++ normal_distribution; y from a fresh distribution per
    vector (tests/fixtures.hpp:42-47) sharing the same engine.
    """
    rng = MT19937_64(seed)
    dist = StdNormal(rng)
    scale = math.sqrt(2.0 * rows)
    ops, ys = [], []
    for _ in range(q_count):
        a = np.empty((rows, cols), dtype=np.complex128)
        for r in range(rows):
            for c in range(cols):
                re = dist()
                im = dist()
                a[r, c] = complex(re / scale, im / scale)
        ops.append(a)
        fresh = StdNormal(rng)
        y = np.empty(rows, dtype=np.complex128)
        for i in range(rows):
            re = fresh()
            im = fresh()
            y[i] = complex(re, im)
        ys.append(y)
    return ops, ys


# --------------------------------------------------------------------------
# BASELINE.json dechirped-LFM workloads (configs 1-5)
# --------------------------------------------------------------------------
@dataclass
class BaselineConfig:
    name: str
    Q: int
    M: int
    K: int
    nside: int
    scene_size: float
    radius: float
    fc: float = 79e9
    bw: float = 1e9
    pulse: float = 50e-6
    n_targets: int = 10
    snr_db: float = 20.0
    seed: int = 1
    mu: float = 1.0
    beta: float = 1.0
    lambda_frac: float = 0.05
    eps_abs: float = 1e-4
    eps_rel: float = 1e-2
    max_iter: int = 300
    fixed_iterations: bool = True
    frame: int = 0

    @property
    def N(self) -> int:
        return self.nside * self.nside

    @property
    def KM(self) -> int:
        return self.K * self.M


def baseline_config(which: str, **overrides) -> BaselineConfig:
    """Configs of BASELINE.json (plus the builder pins recorded in DESIGN.md)."""
    table = {
        "c1": BaselineConfig("c1", Q=4, M=4, K=64, nside=32, scene_size=4.0, radius=10.0,
                             bw=1e9, n_targets=10, snr_db=20.0, max_iter=300,
                             fixed_iterations=True),
        "c2": BaselineConfig("c2", Q=8, M=8, K=256, nside=128, scene_size=8.0, radius=20.0,
                             bw=2e9, n_targets=60, snr_db=20.0, eps_abs=1e-12, eps_rel=1e-5,
                             max_iter=2000, fixed_iterations=False),
        "c3": BaselineConfig("c3", Q=32, M=16, K=512, nside=256, scene_size=16.0, radius=20.0,
                             bw=2e9, n_targets=200, snr_db=15.0, max_iter=500,
                             fixed_iterations=True),
    }
    if which in ("c4_sparse", "c4_dense"):
        base = table["c2"]
        frac = 0.001 if which == "c4_sparse" else 0.05
        cfg = BaselineConfig(**{**base.__dict__, "name": which,
                                "n_targets": int(round(frac * base.N))})
    elif which.startswith("c5"):
        cfg = BaselineConfig(**{**table["c2"].__dict__, "name": which})
    else:
        cfg = BaselineConfig(**table[which].__dict__)
    for k, v in overrides.items():
        setattr(cfg, k, v)
    return cfg


def baseline_geometry(cfg: BaselineConfig):
    """Pixel centres, tx and rx positions (builder-pinned).

    Pixels: centred square grid, n = iy*nside + ix, centre
    (-L/2 + (ix+0.5)L/nside, -L/2 + (iy+0.5)L/nside, 0).  Sensor q (0-based)
    sits on the radius-R arc at theta_q = pi*q/(Q-1); tx at the arc point;
    M receivers on a lambda/2 ULA tangential to the arc, centred on tx.
    """
    L, n = cfg.scene_size, cfg.nside
    cell = L / n
    idx = np.arange(cfg.N)
    ix, iy = idx % n, idx // n
    pix = np.stack([-L / 2 + (ix + 0.5) * cell, -L / 2 + (iy + 0.5) * cell, np.zeros(cfg.N)], axis=1)
    lam = SPEED_OF_LIGHT / cfg.fc
    tx = np.empty((cfg.Q, 3))
    rx = np.empty((cfg.Q, cfg.M, 3))
    for q in range(cfg.Q):
        th = PI * q / (cfg.Q - 1) if cfg.Q > 1 else 0.5 * PI
        c = np.array([cfg.radius * math.cos(th), cfg.radius * math.sin(th), 0.0])
        t = np.array([-math.sin(th), math.cos(th), 0.0])
        tx[q] = c
        for m in range(cfg.M):
            rx[q, m] = c + (m - 0.5 * (cfg.M - 1)) * (0.5 * lam) * t
    return pix, tx, rx


def baseline_phases(cfg: BaselineConfig, q: int) -> np.ndarray:
    """phi_qn = 2 pi u_qn, u_qn ~ U(0, 1) from stream mix_seed(seed, 1000 + q),
    returned in turns (u_qn): the generators add it to the cycle count before
    the portable sincos, so no 2 pi rounding enters the phase."""
    return uniform01(MT19937_64(mix_seed(cfg.seed, 1000 + q)), cfg.N)


# Taylor coefficients of sin(x)/x - 1 (x^2 .. x^16) and cos(x) - 1 (x^2 .. x^18);
# the CUDA generator (kernels_dense.cuh, sincos_turns) carries the same literals.
_SIN_COEF = [(-1.0) ** k / math.factorial(2 * k + 1) for k in range(1, 9)]
_COS_COEF = [(-1.0) ** k / math.factorial(2 * k) for k in range(1, 10)]
_PI_4 = 0.7853981633974483


def sincos_turns(t: np.ndarray):
    """(cos 2 pi t, sin 2 pi t) for t in [0, 1), from IEEE +, -, *, floor only.

    Octant reduction (exact: t*8 and t8 - floor(t8)) and Taylor polynomials on
    [0, pi/4] in Horner form, every operation a separately rounded fp64 op.
    The device generator performs the same operations in the same order with
    __dmul_rn/__dadd_rn (no FMA contraction), so host and device operators are
    bitwise identical on any machine -- which libm sin/cos are not -- and the
    committed oracle fixtures (tests/golden/) can be checked against operators
    generated on the GPU.  Error < 2 ulp of fp64 (tests/test_oracle_pins.py)."""
    t8 = t * 8.0
    o = np.floor(t8)
    f = t8 - o
    oi = o.astype(np.int64)
    odd = (oi & 1) == 1
    h = np.where(odd, 1.0 - f, f)
    x = h * _PI_4
    x2 = x * x
    p = np.full_like(x, _SIN_COEF[-1])
    for c in reversed(_SIN_COEF[:-1]):
        p = c + x2 * p
    sx = x + (x * x2) * p
    r = np.full_like(x, _COS_COEF[-1])
    for c in reversed(_COS_COEF[:-1]):
        r = c + x2 * r
    cx = 1.0 + x2 * r
    # angle = o pi/4 + f pi/4; odd octants use x' = (1 - f) pi/4 from the next axis
    sw = ((oi + 1) >> 1) & 1 == 1          # octants 1, 2, 5, 6: sin <-> cos
    s_abs = np.where(sw, cx, sx)
    c_abs = np.where(sw, sx, cx)
    s_neg = oi >= 4                        # octants 4..7: sin < 0
    c_neg = (oi >= 2) & (oi <= 5)          # octants 2..5: cos < 0
    return np.where(c_neg, -c_abs, c_abs), np.where(s_neg, -s_abs, s_abs)


def baseline_operator(cfg: BaselineConfig, q: int) -> np.ndarray:
    """A_q[m*K+k, n] = exp(j 2 pi (alpha tau t_k + fc tau + u_qn)), complex64.

    t_k = k T / K; the cycle count is reduced modulo one turn in fp64, the
    per-pixel phase u_qn (turns) added and reduced again, then the portable
    ``sincos_turns`` -- bitwise equal to the device generator
    (radmm_generate_dechirp_operator)."""
    pix, tx, rx = baseline_geometry(cfg)
    u = baseline_phases(cfg, q)
    alpha = cfg.bw / cfg.pulse
    tk = np.arange(cfg.K, dtype=np.float64) * (cfg.pulse / cfg.K)
    a = np.empty((cfg.KM, cfg.N), dtype=np.complex64)
    d_tx = _dist(tx[q][None, :], pix)
    for m in range(cfg.M):
        tau = (d_tx + _dist(rx[q, m][None, :], pix)) / SPEED_OF_LIGHT
        cyc = (alpha * tau)[None, :] * tk[:, None] + (cfg.fc * tau)[None, :]
        cyc = cyc - np.floor(cyc)
        t = cyc + u[None, :]
        t = t - np.floor(t)
        c, s = sincos_turns(t)
        blk = a[m * cfg.K:(m + 1) * cfg.K]
        blk.real = c.astype(np.float32)
        blk.imag = s.astype(np.float32)
    return a


def baseline_scene(cfg: BaselineConfig):
    """Targets at distinct seeded pixels; x_q[n] = U(0.5,1) * U(0.2,1).

    Stream mix_seed(seed, 2000 + 7919*frame): per target a pixel (rejecting
    repeats) and a base amplitude; then per (target, sensor) an aspect scale.
    """
    rng = MT19937_64(mix_seed(cfg.seed, 2000 + 7919 * cfg.frame))
    chosen, base = [], []
    taken = set()
    while len(chosen) < cfg.n_targets:
        p = int(uniform01(rng, 1)[0] * cfg.N)
        if p in taken:
            continue
        taken.add(p)
        chosen.append(p)
        base.append(0.5 + 0.5 * uniform01(rng, 1)[0])
    aspect = 0.2 + 0.8 * uniform01(rng, cfg.n_targets * cfg.Q).reshape(cfg.n_targets, cfg.Q)
    per_sensor = []
    for q in range(cfg.Q):
        x = np.zeros(cfg.N)
        for t, p in enumerate(chosen):
            x[p] = base[t] * aspect[t, q]
        per_sensor.append(x)
    return per_sensor


def baseline_measurements(cfg: BaselineConfig, ops, per_sensor):
    """Noise as scene.hpp:147-156 with seeds mix_seed(seed', q+1)."""
    seed = cfg.seed if cfg.frame == 0 else mix_seed(cfg.seed, 10000 + cfg.frame)
    return simulate_measurements(ops, per_sensor, cfg.snr_db, seed)


def baseline_lambda(cfg: BaselineConfig, ops, ys) -> float:
    """lambda = lambda_frac * max_q |A_q^H y_q|_inf (BASELINE.json)."""
    m = 0.0
    for a, y in zip(ops, ys):
        m = max(m, float(np.abs(np.conj(a.astype(np.complex128)).T @ y).max()))
    return cfg.lambda_frac * m


def baseline_hyper(cfg: BaselineConfig, lam: float) -> dict:
    return dict(mu=cfg.mu, lambda_=lam, beta=cfg.beta, eps_abs=cfg.eps_abs,
                eps_rel=cfg.eps_rel, screening_window=5, screening_tol=1e-5,
                max_iter=cfg.max_iter)


def baseline_problem(cfg: BaselineConfig):
    """Host-built operators (complex64), measurements (complex128), truth, hyper."""
    ops = [baseline_operator(cfg, q) for q in range(cfg.Q)]
    per_sensor = baseline_scene(cfg)
    ys = baseline_measurements(cfg, ops, per_sensor)
    lam = baseline_lambda(cfg, ops, ys)
    return ops, ys, per_sensor, baseline_hyper(cfg, lam)
