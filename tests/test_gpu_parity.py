"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle.

Mirrors the reference's own tests for this path (tests/test_solver_core.cpp,
tests/test_admm.cpp, tests/test_screening_scenario.cpp, tests/acceptance.cpp)
plus full-state / mask parity on the BASELINE configurations.

Tolerances: both sides compute in fp64 from the same complex64 operator
values, so states agree to ~1e-10 relative unless a screening decision flips
on a pixel whose criterion sits within round-off of the threshold (counted).
The north-star bar (relative L2 1e-4 on images after a fixed iteration
count) is asserted everywhere; tighter bars are asserted where no mask can
flip.
"""
import math

import numpy as np
import pytest

from oracle import admm_ref
from paper_2307_08606_b200 import api, scenario

from ._parity import compare_masks, gpu_masks, gpu_run, oracle_run, quantize, rel, state_errors

pytestmark = pytest.mark.gpu

NORTH_STAR_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _lib(built_lib):
    return built_lib


# ---- soft_threshold (test_solver_core.cpp:23-58) ------------------------------
def test_soft_threshold_analytic():
    out = api.soft_threshold(np.array([0.5, 0.1, 0.0], dtype=complex), 0.2)
    assert out[0] == 0.3 + 0j or abs(out[0] - 0.3) < 1e-16
    assert out[1] == 0 and out[2] == 0


def test_soft_threshold_phase_and_identity():
    for theta in (0.0, 0.7, 2.5, -1.2):
        out = api.soft_threshold(np.array([3.0 * np.exp(1j * theta)]), 1.0)
        assert abs(out[0] - 2.0 * np.exp(1j * theta)) < 1e-14
    v = np.array([1 - 2j, 0j])
    assert np.array_equal(api.soft_threshold(v, 0.0), v)
    with pytest.raises(api.InvalidArgument):
        api.soft_threshold(np.zeros(2, complex), -0.1)


def test_soft_threshold_matches_oracle_and_non_expansive():
    rng = np.random.default_rng(17)
    for _ in range(100):
        u = rng.normal(size=16) + 1j * rng.normal(size=16)
        v = rng.normal(size=16) + 1j * rng.normal(size=16)
        k = rng.uniform(0, 2)
        su, sv = api.soft_threshold(u, k), api.soft_threshold(v, k)
        assert np.linalg.norm(su - sv) <= np.linalg.norm(u - v) + 1e-14
        assert np.max(np.abs(su - admm_ref.soft_threshold(u, k))) < 1e-15


# ---- LocalSolveCache (test_solver_core.cpp:60-117) --------------------------------
def _q(a):
    return np.asarray(a).astype(np.complex64).astype(np.complex128)


def test_zero_matrix_solve_is_division_by_beta():
    cache = api.factorize(np.zeros((6, 4), complex), 3.0, 100.0)
    rhs = np.random.default_rng(5).normal(size=4) + 1j
    assert np.linalg.norm(cache.solve(rhs) - rhs / 100.0) < 1e-14 * np.linalg.norm(rhs)


def test_scalar_solve_closed_form():
    cache = api.factorize(np.array([[2.0 - 1.0j]]), 3.0, 100.0)
    x = cache.solve(np.array([5.0 + 4.0j]))
    assert abs(x[0] - (5 + 4j) / (3.0 * 5.0 + 100.0)) < 1e-14


@pytest.mark.parametrize("rows,cols", [(8, 5), (5, 8), (40, 25), (24, 96)])
def test_random_solves_match_inverse(rows, cols):
    rng = np.random.default_rng(23)
    a = rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))
    mu, beta = 3.0, 0.5
    cache = api.factorize(a, mu, beta)
    aq = _q(a)
    system = mu * aq.conj().T @ aq + beta * np.eye(cols)
    inv = np.linalg.inv(system)
    for _ in range(5):
        rhs = rng.normal(size=cols) + 1j * rng.normal(size=cols)
        x = cache.solve(rhs)
        assert np.linalg.norm(x - inv @ rhs) < 1e-8 * np.linalg.norm(rhs)
        assert np.linalg.norm(system @ x - rhs) < 1e-8 * np.linalg.norm(rhs)


@pytest.mark.parametrize("herm", ["0", "1", "2", "1-split"])
@pytest.mark.parametrize("rows,cols", [(130, 700), (256, 1024), (64, 65)])
def test_dual_solves_hermitian_apply(rows, cols, herm, monkeypatch):
    """Dual-form solves (cols > rows) through each G-apply variant (RADMM_HERM:
    0 full-matrix column dots, 1 lower-triangle registers, 2 lower-triangle
    TMA ring; "-split": row-segmented adjoint, 64-row segments) against the
    exact inverse; includes the C1 operator shape."""
    if herm.endswith("-split"):
        herm = herm.split("-")[0]
        monkeypatch.setenv("RADMM_ADJ_SPLIT_ROWS", "64")
        monkeypatch.setenv("RADMM_ADJ_SEG", "64")
    monkeypatch.setenv("RADMM_HERM", herm)
    monkeypatch.setenv("RADMM_HERM_MIN_ROWS", "0")  # the triangle kernels even at these small orders
    rng = np.random.default_rng(rows + cols)
    if (rows, cols) == (256, 1024):
        cfg = scenario.baseline_config("c1")
        a = scenario.baseline_operator(cfg, 0).astype(np.complex128)
        mu, beta = 1.0, 1.0
    else:
        a = rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))
        mu, beta = 3.0, 0.5
    cache = api.factorize(a, mu, beta)
    aq = _q(a)
    cap = beta * np.eye(rows) + mu * aq @ aq.conj().T
    for _ in range(3):
        rhs = rng.normal(size=cols) + 1j * rng.normal(size=cols)
        ref = (rhs - mu * aq.conj().T @ np.linalg.solve(cap, aq @ rhs)) / beta
        x = cache.solve(rhs)
        assert np.linalg.norm(x - ref) < 1e-9 * np.linalg.norm(ref), np.linalg.norm(x - ref) / np.linalg.norm(ref)


@pytest.mark.parametrize("rows,cols", [(300, 900), (700, 260)])
def test_gauss_jordan_update_kernels_bitwise_equal(rows, cols, monkeypatch):
    """The shared-memory Gauss-Jordan update (gj_update_kernel) and the general
    DMMA GEMM epilogue it replaces give bit-identical factors (dual and primal
    forms, a ragged last pivot block)."""
    rng = np.random.default_rng(rows)
    a = rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))
    rhs = rng.normal(size=cols) + 1j * rng.normal(size=cols)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("RADMM_GJ_UPDATE", flag)
        outs.append(api.factorize(a, 2.0, 0.5).solve(rhs))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("rows,cols", [(300, 1000), (256, 4096), (130, 700)])
def test_ozaki_tcgen05_gram_matches_fp64_gram(rows, cols, monkeypatch):
    """The capacitance Gram from exact int8 slices on the tcgen05 tensor cores
    (kernels_ozaki.cuh) against the fp64 DMMA Gram: solves agree far inside the
    dual form's conditioning floor (ragged row counts: padded 128-row tiles)."""
    rng = np.random.default_rng(rows + cols)
    a = (rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))).astype(np.complex64)
    rhs = rng.normal(size=cols) + 1j * rng.normal(size=cols)
    outs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RADMM_OZAKI", flag)
        outs[flag] = api.factorize(a.astype(np.complex128), 1.0, 1.0).solve(rhs)
    assert rel(outs["1"], outs["0"]) < 1e-8, rel(outs["1"], outs["0"])


@pytest.mark.parametrize("rows,cols", [(300, 1000), (256, 20000), (130, 700), (1100, 9000)])
def test_ozaki_chunked_gram_matches_fp64_gram(rows, cols, monkeypatch):
    """The chunked Gram (RADMM_OZ_CHUNK=2: 8192-pixel chunks, one CTA per tile
    walking all slice pairs, four real int8 products per stage, fp64
    accumulation across chunks; config 3's upload-time Gram) against the fp64
    DMMA Gram: one chunk, several chunks with a short last one, ragged rows."""
    rng = np.random.default_rng(rows + cols)
    a = (rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))).astype(np.complex64)
    a[:, ::7] *= 1e-3  # columns of very different magnitude: deep slices matter
    rhs = rng.normal(size=cols) + 1j * rng.normal(size=cols)
    outs = {}
    monkeypatch.setenv("RADMM_OZ_CHUNK", "2")
    for flag in ("1", "0"):
        monkeypatch.setenv("RADMM_OZAKI", flag)
        outs[flag] = api.factorize(a.astype(np.complex128), 1.0, 1.0).solve(rhs)
    assert rel(outs["1"], outs["0"]) < 1e-8, rel(outs["1"], outs["0"])
    cap = np.eye(rows) + a.astype(np.complex128) @ a.astype(np.complex128).conj().T
    ref = rhs - a.astype(np.complex128).conj().T @ np.linalg.solve(cap, a.astype(np.complex128) @ rhs)
    assert rel(outs["1"], ref) < 1e-8, rel(outs["1"], ref)


@pytest.mark.parametrize("rows,cols", [(1100, 3000), (576, 2000), (2048, 4096)])
def test_hermitian_sweep_matches_general_sweep(rows, cols, monkeypatch):
    """Packed dual factors are inverted by the Hermitian sweep (lower tiles
    only, half the DMMA work of the general Gauss-Jordan sweep): same solves
    as the general sweep + projection and as a dense LAPACK solve (ragged last
    pivot block, odd tile counts)."""
    rng = np.random.default_rng(rows)
    a = (rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))).astype(np.complex64).astype(np.complex128)
    rhs = rng.normal(size=cols) + 1j * rng.normal(size=cols)
    outs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RADMM_GJ_HERM", flag)
        outs[flag] = api.factorize(a, 0.7, 1.3).solve(rhs)
    cap = 1.3 * np.eye(rows) + 0.7 * a @ a.conj().T
    ref = (rhs - 0.7 * a.conj().T @ np.linalg.solve(cap, a @ rhs)) / 1.3
    assert rel(outs["1"], ref) < 1e-9, rel(outs["1"], ref)
    assert rel(outs["0"], ref) < 1e-9, rel(outs["0"], ref)


def test_hermitian_sweep_ill_conditioned(monkeypatch):
    """The Hermitian sweep on a capacitance of condition ~3e5 (config 2's is
    2e5): with the pivot inverses made exactly Hermitian it is as accurate as
    the general sweep (without that it diverges: |G C - I| ~ 1e3)."""
    rng = np.random.default_rng(77)
    rows, cols = 1024, 3000
    u, _, vh = np.linalg.svd(rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols)), full_matrices=False)
    a = ((u * np.logspace(2.75, 0, rows)) @ vh).astype(np.complex64).astype(np.complex128)
    rhs = rng.normal(size=cols) + 1j * rng.normal(size=cols)
    cap = np.eye(rows) + a @ a.conj().T
    ref = rhs - a.conj().T @ np.linalg.solve(cap, a @ rhs)
    errs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RADMM_GJ_HERM", flag)
        errs[flag] = rel(api.factorize(a, 1.0, 1.0).solve(rhs), ref)
    print(f"cond {np.linalg.cond(cap):.2e}: Hermitian sweep {errs['1']:.2e}, general sweep {errs['0']:.2e}")
    assert errs["1"] < 1e-8 and errs["0"] < 1e-8, errs


def test_tall_operator_dual_solve_matches_dense():
    """A dual solve on an operator taller than 4096 rows (1024-thread forward
    tiles, as at config 3) against a dense complex128 solve."""
    rng = np.random.default_rng(9)
    rows, cols, mu, beta = 4608, 5200, 1.0, 2.0
    a = (rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))).astype(np.complex64).astype(np.complex128)
    rhs = rng.normal(size=cols) + 1j * rng.normal(size=cols)
    x = api.factorize(a, mu, beta).solve(rhs)
    cap = beta * np.eye(rows) + mu * a @ a.conj().T
    ref = (rhs - mu * a.conj().T @ np.linalg.solve(cap, a @ rhs)) / beta
    assert rel(x, ref) < 1e-8, rel(x, ref)


def test_cached_solves_bitwise_reproducible():
    rng = np.random.default_rng(31)
    a = rng.normal(size=(10, 7)) + 1j * rng.normal(size=(10, 7))
    rhs = rng.normal(size=7) + 1j * rng.normal(size=7)
    c1 = api.factorize(a, 1.5, 2.0)
    first = c1.solve(rhs)
    assert np.array_equal(first, c1.solve(rhs))
    assert np.array_equal(api.factorize(a, 1.5, 2.0).solve(rhs), first)


def test_factorization_rejects_bad_input():
    with pytest.raises(api.InvalidArgument):
        api.factorize(np.zeros((2, 2)), 0.0, 1.0)
    with pytest.raises(api.InvalidArgument):
        api.factorize(np.zeros((2, 2)), 1.0, 0.0)
    bad = np.zeros((2, 2), complex)
    bad[0, 0] = np.nan
    with pytest.raises(api.InvalidArgument):
        api.factorize(bad, 1.0, 1.0)
    with pytest.raises(api.InvalidArgument):
        api.factorize(np.zeros((3, 3)), 1.0, 1.0).solve(np.zeros(4))


# ---- engine semantics (test_admm.cpp) -----------------------------------------------
def _tiny(snr, seed):
    sim = scenario.tiny_scenario(snr, seed)
    return quantize(sim.ops), sim.ys


def test_tiny_sadmm_and_asadmm_match_oracle():
    ops, ys = _tiny(3.0, 11)
    h = dict()
    for asadmm in (False, True):
        g = gpu_run(ops, ys, h, asadmm)
        o = oracle_run(ops, ys, h, asadmm)
        assert g.iterations == o.iterations and g.converged == o.converged
        errs = state_errors(g, o)
        assert max(errs.values()) < 1e-9, errs
        for rg, ro in zip(g.report.iterations, o.records):
            assert rg.active_sizes == ro.active_sizes
            assert rg.bytes_sent == ro.bytes_sent
            assert abs(rg.pri_res - ro.pri_res) <= 1e-9 * max(1.0, ro.pri_res)


def test_disabled_screening_matches_plain_mode_bitwise():
    ops, ys = _tiny(3.0, 11)
    prob = api.Problem([api.ForwardOperator.from_matrix(a) for a in ops], ys)
    h = api.Hyperparams()
    plain, accel = [], []
    rp = api.run(prob, h, api.Mode.SADMM, lambda v: plain.append((v.x_global, v.s, v.sigma)))
    ra = api.run(prob, h, api.Mode.ASADMM, lambda v: accel.append((v.x_global, v.s, v.sigma)),
                 disable_screening=True)
    assert rp.iterations == ra.iterations and len(plain) == len(accel)
    for a, b in zip(plain, accel):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    assert np.array_equal(rp.image, ra.image)


def test_converged_state_contracts():
    ops, ys = _tiny(3.0, 31)
    h = api.Hyperparams()
    prob = api.Problem([api.ForwardOperator.from_matrix(a) for a in ops], ys)
    for mode in (api.Mode.SADMM, api.Mode.ASADMM):
        r = api.run(prob, h, mode)
        assert r.converged
        last = r.report.iterations[-1]
        assert np.linalg.norm(r.s - r.x_global) <= last.eps_pri
        assert last.pri_res <= last.eps_pri and last.dual_res <= last.eps_dual
        # x_G is exactly the threshold of what it saw (test_admm.cpp:316-319)
        assert np.array_equal(api.soft_threshold(r.s + admm_ref.cdiv(r.sigma_pre_global, h.beta),
                                                 h.lambda_ / h.beta), r.x_global)
        # the aggregate is the average of the sensor images (test_admm.cpp:320-324)
        total = np.zeros_like(r.s)
        for xq in r.sensor_images:
            total = total + xq
        assert np.array_equal(admm_ref.cdiv(total, len(r.sensor_images)), r.s)


def test_iteration_cap_and_csv():
    ops, ys = _tiny(3.0, 51)
    r = gpu_run(ops, ys, dict(max_iter=3), False)
    assert not r.converged and r.iterations == 3 and len(r.report.iterations) == 3
    lines = r.report.csv().splitlines()
    assert lines[0] == "iter,pri_res,dual_res,eps_pri,eps_dual,active_frac,ms_elapsed,bytes_sent"
    assert len(lines) == 4 and all(l.count(",") == 7 for l in lines[1:])


def test_zero_measurements_collapse():
    ops, ys = _tiny(math.inf, 0)
    r = gpu_run(ops, [np.zeros_like(y) for y in ys], {}, False)
    assert r.converged and r.iterations <= 2 and np.linalg.norm(r.image) == 0.0


def test_accelerated_runs_shrink_monotonically():
    ops, ys = _tiny(3.0, 41)
    h = dict(screening_tol=1e-3)
    g = gpu_run(ops, ys, h, True)
    o = oracle_run(ops, ys, h, True)
    p = gpu_run(ops, ys, h, False)
    assert g.converged and p.converged
    for k in range(1, len(g.report.iterations)):
        for q in range(2):
            assert g.report.iterations[k].active_sizes[q] <= g.report.iterations[k - 1].active_sizes[q]
    assert g.report.iterations[-1].active_sizes != g.report.iterations[0].active_sizes
    assert g.report.total_active_solves < p.report.total_active_solves
    bad, near = compare_masks(g, o, 1e-3, 5)
    assert bad == 0, (bad, near)
    assert g.iterations == o.iterations
    assert max(state_errors(g, o).values()) < 1e-8


def test_over_aggressive_tolerance_stalls():
    ops, ys = _tiny(3.0, 41)
    h = dict(screening_tol=0.1)
    a = gpu_run(ops, ys, h, True)
    p = gpu_run(ops, ys, h, False)
    assert a.screening_stalled and a.converged
    assert all(r.active_fraction == 1.0 for r in a.report.iterations)
    assert a.iterations == p.iterations and np.array_equal(a.image, p.image)


def test_criterion4_objective():
    ops, ys = scenario.gaussian_instance(40, 25, 2, 9)
    ops64 = quantize(ops)
    h = dict(mu=2.0, lambda_=0.05, beta=1.0, eps_abs=1e-9, eps_rel=1e-7, max_iter=100000)
    g = gpu_run(ops64, ys, h, False)
    o = oracle_run(ops64, ys, h, False)
    assert g.converged and g.iterations == o.iterations
    prob_ops = [a.astype(np.complex128) for a in ops64]
    fg = admm_ref.objective_value(prob_ops, ys, g.sensor_images, 2.0, 0.05)
    fo = admm_ref.objective_value(prob_ops, ys, o.sensor_images, 2.0, 0.05)
    assert abs(fg - fo) / fo < 1e-10
    assert abs(fg - 65.584653039) / 65.584653039 < 1e-5  # published, on complex128 inputs


# ---- reference scenarios ----------------------------------------------------------
@pytest.fixture(scope="module")
def desk():
    sim = scenario.build_simulation(scenario.desk_scenario())
    return quantize(sim.ops), sim.ys, sim.composite


def test_desk_parity(desk):
    ops, ys, truth = desk
    g = gpu_run(ops, ys, {}, True)
    o = oracle_run(ops, ys, {}, True)
    assert g.iterations == o.iterations == 17
    errs = state_errors(g, o)
    assert max(errs.values()) < 1e-9, errs
    assert abs(api.nmse_db(g.image, truth) - (-13.70)) < 0.01


def test_device_echo_operator_matches_host():
    """EchoKernel::entry on the device (forward_model.hpp:64-71, dense
    assembly :91-114) against the host restatement on the reference's desk
    scenario: the same fp64 phase, sincos within an ulp, stored as complex64
    -- entries equal up to one fp32 rounding, on a vanishing fraction."""
    sc = scenario.desk_scenario()
    sim = scenario.build_simulation(sc)
    s = api.Solver(sc.grid.pixel_count, len(sc.sensors))
    try:
        for q, sensor in enumerate(sc.sensors):
            s.generate_echo_operator(q, sc.grid, sensor, sc.waveform)
            dev = s.get_operator(q)
            host = np.asarray(sim.ops[q]).astype(np.complex64)
            assert dev.shape == host.shape  # K = derive_sample_count (6142/6105/6105/6142)
            d = np.abs(dev.astype(np.complex128) - host.astype(np.complex128))
            assert d.max() <= 2.0 ** -23, d.max()
            assert np.count_nonzero(d) <= 1e-5 * d.size, np.count_nonzero(d)
    finally:
        s.close()


def test_desk_pin_with_device_built_operators():
    """The reference's published desk numbers (17 iterations, NMSE -13.70 dB,
    proj/test_output.txt:21-23) with the operators assembled on the GPU."""
    sc = scenario.desk_scenario()
    sim = scenario.build_simulation(sc)
    s = api.Solver(sc.grid.pixel_count, len(sc.sensors))
    try:
        for q, sensor in enumerate(sc.sensors):
            s.generate_echo_operator(q, sc.grid, sensor, sc.waveform)
            s.set_measurement(q, sim.ys[q])
        r = s.run(api.Hyperparams(**sc.hyper), api.Mode.ASADMM)
    finally:
        s.close()
    assert r.iterations == 17 and r.converged
    assert abs(api.nmse_db(r.image, sim.composite) - (-13.70)) < 0.01


def test_back_projection_desk(desk):
    """back_projection on the GPU (forward_model.hpp:201-220) against the host
    restatement on the same complex64 operators: the desk's published BP NMSE
    is -5.92 dB (proj/test_output.txt:21)."""
    ops, ys, truth = desk
    img = api.back_projection(ops, ys)
    ref = scenario.back_projection([a.astype(np.complex128) for a in ops], ys)
    assert rel(img, ref) < 1e-12
    assert img.max() == 1.0
    assert abs(api.nmse_db(img, truth) - (-5.92)) < 0.01
    zero = api.back_projection(ops, [np.zeros_like(y) for y in ys])
    assert not zero.any()  # an all-zero result stays all-zero
    with pytest.raises(api.InvalidArgument):
        api.back_projection(ops, ys[:-1])


def test_clean_desk_screening_parity():
    sc = scenario.desk_scenario()
    sc.snr_db = math.inf
    for t in sc.targets:
        t.base_amplitude *= 10
    sim = scenario.build_simulation(sc)
    ops = quantize(sim.ops)
    h = dict(screening_tol=1e-3)
    g = gpu_run(ops, sim.ys, h, True)
    o = oracle_run(ops, sim.ys, h, True)
    assert g.converged and not g.screening_stalled
    bad, near = compare_masks(g, o, 1e-3, 5)
    assert bad == 0, (bad, near)
    assert g.iterations == o.iterations
    assert g.report.iterations[-1].active_fraction < 0.6
    assert g.report.total_active_solves < g.iterations * 4 * 256 * 3 // 4
    assert api.nmse_db(g.image, sim.composite) < -40
    assert max(state_errors(g, o).values()) < NORTH_STAR_TOL


def test_full_scenario_dual_form_parity():
    sim = scenario.build_simulation(scenario.full_scenario())
    ops = quantize(sim.ops)
    h = dict(max_iter=8)
    g = gpu_run(ops, sim.ys, h, True, fixed_iterations=True)
    o = oracle_run(ops, sim.ys, h, True, fixed_iterations=True)
    errs = state_errors(g, o)
    assert max(errs.values()) < 1e-8, errs


# ---- BASELINE configs -------------------------------------------------------------
def test_device_generator_matches_host():
    cfg = scenario.baseline_config("c1", nside=16, K=32)
    pix, tx, rx = scenario.baseline_geometry(cfg)
    s = api.Solver(cfg.N, cfg.Q)
    for q in range(cfg.Q):
        s.generate_dechirp_operator(q, cfg.M, cfg.K, pix, tx[q], rx[q], scenario.baseline_phases(cfg, q),
                                    cfg.fc, cfg.bw, cfg.pulse)
        dev = s.get_operator(q)
        host = scenario.baseline_operator(cfg, q)
        # portable sincos (IEEE basic ops only): bitwise, not "within ulps"
        assert np.array_equal(np.ascontiguousarray(dev).view(np.uint32), np.ascontiguousarray(host).view(np.uint32))
    s.close()


@pytest.mark.parametrize("adj_split", [False, True])
def test_c1_fixed_iterations_parity(adj_split, monkeypatch):
    """adj_split forces the row-segmented adjoint (used for KM > 6144, config 3)
    with four 64-row segments."""
    if adj_split:
        monkeypatch.setenv("RADMM_ADJ_SPLIT_ROWS", "64")
        monkeypatch.setenv("RADMM_ADJ_SEG", "64")
    cfg = scenario.baseline_config("c1")
    ops, ys, _, hyper = scenario.baseline_problem(cfg)
    g = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    o = oracle_run(ops, ys, hyper, True, fixed_iterations=True)
    assert g.iterations == o.iterations == cfg.max_iter
    bad, near = compare_masks(g, o, hyper["screening_tol"], 5)
    errs = state_errors(g, o)
    print("c1 mask mismatches", bad, "near-threshold", near, "errors", errs)
    assert bad == 0
    for k in ("sensor_images", "s", "sigma", "x_global"):
        assert errs[k] < NORTH_STAR_TOL, errs


# ---- event paths: downdates, form switch, rebuild, sharded context ------------------
def _small_c1(**kw):
    cfg = scenario.baseline_config("c1", **kw)
    ops, ys, _, hyper = scenario.baseline_problem(cfg)
    return ops, ys, hyper


DOWNDATE_VARIANTS = {
    "lazy": {},                        # default: columns accumulate in P = G A_D, folded at 64
    "lazy_herm": {"RADMM_HERM_MIN_ROWS": "0"},  # up to 3 columns ride the triangle G-apply (NR = 2 / 4)
    "lazy_herm_ride1": {"RADMM_HERM_MIN_ROWS": "0", "RADMM_LAZY_RIDE": "1"},  # one rides, more in extra passes
    "lazy_herm_no_ride": {"RADMM_HERM_MIN_ROWS": "0", "RADMM_LAZY_RIDE": "0"},  # every column in extra passes
    "lazy_two_launch": {"RADMM_LAZY_FUSED": "0"},  # lazy terms as dot + axpy launches (not the cluster kernel)
    "lazy_folds": {"RADMM_LAZY_MAX": "3", "RADMM_HERM_MIN_ROWS": "0"},  # fold into G every few events
    "lazy_full_gapply": {"RADMM_HERM": "0"},  # every column through the column-dot G-apply
    "eager": {"RADMM_LAZY": "0"},      # G rewritten at every event
    "three_kernel_screen": {"RADMM_SCREEN_FUSED": "0"},  # flags / scan / scatter instead of the cluster kernel
}


@pytest.mark.parametrize("variant", list(DOWNDATE_VARIANTS))
@pytest.mark.parametrize("nside,K,tol,iters", [(16, 16, 1e-3, 150), (12, 8, 3e-3, 150), (16, 64, 1e-3, 120)])
def test_elimination_event_paths_match_oracle(nside, K, tol, iters, variant, monkeypatch):
    """Aggressive screening drives the active sets through low-rank downdates
    (lazy Woodbury columns, folds, eager rewrites), dual->primal form switches
    and large-removal rebuilds; masks and states must track the oracle at
    every step."""
    ops, ys, hyper = _small_c1(nside=nside, K=K, n_targets=4, max_iter=iters)
    hyper = dict(hyper, screening_tol=tol)
    for k, v in DOWNDATE_VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    g = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    o = oracle_run(ops, ys, hyper, True, fixed_iterations=True)
    print(f"nside={nside} K={K}: rebuilds={g.rebuilds} downdates={g.downdates} "
          f"final sizes={g.report.iterations[-1].active_sizes} rows={ops[0].shape[0]}")
    assert g.downdates + g.rebuilds > len(ops)  # events beyond the initial factorisations
    bad, near = compare_masks(g, o, tol, 5)
    assert bad == 0, (bad, near)
    for rg, ro in zip(g.report.iterations, o.records):
        assert rg.active_sizes == ro.active_sizes
    errs = state_errors(g, o)
    assert max(errs[k] for k in ("sensor_images", "sigma")) < 1e-6, errs


def test_eager_upload_gram_is_bitwise_identical(monkeypatch):
    """The full-set Gram formed right after each operator upload (overlapping
    the next sensor's upload) and scaled at run time gives the same factor,
    bit for bit, as forming beta I + mu A A^H at run time."""
    ops, ys, hyper = _small_c1(nside=16, K=16, n_targets=4, max_iter=60)
    hyper = dict(hyper, screening_tol=1e-3)
    eager = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    monkeypatch.setenv("RADMM_EAGER_GRAM", "0")
    late = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    for a, b in zip(eager.sensor_images, late.sensor_images):
        assert np.array_equal(a, b)
    assert np.array_equal(eager.sigma, late.sigma)


@pytest.mark.parametrize("nside,tol", [(100, 3e-4), (181, 1e-4)])
def test_fused_screening_equals_three_kernel_path(nside, tol, monkeypatch):
    """The one-launch cluster screening (several 1024-entry rounds per CTA,
    ragged last CTA: N = 10000 and 32761) compacts exactly like the
    flags / scan / scatter kernels: same active sets, same states bit for bit,
    and the sets track the oracle's."""
    ops, ys, hyper = _small_c1(nside=nside, K=8, n_targets=6, max_iter=40)
    hyper = dict(hyper, screening_tol=tol)
    runs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RADMM_SCREEN_FUSED", flag)
        runs[flag] = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    f, t = runs["1"], runs["0"]
    assert f.downdates + f.rebuilds > len(ops)
    for rf, rt in zip(f.report.iterations, t.report.iterations):
        assert rf.active_sizes == rt.active_sizes
    for a, b in zip(f.sensor_images, t.sensor_images):
        assert np.array_equal(a, b)
    assert np.array_equal(f.sigma, t.sigma) and np.array_equal(f.x_global, t.x_global)
    o = oracle_run(ops, ys, hyper, True, fixed_iterations=True)
    bad, near = compare_masks(f, o, hyper["screening_tol"], 5)
    assert bad == 0, (bad, near)


def test_sharded_context_world1_equals_plain():
    from paper_2307_08606_b200 import distributed as D
    ops, ys, hyper = _small_c1(nside=16, K=16, max_iter=40)
    h = api.Hyperparams(**hyper)
    plain = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    s = D.sharded_solver(ops[0].shape[1], len(ops), 0, 1, 0, None)
    for q, (a, y) in enumerate(zip(ops, ys)):
        s.set_operator(q, a)
        s.set_measurement(q, y)
    r = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
    s.close()
    assert np.array_equal(r.x_global, plain.x_global) and np.array_equal(r.sigma, plain.sigma)


def test_nccl_exchange_path_one_rank_equals_plain(monkeypatch):
    """The multi-GPU exchange path on real hardware: a one-rank NCCL
    communicator (RADMM_FORCE_NCCL) runs the same per-iteration all-gather of
    the sensor images and the fusion over the gathered buffer as a G-rank run
    does, plus the end-of-run record gather; results equal the plain
    single-GPU run bitwise."""
    from paper_2307_08606_b200 import distributed as D
    ops, ys, hyper = _small_c1(nside=16, K=16, n_targets=4, max_iter=60)
    hyper = dict(hyper, screening_tol=1e-3)
    h = api.Hyperparams(**hyper)
    plain = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    monkeypatch.setenv("RADMM_FORCE_NCCL", "1")
    s = D.sharded_solver(ops[0].shape[1], len(ops), 0, 1, 0, D.nccl_unique_id())
    for q, (a, y) in enumerate(zip(ops, ys)):
        s.set_operator(q, a)
        s.set_measurement(q, y)
    r = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
    s.close()
    assert plain.downdates + plain.rebuilds > len(ops)  # eliminations happened
    assert np.array_equal(r.x_global, plain.x_global) and np.array_equal(r.sigma, plain.sigma)
    for a, b in zip(r.sensor_images, plain.sensor_images):
        assert np.array_equal(a, b)
    assert [rec.active_sizes for rec in r.report.iterations] == [rec.active_sizes for rec in plain.report.iterations]


def test_apply_and_adjoint_match_host():
    ops, ys, hyper = _small_c1(nside=16, K=16)
    s = api.Solver(ops[0].shape[1], len(ops))
    rng = np.random.default_rng(3)
    for q, a in enumerate(ops):
        s.set_operator(q, a)
        x = rng.normal(size=a.shape[1]) + 1j * rng.normal(size=a.shape[1])
        y = rng.normal(size=a.shape[0]) + 1j * rng.normal(size=a.shape[0])
        a128 = a.astype(np.complex128)
        assert rel(s.apply(q, x), a128 @ x) < 1e-13
        assert rel(s.apply_adjoint(q, y), a128.conj().T @ y) < 1e-13
        # adjoint identity <Ax, y> = <x, A^H y> (forward_model tests, 1e-10)
        lhs, rhs = np.vdot(y, s.apply(q, x)), np.vdot(s.apply_adjoint(q, y), x)
        assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(a128 @ x) * np.linalg.norm(y)
    s.close()


@pytest.mark.parametrize("fused", ["1", "2", "3", "4", "5"])
def test_fused_sweeps_match_oracle(fused, monkeypatch):
    """The parked single-kernel sweeps (RADMM_FUSED=1..5)
    reproduce the oracle, including elimination (masks) -- on a shape every
    variant accepts (Q=4 dual sensors, KM=512, N=1024).  Only in a library
    built with RADMM_EXPERIMENTAL=1; the shipped one does not contain them."""
    from paper_2307_08606_b200 import _lib
    if not _lib.lib().radmm_build_features() & 1:
        pytest.skip("parked experiment not compiled (RADMM_EXPERIMENTAL=0)")
    ops, ys, hyper = _small_c1(nside=32, K=64, M=8, n_targets=6, max_iter=120)
    hyper = dict(hyper, screening_tol=1e-3)
    monkeypatch.setenv("RADMM_FUSED", fused)
    g = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    monkeypatch.delenv("RADMM_FUSED")
    o = oracle_run(ops, ys, hyper, True, fixed_iterations=True)
    bad, near = compare_masks(g, o, 1e-3, 5)
    assert bad == 0, (bad, near)
    errs = state_errors(g, o)
    assert max(errs[k] for k in ("sensor_images", "sigma")) < 1e-6, errs


def test_multi_frame_shared_operator_matches_oracle():
    """BASELINE config 5 at reduced size: frames with fresh targets and noise
    over the SAME operators, solved one after another on one resident problem
    (the cached full-set factor is reused after the first frame)."""
    cfg = scenario.baseline_config("c1", nside=16, K=32, n_targets=5, max_iter=60)
    ops = [scenario.baseline_operator(cfg, q) for q in range(cfg.Q)]
    s = api.Solver(cfg.N, cfg.Q)
    for q, a in enumerate(ops):
        s.set_operator(q, a)
    for frame in range(3):
        cfg.frame = frame
        per_sensor = scenario.baseline_scene(cfg)
        ys = scenario.baseline_measurements(cfg, ops, per_sensor)
        hyper = scenario.baseline_hyper(cfg, scenario.baseline_lambda(cfg, ops, ys))
        for q, y in enumerate(ys):
            s.set_measurement(q, y)
        g = s.run(api.Hyperparams(**hyper), api.Mode.ASADMM, fixed_iterations=True)
        assert g.rebuilds == (cfg.Q if frame == 0 else 0)  # factor reused from frame 1 on
        o = oracle_run(ops, ys, hyper, True, fixed_iterations=True)
        errs = state_errors(g, o)
        assert max(errs[k] for k in ("sensor_images", "sigma")) < 1e-8, (frame, errs)
    s.close()


def test_mask_replay_event_paths():
    """Mask replay: the GPU runs free; the oracle adopts the GPU's
    active set at every screening step (oracle/admm_ref.py forced_masks) and
    the iterates are compared at EVERY iteration -- sigma and the residual
    records -- so a divergence is localised to the step it appears.  The
    oracle's own decisions are reported: wherever they differ from the
    replayed ones, the pixel's zeta must sit within round-off of tol."""
    tol = 1e-3
    ops, ys, hyper = _small_c1(nside=16, K=16, n_targets=4, max_iter=120)
    hyper = dict(hyper, screening_tol=tol)
    g_sig = []
    g = gpu_run(ops, ys, hyper, True, fixed_iterations=True,
                observer=lambda v: g_sig.append(v.sigma.copy()))
    gm = gpu_masks(g, len(ops))
    active = [np.arange(ops[0].shape[1]) for _ in ops]

    def forced(k, q):
        rem = gm.get((k, q))
        if rem is not None and rem.size:
            active[q] = np.setdiff1d(active[q], rem)
        return active[q]

    o_sig = []
    o = oracle_run(ops, ys, hyper, True, fixed_iterations=True, forced_masks=forced,
                   observer=lambda k, f, s: o_sig.append(f.sigma.copy()))
    assert g.downdates + g.rebuilds > len(ops)
    assert len(g_sig) == len(o_sig) == g.iterations
    worst = max(rel(a, b) for a, b in zip(g_sig, o_sig))
    for rg, ro in zip(g.report.iterations, o.records):
        assert rg.active_sizes == ro.active_sizes
        assert abs(rg.pri_res - ro.pri_res) <= 1e-6 * max(ro.pri_res, 1e-300)
    own_diff = sum(len(set(e.own_removed.tolist()) ^ set(e.removed.tolist())) for e in o.events)
    print(f"mask replay: worst per-iteration sigma rel {worst:.2e}; own-decision differences {own_diff}")
    assert worst < 1e-6
    bad, _ = compare_masks(g, o, tol, 5)  # replayed decisions == oracle's own, up to round-off
    assert bad == 0


# ---- multi-frame batches (BASELINE config 5) ---------------------------------------
def _frames_problem(n_frames, **kw):
    cfg = scenario.baseline_config("c1", **kw)
    ops = [scenario.baseline_operator(cfg, q) for q in range(cfg.Q)]
    frames = []
    for f in range(n_frames):
        cfg.frame = f
        per = scenario.baseline_scene(cfg)
        ys = scenario.baseline_measurements(cfg, ops, per)
        frames.append((ys, scenario.baseline_hyper(cfg, scenario.baseline_lambda(cfg, ops, ys))))
    return cfg, ops, frames


@pytest.mark.parametrize("batched", [False, True])
@pytest.mark.parametrize("fixed", [True, False])
def test_frames_match_separate_runs(fixed, batched, monkeypatch):
    """run_frames (frames in lockstep on shared operators) against a separate
    run per frame.  Per-frame kernels (RADMM_FRAME_BATCH=0): every state
    vector, record and removal log bitwise equal, including frames that stop
    at different iterations.  Batched contractions (frames that still share
    the full active set go through one DMMA GEMM per operator): same
    iterations and masks, states within the oracle-parity bar (the
    degenerate BASELINE objective amplifies fp64 summation-order differences
    in s and sigma to ~1e-5 / 5e-8, exactly as between the GPU and the
    oracle in test_c1_fixed_iterations_parity)."""
    monkeypatch.setenv("RADMM_FRAME_BATCH", "1" if batched else "0")
    cfg, ops, frames = _frames_problem(3, max_iter=150 if fixed else 400)
    s = api.Solver(cfg.N, cfg.Q)
    for q in range(cfg.Q):
        s.set_operator(q, ops[q])
    for f, (ys, _) in enumerate(frames):
        for q in range(cfg.Q):
            s.set_frame_measurement(f, q, ys[q])
    hypers = [api.Hyperparams(**h) for _, h in frames]
    batch = s.run_frames(hypers, api.Mode.ASADMM, fixed_iterations=fixed)
    iters = set()
    for f, (ys, h) in enumerate(frames):
        one = gpu_run(ops, ys, h, True, fixed_iterations=fixed)
        b = batch[f]
        iters.add(b.iterations)
        assert b.iterations == one.iterations and b.converged == one.converged
        if batched:
            errs = state_errors(b, one)
            for k in ("sensor_images", "s", "sigma", "x_global"):
                assert errs[k] < NORTH_STAR_TOL, errs
            assert errs["sensor_images"] < 1e-8, errs
            assert [r.active_sizes for r in b.report.iterations] == [r.active_sizes for r in one.report.iterations]
            assert np.array_equal(np.asarray(b.removal_log), np.asarray(one.removal_log))
            continue
        for k in ("x_global", "s", "sigma", "image"):
            assert np.array_equal(getattr(b, k), getattr(one, k)), (f, k)
        for xa, xb in zip(b.sensor_images, one.sensor_images):
            assert np.array_equal(xa, xb)
        assert [r.pri_res for r in b.report.iterations] == [r.pri_res for r in one.report.iterations]
        assert [r.active_sizes for r in b.report.iterations] == [r.active_sizes for r in one.report.iterations]
        assert np.array_equal(np.asarray(b.removal_log), np.asarray(one.removal_log))
    if fixed:
        assert sum(len(x.removal_log) for x in batch) > 0  # elimination happened
    s.close()


def test_frames_reject_bad_use():
    cfg, ops, frames = _frames_problem(1)
    s = api.Solver(cfg.N, cfg.Q)
    with pytest.raises(api.InvalidArgument):  # operators first
        s.set_frame_measurement(0, 0, frames[0][0][0])
    for q in range(cfg.Q):
        s.set_operator(q, ops[q])
    s.set_frame_measurement(0, 0, frames[0][0][0])
    with pytest.raises(api.InvalidArgument):  # sensor 1 of frame 0 has no measurement
        s.run_frames([api.Hyperparams(**frames[0][1])])
    s.close()


# ---- ragged shapes and full-size properties ------------------------------------------
def _ragged_problem(seed=3, n=700, rows=(130, 256, 65, 200), n_targets=6):
    rng = np.random.default_rng(seed)
    ops = [(rng.normal(size=(r, n)) + 1j * rng.normal(size=(r, n))).astype(np.complex64) / np.sqrt(r) for r in rows]
    x = np.zeros(n)
    x[rng.choice(n, n_targets, replace=False)] = rng.uniform(0.5, 1.0, n_targets)
    ys = [a.astype(np.complex128) @ x + 0.01 * (rng.normal(size=a.shape[0]) + 1j * rng.normal(size=a.shape[0]))
          for a in ops]
    return ops, ys


@pytest.mark.parametrize("variant", ["default", "full_gapply", "adj_segments", "simt_gram"])
def test_ragged_dual_sensors_match_oracle(variant, monkeypatch):
    """Ragged sensors (KM = 130/256/65/200, N = 700: no shape a multiple of the
    64 / 128 tiles) in the dual form with elimination, through every kernel
    variant's padding paths, against the oracle at every step."""
    env = {"full_gapply": {"RADMM_HERM": "0"}, "adj_segments": {"RADMM_ADJ_SPLIT_ROWS": "64", "RADMM_ADJ_SEG": "64"},
           "simt_gram": {"RADMM_GRAM": "0", "RADMM_GEMM_BIG": "0"}}.get(variant, {})
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    ops, ys = _ragged_problem()
    # trigger at iteration ~10, then gradual elimination through dual downdates,
    # rebuilds and the dual -> primal switch (700 -> ~40 -> a few pixels)
    hyper = dict(mu=1.0, lambda_=0.05, beta=1.0, eps_abs=1e-3, eps_rel=1e-2, screening_tol=1e-4, max_iter=60)
    g = gpu_run(ops, ys, hyper, True, fixed_iterations=True)
    o = oracle_run(ops, ys, hyper, True, fixed_iterations=True)
    assert g.downdates + g.rebuilds > len(ops)  # elimination events happened
    bad, near = compare_masks(g, o, hyper["screening_tol"], 5)
    assert bad == 0, (bad, near)
    errs = state_errors(g, o)
    assert max(errs[k] for k in ("sensor_images", "sigma", "s")) < 1e-6, errs


def test_ragged_frames_batched_match_separate(monkeypatch):
    """Frame-batched contractions on ragged sensors (padding in every tile)."""
    ops, ys0 = _ragged_problem()
    frames = [ys0, _ragged_problem(seed=4)[1]]
    rng = np.random.default_rng(11)
    frames.append([y + 0.05 * (rng.normal(size=y.shape) + 1j * rng.normal(size=y.shape)) for y in ys0])
    hyper = dict(mu=1.0, lambda_=0.05, beta=1.0, eps_abs=1e-6, eps_rel=1e-4, max_iter=40)
    s = api.Solver(ops[0].shape[1], len(ops))
    for q, a in enumerate(ops):
        s.set_operator(q, a)
    for f, ys in enumerate(frames):
        for q in range(len(ops)):
            s.set_frame_measurement(f, q, ys[q])
    res = s.run_frames([api.Hyperparams(**hyper)] * len(frames), api.Mode.SADMM, fixed_iterations=True)
    for f, ys in enumerate(frames):
        one = gpu_run(ops, ys, hyper, False, fixed_iterations=True)
        errs = state_errors(res[f], one)
        assert errs["sensor_images"] < 1e-9 and errs["sigma"] < 1e-9, errs
    s.close()


@pytest.fixture(scope="module")
def c2_solver():
    cfg = scenario.baseline_config("c2")
    s = api.Solver(cfg.N, cfg.Q)
    pix, tx, rx = scenario.baseline_geometry(cfg)
    for q in range(cfg.Q):
        s.generate_dechirp_operator(q, cfg.M, cfg.K, pix, tx[q], rx[q], scenario.baseline_phases(cfg, q),
                                    cfg.fc, cfg.bw, cfg.pulse)
    xs = scenario.baseline_scene(cfg)
    ys = []
    for q in range(cfg.Q):
        y = s.apply(q, xs[q].astype(np.complex128))
        ys.append(y)
        s.set_measurement(q, y)
    yield cfg, s, ys
    s.close()


def test_c2_full_size_disabled_screening_is_sadmm(c2_solver):
    """Size-independent property at BASELINE config 2's full size: ASADMM with
    screening disabled is SADMM, bitwise (test_admm.cpp:266-288)."""
    cfg, s, _ = c2_solver
    h = api.Hyperparams(mu=1.0, lambda_=100.0, beta=1.0, eps_abs=1e-12, eps_rel=1e-5, max_iter=12)
    a = s.run(h, api.Mode.ASADMM, disable_screening=True, fixed_iterations=True)
    b = s.run(h, api.Mode.SADMM, fixed_iterations=True)
    for k in ("x_global", "s", "sigma"):
        assert np.array_equal(getattr(a, k), getattr(b, k))
    assert all(np.array_equal(x, y) for x, y in zip(a.sensor_images, b.sensor_images))


def test_c2_full_size_woodbury_solve_accuracy(c2_solver):
    """At full size (KM = 2048, N = 16384, mu sigma_max^2 / beta = 2.1e5) the
    cached solve of (mu A^H A + beta I) x = rhs (solver_core.hpp:39-51):
    forward error estimated by one step of iterative refinement < 1e-9
    relative; residual within the Woodbury form's backward-error bound
    (the dominant directions cancel to ~eps mu sigma^2 / beta: ~1e-6)."""
    cfg, s, _ = c2_solver
    a = s.get_operator(0)
    cache = api.factorize(a.astype(np.complex128), 1.0, 1.0)
    rng = np.random.default_rng(2)
    rhs = rng.normal(size=cfg.N) + 1j * rng.normal(size=cfg.N)
    x = cache.solve(rhs)
    resid = s.apply_adjoint(0, s.apply(0, x)) + x - rhs
    dx = cache.solve(resid)
    assert np.linalg.norm(dx) < 1e-9 * np.linalg.norm(x)
    assert np.linalg.norm(resid) < 1e-5 * np.linalg.norm(rhs)


def test_c2_full_size_batched_frames_agree(c2_solver, monkeypatch):
    """Two frames at full size through the frame-batched tensor-core
    contractions vs separate runs (10 iterations).  At this conditioning
    (cond(C) = 2.1e5) the dual solve's fp64 forward error is ~eps cond^2 in the
    dominant directions, so ANY change of summation order moves the iterates
    by ~1e-6: the bar is the spread between the two
    G-apply variants (full-matrix vs lower-triangle) measured here."""
    cfg, s, ys = c2_solver
    rng = np.random.default_rng(5)
    frames = [ys, [y + 1e-3 * (rng.normal(size=y.shape) + 1j * rng.normal(size=y.shape)) for y in ys]]
    for f, yf in enumerate(frames):
        for q in range(cfg.Q):
            s.set_frame_measurement(f, q, yf[q])
    h = api.Hyperparams(mu=1.0, lambda_=100.0, beta=1.0, eps_abs=1e-12, eps_rel=1e-5, max_iter=10)
    res = s.run_frames([h, h], api.Mode.ASADMM, fixed_iterations=True)
    for f, yf in enumerate(frames):
        for q in range(cfg.Q):
            s.set_measurement(q, yf[q])
        one = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
        monkeypatch.setenv("RADMM_HERM", "0")
        alt = s.run(h, api.Mode.ASADMM, fixed_iterations=True)
        monkeypatch.delenv("RADMM_HERM")
        dev, spread = state_errors(res[f], one), state_errors(alt, one)
        for k in ("sensor_images", "sigma"):
            assert dev[k] < 10 * spread[k] + 1e-12, (k, dev, spread)


def test_c2_full_size_first_iterations_match_oracle(c2_solver):
    """BASELINE config 2 at full size (8 x 2048 x 16384) against the fp64
    oracle on the same complex64 operators: the first iterations' sensor
    images, s and sigma agree to the north-star 1e-4 (DESIGN.md section 3 gives
    the fp64 conditioning floor of the Woodbury form at this size, ~1e-6 per
    solve, which is what the differences measure)."""
    cfg, s, ys = c2_solver
    for q, y in enumerate(ys):  # earlier tests on this fixture leave other measurements set
        s.set_measurement(q, y)
    iters = 3
    hyper = dict(mu=1.0, lambda_=100.0, beta=1.0, eps_abs=1e-12, eps_rel=1e-5, max_iter=iters)
    g = s.run(api.Hyperparams(**hyper), api.Mode.ASADMM, fixed_iterations=True)
    ops = [s.get_operator(q) for q in range(cfg.Q)]
    o = oracle_run(ops, ys, hyper, True, fixed_iterations=True)
    errs = state_errors(g, o)
    print(f"C2 full size, {iters} iterations: {errs}")
    assert g.iterations == o.iterations == iters
    for k in ("sensor_images", "s", "sigma"):
        assert errs[k] < 1e-4, errs  # measured ~1e-5 (tools/c2_oracle_diag.py: 6.4e-6 / 4.5e-6 / 1.2e-5)
    for rg, ro in zip(g.report.iterations, o.records):
        assert abs(rg.pri_res - ro.pri_res) <= 1e-6 * ro.pri_res


# ---- round-2 switches and ABI additions ------------------------------------------
def test_factor_layouts_and_tuning_api_agree_with_oracle():
    """The packed lower-tile factor (default for >= 512 rows) and the full
    column-major factor (RADMM_GPACK=0 through radmm_set_tuning) both match
    the oracle; the shipped library carries no parked experiments."""
    from paper_2307_08606_b200 import _lib
    assert _lib.lib().radmm_build_features() & 1 == 0
    cfg = scenario.baseline_config("c1", nside=32, K=128, M=4, n_targets=6, max_iter=40)  # KM = 512: packed
    ops, ys, _, hyper = scenario.baseline_problem(cfg)
    hyper = dict(hyper, screening_tol=1e-3)
    o = oracle_run(quantize(ops), ys, hyper, True, fixed_iterations=True)
    res = {}
    for gpack in (1, 0):
        api.set_tuning("RADMM_GPACK", gpack)
        try:
            res[gpack] = gpu_run(quantize(ops), ys, hyper, True, fixed_iterations=True)
        finally:
            api.set_tuning("RADMM_GPACK", None)
        bad, near = compare_masks(res[gpack], o, 1e-3, 5)
        assert bad == 0, (gpack, bad, near)
        errs = state_errors(res[gpack], o)
        assert errs["sensor_images"] < 1e-8, (gpack, errs)
    assert rel(np.concatenate(res[0].sensor_images), np.concatenate(res[1].sensor_images)) < 1e-9


def test_pinned_host_buffer_feeds_the_solver():
    """api.PinnedBuffer (radmm_host_alloc): page-locked operators upload and
    solve exactly like pageable ones."""
    cfg = scenario.baseline_config("c1", nside=16, K=32, n_targets=4, max_iter=15)
    ops, ys, _, hyper = scenario.baseline_problem(cfg)
    buf = api.PinnedBuffer((cfg.Q, cfg.N, cfg.KM), np.complex64)
    try:
        for q, a in enumerate(ops):
            buf.array[q][:] = np.asarray(a).T
        pinned = gpu_run([buf.array[q].T for q in range(cfg.Q)], ys, hyper, True, fixed_iterations=True)
        plain = gpu_run(quantize(ops), ys, hyper, True, fixed_iterations=True)
    finally:
        buf.free()
    assert np.array_equal(np.concatenate(pinned.sensor_images), np.concatenate(plain.sensor_images))


def test_transport_timeout_setter_and_validation():
    """radmm_set_transport_timeout (run_distributed's tcp_timeout_ms): accepted
    on a sharded context, rejected when < 1 ms."""
    from paper_2307_08606_b200 import _lib, distributed as D
    import ctypes as C
    s = D.sharded_solver(64, 2, 0, 1, 0, D.nccl_unique_id(), tcp_timeout_ms=5000)
    try:
        with pytest.raises(api.InvalidArgument):
            _lib.check(_lib.lib().radmm_set_transport_timeout(s._h, 0))
    finally:
        s.close()
    del C


def test_sharded_observer_run_sees_every_iteration(monkeypatch):
    """Observer runs of a sharded context take the per-iteration metadata
    all-gather (pinned double-buffered slots): the views and records equal the
    plain run's, eliminations included."""
    from paper_2307_08606_b200 import distributed as D
    ops, ys, hyper = _small_c1(nside=16, K=16, n_targets=4, max_iter=40)
    hyper = dict(hyper, screening_tol=1e-3)
    h = api.Hyperparams(**hyper)
    seen_plain, seen_sharded = [], []
    plain = api.Solver(ops[0].shape[1], len(ops))
    try:
        for q, (a, y) in enumerate(zip(ops, ys)):
            plain.set_operator(q, a)
            plain.set_measurement(q, y)
        rp = plain.run(h, api.Mode.ASADMM, observer=lambda v: seen_plain.append(list(v.active_sizes)),
                       fixed_iterations=True)
    finally:
        plain.close()
    monkeypatch.setenv("RADMM_FORCE_NCCL", "1")
    s = D.sharded_solver(ops[0].shape[1], len(ops), 0, 1, 0, D.nccl_unique_id())
    try:
        for q, (a, y) in enumerate(zip(ops, ys)):
            s.set_operator(q, a)
            s.set_measurement(q, y)
        rs = s.run(h, api.Mode.ASADMM, observer=lambda v: seen_sharded.append(list(v.active_sizes)),
                   fixed_iterations=True)
    finally:
        s.close()
    assert seen_sharded == seen_plain and len(seen_plain) == 40
    assert any(sz != seen_plain[0] for sz in seen_plain)  # eliminations happened
    assert [r.bytes_sent for r in rs.report.iterations] == [r.bytes_sent for r in rp.report.iterations]
    assert np.array_equal(rs.sigma, rp.sigma)


def test_pool_trim_returns_memory_after_close():
    """Solver.close() hands the device memory back to the library's pool and a
    background thread returns it to the driver; api.pool_trim() waits for that
    and trims synchronously, after which the driver sees the memory free."""
    import torch
    rng = np.random.default_rng(5)
    n, rows, q = 4096, 1024, 24  # ~0.8 GB of operators
    s = api.Solver(n, q)
    a = (rng.normal(size=(rows, n)) + 1j * rng.normal(size=(rows, n))).astype(np.complex64)
    for i in range(q):
        s.set_operator(i, a)
    used_free, _ = torch.cuda.mem_get_info()
    s.close()
    api.set_tuning("RADMM_POOL_KEEP_GB", 0)
    try:
        api.pool_trim(0)
        free_after, _ = torch.cuda.mem_get_info()
    finally:
        api.set_tuning("RADMM_POOL_KEEP_GB", None)
    assert free_after - used_free > 0.5 * q * a.nbytes, (used_free, free_after)
