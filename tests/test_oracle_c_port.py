"""The compiled OpenMP operator passes used for the CPU-baseline figure
(oracle/local_update.c) against the NumPy oracle they restate."""
import numpy as np

from oracle import admm_ref, local_update as lu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_compiled_passes_match_numpy():
    rng = np.random.default_rng(3)
    rows, n = 96, 700
    a = np.asfortranarray((rng.normal(size=(rows, n)) + 1j * rng.normal(size=(rows, n))).astype(np.complex64))
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    w = rng.normal(size=rows) + 1j * rng.normal(size=rows)
    a128 = a.astype(np.complex128)
    assert rel(lu.forward(a, x), a128 @ x) < 1e-14
    assert rel(lu.adjoint(a, w), a128.conj().T @ w) < 1e-14
    cols = np.sort(rng.choice(n, 333, replace=False))
    assert rel(lu.forward(a, x[:333], cols), a128[:, cols] @ x[:333]) < 1e-14
    assert rel(lu.adjoint(a, w, cols), a128[:, cols].conj().T @ w) < 1e-14
    nmax = lu.threads()
    for t in (1, 3):  # reproducible for a given thread count, any count within rounding
        lu.set_threads(t)
        v1, v2 = lu.forward(a, x), lu.forward(a, x)
        assert np.array_equal(v1, v2) and rel(v1, a128 @ x) < 1e-14
    lu.set_threads(nmax)


def test_compiled_cholesky_solve_matches_lapack():
    import scipy.linalg as sla
    rng = np.random.default_rng(6)
    n = 150
    m = rng.normal(size=(n, 2 * n)) + 1j * rng.normal(size=(n, 2 * n))
    cap = m @ m.conj().T + np.eye(n)
    fac = sla.cho_factor(cap, lower=True)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    assert rel(lu.chol_solve(np.asfortranarray(fac[0]), b), sla.cho_solve(fac, b)) < 1e-12


def test_compiled_local_update_tracks_the_oracle():
    rng = np.random.default_rng(4)
    rows, n, q = 64, 400, 3
    h = admm_ref.Hyper(mu=1.0, lambda_=0.3, beta=1.0, max_iter=50)
    ops = [np.asfortranarray((rng.normal(size=(rows, n)) + 1j * rng.normal(size=(rows, n))).astype(np.complex64))
           for _ in range(q)]
    ys = [rng.normal(size=rows) + 1j * rng.normal(size=rows) for _ in range(q)]
    ref = [admm_ref.SensorRef(a.astype(np.complex128), y, h) for a, y in zip(ops, ys)]
    alt = [admm_ref.SensorRef(a.astype(np.complex128), y, h) for a, y in zip(ops, ys)]
    f_ref, f_alt = admm_ref.FusionRef(n, q, h), admm_ref.FusionRef(n, q, h)
    for _ in range(15):
        for s in ref:
            s.local_update(f_ref.gap, f_ref.sigma)
        for s, a in zip(alt, ops):
            lu.local_update(s, a, f_alt.gap, f_alt.sigma)
        for fus, sens in ((f_ref, ref), (f_alt, alt)):
            for k, s in enumerate(sens):
                fus.set_contribution(k + 1, s.active, s.x_hat)
            fus.round()
    assert rel(np.concatenate([s.x_hat for s in alt]), np.concatenate([s.x_hat for s in ref])) < 1e-11
    assert rel(f_alt.sigma, f_ref.sigma) < 1e-9  # sigma accumulates beta (s - x_G): a cancelling quantity
