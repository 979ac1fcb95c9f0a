"""CPU checks of the linear algebra behind the GPU's lazy Woodbury downdates
(kernels lazy_*_kernel in csrc/kernels_batched.cuh).

The reference refactorises mu A_J^H A_J + beta I whenever the active set J
shrinks (admm.hpp:171-179, solver_core.hpp:34-45).  The GPU keeps the inverse
G of the base capacitance C = beta I + mu A A^H and accumulates the removed
columns D:  C_D^{-1} v = G v + mu P Sinv (A_D^H G v),  P = G A_D,
Sinv = (I - mu A_D^H P)^{-1}, with Sinv grown by a bordered (Schur complement)
update per event.  These tests restate that algebra in NumPy (fp64) and check
it against a direct solve of the downdated system and against the oracle's
x-update on the same active set -- no GPU involved.
"""
import numpy as np

from oracle import admm_ref


def _border(sinv_old, a_old, a_new, p_new, mu):
    """The bordered update lazy_border_inv_kernel performs."""
    s12 = -mu * (a_old.conj().T @ p_new)
    s22 = np.eye(a_new.shape[1]) - mu * (a_new.conj().T @ p_new)
    w = sinv_old @ s12
    z = s22 - s12.conj().T @ w
    zinv = np.linalg.inv(z)
    x = w @ zinv
    d0, r = sinv_old.shape[0], a_new.shape[1]
    out = np.zeros((d0 + r, d0 + r), dtype=complex)
    out[:d0, :d0] = sinv_old + x @ w.conj().T
    out[:d0, d0:] = -x
    out[d0:, :d0] = -x.conj().T
    out[d0:, d0:] = zinv
    return out


def test_bordered_inverse_and_correction_match_direct_solve():
    rng = np.random.default_rng(7)
    km, n, mu, beta = 48, 160, 1.5, 0.7
    a = rng.normal(size=(km, n)) + 1j * rng.normal(size=(km, n))
    c = beta * np.eye(km) + mu * a @ a.conj().T
    g = np.linalg.inv(c)
    g = (g + g.conj().T) / 2  # the Hermitian projection of the GPU factor
    removed = []
    sinv = np.zeros((0, 0), dtype=complex)
    for event in ([3], [17, 40], [5], [90, 91, 120], [0]):  # r = 1 and r > 1 events
        a_old = a[:, removed]
        a_new = a[:, event]
        p_new = g @ a_new
        sinv = _border(sinv, a_old, a_new, p_new, mu)
        removed += event
        ad = a[:, removed]
        p = g @ ad
        # Sinv really is (I - mu A_D^H P)^{-1}
        direct = np.linalg.inv(np.eye(len(removed)) - mu * ad.conj().T @ p)
        assert np.abs(sinv - direct).max() < 1e-10 * np.abs(direct).max()
        # the corrected apply equals the downdated capacitance's inverse
        keep = [j for j in range(n) if j not in removed]
        ck = beta * np.eye(km) + mu * a[:, keep] @ a[:, keep].conj().T
        v = rng.normal(size=km) + 1j * rng.normal(size=km)
        u = g @ v
        w = u + mu * p @ (sinv @ (ad.conj().T @ u))
        ref = np.linalg.solve(ck, v)
        assert np.linalg.norm(w - ref) < 1e-10 * np.linalg.norm(ref)


def test_lazy_x_update_equals_oracle_local_solve():
    """x = (rhs - mu A_J^H C_J^{-1} A_J rhs) / beta with C_J^{-1} applied lazily
    equals the oracle's cached solve on the shrunken active set."""
    rng = np.random.default_rng(11)
    km, n, mu, beta = 32, 96, 3.0, 100.0  # reference defaults mu=3, beta=100 (admm.hpp:32-34)
    a = rng.normal(size=(km, n)) + 1j * rng.normal(size=(km, n))
    removed = [4, 9, 10, 50, 77]
    keep = np.array([j for j in range(n) if j not in removed])
    g = np.linalg.inv(beta * np.eye(km) + mu * a @ a.conj().T)
    ad = a[:, removed]
    p = g @ ad
    sinv = np.linalg.inv(np.eye(len(removed)) - mu * ad.conj().T @ p)
    aj = a[:, keep]
    rhs = rng.normal(size=keep.size) + 1j * rng.normal(size=keep.size)
    u = g @ (aj @ rhs)
    w = u + mu * p @ (sinv @ (ad.conj().T @ u))
    x_lazy = (rhs - mu * aj.conj().T @ w) / beta
    cache = admm_ref.LocalSolve(aj, mu, beta, form="primal")
    x_ref = cache.solve(rhs)
    assert np.linalg.norm(x_lazy - x_ref) < 1e-10 * np.linalg.norm(x_ref)
