"""CPU restatements of the two setup algorithms added for config 3
(DESIGN.md sections 3 and 9d), checked in NumPy:

* the Hermitian (symmetric) blocked Gauss-Jordan sweep that inverts the packed
  dual capacitances from their lower tiles only -- including the measured
  reason its pivot inverses must be made exactly Hermitian;
* the band-ordered tile enumeration of the chunked Ozaki Gram, and the int32
  exactness bound of its weight groups.
"""
import numpy as np

from oracle import gen
from paper_2307_08606_b200 import scenario


def herm_sweep(cap, hermitize, kb=64, bm=128, bn=64):
    """gj_invert(..., herm=true): only tiles with n0 < m0 + bm are maintained
    (the others are poisoned here to prove they are never read)."""
    n = cap.shape[0]
    m = cap.copy()
    for m0 in range(0, n, bm):
        for n0 in range(0, n, bn):
            if n0 >= m0 + bm:
                m[m0:m0 + bm, n0:n0 + bn] = np.nan
    for k0 in range(0, n, kb):
        k1 = min(n, k0 + kb)
        d = m[k0:k1, k0:k1]
        if hermitize:
            d = (d + d.conj().T) / 2
        p = np.linalg.inv(d)
        if hermitize:
            p = (p + p.conj().T) / 2
        f = np.empty((n, k1 - k0), complex)
        f[k0:] = m[k0:, k0:k1]                 # gj_hpanel_kernel: rows at / below the pivot block
        f[:k0] = m[k0:k1, :k0].conj().T        # rows above: conjugate of the pivot rows
        t = f @ p
        for m0 in range(0, n, bm):             # gj_update_kernel<true>
            for n0 in range(0, n, bn):
                if n0 < m0 + bm:
                    m[m0:m0 + bm, n0:n0 + bn] -= t[m0:m0 + bm] @ f[n0:n0 + bn].conj().T
        m[k1:, k0:k1] = t[k1:]                 # gj_hfix_kernel
        m[k0:k1, :k0] = t[:k0].conj().T
        m[k0:k1, k0:k1] = -p
    g = -np.tril(m)                            # gj_hfinish_kernel
    return g + np.tril(g, -1).conj().T


def general_sweep(cap, kb=64):
    n = cap.shape[0]
    m = cap.copy()
    for k0 in range(0, n, kb):
        k1 = min(n, k0 + kb)
        p = np.linalg.inv(m[k0:k1, k0:k1])
        f = m[:, k0:k1].copy()
        r = p @ m[k0:k1, :]
        r[:, k0:k1] = p
        m2 = m.copy()
        m2[:, k0:k1] = 0
        m2 -= f @ r
        m2[k0:k1, :] = r
        m = m2
    return m


def test_hermitian_sweep_needs_hermitian_pivot_inverses():
    cfg = scenario.baseline_config("c2")
    a = gen.baseline_operator(cfg, 0)[:512, :4096].astype(np.complex128)
    cap = np.eye(512) + a @ a.conj().T
    eye = np.eye(512)
    err = {name: np.linalg.norm(g @ cap - eye, 2)
           for name, g in (("general", general_sweep(cap)), ("hermitian", herm_sweep(cap, True)),
                           ("hermitian, raw pivots", herm_sweep(cap, False)))}
    print(f"cond {np.linalg.cond(cap):.2e}: {err}")
    assert not np.isnan(herm_sweep(cap, True)).any()  # the unmaintained upper tiles are never read
    assert err["hermitian"] < 10 * err["general"] + 1e-9
    assert err["hermitian, raw pivots"] > 20 * err["hermitian"]


def band_tile(idx, t, band=12):
    """oz_gram_chunk_kernel's blockIdx.x -> (I, J) map."""
    r0, h = 0, min(band, t)
    while True:
        cnt = h * r0 + h * (h + 1) // 2
        if idx < cnt:
            break
        idx -= cnt
        r0 += h
        h = min(band, t - r0)
    full = (r0 + 1) * h
    if idx < full:
        return r0 + idx % h, idx // h
    idx -= full
    col = 1
    while idx >= h - col:
        idx -= h - col
        col += 1
    return r0 + col + idx, r0 + col


def test_band_ordered_tiles_cover_the_lower_triangle_once():
    for t in (1, 2, 5, 12, 13, 25, 64):
        n = t * (t + 1) // 2
        got = sorted(band_tile(i, t) for i in range(n))
        assert got == sorted((i, j) for i in range(t) for j in range(i + 1)), t
    # the CTAs resident together (148 consecutive indices) share few row blocks
    # (a window inside the fifth band's full columns: rows 48..59)
    t = 64
    wave = [band_tile(i, t) for i in range(1200, 1348)]
    assert len({i for i, _ in wave}) <= 12 and len({j for _, j in wave}) <= 14
    rowmajor = [(i, j) for i in range(t) for j in range(i + 1)][1200:1348]
    assert len({j for _, j in rowmajor}) > 40


def test_weight_groups_are_exact_in_int32():
    slices, max_sum, chunk = 7, 10, 8192
    for t in range(2, max_sum + 1):
        pairs = sum(1 for s1 in range(1, slices + 1) if 1 <= t - s1 <= slices)
        assert pairs * 2 * chunk * 127 * 127 < 2 ** 31, (t, pairs)
