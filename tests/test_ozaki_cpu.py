"""CPU restatement of the Ozaki slicing behind the tcgen05 int8 Gram
(csrc/kernels_ozaki.cuh): per-row power-of-two scaling, seven exact int8
truncation slices, slice pairs with s1 + s2 <= 10, fp64 combination.  Checks
the representation error and the Gram error against the exact complex128
product -- no GPU involved."""
import numpy as np

S = 7
MAX_SUM = S + 3


def _slices(v):
    """v: real array with |v| < 1 -> S int8 slices (exact truncation residuals)."""
    out = []
    r = v.astype(np.float64).copy()
    for _ in range(S):
        d = np.trunc(r * 128.0)
        out.append(d.astype(np.int8))
        r = r * 128.0 - d
    return out


def _gram(a):
    rows = a.shape[0]
    m = np.maximum(np.abs(a.real), np.abs(a.imag)).max(axis=1)
    e = np.where(m > 0, np.floor(np.log2(m)).astype(int) + 1, 0)  # ilogb + 1: |v| < 1
    v = a / np.ldexp(1.0, e)[:, None]
    sr, si = _slices(v.real), _slices(v.imag)
    P = [np.concatenate([r, i], axis=1).astype(np.int64) for r, i in zip(sr, si)]
    Q = [np.concatenate([i, -r], axis=1).astype(np.int64) for r, i in zip(sr, si)]
    re = np.zeros((rows, rows))
    im = np.zeros((rows, rows))
    for t in range(2, MAX_SUM + 1):
        for s1 in range(1, S + 1):
            s2 = t - s1
            if not 1 <= s2 <= S:
                continue
            re += np.ldexp(1.0, -7 * t) * (P[s1 - 1] @ P[s2 - 1].T)
            im += np.ldexp(1.0, -7 * t) * (Q[s1 - 1] @ P[s2 - 1].T)
    scale = np.ldexp(1.0, e[:, None] + e[None, :])
    return (re + 1j * im) * scale, v, sr, si


def test_slices_represent_values_to_2_pow_minus_49():
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, size=4096) * 0.999
    d = _slices(v)
    approx = sum(x.astype(np.float64) * np.ldexp(1.0, -7 * (k + 1)) for k, x in enumerate(d))
    assert np.abs(approx - v).max() < 2.0 ** -49
    assert all(np.abs(x).max() <= 127 for x in d)


def test_sliced_gram_matches_complex128_gram():
    rng = np.random.default_rng(1)
    a = (np.exp(2j * np.pi * rng.uniform(size=(48, 700)))).astype(np.complex64)  # unit modulus, like the dechirp operator
    g, *_ = _gram(a)
    ref = a.astype(np.complex128) @ a.astype(np.complex128).conj().T
    # fp64-grade: the KM-space refinement of the dual solve takes its residual
    # with this C (a 6-slice, s1 + s2 <= 7 Gram was only ~1e-12 relative)
    assert np.abs(g - ref).max() < 1e-14 * np.abs(ref).max()
    # complex64 entries are represented exactly (24-bit mantissas within 2^-25
    # of the row maximum): the slice Gram equals the exact product's rounding
    exact = (a.astype(np.clongdouble) @ a.astype(np.clongdouble).conj().T)
    assert np.abs(g - exact).max() <= 4 * np.finfo(np.float64).eps * np.abs(ref).max()
    # the int32 pair sums cannot overflow: |sum| <= 2N * 127^2 < 2^31 for N <= 65536
    assert 2 * 65536 * 127 * 127 < 2 ** 31
