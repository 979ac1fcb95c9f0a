"""Bit-exact random streams used by the reference's input generators.

Host-side input generation (setup, not the hot path): restates the random
number generation the reference relies on so the CUDA path and the CPU
oracle can be fed the very inputs the reference would build.

* ``MT19937_64``      -- the C++ ``std::mt19937_64`` engine (the reference
                         seeds it directly, ``scene.hpp:103-116``).
* ``mix_seed``        -- splitmix64 finaliser, ``scene.hpp:93-98``.
* ``ComplexGaussian`` -- hand Box-Muller on top of mt19937_64,
                         ``scene.hpp:103-116`` (note sqrt(-ln u1), i.e. unit
                         complex variance).
* ``StdNormal``       -- libstdc++'s ``std::normal_distribution<double>``
                         (Marsaglia polar method with a cached second
                         sample) on ``generate_canonical<double,53>``; the
                         reference tests draw their Gaussian fixtures from
                         it (``tests/fixtures.hpp:42-47``,
                         ``tests/acceptance.cpp:70-84``).

Pinned by ``tests/golden/rng_golden.json`` which ``tests/golden/gen_rng_golden.cpp``
produced with g++ 13 / libstdc++ in this container.
"""
from __future__ import annotations

import math

import numpy as np

_MASK64 = (1 << 64) - 1
_N = 312
_M = 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x7FFFFFFF)


class MT19937_64:
    """std::mt19937_64 (w=64, n=312, m=156, r=31), vectorised twist."""

    def __init__(self, seed: int = 5489):
        mt = [0] * _N
        mt[0] = seed & _MASK64
        for i in range(1, _N):
            prev = mt[i - 1]
            mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK64
        self._mt = np.array(mt, dtype=np.uint64)
        self._buf = np.empty(0, dtype=np.uint64)
        self._pos = 0

    def _twist(self) -> None:
        mt = self._mt
        one = np.uint64(1)

        def step(lo, hi, partner):
            x = (mt[lo:hi] & _UPPER) | (mt[lo + 1:hi + 1] & _LOWER)
            xa = x >> one
            xa = np.where((x & one) == one, xa ^ _MATRIX_A, xa)
            mt[lo:hi] = partner ^ xa

        # i in [0, 156): partner mt[i+156] still holds the old value.
        step(0, _M, mt[_M:_N].copy())
        # i in [156, 311): partner mt[i-156] was refreshed above.
        step(_M, _N - 1, mt[0:_N - 1 - _M].copy())
        # i = 311 wraps to mt[0] (new) and partner mt[155] (new).
        x = (int(mt[_N - 1]) & 0xFFFFFFFF80000000) | (int(mt[0]) & 0x7FFFFFFF)
        xa = x >> 1
        if x & 1:
            xa ^= 0xB5026F5AA96619E9
        mt[_N - 1] = np.uint64(int(mt[_M - 1]) ^ xa)

        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self._buf = y
        self._pos = 0

    def next_u64_array(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        filled = 0
        while filled < count:
            if self._pos >= self._buf.size:
                self._twist()
            take = min(count - filled, self._buf.size - self._pos)
            out[filled:filled + take] = self._buf[self._pos:self._pos + take]
            self._pos += take
            filled += take
        return out

    def __call__(self) -> int:
        if self._pos >= self._buf.size:
            self._twist()
        v = int(self._buf[self._pos])
        self._pos += 1
        return v


def mix_seed(base: int, stream: int) -> int:
    """splitmix64 finaliser (scene.hpp:93-98)."""
    z = (base + stream * 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


class ComplexGaussian:
    """Unit-variance circular complex Gaussian (scene.hpp:103-116).

    u1 = ((r >> 11) + 1) * 2^-53, u2 = (r >> 11) * 2^-53,
    value = polar(sqrt(-ln u1), 2*pi*u2).  Scalar libm calls (math.*) are used
    so every sample is the one glibc computes for the reference.
    """

    def __init__(self, seed: int):
        self._rng = MT19937_64(seed)

    def draw(self, count: int) -> np.ndarray:
        raw = self._rng.next_u64_array(2 * count)
        out = np.empty(count, dtype=np.complex128)
        scale = 2.0 ** -53
        two_pi = 2.0 * 3.141592653589793238462643383279502884
        for i in range(count):
            u1 = (float(int(raw[2 * i]) >> 11) + 1.0) * scale
            u2 = float(int(raw[2 * i + 1]) >> 11) * scale
            rad = math.sqrt(-math.log(u1))
            th = two_pi * u2
            out[i] = complex(rad * math.cos(th), rad * math.sin(th))
        return out


class StdNormal:
    """libstdc++ std::normal_distribution<double>(0, 1) on an mt19937_64.

    generate_canonical<double, 53>: one 64-bit draw, (double)r / 2^64, clamped
    below 1.  Marsaglia polar: x, y = 2U-1; reject r2 > 1 or r2 == 0;
    mult = sqrt(-2 ln r2 / r2); cache x*mult, return y*mult.
    """

    def __init__(self, rng: MT19937_64):
        self._rng = rng
        self._saved = None

    def reset(self) -> None:
        self._saved = None

    def _canonical(self) -> float:
        r = float(self._rng())  # rounds to nearest like the (double) cast
        v = r / 18446744073709551616.0
        if v >= 1.0:
            v = math.nextafter(1.0, 0.0)
        return v

    def __call__(self) -> float:
        if self._saved is not None:
            v = self._saved
            self._saved = None
            return v
        while True:
            x = 2.0 * self._canonical() - 1.0
            y = 2.0 * self._canonical() - 1.0
            r2 = x * x + y * y
            if not (r2 > 1.0 or r2 == 0.0):
                break
        mult = math.sqrt(-2.0 * math.log(r2) / r2)
        self._saved = x * mult
        return y * mult


def uniform01(rng: MT19937_64, count: int) -> np.ndarray:
    """53-bit uniforms in [0, 1): (r >> 11) * 2^-53 (builder-pinned helper)."""
    raw = rng.next_u64_array(count)
    return (raw >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
