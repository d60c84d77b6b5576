"""Seeded synthetic inputs, restating the reference test suite's generators
(proj/tests/test_support.hpp:15-106) on numpy, draw-for-draw:

* ``Rng``            std::mt19937_64 + rng.hpp's draw helpers (rng.hpp:15-24),
                     with a vectorised twist (the 312-word state splits into
                     two halves whose updates are independent).
* ``random_set``     test_support.hpp:15-30 (mu, theta, s1, s2, r, g, b order)
* ``photo_like_image`` / ``texture_like_image`` / ``random_image``
* ``init_set``       the fit's starting state (sampling.cpp:154-174 shape:
                     theta = 0, s = 2/max(H, W)) at uniform random pixel
                     centres -- the worst case for culling.

Used by bench.py and smoke(); tests check them against the oracle.
"""
from __future__ import annotations

import numpy as np

_N, _M = 312, 156
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x7FFFFFFF)
_MAG = np.uint64(0xB5026F5AA96619E9)


class Rng:
    def __init__(self, seed: int):
        mt = np.zeros(_N, dtype=np.uint64)
        x = seed & 0xFFFFFFFFFFFFFFFF
        mt[0] = x
        for i in range(1, _N):
            x = (6364136223846793005 * (x ^ (x >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
            mt[i] = x
        self.mt = mt
        self.buf = np.zeros(0, dtype=np.uint64)
        self.pos = 0

    def _twist(self):
        mt = self.mt
        one = np.uint64(1)
        # i = 0..155: every operand is an old word
        y = (mt[0:_M] & _UPPER) | (mt[1:_M + 1] & _LOWER)
        new_lo = mt[_M:_N] ^ (y >> one) ^ np.where((y & one) == one, _MAG, np.uint64(0))
        # i = 156..310: mt[i-156] is new
        y2 = (mt[_M:_N - 1] & _UPPER) | (mt[_M + 1:_N] & _LOWER)
        new_hi = new_lo[0:_M - 1] ^ (y2 >> one) ^ np.where((y2 & one) == one, _MAG, np.uint64(0))
        # i = 311: wraps to the new mt[0]
        y3 = (mt[_N - 1] & _UPPER) | (new_lo[0] & _LOWER)
        last = new_lo[_M - 1] ^ (y3 >> one) ^ (_MAG if (int(y3) & 1) else np.uint64(0))
        mt = np.concatenate([new_lo, new_hi, np.array([last], dtype=np.uint64)])
        self.mt = mt
        x = mt.copy()
        x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
        x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        x ^= x >> np.uint64(43)
        return x

    def u64(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        filled = 0
        while filled < count:
            if self.pos >= self.buf.size:
                blocks = max(1, (count - filled + _N - 1) // _N)
                self.buf = np.concatenate([self._twist() for _ in range(min(blocks, 4096))])
                self.pos = 0
            take = min(count - filled, self.buf.size - self.pos)
            out[filled:filled + take] = self.buf[self.pos:self.pos + take]
            self.pos += take
            filled += take
        return out

    def doubles(self, count: int) -> np.ndarray:
        """next_double() x count: (u64 >> 11) * 2^-53 (rng.hpp:18)."""
        return (self.u64(count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def random_set(n: int, seed: int, smin: float = 0.01, smax: float = 0.3) -> np.ndarray:
    """test_support.hpp:24-30; next_range(lo, hi) = lo + (hi - lo) * d."""
    d = Rng(seed).doubles(8 * n).reshape(n, 8)
    out = np.empty((n, 8))
    out[:, 0] = d[:, 0]
    out[:, 1] = d[:, 1]
    out[:, 2] = 0.0 + (3.141592653589793 - 0.0) * d[:, 2]
    out[:, 3] = smin + (smax - smin) * d[:, 3]
    out[:, 4] = smin + (smax - smin) * d[:, 4]
    out[:, 5:8] = d[:, 5:8]
    return out


def random_local_set(n: int, width: int, height: int, seed: int = 7) -> np.ndarray:
    """SURVEY.md 8d "random-local": sigma 2..16 px at the given raster."""
    m = max(width, height)
    return random_set(n, seed, 2.0 / m, 16.0 / m)


def init_set(n: int, width: int, height: int, seed: int = 11) -> np.ndarray:
    """Fit-start state (sampling.cpp:159-171 shape) at uniform pixel centres."""
    r = Rng(seed)
    flat = (r.u64(n) % np.uint64(width * height)).astype(np.int64)
    h, w = flat // width, flat % width
    d = r.doubles(3 * n).reshape(n, 3)
    out = np.empty((n, 8))
    out[:, 0] = (w + 0.5) / width
    out[:, 1] = (h + 0.5) / height
    out[:, 2] = 0.0
    out[:, 3] = out[:, 4] = 2.0 / max(width, height)
    out[:, 5:8] = d
    return out


def _centers(width, height):
    u = (np.arange(width) + 0.5) / width
    v = (np.arange(height) + 0.5) / height
    return np.meshgrid(u, v)


def photo_like_image(width: int, height: int, seed: int) -> np.ndarray:
    """test_support.hpp:42-65 (12 blobs over a ramp)."""
    d = Rng(seed).doubles(12 * 6).reshape(12, 6)
    U, V = _centers(width, height)
    c = np.stack([0.2 + 0.6 * U, 0.3 + 0.4 * V, np.full_like(U, 0.5)], axis=-1)
    for cx, cy, rr, r, g, b in d:
        rr = 0.05 + (0.3 - 0.05) * rr
        d2 = (U - cx) * (U - cx) + (V - cy) * (V - cy)
        wgt = np.exp(-d2 / (2.0 * rr * rr))[..., None]
        c = c * (1.0 - wgt) + np.array([r, g, b]) * wgt
    return c.astype(np.float32)


def texture_like_image(width: int, height: int, seed: int) -> np.ndarray:
    """test_support.hpp:93-106 (sinusoids)."""
    d = Rng(seed).doubles(4)
    p1 = 15.0 + 10.0 * d[0]
    p2 = 25.0 + 15.0 * d[1]
    ph1 = 0.0 + 6.28 * d[2]
    ph2 = 0.0 + 6.28 * d[3]
    U, V = _centers(width, height)
    a = 0.5 + 0.5 * np.sin(p1 * U + ph1) * np.cos(p2 * V + ph2)
    b = 0.5 + 0.5 * np.sin(p2 * (U + V) + ph2)
    return np.stack([a, b, 0.5 + 0.25 * (a - b)], axis=-1).astype(np.float32)


def random_image(width: int, height: int, seed: int) -> np.ndarray:
    """test_support.hpp:32-39."""
    return Rng(seed).doubles(width * height * 3).reshape(height, width, 3).astype(np.float32)


def sample_indices(n: int, width: int, height: int, seed: int = 99, steps: int = 1) -> np.ndarray:
    """Uniform flat pixel indices (steps x n) for training benchmarks."""
    r = Rng(seed)
    return (r.u64(steps * n) % np.uint64(width * height)).astype(np.uint32).reshape(steps, n)
