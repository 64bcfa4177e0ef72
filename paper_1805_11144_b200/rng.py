"""Deterministic splitmix64 stream with Box-Muller normals — the reference's
model-sampling RNG (proj/src/frontend.cpp:15-36), restated so seeded
workloads are reproducible without any library distribution code.
Scalar methods match the reference bit-for-bit; the vectorised numpy
variants produce the same integer stream (the float transforms may differ
from libm in the last ulp, which is irrelevant for workload construction:
every engine consumes the same BuiltModel)."""
from __future__ import annotations

import math

import numpy as np

_M64 = (1 << 64) - 1
_GOLD = 0x9E3779B97F4A7C15
_TWO_PI = 6.283185307179586


class Rng:
    def __init__(self, seed: int):
        self.state = seed & _M64

    def next_u64(self) -> int:
        self.state = (self.state + _GOLD) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self, lo: float = None, hi: float = None) -> float:
        u = float(self.next_u64() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def gaussian(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log1p(-u1)) * math.cos(_TWO_PI * u2)

    # -- vectorised (same integer stream) ---------------------------------
    def u64_array(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            k = np.arange(1, n + 1, dtype=np.uint64)
            s = np.uint64(self.state) + k * np.uint64(_GOLD)
            z = s
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * _GOLD) & _M64
        return z

    def uniform_array(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        u = (self.u64_array(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return lo + (hi - lo) * u

    def gaussian_array(self, n: int) -> np.ndarray:
        u = self.uniform_array(2 * n).reshape(n, 2)
        return np.sqrt(-2.0 * np.log1p(-u[:, 0])) * np.cos(_TWO_PI * u[:, 1])


def derive_seed(base: int, stream: int) -> int:
    """Child stream k of a base seed (frontend.cpp:33-36)."""
    mix = Rng(base ^ ((stream * _GOLD + 0xD1B54A32D192ED03) & _M64))
    return mix.next_u64()
