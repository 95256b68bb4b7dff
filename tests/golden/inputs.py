"""Input definitions shared by the golden generator and the parity tests.

These restate the reference tests' fixtures: TestRng (proj/tests/test_helpers.hpp:44-71),
the find_extrema / envelope unit cases (proj/tests/test_emd.cpp:13-112) and
BASELINE.json configs 1-3.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1

# BASELINE.json configs 1-3: the pick-up-mask signals serialized with interval D.
C_CONFIGS = {
    "c1_emd_D50": dict(algo=0, D=50, iters=1000, imfs=0, nr=1),
    "c2_eemd_D1": dict(algo=1, D=1, iters=300, imfs=10, nr=100),
    "c2_eemd_D50": dict(algo=1, D=50, iters=300, imfs=10, nr=100),
    "c2_eemd_D500": dict(algo=1, D=500, iters=300, imfs=10, nr=100),
    "c3_ceemdan_D50": dict(algo=2, D=50, iters=5000, imfs=0, nr=500),
}


class TestRng:
    """test_helpers.hpp:44-71 -- LCG state + splitmix finaliser, uniform in [-1, 1)."""

    __test__ = False

    def __init__(self, seed: int):
        self.state = (seed ^ 0x853C49E6748FEA9B) & MASK64

    def next_u64(self) -> int:
        self.state = (self.state * 6364136223846793005 + 1442695040888963407) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return 2.0 * (float(self.next_u64() >> 11) * 2.0 ** -53) - 1.0

    def range(self, lo: int, hi: int) -> int:
        return lo + self.next_u64() % (hi - lo + 1)


def rng_signal(seed: int, n: int) -> np.ndarray:
    g = TestRng(seed)
    return np.array([g.uniform() for _ in range(n)], dtype=np.float64)


def sine(f: float, n: int, fs: float) -> np.ndarray:
    import math
    two_pi = 6.283185307179586476925286766559
    return np.array([math.sin(two_pi * f * float(k) / fs) for k in range(n)])


def kat_extrema_cases():
    yield "single_oscillation", np.array([0.0, 1.0, 0.0, -1.0, 0.0])
    yield "constant", np.full(16, 3.5)
    yield "endpoints", np.array([5.0, 1.0, 2.0, 1.0, 9.0])
    yield "plateau2", np.array([0.0, 1.0, 1.0, 0.0])
    yield "plateau3", np.array([0.0, 2.0, 2.0, 2.0, 0.0])
    yield "shoulder", np.array([0.0, 1.0, 1.0, 2.0, 0.0])
    yield "tone32", sine(32.0, 1000, 1000.0)
    yield "edge_plateaus", np.array([1.0, 1.0, 0.0, 2.0, 2.0, 2.0, 2.0, 0.0, 0.0, 3.0, 3.0])
    yield "ramp", np.arange(64) * 0.25
    yield "min3", np.array([1.0, 0.0, 1.0])


def kat_envelope_cases(backend):
    yield "two_equal", [0, 9], [1.0, 1.0], 10
    yield "interp4", [0, 3, 5, 10], [0.0, 7.0, 2.0, 10.0], 11
    yield "collinear", [0, 5, 10], [0.0, 5.0, 10.0], 11
    s = sine(8.0, 1000, 1000.0)
    mi, mv, _, _ = backend.find_extrema(s)
    yield "sine8_max", mi.tolist(), mv.tolist(), 1000
    yield "mirror_quirk", [3, 7, 12, 16], [1.0, -2.0, 0.5, 3.0], 20
    yield "left_anchored", [0, 4, 9], [2.0, -1.0, 4.0], 15
    yield "right_anchored", [2, 6, 14], [2.0, -1.0, 4.0], 15
    yield "three_knots", [5, 9, 13], [1.0, 2.0, 0.5], 20


def pickup_serialized(backend, D: int) -> np.ndarray:
    x6 = backend.multivariate_sinusoids(1000, 1000.0)
    return backend.concatenate(x6, 1000, 6, D)
