"""The M-step's division by a constant (kernels_mstep.cu div_rcp): with y = RN(1/b),
q0 = RN(a y), two FMA corrections q <- RN(q + RN-exact(a - b q) y) give RN(a / b)
(Markstein's theorem for the second step).  The kernels rely on it for
count / m_t and (rho cand) / total -- bit-identity with the reference's
division.  Restated here with exact rational arithmetic (Fraction -> float is
correctly rounded, so fma(x, y, z) = float(Fraction(x) * y + z)) and checked
against IEEE division on counts (small, random, up to 2^40) and the m_t values
the schedules produce, plus random divisors and random real numerators."""
from __future__ import annotations

import random
from fractions import Fraction

import numpy as np
import pytest


def fma(x: float, y: float, z: float) -> float:
    return float(Fraction(x) * Fraction(y) + Fraction(z))


def div_rcp(a: float, b: float) -> float:
    y = 1.0 / b
    q0 = a * y
    q1 = fma(fma(-q0, b, a), y, q0)
    return fma(fma(-q1, b, a), y, q1)


M_T = [100.0, 10.0, 1.0, 99.0, 50.0, 0.37, 1e-3, 1e4, 3.0, 7.0, 1.0 / 3, 2.0 * 50 * 7 / 101.0,
       100.0 * 33 / 101.0, 19.999999999999996]


@pytest.mark.parametrize("b", M_T)
def test_counts_over_m_t(b):
    rng = random.Random(int(b * 1000) + 1)
    counts = list(range(0, 600)) + [rng.randrange(1 << 40) for _ in range(1500)]
    for a in counts:
        assert div_rcp(float(a), b) == float(a) / b, (a, b)


def test_random_divisors_and_numerators():
    rng = np.random.default_rng(5)
    bs = np.exp(rng.uniform(-20, 20, 300)) * (1 + rng.random(300))
    for b in bs:
        for a in np.exp(rng.uniform(-30, 30, 40)):
            assert div_rcp(float(a), float(b)) == float(a) / float(b), (a, b)
