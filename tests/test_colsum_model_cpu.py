"""CPU model of the exact parallel column-sum scan (kernels_mstep.cu,
k_colsum_partial / _program / _resolve): the algorithm restated in Python
with exact integer arithmetic and checked bit for bit against the sequential
f64 sum it replaces (sampler.cpp:214-218).  The GPU implementation is checked
against the same sums in tests/test_colsum_gpu.py; this pins the design --
binade segments composed as parity-dependent ulp increments, explicit adds at
binade changes -- independently of the kernels."""
from __future__ import annotations

import math
import struct

import numpy as np
import pytest

ROWS = 16  # sub-range length (the kernels use 256)


def bits(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", x))[0]


def hi_fields(s: float):
    h = bits(s) >> 32
    return (h >> 20) & 0x7FF, h & 0xFFFFF


def explicit(sa: float, v: float, sn: float) -> bool:
    es, fs = hi_fields(sa)
    en, fn = hi_fields(sn)
    return (not (0.0 < v < 1e300) or es != en or fs in (0, 0xFFFFF) or fn in (0, 0xFFFFF)
            or es < 123 or es > 1923)


def program(x: np.ndarray, r: int, approx_start: float):
    """k_colsum_program for one (topic, sub-range): items (d0, d1)."""
    items = []
    sa = approx_start
    seg = None  # [biased exponent, n0, nd]

    def close():
        if seg is not None:
            e = seg[0] - 1023
            ulp = math.ldexp(1.0, e - 52)
            items.append((seg[1] * ulp, (seg[1] + seg[2]) * ulp, "seg"))

    for w in range(r * ROWS, min((r + 1) * ROWS, len(x))):
        v = float(x[w])
        sn = sa + v
        es = hi_fields(sa)[0]
        if explicit(sa, v, sn):
            close()
            seg = None
            items.append((v, v, "term"))
        else:
            if seg is None or seg[0] != es:
                close()
                seg = [es, 0, 0]
            y = v * math.ldexp(1.0, 52 - (es - 1023))  # exact
            q = math.floor(y)
            f = y - q
            if f == 0.5:
                a0 = (seg[1] + q) & 1
                a1 = (1 + seg[1] + seg[2] + q) & 1
                seg[1] += q + a0
                seg[2] += a1 - a0
            else:
                seg[1] += q + (1 if f > 0.5 else 0)
        sa = sn
    close()
    return items


def scan_sum(x: np.ndarray) -> float:
    nsub = (len(x) + ROWS - 1) // ROWS
    part = [float(np.sum(x[r * ROWS:(r + 1) * ROWS][::-1])) for r in range(nsub)]  # any order
    s = 0.0
    for r in range(nsub):
        for d0, d1, _ in program(x, r, float(sum(part[:r]))):
            s = s + (d1 if bits(s) & 1 else d0)
    return s


def seq_sum(x: np.ndarray) -> float:
    s = 0.0
    for v in x:
        s = s + float(v)
    return s


def column(kind: str, n: int, rng) -> np.ndarray:
    if kind == "counts":
        return rng.poisson(rng.gamma(0.3, 3.0, n)) / 37.0 + 0.01
    if kind == "ties":
        return rng.integers(1, 9, n) * 2.0 ** rng.integers(-3, 3, n)
    if kind == "jumps":
        x = rng.random(n) * 1e-3 + 1e-6
        x[rng.random(n) < 0.02] *= 1e9
        return x
    if kind == "tiny_start":
        x = rng.random(n) + 1e-3
        x[: n // 3] *= 1e-280
        return x
    if kind == "pow2":
        return np.full(n, 0.25) + (rng.random(n) < 0.05) * 2.0 ** -40
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["counts", "ties", "jumps", "tiny_start", "pow2"])
@pytest.mark.parametrize("n", [1, 17, 300, 2000])
def test_scan_model_equals_sequential_sum(kind, n):
    rng = np.random.default_rng(n * 7 + len(kind))
    for _ in range(3):
        x = column(kind, n, rng)
        assert scan_sum(x) == seq_sum(x)


def test_segment_items_are_exact_increments():
    """A segment's add is exact (s stays on its binade's grid: no rounding),
    and segments carry almost all rows -- explicit adds are the binade
    changes only."""
    rng = np.random.default_rng(3)
    x = column("counts", 3000, rng)
    s = 0.0
    n_seg = n_term = 0
    nsub = (len(x) + ROWS - 1) // ROWS
    part = [float(np.sum(x[r * ROWS:(r + 1) * ROWS])) for r in range(nsub)]
    for r in range(nsub):
        for d0, d1, kind in program(x, r, float(sum(part[:r]))):
            d = d1 if bits(s) & 1 else d0
            t = s + d
            if kind == "seg":
                assert t - s == d and math.frexp(t)[1] == math.frexp(s)[1]
                n_seg += 1
            else:
                n_term += 1
            s = t
    assert s == seq_sum(x)
    assert n_term < 40 and n_seg >= nsub - 1
