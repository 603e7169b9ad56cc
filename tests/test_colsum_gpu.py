"""The exact parallel column-sum scan (k_colsum_*, kernels_mstep.cu) against
the sequential f64 sum it replaces (sampler.cpp:214-218's row normaliser):
bit-equal on realistic and adversarial columns -- ties at half an ulp, sums
crossing powers of two, huge and tiny terms, a column that starts tiny."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_1409_5402_b200 import samelda
    lib = samelda.load_library()
    lib.samelda_debug_col_sums.restype = C.c_int
    lib.samelda_debug_col_sums.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    return lib


def seq_sums(x):
    """The reference's loop: total += x[w, k] in w order, f64."""
    tot = np.zeros(x.shape[1])
    for w in range(x.shape[0]):
        tot = tot + x[w]
    return tot


def gpu_sums(lib, x, mode):
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(x.shape[1])
    rc = lib.samelda_debug_col_sums(x.ctypes.data, x.shape[0], x.shape[1], mode, out.ctypes.data)
    assert rc == 0
    return out


def columns(kind, W, K, rng):
    if kind == "counts":  # count / m_t + beta, the M-step's candidate
        c = rng.poisson(rng.gamma(0.3, 3.0, size=(W, K)))
        return c / 37.0 + 0.01
    if kind == "ties":  # many exact half-ulp ties: dyadic terms comparable to the sum
        return rng.integers(1, 9, size=(W, K)) * 2.0 ** rng.integers(-3, 3, size=(W, K))
    if kind == "jumps":  # rare huge terms force binade jumps mid-column
        x = rng.random((W, K)) * 1e-3 + 1e-6
        x[rng.random((W, K)) < 1e-3] *= 1e9
        return x
    if kind == "tiny_start":  # the running sum spends many rows at tiny magnitudes
        x = rng.random((W, K)) + 1e-3
        x[: W // 3] *= 1e-280
        return x
    if kind == "pow2":  # partial sums landing exactly on powers of two
        return np.full((W, K), 0.25) + (rng.random((W, K)) < 0.01) * 2.0 ** -40
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["counts", "ties", "jumps", "tiny_start", "pow2"])
@pytest.mark.parametrize("W,K", [(5000, 32), (3001, 40), (700, 256), (1, 7), (513, 1)])
def test_scan_equals_sequential_sum(lib, kind, W, K):
    rng = np.random.default_rng(W * 131 + K)
    x = columns(kind, W, K, rng)
    ref = seq_sums(x)
    np.testing.assert_array_equal(gpu_sums(lib, x, 1), ref)  # the sequential chain kernel
    np.testing.assert_array_equal(gpu_sums(lib, x, 0), ref)  # the parallel scan


def test_scan_nytimes_shape(lib):
    rng = np.random.default_rng(7)
    W, K = 102660, 256
    c = rng.poisson(rng.gamma(0.2, 2.0, size=(W, K)).astype(np.float64))
    x = c / 100.0 + 0.01
    ref = seq_sums(x)  # the reference's sequential loop, in numpy (IEEE f64 adds, no FMA)
    np.testing.assert_array_equal(gpu_sums(lib, x, 0), ref)
    np.testing.assert_array_equal(gpu_sums(lib, x, 1), ref)
