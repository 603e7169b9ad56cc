"""libsamelda_cuda.so without a GPU: it loads, exports every entry point that
include/samelda_cu.h declares, and its host-side logic (MinibatchStream,
anneal_m, rho_schedule, config validation) matches the reference fixtures."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1409_5402_b200 import samelda

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("samelda_cu.h", "samelda_io.h")]


def declared_symbols():
    names = set()
    for h in HEADERS:
        text = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names |= set(re.findall(r"\b(samelda_(?:cu|io)_\w+)\s*\(", text))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = samelda.load_library()
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    bound = {s[0] for s in samelda.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_version():
    assert samelda.load_library().samelda_cu_version() >= 1


def test_minibatch_stream_matches_reference(golden):
    s = samelda.MinibatchStream(97, 0.1, 77)
    assert s.batch_size == 10 and s.batches_per_pass() == 10
    got = [s.next() for _ in range(len(golden["minibatch_sizes"]))]
    np.testing.assert_array_equal([len(b) for b in got], golden["minibatch_sizes"])
    np.testing.assert_array_equal(np.concatenate(got), golden["minibatch_ids"])
    with pytest.raises(samelda.ConfigError):
        samelda.MinibatchStream(10, 0.0, 1)


def test_schedules_match_reference(golden):
    for s, t, tmax, v in golden["anneal_grid"]:
        assert samelda.anneal_m(int(s), int(t), int(tmax), 100.0) == v
    for t, tau, gm, v in golden["rho_grid"]:
        assert samelda.rho_schedule(int(t), tau, gm) == v
    # test_sampler.cpp:113-135 documented points and errors
    assert samelda.rho_schedule(3, 1.0, 0.5) == pytest.approx(0.5, rel=1e-15)
    assert samelda.rho_schedule(0, 64.0, 0.7) == pytest.approx(0.054409410206007759, rel=1e-14)
    for bad in [(0, 0.5, 0.5), (0, 1.0, 0.3), (0, 1.0, 1.2), (-1, 1.0, 0.5)]:
        with pytest.raises(samelda.ConfigError):
            samelda.rho_schedule(*bad)
    assert samelda.anneal_m("linear", 1, 20, 100.0) == pytest.approx(9.5238095238095238, rel=1e-13)
    assert samelda.anneal_m("log", 1, 37, 100.0) == 0.01
    assert samelda.anneal_m("log", 1, 1, 100.0) == 100.0
    for bad in [(0, 20), (21, 20)]:
        with pytest.raises(samelda.ConfigError):
            samelda.anneal_m("linear", bad[0], bad[1], 100.0)
    with pytest.raises(samelda.ConfigError):
        samelda.parse_schedule("bogus")


def test_schedules_conserve_mass():
    # test_sampler.cpp:137-158
    t_max, m = 37, 100.0
    for s in ("constant", "linear", "invlinear"):
        total = sum(samelda.anneal_m(s, t, t_max, m) for t in range(1, t_max + 1))
        assert abs(total - m * t_max) < 1e-9 * m * t_max
    total = sum(samelda.anneal_m("log", t, t_max, m) for t in range(1, t_max + 1))
    assert abs(total - m * t_max) < 0.01 + 1e-9 * m * t_max


def test_no_device_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(samelda.CudaError):
        samelda.Context(0)
