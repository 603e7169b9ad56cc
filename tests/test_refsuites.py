"""The reference's OWN unit suites (proj/tests/test_{rng,corpus,model,sampler,cgs,eval}.cpp,
79 doctest cases) compiled unmodified by oracle/Makefile `refsuites` with the
doctest-compatible runner oracle/doctest/doctest.h (test infrastructure: the
reference does not vendor doctest):

  samelda_unit_ref   against the stock reference library -- runs here, on the CPU, and
                     pins the runner itself (every case passes, as in proj/test_output.txt)
  samelda_unit_cuda  with sampler.cpp / eval.cpp replaced by the drop-in shim over
                     libsamelda_cuda.so (GPU): the suites exercise sddmm, sample_counts,
                     update_model, rho / anneal, train, fold_in_theta, perword_loglik
                     and cgs_train's evaluation through the C ABI -- on one device, and
                     with train() sharded over a three-member device group.

test_cli.cpp needs the reference CLI binary (tools/main.cpp: CLI11, absent)."""
from __future__ import annotations

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "samelda_unit_ref")
CUDA_BIN = os.path.join(ROOT, "oracle", "_ref", "samelda_unit_cuda")
SUITES = {"rng": 15, "corpus": 14, "model": 4, "sampler": 24, "eval": 12, "cgs": 10}


def _run(binary, suite, env=None):
    r = subprocess.run([binary, f"-ts={suite}"], capture_output=True, text=True, timeout=900,
                       env=env)
    out = r.stdout + r.stderr
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert m, out[-3000:]
    return r.returncode, int(m.group(1)), int(m.group(3)), out


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="built only where /root/reference exists")
@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_on_reference(suite):
    rc, ran, failed, out = _run(REF_BIN, suite)
    assert rc == 0 and failed == 0 and ran == SUITES[suite], out[-3000:]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(CUDA_BIN), reason="built only where /root/reference exists")
@pytest.mark.parametrize("devices", ["0", "0,0,0"], ids=["one-gpu", "group3"])
@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_on_drop_in(suite, devices):
    env = dict(os.environ, SAMELDA_CU_DEVICES=devices)
    rc, ran, failed, out = _run(CUDA_BIN, suite, env)
    assert rc == 0 and failed == 0 and ran == SUITES[suite], out[-3000:]
