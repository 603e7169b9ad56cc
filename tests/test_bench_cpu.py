"""bench.py's reference arm (the compiled reference on the host cores) runs
without a GPU: the driver's `bench.py --impl reference` line carries the
contract keys (impl, metric, value, unit, cpu_baseline, e2e with zero
transfer bytes) on the same metric and config as our arm."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from oracle import have_ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref (compiled reference) not built")
def test_reference_arm_json_line():
    env = dict(os.environ, BENCH_REF_BUDGET_S="2")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference"
    assert line["metric"] == "sampled tokens/sec (x m replicas)" and line["unit"] == "samples/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["K"] == 256 and line["config"]["m"] == 100.0


def test_reference_arm_expected_config_unavailable():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config",
                          "nytimes-expected"], cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and "unavailable" in line


def test_run_horizon_covers_every_period():
    """The annealing horizon T must cover warm-up + timed + profiled + end-to-end
    periods (anneal_m rejects t > T): the driver's --steps 20 run once failed here."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    for warmup, steps in ((3, 10), (5, 20), (1, 1), (3, 50)):
        args = argparse.Namespace(warmup=warmup, steps=steps)
        prof = max(1, min(steps, 10))
        used = warmup + steps + prof + max(1, steps)
        for name in ("nytimes", "c3"):
            assert bench.run_t_max(bench.CONFIGS[name], args) >= used
