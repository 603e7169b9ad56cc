"""Phases of the drop-in train() at the bench shape on a fresh context: corpus
upload + init, held-out split, 20 periods, one evaluation, model download.

    python tools/dropin_phases.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1409_5402_b200 import samelda as S  # noqa: E402

cfg = bench.CONFIGS["nytimes"]
train, heldout = bench.single_gpu_corpus("nytimes")
for rep in range(3):
    ctx = S.Context(0)
    scfg = S.SamplerConfig(n_topics=256, m=100.0, batch_fraction=cfg["batch_fraction"], t_max=20, seed=1)
    ph = {}
    t0 = time.perf_counter()
    tr = S.Trainer(train, scfg, ctx=ctx)
    ctx.synchronize()
    ph["upload+init"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    tr.set_heldout(heldout, seed=1)
    ctx.synchronize()
    ph["heldout"] = time.perf_counter() - t0
    stream = S.MinibatchStream(train.n_docs, cfg["batch_fraction"], 1)
    t0 = time.perf_counter()
    for t in range(20):
        tr.period(stream.next(), t, 100.0, S.rho_schedule(t, 1.0, 0.5))
    ctx.synchronize()
    ph["20 periods"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    tr.evaluate()
    ph["eval"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    tr.model()
    ph["download"] = time.perf_counter() - t0
    ctx.close()
    print(" ".join(f"{k}={1e3 * v:.1f}ms" for k, v in ph.items()), flush=True)
