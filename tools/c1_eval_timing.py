"""C1 (BASELINE configs[0]) end to end as bench.py's e2e leg times it: a fresh
context per train() call (corpus upload, init, 20 full-batch periods, eval
every 5, model download), per held-out evaluation mode.

    python tools/c1_eval_timing.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1409_5402_b200 import samelda as S  # noqa: E402

tr, te = bench.single_gpu_corpus("c1")
cfg = S.SamplerConfig(n_topics=32, m=10.0, t_max=20, batch_fraction=1.0, seed=1)
for exact in (False, True, False):
    runs, runs_noeval = [], []
    for _ in range(3):
        ctx = S.Context(0)
        ctx.set_eval_exact(exact)
        t0 = time.perf_counter()
        S.train(tr, cfg, te, 5, ctx=ctx)
        runs.append(time.perf_counter() - t0)
        ctx.close()
        ctx = S.Context(0)
        t0 = time.perf_counter()
        S.train(tr, cfg, None, 0, ctx=ctx)
        runs_noeval.append(time.perf_counter() - t0)
        ctx.close()
    print(f"exact={exact}: fresh-context train()+eval best {1e3 * min(runs):.1f} ms "
          f"(runs {[round(1e3 * r, 1) for r in runs]}), without eval {1e3 * min(runs_noeval):.1f} ms",
          flush=True)
