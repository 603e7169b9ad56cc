"""Held-out evaluation (perword_loglik) timing on the bench workload, for the
kernel variant the environment selects (SAMELDA_EVAL=cta|warp,
SAMELDA_EVAL_CTAS_PER_SM=n; read once per process).

    python tools/eval_timing.py [--config nytimes] [--periods 6]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1409_5402_b200 import samelda as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="nytimes")
ap.add_argument("--periods", type=int, default=6)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
train, heldout = bench.single_gpu_corpus(args.config)
scfg = S.SamplerConfig(n_topics=cfg["n_topics"], m=cfg["m"], batch_fraction=cfg["batch_fraction"],
                       inner_sweeps=cfg["inner_sweeps"], t_max=args.periods, seed=1)
tr = S.Trainer(train, scfg)
tr.set_heldout(heldout, seed=1)
stream = S.MinibatchStream(train.n_docs, cfg["batch_fraction"], 1)
for t in range(args.periods):
    tr.period(stream.next(), t, cfg["m"], S.rho_schedule(t, 1.0, 0.5))
tr.ctx.synchronize()
# default fold-in kernel (k_eval_fold) and the reference-order exact mode
# (variant of the exact mode: SAMELDA_EVAL=cta|warp, SAMELDA_EVAL_CTAS_PER_SM=n)
tr.evaluate()  # warm (split computed once)
for exact in (False, True):
    tr.ctx.set_eval_exact(exact)
    tr.evaluate()
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        ll = tr.evaluate()
        times.append(time.perf_counter() - t0)
    variant = ("exact:" + os.environ.get("SAMELDA_EVAL", "stage") + "/" +
               os.environ.get("SAMELDA_EVAL_CTAS_PER_SM", "-")) if exact else "fast (k_eval_fold)"
    print(f"{variant}: ll={ll!r} best {min(times) * 1e3:.2f} ms  (test docs {heldout.n_docs}, "
          f"nnz {heldout.nnz})", flush=True)
