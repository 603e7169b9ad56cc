"""Train P periods of the bench workload (untimed), then run 2 more periods --
the kernels of those two periods are the ones to profile (ncu --launch-skip)
at a late, converged model state.

    python tools/late_period.py [--periods 100]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1409_5402_b200 import samelda as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="nytimes")
ap.add_argument("--periods", type=int, default=100)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
train, heldout = bench.single_gpu_corpus(args.config)
scfg = S.SamplerConfig(n_topics=cfg["n_topics"], m=cfg["m"], batch_fraction=cfg["batch_fraction"],
                       inner_sweeps=cfg["inner_sweeps"], t_max=args.periods + 2, seed=1)
tr = S.Trainer(train, scfg)
stream = S.MinibatchStream(train.n_docs, cfg["batch_fraction"], 1)
for t in range(args.periods + 2):
    tr.period(stream.next(), t, cfg["m"], S.rho_schedule(t, 1.0, 0.5))
tr.ctx.synchronize()
print("launches", tr.ctx.launches)
