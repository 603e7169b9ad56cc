"""Fold-in sweep statistics of the held-out evaluation at the bench workload:
how many of the (at most 50) fold-in sweeps documents run before
||delta||_inf < 1e-12 (eval.cpp:19-64), and their fold-cell counts -- the
numbers that size the evaluation kernel.  numpy restatement (order-insensitive
statistic), on a sample of held-out documents with a device-trained model.

    python tools/eval_sweeps.py [--periods 6] [--docs 400]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1409_5402_b200 import samelda as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--periods", type=int, default=6)
ap.add_argument("--docs", type=int, default=400)
args = ap.parse_args()
cfg = bench.CONFIGS["nytimes"]
train, heldout = bench.single_gpu_corpus("nytimes")
tr = S.Trainer(train, S.SamplerConfig(n_topics=256, m=100.0, batch_fraction=0.05,
                                      t_max=args.periods, seed=1))
stream = S.MinibatchStream(train.n_docs, 0.05, 1)
for t in range(args.periods):
    tr.period(stream.next(), t, 100.0, S.rho_schedule(t, 1.0, 0.5))
phi = tr.model(with_theta=False).phi  # K x W
rng = np.random.default_rng(0)
sweeps, cells, fold = [], [], []
o = heldout.doc_offsets
for d in rng.choice(heldout.n_docs, size=args.docs, replace=False):
    w = heldout.word_ids[o[d]:o[d + 1]]
    c = heldout.counts[o[d]:o[d + 1]]
    # approximate 50/50 split: each token to fold with p = 1/2
    fc = rng.binomial(c, 0.5)
    keep = fc > 0
    w, fc = w[keep], fc[keep].astype(np.float64)
    P = phi[:, w].T  # cells x K
    th = np.full(256, 1.0 / 256)
    n = 0
    for s in range(50):
        mu = P @ th
        nx = 0.1 + ((fc / mu)[:, None] * P * th[None, :]).sum(0)
        new = nx / nx.sum()
        n = s + 1
        delta = np.abs(new - th).max()
        th = new
        if delta < 1e-12:
            break
    sweeps.append(n)
    cells.append(len(o[d:d + 2]) and o[d + 1] - o[d])
    fold.append(int(keep.sum()))
sweeps, fold, cells = map(np.array, (sweeps, fold, cells))
print(f"sweeps: mean {sweeps.mean():.1f} median {np.median(sweeps):.0f} "
      f"frac at 50 {np.mean(sweeps == 50):.2f}")
print(f"fold cells: mean {fold.mean():.1f} p50 {np.percentile(fold, 50):.0f} "
      f"p90 {np.percentile(fold, 90):.0f} p99 {np.percentile(fold, 99):.0f} max {fold.max()}")
print(f"cells: mean {cells.mean():.1f}; sweep-weighted fold cells {np.sum(sweeps * fold) / sweeps.sum():.1f}")
for R in (25, 45, 64, 95, 128, 190):
    print(f"  rows beyond {R} resident, per sweep (sweep-weighted mean): "
          f"{np.sum(sweeps * np.maximum(fold - R, 0)) / sweeps.sum():.1f}")
