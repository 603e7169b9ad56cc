"""Per-period timing of the device-resident trainer on the bench workload.

    python tools/period_timing.py [--config nytimes] [--periods 12]
Prints per period: sample ms (fast + deferred), M-step ms, deferred records.
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
ap.add_argument("--periods", type=int, default=12)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--every", type=int, default=1, help="print every n-th period")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
train, heldout = bench.single_gpu_corpus(args.config)
scfg = S.SamplerConfig(n_topics=cfg["n_topics"], m=cfg["m"], batch_fraction=cfg["batch_fraction"],
                       inner_sweeps=cfg["inner_sweeps"], t_max=args.periods, seed=1, mode=args.mode)
tr = S.Trainer(train, scfg)
stream = S.MinibatchStream(train.n_docs, cfg["batch_fraction"], 1)
for t in range(args.periods):
    batch = stream.next()
    tr.profile(True)
    t0 = time.perf_counter()
    tr.period(batch, t, cfg["m"], S.rho_schedule(t, 1.0, 0.5))
    tr.ctx.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    p = tr.profile_read()
    if t % args.every:
        continue
    print(f"t={t:3d} wall={wall:8.2f}ms sample={p['sample_ms']:8.2f}ms mstep={p['mstep_ms']:6.2f}ms "
          f"first={p['sample_first_ms']:7.2f} last={p['sample_last_ms']:7.2f} nnz={p['nnz']} deferred={p['deferred']} ({p['deferred'] / max(p['nnz'], 1) * 100:.2f}%)",
          flush=True)
