"""Held-out evaluation (perword_loglik) timing on the bench workload, for the
CTA-per-document kernel and the warp-per-document one (SAMELDA_EVAL_WARP=1).

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
corpus = bench.make_corpus(cfg["corpus"], 0)
train, heldout = bench.split_heldout(corpus)
scfg = S.SamplerConfig(n_topics=cfg["n_topics"], m=cfg["m"], batch_fraction=cfg["batch_fraction"],
                       inner_sweeps=cfg["inner_sweeps"], t_max=args.periods, seed=1)
tr = S.Trainer(train, scfg)
tr.set_heldout(heldout, seed=1)
stream = S.MinibatchStream(train.n_docs, cfg["batch_fraction"], 1)
for t in range(args.periods):
    tr.period(stream.next(), t, cfg["m"], S.rho_schedule(t, 1.0, 0.5))
tr.ctx.synchronize()
res = {}
for name, env in (("cta", None), ("warp", "1")):
    if env:
        os.environ["SAMELDA_EVAL_WARP"] = env
    else:
        os.environ.pop("SAMELDA_EVAL_WARP", None)
    tr.evaluate()  # warm (split computed once)
    t0 = time.perf_counter()
    ll = tr.evaluate()
    dt = time.perf_counter() - t0
    res[name] = ll
    print(f"{name}: ll={ll!r} {dt * 1e3:.2f} ms  (test docs {heldout.n_docs}, nnz {heldout.nnz})",
          flush=True)
print("rel diff", abs(res["cta"] - res["warp"]) / abs(res["warp"]))
