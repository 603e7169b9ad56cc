"""Held-out evaluation (perword_loglik) timing on the bench workload: the
staged-row kernel (1, 2, 3 CTAs per SM), the CTA-per-document kernel and the
warp-per-document one (SAMELDA_EVAL=cta|warp).

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
res = {}
variants = (("stage3", {}), ("stage1", {"SAMELDA_EVAL_CTAS_PER_SM": "1"}),
            ("stage2", {"SAMELDA_EVAL_CTAS_PER_SM": "2"}),
            ("stage4", {"SAMELDA_EVAL_CTAS_PER_SM": "4"}), ("cta", {"SAMELDA_EVAL": "cta"}),
            ("warp", {"SAMELDA_EVAL": "warp"}))
for name, env in variants:
    for key in ("SAMELDA_EVAL", "SAMELDA_EVAL_CTAS_PER_SM"):
        os.environ.pop(key, None)
    os.environ.update(env)
    tr.evaluate()  # warm (split computed once)
    t0 = time.perf_counter()
    ll = tr.evaluate()
    dt = time.perf_counter() - t0
    res[name] = ll
    print(f"{name}: ll={ll!r} {dt * 1e3:.2f} ms  (test docs {heldout.n_docs}, nnz {heldout.nnz})",
          flush=True)
print("max rel diff vs warp", max(abs(v - res["warp"]) / abs(res["warp"]) for v in res.values()))
