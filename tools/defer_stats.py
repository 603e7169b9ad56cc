"""Why do fast-path draws defer?  Needs libsamelda_cuda_stats.so (tools/defer_stats.sh).

    python tools/defer_stats.py [--config nytimes] [--periods 6]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["SAMELDA_CUDA_LIB"] = os.path.join(ROOT, "paper_1409_5402_b200", "libsamelda_cuda_stats.so")
sys.path.insert(0, ROOT)
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
lib = S.load_library()
stats = (C.c_ulonglong * 96)()
stream = S.MinibatchStream(train.n_docs, cfg["batch_fraction"], 1)
for t in range(args.periods):
    batch = stream.next()
    tr.profile(True)
    tr.period(batch, t, cfg["m"], S.rho_schedule(t, 1.0, 0.5))
    tr.ctx.synchronize()
    p = tr.profile_read()
    lib.samelda_debug_defer_stats(stats, 1)
    v = list(stats)
    draws = p["nnz"] * cfg["n_topics"]
    print(f"t={t} nnz={p['nnz']} records={p['deferred']} draws={draws} deferred draws="
          f"{sum(v[0:4])}  nz_exact={v[0]} tiny={v[1]} lam>=10={v[2]} band={v[3]}")
    for b in range(40):
        if v[48 + b] or v[8 + b]:
            print(f"   lambda in [2^{b - 20}, 2^{b - 19}): draws {v[48 + b]:>12d}  deferred {v[8 + b]:>10d}"
                  f"  ({v[8 + b] / max(v[48 + b], 1):.2e})")
