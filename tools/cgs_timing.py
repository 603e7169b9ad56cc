"""CGS baseline timing on BASELINE configs[0]'s corpus (the reference's make_corpus(10000,
5000, 32, 100, 1), split_holdout(0.1, 1)): sweeps on the device (one warp, the reference's
sequential chain) against the compiled reference's cgs_train on the host.

    python tools/cgs_timing.py [--sweeps 5] [--K 32]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1409_5402_b200 import samelda as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sweeps", type=int, default=5)
ap.add_argument("--K", type=int, default=32)
args = ap.parse_args()
train, test = bench.single_gpu_corpus("c1")
ctx = S.Context(0)
S.cgs_train(train, args.K, 0.1, 0.01, 1, 1, ctx=ctx)  # warm
t0 = time.perf_counter()
model, _ = S.cgs_train(train, args.K, 0.1, 0.01, args.sweeps, 1, ctx=ctx)
dev = time.perf_counter() - t0
tokens = train.n_tokens * args.sweeps
print(f"device: {args.sweeps} sweeps {dev:.3f}s  {tokens / dev:.3e} token samples/s "
      f"({dev / tokens * 1e9:.0f} ns/token)")
try:
    from oracle import CorpusArrays, Ref
    ref = Ref()
    c = CorpusArrays(train.doc_offsets, train.word_ids, train.counts, train.n_words)
    t0 = time.perf_counter()
    phi, theta, _ = ref.cgs_train(c, args.K, 0.1, 0.01, args.sweeps, 1)
    host = time.perf_counter() - t0
    import numpy as np
    print(f"reference (host, sequential): {host:.3f}s  {tokens / host:.3e} token samples/s; "
          f"phi bit-equal: {np.array_equal(phi, model.phi)}")
except Exception as e:  # noqa: BLE001
    print("reference unavailable:", e)
