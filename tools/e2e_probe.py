"""Where the end-to-end period time goes (bench.py's e2e leg): host time per period
(Python + C ABI enqueue), device time per period, and the e2e wall time, for a few
step counts.

    python tools/e2e_probe.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1409_5402_b200 import distributed as DIST  # noqa: E402
from paper_1409_5402_b200 import samelda as S  # noqa: E402

train, heldout = bench.single_gpu_corpus("nytimes")
ctx = S.Context(0)
stream = torch.cuda.Stream(device=0)
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
T = 200
tr = S.Trainer(train, S.SamplerConfig(n_topics=256, m=100.0, batch_fraction=0.05, t_max=T, seed=1),
               ctx=ctx)
eng = DIST.CudaEngine(tr, 0)
st = DIST.ShardedTrainer(eng, train.n_docs, 0, train.n_docs, train.doc_tokens(), 0.05, 1, 100.0,
                         "constant", T)
bufs = [torch.empty(20000 * 256, dtype=torch.float64, pin_memory=True).numpy() for _ in range(40)]
for _ in range(5):
    st.period()
torch.cuda.synchronize()
for n, copies in ((10, True), (20, True), (40, True), (20, False)):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    host = []
    t0 = time.perf_counter()
    ev0.record(stream)
    for i in range(n):
        h0 = time.perf_counter()
        s = st.period()
        if copies:
            tr.batch_theta_async(s.owned_docs, bufs[i])
        host.append(time.perf_counter() - h0)
    ev1.record(stream)
    t_enq = time.perf_counter() - t0
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev = ev0.elapsed_time(ev1) / 1e3
    print(f"n={n:3d} copies={copies}: wall {wall / n * 1e3:.3f} ms/period, device {dev / n * 1e3:.3f}, "
          f"host enqueue {np.mean(host) * 1e3:.3f} (max {np.max(host) * 1e3:.3f}), "
          f"enqueue total {t_enq / n * 1e3:.3f}", flush=True)
