"""Where does a period's host time go?  Times each host call of the bench loop."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, '.')
import bench
from paper_1409_5402_b200 import samelda as S, distributed as D

cfg = bench.CONFIGS["nytimes"]
train, _ = bench.single_gpu_corpus("nytimes")
ctx = S.Context(0)
stream = torch.cuda.Stream(device=0)
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
scfg = S.SamplerConfig(n_topics=256, m=100.0, batch_fraction=0.05, inner_sweeps=2, t_max=40, seed=1)
tr = S.Trainer(train, scfg, ctx=ctx)
batches = S.MinibatchStream(train.n_docs, 0.05, 1)
acc = {}
def tick(name, t0):
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
for t in range(30):
    if t == 5:
        torch.cuda.synchronize(); acc.clear(); T0 = time.perf_counter()
    t0 = time.perf_counter(); b = batches.next(); tick("next", t0)
    t0 = time.perf_counter(); m_t = S.anneal_m("constant", t + 1, 40, 100.0); rho = S.rho_schedule(t, 1.0, 0.5); tick("sched", t0)
    t0 = time.perf_counter(); tr.period_sample(b, t, m_t); tick("period_sample", t0)
    t0 = time.perf_counter(); tr.period_update(rho); tick("period_update", t0)
torch.cuda.synchronize()
wall = time.perf_counter() - T0
print(f"25 periods wall {wall*1e3:.1f} ms -> {wall/25*1e3:.2f} ms/period")
for k, v in acc.items(): print(f"  {k:14s} {v/25*1e3:8.3f} ms/period")
