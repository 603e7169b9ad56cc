import sys, time, os
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_1409_5402_b200 import samelda as S, distributed as DIST
train, heldout = bench.single_gpu_corpus("nytimes")
ctx = S.Context(0)
stream = torch.cuda.Stream(device=0); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
T = 100
MODE = int(os.environ.get("MODE", "0"))
tr = S.Trainer(train, S.SamplerConfig(n_topics=256, m=100.0, batch_fraction=0.05, t_max=T, seed=1, mode=MODE), ctx=ctx)
tr.set_heldout(heldout, seed=1)
eng = DIST.CudaEngine(tr, 0)
st = DIST.ShardedTrainer(eng, train.n_docs, 0, train.n_docs, train.doc_tokens(), 0.05, 1, 100.0, "constant", T)
for _ in range(5): st.period()
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(stream)
for _ in range(20): st.period()
ev1.record(stream); torch.cuda.synchronize()
print("timed device ms/period", ev0.elapsed_time(ev1)/20)
bmax = int(1.25 * 0.05 * train.n_docs) + 64
bufs = [torch.empty(bmax * 256, dtype=torch.float64, pin_memory=True).numpy() for _ in range(20)]
torch.cuda.synchronize()
t0 = time.perf_counter(); hs=[]
ev0.record(stream)
for i in range(20):
    h0=time.perf_counter()
    s = st.period()
    tr.batch_theta_async(s.owned_docs, bufs[i])
    hs.append(1e3*(time.perf_counter()-h0))
ev1.record(stream)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print("e2e wall ms/period", 1e3*wall/20, "device", ev0.elapsed_time(ev1)/20, "host per call", [round(x,2) for x in hs])
