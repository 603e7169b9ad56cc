import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_1409_5402_b200 import samelda as S, distributed as D
from oracle import Port
g = Port().make_corpus(40, 30, 3, 20.0, 3)
tr = S.Trainer(g, S.SamplerConfig(n_topics=4, m=5.0, t_max=3, batch_fraction=1.0, seed=1))
tr.period_sample(np.arange(g.n_docs, dtype=np.int32), 0, 5.0)
eng = D.CudaEngine(tr, 0)
t = eng.counts()
print("sum via torch", int(t.sum()), "totals via C ABI", tr.count_totals())
t.zero_()
torch.cuda.synchronize()
print("after torch zero_: C ABI sees", tr.count_totals())
ptr = tr.phi_counts_device()[0]
print("ptr", hex(ptr), "torch data_ptr", hex(t.data_ptr()))
