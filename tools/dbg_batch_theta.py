import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1409_5402_b200 import samelda as S
from oracle import Port
rng = np.random.default_rng(0)
port = Port()
corpus = port.make_corpus(60, 40, 4, 9, 5)
tr = corpus
cfg = S.SamplerConfig(n_topics=8, m=5.0, t_max=4, batch_fraction=0.3, seed=3)
a, b = S.Trainer(tr, cfg), S.Trainer(tr, cfg)
sa = S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed)
sb = S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed)
for t in range(3):
    m_t, rho = S.anneal_m("constant", t + 1, 4, cfg.m), S.rho_schedule(t, 1.0, 0.5)
    ba, bb = sa.next(), sb.next()
    print("batches equal", np.array_equal(ba, bb), len(ba))
    a.period(ba, t, m_t, rho)
    b.period(bb, t, m_t, rho)
    ra = a.batch_theta(len(ba))
    rb = b.batch_theta(len(bb))
    buf = np.full(len(ba) * 8, np.nan)
    rasync = a.batch_theta_async(len(ba), buf); a.ctx.synchronize()
    ma = a.model().theta[ba]; mb = b.model().theta[bb]
    print(t, "a==b sync", np.array_equal(ra, rb), "async==sync", np.array_equal(rasync, ra),
          "model a==b", np.array_equal(ma, mb), "sync==model", np.array_equal(ra, ma))

print("--- test order")
a, b = S.Trainer(tr, cfg), S.Trainer(tr, cfg)
sa = S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed)
sb = S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed)
bufs, sync_rows, pinned = [], [], []
import torch
for t in range(4):
    m_t, rho = S.anneal_m("constant", t + 1, 4, cfg.m), S.rho_schedule(t, 1.0, 0.5)
    batch = sa.next()
    a.period(batch, t, m_t, rho)
    buf = np.full(len(batch) * 8 + 3, np.nan)
    bufs.append(a.batch_theta_async(len(batch), buf))
    pb = torch.full((len(batch) * 8,), float("nan"), dtype=torch.float64, pin_memory=True).numpy()
    pinned.append(a.batch_theta_async(len(batch), pb))
    b.period(sb.next(), t, m_t, rho)
    sync_rows.append(b.batch_theta(len(batch)))
    print(t, "immediately: pageable==sync", np.array_equal(bufs[-1], sync_rows[-1]))
a.ctx.synchronize()
for t in range(4):
    print(t, "pageable==sync", np.array_equal(bufs[t], sync_rows[t]), "pinned==sync", np.array_equal(pinned[t], sync_rows[t]))
