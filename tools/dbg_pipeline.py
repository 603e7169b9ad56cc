import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1409_5402_b200 import samelda as S
from oracle import Port
port = Port()
tr = port.make_corpus(60, 40, 4, 9, 5)
cfg = S.SamplerConfig(n_topics=8, m=5.0, t_max=4, batch_fraction=0.3, seed=3)

def run(sync_each, async_each, other=None):
    a = S.Trainer(tr, cfg)
    s = S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed)
    for t in range(4):
        m_t, rho = S.anneal_m("constant", t + 1, 4, cfg.m), S.rho_schedule(t, 1.0, 0.5)
        batch = s.next()
        a.period(batch, t, m_t, rho)
        if async_each:
            a.batch_theta_async(len(batch), np.zeros(len(batch) * 8))
        if other is not None:
            other(t)
        if sync_each:
            a.ctx.synchronize()
    return a.model().theta

ref = run(True, False)
print("nosync            ", np.array_equal(run(False, False), ref))
print("nosync+async      ", np.array_equal(run(False, True), ref))
b = S.Trainer(tr, cfg)
sb = S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed)
def other(t):
    m_t, rho = S.anneal_m("constant", t + 1, 4, cfg.m), S.rho_schedule(t, 1.0, 0.5)
    b.period(sb.next(), t, m_t, rho)
print("nosync+other ctx  ", np.array_equal(run(False, False, other), ref))
b = S.Trainer(tr, cfg); sb = S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed)
print("sync+other ctx    ", np.array_equal(run(True, False, other), ref))
print("b (other) correct ", np.array_equal(b.model().theta, ref))
