"""Debug: per-call throughput sample_counts vs the period path's first sweep."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import Port
from paper_1409_5402_b200 import samelda as S
sys.path.insert(0, "tests")
from test_throughput_gpu import _phi_counts

port = Port()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = port.make_corpus(50, 90, 4, 30.0, 3)
m_t, seed, t = 40.0, 21, 5
tr = S.Trainer(g, S.SamplerConfig(n_topics=K, m=m_t, t_max=1, batch_fraction=1.0, seed=seed,
                                  inner_sweeps=1, mode=S.MODE_THROUGHPUT))
batch = np.random.default_rng(1).permutation(g.n_docs).astype(np.int32)
tr.period_sample(batch, t, m_t)
pcp = _phi_counts(tr, g.n_words, K)
tcp, pcpt = tr.count_totals()
m = tr.model()
tb = m.theta[batch]
mu = port.sddmm(tb, m.phi, g, batch)
a = S.sample_counts(tb, m.phi, mu, g, batch, m_t, seed, t, 0, mode=S.MODE_THROUGHPUT)
d = a.phi_counts - pcp
print("totals period", tcp, pcpt, "per-call", a.theta_total(), a.phi_total(), "pcp sum", pcp.sum())
nz = np.argwhere(d != 0)
print("diff cells", len(nz), "words", np.unique(nz[:, 0])[:20], "topics", np.unique(nz[:, 1])[:40])
print("theta rows equal?", np.unique(tb).size, "phi range", m.phi.min(), m.phi.max())
