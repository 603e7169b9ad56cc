"""Debug: sharded periods in ONE process (two contexts, counts summed by hand) vs train()."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1409_5402_b200 import samelda as S, distributed as D
from oracle import Port
K, SEED, M, T_MAX, BF = 8, 7, 20.0, 5, 0.25
g = S.Corpus.of(Port().make_corpus(120, 60, 4, 30.0, 3))
cfg = S.SamplerConfig(n_topics=K, m=M, schedule="invlinear", t_max=T_MAX, batch_fraction=BF, seed=SEED)
ref, _ = S.train(g, cfg)
# world = 1 through ShardedTrainer
tr = S.Trainer(g, cfg)
st = D.ShardedTrainer(D.CudaEngine(tr, 0), g.n_docs, 0, g.n_docs, g.doc_tokens(), BF, SEED, M, "invlinear", T_MAX)
for _ in range(T_MAX): st.period()
print("world1 equal:", np.array_equal(tr.model().phi, ref.phi))
# two shards by hand
ranges = D.shard_ranges(g.doc_offsets, 2)
trs, engs = [], []
for lo, hi in ranges:
    offs = g.doc_offsets[lo:hi + 1] - g.doc_offsets[lo]
    local = S.Corpus(offs, g.word_ids[g.doc_offsets[lo]:g.doc_offsets[hi]], g.counts[g.doc_offsets[lo]:g.doc_offsets[hi]], g.n_words)
    t_ = S.Trainer(local, cfg, ctx=S.Context(0)); t_.set_doc_base(lo); trs.append(t_); engs.append(D.CudaEngine(t_, 0))
stream = S.MinibatchStream(g.n_docs, BF, SEED)
for t in range(T_MAX):
    batch = stream.next()
    m_t = S.anneal_m("invlinear", t + 1, T_MAX, M); rho = S.rho_schedule(t, 1.0, 0.5)
    for (lo, hi), e in zip(ranges, engs):
        e.sample(D.owned(batch, lo, hi), t, m_t)
    torch.cuda.synchronize()
    tot = sum(e.counts().clone() for e in engs)
    for e in engs:
        e.counts().copy_(tot)
    torch.cuda.synchronize()
    for e in engs:
        e.update(rho)
    print(t, "phi equal rank0/rank1:", np.array_equal(trs[0].model(False).phi, trs[1].model(False).phi))
print("sharded equal:", np.array_equal(trs[0].model(False).phi, ref.phi))
