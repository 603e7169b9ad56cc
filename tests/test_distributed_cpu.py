"""World-size-2 doc-sharded training on CPU (gloo): the product's sharding and
exchange logic (paper_1409_5402_b200/distributed.py) driving an oracle engine
per rank must reproduce single-process train() bit for bit -- the property
that makes the NCCL run on B200s identical to one GPU."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1409_5402_b200 import distributed as D

K, SEED, M, T_MAX, BF = 4, 31, 10.0, 6, 0.3


class OracleEngine:
    """Per-rank compute on the C restatement (test infrastructure)."""

    def __init__(self, port, corpus, lo, hi):
        self.port, self.corpus, self.lo, self.hi = port, corpus, lo, hi
        W = corpus.n_words
        self.phi = port.init_phi(K, W, 0.1, SEED)
        self.theta = np.full((corpus.n_docs, K), 0.1 + 1.0 / K)
        self.counts_t = torch.zeros(W * K, dtype=torch.int64)

    def sample(self, local_ids, t, m_t):
        ids = (local_ids.astype(np.int64) + self.lo).astype(np.int32)  # global doc ids
        self.ids = ids
        tb = self.theta[ids]
        tc = np.zeros((0, K), np.int64)
        pc = np.zeros((self.corpus.n_words, K), np.int64)
        for sweep in range(2):
            if len(ids):
                mu = self.port.sddmm(tb, self.phi, self.corpus, ids)
                tc, pc = self.port.sample_counts(tb, self.phi, mu, self.corpus, ids, m_t, SEED,
                                                 t, sweep)
                tb = tc / m_t + 0.1
        self.tc, self.m_t = tc, m_t
        self.counts_t.copy_(torch.from_numpy(pc.reshape(-1)))

    def counts(self):
        return self.counts_t

    def update(self, rho):
        pc = self.counts_t.numpy().reshape(self.corpus.n_words, K)
        tc = self.tc if len(self.ids) else np.zeros((0, K), np.int64)
        self.theta, self.phi = self.port.update_model(self.theta, self.phi, self.ids, tc, pc,
                                                      self.m_t, rho, 0.1, 0.01)


def _corpus():
    from oracle import Port
    port = Port()
    return port, port.make_corpus(40, 25, 3, 15.0, 8)


def _worker(rank, world, port_no, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port, corpus = _corpus()
    lo, hi = D.shard_ranges(corpus.doc_offsets, world)[rank]
    eng = OracleEngine(port, corpus, lo, hi)
    toks = np.array([corpus.counts[corpus.doc_offsets[d]:corpus.doc_offsets[d + 1]].sum()
                     for d in range(lo, hi)])
    tr = D.ShardedTrainer(eng, corpus.n_docs, lo, hi, toks, BF, SEED, M, "linear", T_MAX)
    for _ in range(T_MAX):
        tr.period()
    # gather owned theta rows on rank 0 (each rank holds its own rows)
    theta_rows = torch.from_numpy(eng.theta[lo:hi].copy())
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([hi - lo]))
    if rank == 0:
        parts = [theta_rows] + [torch.zeros((int(s.item()), K), dtype=torch.float64)
                                for s in sizes[1:]]
        for r in range(1, world):
            dist.recv(parts[r], src=r)
        np.savez(out_path, phi=eng.phi, theta=torch.cat(parts).numpy())
    else:
        dist.send(theta_rows, dst=0)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_balance_and_cover():
    offs = np.array([0, 5, 6, 30, 31, 40, 80, 81, 100], np.int64)
    for world in (1, 2, 3, 8):
        r = D.shard_ranges(offs, world)
        assert r[0][0] == 0 and r[-1][1] == len(offs) - 1
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))


def test_owned_preserves_batch_order():
    np.testing.assert_array_equal(D.owned(np.array([7, 2, 9, 4, 5]), 3, 8), [4, 1, 2])


@pytest.mark.timeout(300)
def test_two_rank_training_equals_single_process(tmp_path):
    from oracle import TrainConfig
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn")
    got = np.load(out)
    port, corpus = _corpus()
    cfg = TrainConfig(n_topics=K, m=M, schedule="linear", t_max=T_MAX, batch_fraction=BF,
                      seed=SEED, inner_sweeps=2)
    phi, theta, _ = port.train(corpus, cfg)
    np.testing.assert_array_equal(got["phi"], phi)
    np.testing.assert_array_equal(got["theta"], theta)
