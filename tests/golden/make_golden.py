"""Generate the golden parity fixtures from the COMPILED REFERENCE (oracle/_ref).

    make -C oracle && python tests/golden/make_golden.py

Every array in golden.npz / c1_train.json is produced by the reference's own
code (proj/src via oracle/_ref/libsamelda_ref.so), never by the code under
test.  The fixtures pin:
  * the Philox stream words, uniforms and uniform_below (rng.cpp:24-133)
  * Poisson draws across the inversion / PTRS boundary (rng.cpp:39-150)
  * sddmm / sample_counts / update_model on a small synthetic corpus
    (sampler.cpp:88-229), in three (m_t, seed, t, sweep) settings
  * fold_in_theta / perword_loglik (eval.cpp:19-159)
  * MinibatchStream batches and split_holdout (corpus.cpp:231-285)
  * rho_schedule / anneal_m grids (sampler.cpp:231-267)
  * full train() runs: phi, theta and the metrics trace (sampler.cpp:269-353)
  * c1_train.json: BASELINE config 0 (10K docs x 5K vocab, K=32, m=10,
    20 full-batch periods) -- phi digest and ll trace.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Ref, TrainConfig  # noqa: E402

SMALL = dict(n_docs=60, n_words=40, n_topics=4, len_mean=25.0, seed=5)
C1 = dict(n_docs=10000, n_words=5000, n_topics=32, len_mean=100.0, seed=1)
C1_CONFIG = dict(n_topics=32, m=10.0, t_max=20, batch_fraction=1.0, inner_sweeps=2, alpha=0.1,
                 beta=0.01, tau0=1.0, gamma=0.5, init_noise=0.1, seed=1)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(with_c1: bool = True) -> None:
    R = Ref()
    out: dict[str, np.ndarray] = {}
    # --- Philox words / uniforms (SURVEY Appendix A keys + a few more)
    keys = np.array([[0, 0, 0, 0, 0], [0x0123456789abcdef, 7, 123456, 98765, 0],
                     [0x0123456789abcdef, 7, 123456, 98765, 0x101000c8],
                     [42, 3, 17, 92, (1 << 28) | (1 << 20) | 4], [2**64 - 1, 2**32 - 1, 5, 9, 0x60000000]],
                    dtype=np.uint64)
    out["philox_keys"] = keys
    out["philox_words"] = np.stack([R.stream_u32(int(k[0]), int(k[1]), int(k[2]), int(k[3]),
                                                 int(k[4]), 16) for k in keys])
    out["uniform"] = np.stack([R.stream_uniform(int(k[0]), int(k[1]), int(k[2]), int(k[3]),
                                                int(k[4]), 8) for k in keys])
    out["uniform_oo"] = np.stack([R.stream_uniform(int(k[0]), int(k[1]), int(k[2]), int(k[3]),
                                                   int(k[4]), 8, oo=True) for k in keys])
    out["below"] = np.stack([R.stream_below(int(k[0]), int(k[1]), int(k[2]), int(k[3]),
                                            int(k[4]), 1000003, 8) for k in keys])
    # --- Poisson grid (fresh stream per draw, keyed like sample_counts)
    lams = np.array([1e-3, 0.05, 0.3, 1.0, 4.0, 9.5, 9.99, 10.0, 10.5, 57.5, 156.0, 1234.5, 1e5])
    out["poisson_lambdas"] = lams
    out["poisson_draws"] = np.stack([R.poisson_grid(float(l), 1, 0, 5, 17, 0, 0, 256) for l in lams])
    out["poisson_draws_s2"] = np.stack([R.poisson_grid(float(l), 0xdeadbeefcafef00d, 9, 77, 4242, 3,
                                                       1000, 256) for l in lams])
    # --- small synthetic corpus + per-call hot path
    g = R.make_corpus(**SMALL)
    out["small_offsets"], out["small_words"], out["small_counts"] = (g.doc_offsets, g.word_ids,
                                                                     g.counts)
    out["small_phi_true"] = g.phi_true
    K, W, D = SMALL["n_topics"], SMALL["n_words"], SMALL["n_docs"]
    rng = np.random.default_rng(11)
    theta = rng.uniform(0.05, 2.0, size=(D, K))
    phi = rng.uniform(0.0, 1.0, size=(K, W))
    phi /= phi.sum(axis=1, keepdims=True)
    batch = rng.permutation(D)[:37].astype(np.int32)
    theta_b = theta[batch]
    out["small_theta"], out["small_phi"], out["small_batch"] = theta, phi, batch
    mu = R.sddmm(theta_b, phi, g, batch)
    out["small_mu"] = mu
    settings = [(10.0, 1, 0, 0), (100.0, 0x0123456789abcdef, 7, 1), (0.37, 99, 3, 255)]
    out["sample_m_t"] = np.array([s[0] for s in settings], dtype=np.float64)
    out["sample_seed"] = np.array([s[1] for s in settings], dtype=np.uint64)
    out["sample_t_sweep"] = np.array([[s[2], s[3]] for s in settings], dtype=np.int64)
    for i, (m_t, seed, t, sweep) in enumerate(settings):
        tc, pc = R.sample_counts(theta_b, phi, mu, g, batch, m_t, seed, t, sweep)
        out[f"small_tc{i}"], out[f"small_pc{i}"] = tc, pc
        th2, ph2 = R.update_model(theta, phi, batch, tc, pc, m_t, 0.37 + 0.2 * i, 0.1, 0.01)
        out[f"small_upd_theta{i}"], out[f"small_upd_phi{i}"] = th2, ph2
    # large rates: PTRS path inside sample_counts
    big_theta_b = theta_b * 50.0
    mu_big = R.sddmm(big_theta_b, phi, g, batch)
    tc, pc = R.sample_counts(big_theta_b, phi, mu_big, g, batch, 2000.0, 5, 1, 0)
    out["small_big_tc"], out["small_big_pc"] = tc, pc
    # eval
    out["small_ll_true"] = np.array([R.perword_loglik(g.phi_true, g, 0.1, 3)])
    out["small_ll_rand"] = np.array([R.perword_loglik(phi, g, 0.1, 12345)])
    w0 = g.word_ids[g.doc_offsets[0]:g.doc_offsets[1]]
    c0 = g.counts[g.doc_offsets[0]:g.doc_offsets[1]]
    out["small_fold_in"] = R.fold_in_theta(g.phi_true, w0, c0, 0.1, 50)
    out["small_fold_in_5"] = R.fold_in_theta(phi, w0, c0, 0.3, 5)
    # minibatches + split
    mbs = R.minibatches(97, 0.1, 77, 25)
    out["minibatch_sizes"] = np.array([len(b) for b in mbs])
    out["minibatch_ids"] = np.concatenate(mbs)
    tr, te = R.split_holdout(g, 0.2, 9)
    out["split_train_offsets"], out["split_test_offsets"] = tr.doc_offsets, te.doc_offsets
    out["split_train_words"], out["split_test_words"] = tr.word_ids, te.word_ids
    # schedules
    sched = []
    for s in range(4):
        for tmax in (1, 7, 20):
            for t in range(1, tmax + 1):
                sched.append([s, t, tmax, R.anneal_m(s, t, tmax, 100.0)])
    out["anneal_grid"] = np.array(sched)
    out["rho_grid"] = np.array([[t, tau, gm, R.rho_schedule(t, tau, gm)]
                                for t in (0, 1, 3, 17, 1000) for tau in (1.0, 64.0)
                                for gm in (0.5, 0.7, 1.0)])
    # full train() runs on the small corpus
    for name, cfg in {
        "train_a": TrainConfig(n_topics=4, m=10.0, t_max=8, batch_fraction=0.25, seed=31),
        "train_b": TrainConfig(n_topics=4, m=3.5, t_max=6, batch_fraction=1.0, seed=7,
                               schedule="linear", inner_sweeps=3),
        "train_c": TrainConfig(n_topics=4, m=20.0, t_max=5, batch_fraction=0.5, seed=2,
                               schedule="log", init_noise=0.0),
    }.items():
        phi_o, theta_o, trace = R.train(tr, cfg, te, 2)
        out[f"{name}_phi"], out[f"{name}_theta"] = phi_o, theta_o
        out[f"{name}_ll"] = np.array([r["ll"] for r in trace])
        out[f"{name}_spw"] = np.array([r["samples_per_word"] for r in trace])
        out[f"{name}_passes"] = np.array([r["passes"] for r in trace])
        out[f"{name}_cfg"] = np.array([cfg.n_topics, cfg.m, ["constant", "linear", "log",
                                                              "invlinear"].index(cfg.schedule),
                                       cfg.t_max, cfg.batch_fraction, cfg.inner_sweeps, cfg.seed,
                                       cfg.init_noise])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote golden.npz with", len(out), "arrays")

    if with_c1:
        import time
        t0 = time.time()
        g1 = R.make_corpus(**C1)
        tr1, te1 = R.split_holdout(g1, 0.1, 1)
        cfg = TrainConfig(**C1_CONFIG, n_threads=os.cpu_count() or 1)
        phi_o, theta_o, trace = R.train(tr1, cfg, te1, 5)
        rec = dict(corpus=C1, config=C1_CONFIG, split=dict(test_fraction=0.1, seed=1),
                   corpus_digest=dict(offsets=digest(g1.doc_offsets), words=digest(g1.word_ids),
                                      counts=digest(g1.counts)),
                   train_nnz=int(tr1.nnz), train_tokens=int(tr1.n_tokens),
                   phi_digest=digest(phi_o), theta_digest=digest(theta_o),
                   trace=[{k: (v.hex() if isinstance(v, float) else v) for k, v in r.items()
                           if k != "wall_seconds"} for r in trace],
                   seconds=time.time() - t0)
        with open(os.path.join(HERE, "c1_train.json"), "w") as f:
            json.dump(rec, f, indent=1)
        print("wrote c1_train.json", rec["trace"][-1], f"{rec['seconds']:.1f}s")


if __name__ == "__main__":
    main(with_c1="--no-c1" not in sys.argv)
