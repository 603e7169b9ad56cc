"""CUDA path (through the C ABI) against the reference's golden fixtures and the
oracle on seeded inputs.  Bar: bit-exact for counts, ids and the parity-mode
model (f64, reference rounding); 1e-12 relative for ll; 1e-5 relative for the
expected-count path (north_star).  Also the reference's own statistical and
error-convention tests (test_sampler.cpp, test_eval.cpp) ported verbatim."""
from __future__ import annotations

import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import CorpusArrays, TrainConfig

pytestmark = pytest.mark.gpu

S = None


@pytest.fixture(scope="module", autouse=True)
def _samelda(cuda_ctx):
    global S
    from paper_1409_5402_b200 import samelda
    S = samelda
    yield


def tiny(n_docs, n_words, cells):
    """test_sampler.cpp:18-42 make_corpus from (doc, word, count) triplets."""
    offs = np.zeros(n_docs + 1, np.int64)
    words, counts = [], []
    for d, w, c in cells:
        offs[d + 1:] += 1
        words.append(w)
        counts.append(c)
    return CorpusArrays(offs, np.array(words, np.int32), np.array(counts, np.int32), n_words)


def all_docs(c):
    return np.arange(c.n_docs, dtype=np.int32)


# ------------------------------------------------------------ golden parity

def test_sddmm_bit_exact(golden, small):
    tb = golden["small_theta"][golden["small_batch"]]
    mu = S.sddmm(tb, golden["small_phi"], small, golden["small_batch"])
    np.testing.assert_array_equal(mu, golden["small_mu"])


def test_sample_counts_bit_exact(golden, small):
    batch, phi = golden["small_batch"], golden["small_phi"]
    tb = golden["small_theta"][batch]
    for i, (m_t, seed, (t, sweep)) in enumerate(zip(golden["sample_m_t"], golden["sample_seed"],
                                                    golden["sample_t_sweep"])):
        sc = S.sample_counts(tb, phi, golden["small_mu"], small, batch, m_t, int(seed), int(t),
                             int(sweep))
        np.testing.assert_array_equal(sc.theta_counts, golden[f"small_tc{i}"])
        np.testing.assert_array_equal(sc.phi_counts, golden[f"small_pc{i}"])
        assert sc.theta_total() == sc.phi_total()


def test_sample_counts_ptrs_bit_exact(golden, small):
    batch, phi = golden["small_batch"], golden["small_phi"]
    big = golden["small_theta"][batch] * 50.0
    mu = S.sddmm(big, phi, small, batch)
    sc = S.sample_counts(big, phi, mu, small, batch, 2000.0, 5, 1, 0)
    np.testing.assert_array_equal(sc.theta_counts, golden["small_big_tc"])
    np.testing.assert_array_equal(sc.phi_counts, golden["small_big_pc"])


def test_update_model_bit_exact(golden):
    batch, theta, phi = golden["small_batch"], golden["small_theta"], golden["small_phi"]
    K, W = phi.shape
    for i, m_t in enumerate(golden["sample_m_t"]):
        model = S.Model(K, W, 0.1, 0.01, phi.copy(), theta.copy())
        counts = S.SampledCounts(batch, K, W, float(m_t), golden[f"small_tc{i}"],
                                 golden[f"small_pc{i}"])
        S.update_model(model, counts, 0.37 + 0.2 * i)
        np.testing.assert_array_equal(model.theta, golden[f"small_upd_theta{i}"])
        np.testing.assert_array_equal(model.phi, golden[f"small_upd_phi{i}"])


def test_eval_matches_reference(golden, small):
    ll = S.perword_loglik(small.phi_true, small, 0.1, 3)
    assert ll == pytest.approx(golden["small_ll_true"][0], rel=1e-12, abs=0)
    ll2 = S.perword_loglik(golden["small_phi"], small, 0.1, 12345)
    assert ll2 == pytest.approx(golden["small_ll_rand"][0], rel=1e-12, abs=0)
    w0 = small.word_ids[small.doc_offsets[0]:small.doc_offsets[1]]
    c0 = small.counts[small.doc_offsets[0]:small.doc_offsets[1]]
    np.testing.assert_allclose(S.fold_in_theta(small.phi_true, w0, c0, 0.1, 50),
                               golden["small_fold_in"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(S.fold_in_theta(golden["small_phi"], w0, c0, 0.3, 5),
                               golden["small_fold_in_5"], rtol=1e-12, atol=0)


def _cfg_from(arr, cls):
    n_topics, m, sched, t_max, bf, inner, seed, noise = arr
    return cls(n_topics=int(n_topics), m=float(m),
               schedule=["constant", "linear", "log", "invlinear"][int(sched)], t_max=int(t_max),
               batch_fraction=float(bf), inner_sweeps=int(inner), seed=int(seed),
               init_noise=float(noise))


@pytest.mark.parametrize("name", ["train_a", "train_b", "train_c"])
def test_train_bit_exact(golden, small_split, name):
    tr, te = small_split
    model, trace = S.train(tr, _cfg_from(golden[f"{name}_cfg"], S.SamplerConfig), te, 2)
    np.testing.assert_array_equal(model.phi, golden[f"{name}_phi"])
    np.testing.assert_array_equal(model.theta, golden[f"{name}_theta"])
    np.testing.assert_allclose([r["ll"] for r in trace], golden[f"{name}_ll"], rtol=1e-12, atol=0)
    np.testing.assert_array_equal([r["samples_per_word"] for r in trace], golden[f"{name}_spw"])
    np.testing.assert_array_equal([r["passes"] for r in trace], golden[f"{name}_passes"])


def test_c1_train_matches_reference(port):
    """BASELINE config 0 end to end: 20 full-batch periods, K=32, m=10."""
    rec = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c1_train.json")))
    c = rec["corpus"]
    g = port.make_corpus(c["n_docs"], c["n_words"], c["n_topics"], c["len_mean"], c["seed"])
    tr, te = port.split_holdout(g, 0.1, 1)
    cfg = S.SamplerConfig(**rec["config"])
    model, trace = S.train(tr, cfg, te, 5)
    got = [r["ll"] for r in trace]
    want = [float.fromhex(r["ll"]) for r in rec["trace"]]
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
    assert [r["samples_per_word"].hex() for r in trace] == [r["samples_per_word"]
                                                           for r in rec["trace"]]
    digest = hashlib.sha256(np.ascontiguousarray(model.phi).tobytes()).hexdigest()
    assert digest == rec["phi_digest"]


def test_trainer_periods_equal_composed_calls(port, small_split):
    """samelda_cu_period == sddmm -> sample_counts -> update_model composed by hand."""
    tr, _ = small_split
    cfg = S.SamplerConfig(n_topics=4, m=7.0, t_max=3, batch_fraction=0.3, seed=9)
    trainer = S.Trainer(tr, cfg)
    model = trainer.model()
    stream = S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed)
    for t in range(3):
        batch = stream.next()
        m_t, rho = S.anneal_m("constant", t + 1, 3, cfg.m), S.rho_schedule(t, 1.0, 0.5)
        trainer.period(batch, t, m_t, rho)
        tb = model.theta[batch]
        for sweep in range(cfg.inner_sweeps):
            mu = S.sddmm(tb, model.phi, tr, batch)
            counts = S.sample_counts(tb, model.phi, mu, tr, batch, m_t, cfg.seed, t, sweep)
            tb = counts.theta_counts / m_t + cfg.alpha
        S.update_model(model, counts, rho)
        assert trainer.count_totals() == (counts.theta_total(), counts.phi_total())
        dev = trainer.model()
        np.testing.assert_array_equal(dev.phi, model.phi)
        np.testing.assert_array_equal(dev.theta, model.theta)


def test_batch_theta_async_matches_sync(small_split):
    """Async result copies queued behind later periods equal the sync copies."""
    tr, _ = small_split
    cfg = S.SamplerConfig(n_topics=8, m=5.0, t_max=4, batch_fraction=0.3, seed=3)
    a, b = S.Trainer(tr, cfg), S.Trainer(tr, cfg)
    sa, sb = (S.MinibatchStream(tr.n_docs, cfg.batch_fraction, cfg.seed) for _ in range(2))
    bufs, sync_rows = [], []
    for t in range(4):
        m_t, rho = S.anneal_m("constant", t + 1, 4, cfg.m), S.rho_schedule(t, 1.0, 0.5)
        batch = sa.next()
        a.period(batch, t, m_t, rho)
        buf = np.full(len(batch) * cfg.n_topics + 3, np.nan)
        bufs.append((a.batch_theta_async(len(batch), buf), len(batch)))
        b.period(sb.next(), t, m_t, rho)
        sync_rows.append(b.batch_theta(len(batch)))
    a.ctx.synchronize()
    for (rows, n), ref in zip(bufs, sync_rows):
        np.testing.assert_array_equal(rows, ref)
    with pytest.raises(S.ConfigError):
        a.batch_theta_async(len(batch), np.zeros(2))


def test_trainers_do_not_share_device_state(small_split):
    """Each Trainer owns its context; re-initialising a shared one is loud."""
    tr, _ = small_split
    cfg = S.SamplerConfig(n_topics=4, m=3.0, t_max=2, batch_fraction=0.5, seed=4)
    a, b = S.Trainer(tr, cfg), S.Trainer(tr, cfg)
    assert a.ctx is not b.ctx
    ctx = S.Context(0)
    c = S.Trainer(tr, cfg, ctx=ctx)
    S.Trainer(tr, cfg, ctx=ctx)
    with pytest.raises(S.ConfigError):
        c.period(np.arange(3, dtype=np.int32), 0, 3.0, 1.0)


def test_expected_counts_match_oracle(port, golden, small):
    batch, phi = golden["small_batch"], golden["small_phi"]
    tb = golden["small_theta"][batch]
    mu = golden["small_mu"]
    tf, pf = S.expected_counts(tb, phi, mu, small, batch, 3.0)
    otf, opf = port.expected_counts(tb, phi, mu, small, batch, 3.0)
    np.testing.assert_allclose(tf, otf, rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(pf, opf, rtol=1e-12, atol=1e-300)


def test_expected_train_within_1e5(port, small_split):
    tr, te = small_split
    cfg = S.SamplerConfig(n_topics=4, m=10.0, t_max=6, batch_fraction=0.5, seed=3,
                          mode=S.MODE_EXPECTED)
    model, trace = S.train(tr, cfg, te, 3)
    ocfg = TrainConfig(n_topics=4, m=10.0, t_max=6, batch_fraction=0.5, seed=3)
    ophi, otheta, otrace = port.train(tr, ocfg, te, 3, expected=True)
    np.testing.assert_allclose(model.phi, ophi, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(model.theta, otheta, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose([r["ll"] for r in trace], [r["ll"] for r in otrace], rtol=1e-9)


@pytest.mark.parametrize("K", [256, 200, 300])
def test_expected_train_wide_k_within_1e5(port, K):
    """The period path's expected-count kernel (k_expected: 8 topics per lane,
    fused f64 mu for K <= 256, full and partial slices; K > 256 takes the
    SDDMM's mu) against the oracle."""
    g = port.make_corpus(80, 150, 6, 60.0, 12)
    tr, te = port.split_holdout(g, 0.15, 3)
    kw = dict(n_topics=K, m=20.0, t_max=3, batch_fraction=0.5, seed=5)
    model, trace = S.train(tr, S.SamplerConfig(mode=S.MODE_EXPECTED, **kw), te, 3)
    ophi, otheta, otrace = port.train(tr, TrainConfig(**kw), te, 3, expected=True)
    np.testing.assert_allclose(model.phi, ophi, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(model.theta, otheta, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose([r["ll"] for r in trace], [r["ll"] for r in otrace], rtol=1e-9)


def test_random_larger_case_bit_exact(port):
    """K=256 (8 topics per lane), multi-chunk docs, random theta/phi: counts bit-exact."""
    g = port.make_corpus(300, 700, 8, 120.0, 21)
    rng = np.random.default_rng(5)
    K = 256
    theta = rng.gamma(0.3, 1.0, size=(g.n_docs, K)) + 1e-3
    phi = rng.gamma(0.2, 1.0, size=(K, g.n_words)) + 1e-9
    phi /= phi.sum(1, keepdims=True)
    batch = rng.permutation(g.n_docs)[:211].astype(np.int32)
    tb = theta[batch]
    mu = S.sddmm(tb, phi, g, batch)
    np.testing.assert_array_equal(mu, port.sddmm(tb, phi, g, batch))
    sc = S.sample_counts(tb, phi, mu, g, batch, 100.0, 77, 4, 1)
    otc, opc = port.sample_counts(tb, phi, mu, g, batch, 100.0, 77, 4, 1)
    np.testing.assert_array_equal(sc.theta_counts, otc)
    np.testing.assert_array_equal(sc.phi_counts, opc)
    # per-doc and per-word integer totals
    np.testing.assert_array_equal(sc.theta_counts.sum(1), otc.sum(1))
    np.testing.assert_array_equal(sc.phi_counts.sum(1), opc.sum(1))


@pytest.mark.parametrize("K", [1, 3, 33, 100, 300, 1024])
def test_odd_topic_counts_bit_exact(port, K):
    g = port.make_corpus(40, 90, 5, 30.0, 3 + K)
    rng = np.random.default_rng(K)
    theta = rng.uniform(0.01, 1.0, size=(g.n_docs, K))
    phi = rng.uniform(0.0, 1.0, size=(K, g.n_words))
    phi /= phi.sum(1, keepdims=True)
    batch = all_docs(g)
    mu = S.sddmm(theta, phi, g, batch)
    np.testing.assert_array_equal(mu, port.sddmm(theta, phi, g, batch))
    sc = S.sample_counts(theta, phi, mu, g, batch, 12.5, 3, 2, 0)
    otc, opc = port.sample_counts(theta, phi, mu, g, batch, 12.5, 3, 2, 0)
    np.testing.assert_array_equal(sc.theta_counts, otc)
    np.testing.assert_array_equal(sc.phi_counts, opc)
    ll = S.perword_loglik(phi, g, 0.1, 4)
    assert ll == pytest.approx(port.perword_loglik(phi, g, 0.1, 4), rel=1e-12, abs=0)


# -------------------------------------- reference unit tests (test_sampler.cpp)

def test_sddmm_unit_theta_row():
    c = tiny(1, 2, [(0, 1, 1)])
    mu = S.sddmm(np.array([[1.0, 0.0]]), np.array([[0.3, 0.7], [0.5, 0.5]]), c, [0])
    assert len(mu) == 1 and mu[0] == pytest.approx(0.7, rel=1e-15)


def test_sddmm_empty_and_shape_errors():
    c = tiny(2, 3, [(0, 1, 4)])
    assert len(S.sddmm(np.zeros((0, 2)), np.full((2, 3), 0.5), c, [])) == 0
    c1 = tiny(1, 3, [(0, 0, 1)])
    with pytest.raises(S.ConfigError):
        S.sddmm(np.zeros((1, 2)), np.full((3, 3), 0.5), c1, [0])


def test_single_topic_scaled_poisson():
    # test_sampler.cpp:160-179
    c = tiny(1, 2, [(0, 0, 2), (0, 1, 1)])
    theta, phi, m_t = np.ones((1, 1)), np.full((1, 2), 0.5), 4.0
    mu = S.sddmm(theta, phi, c, [0])
    vals = [S.sample_counts(theta, phi, mu, c, [0], m_t, r, 0, 0).theta_hat(0, 0)
            for r in range(2000)]
    assert abs(np.mean(vals) - 3.0) < 3.0 * math.sqrt(3.0 / m_t / len(vals))


def test_large_m_recovers_responsibilities():
    c = tiny(1, 1, [(0, 0, 1)])
    theta, phi = np.ones((1, 2)), np.array([[0.2], [0.8]])
    mu = S.sddmm(theta, phi, c, [0])
    sc = S.sample_counts(theta, phi, mu, c, [0], 1e4, 9, 0, 0)
    assert sc.theta_hat(0, 0) == pytest.approx(0.2, rel=0.02)
    assert sc.theta_hat(0, 1) == pytest.approx(0.8, rel=0.02)


def test_poisson_splitting():
    # test_sampler.cpp:262-282 (fewer runs)
    c = tiny(1, 1, [(0, 0, 2)])
    theta, phi, m_t = np.ones((1, 4)), np.full((4, 1), 0.25), 5.0
    mu = S.sddmm(theta, phi, c, [0])
    tot = np.array([S.sample_counts(theta, phi, mu, c, [0], m_t, r, 0, 0).theta_total()
                    for r in range(3000)], dtype=float)
    rate = m_t * 2.0
    assert abs(tot.mean() - rate) < 3.0 * math.sqrt(rate / len(tot))


def test_vanishing_mu_uniform_fallback():
    c = tiny(1, 1, [(0, 0, 4)])
    theta, phi = np.zeros((1, 2)), np.full((2, 1), 0.5)
    mu = S.sddmm(theta, phi, c, [0])
    assert mu[0] == 0.0
    sums = np.zeros(2)
    for r in range(1000):
        sc = S.sample_counts(theta, phi, mu, c, [0], 50.0, r, 0, 0)
        sums += [sc.theta_hat(0, 0), sc.theta_hat(0, 1)]
    assert np.all(np.abs(sums / 1000 - 2.0) < 3.0 * math.sqrt(2.0 / 50.0 / 1000) + 1e-9)


def test_nonfinite_rate_raises_numerical_error():
    c = tiny(1, 1, [(0, 0, 1)])
    theta = np.array([[np.inf, 1.0]])
    with pytest.raises(S.NumericalError):
        S.sample_counts(theta, np.full((2, 1), 0.5), [1.0], c, [0], 1.0, 1, 0, 0)


def test_sample_counts_config_errors():
    c = tiny(1, 1, [(0, 0, 1)])
    with pytest.raises(S.ConfigError):
        S.sample_counts(np.ones((1, 2)), np.full((2, 1), 0.5), [1.0], c, [0], 0.0, 1, 0, 0)
    with pytest.raises(S.ConfigError):
        S.sample_counts(np.ones((1, 2)), np.full((2, 1), 0.5), [1.0, 2.0], c, [0], 1.0, 1, 0, 0)


def test_update_model_known_answers():
    # test_sampler.cpp:319-380
    model = S.init_model(2, 3, 1, 0.1, 0.01)
    pc = np.zeros((3, 2), np.int64)
    pc[0, 0], pc[1, 0] = 2, 6
    S.update_model(model, S.SampledCounts(np.array([0], np.int32), 2, 3, 2.0,
                                          np.array([[3, 5]]), pc), 1.0)
    assert model.theta[0, 0] == pytest.approx(1.6, rel=1e-12)
    assert model.theta[0, 1] == pytest.approx(2.6, rel=1e-12)
    total = 4.0 + 3 * 0.01
    assert model.phi[0, 0] == pytest.approx(1.01 / total, rel=1e-12)
    assert model.phi[0, 2] == pytest.approx(0.01 / total, rel=1e-12)
    assert np.allclose(model.phi[1], 1.0 / 3, rtol=1e-12)
    m2 = S.init_model(1, 2, 1, 0.1, 0.01)
    m2.phi[0] = [0.6, 0.4]
    cnt = S.SampledCounts(np.array([0], np.int32), 1, 2, 1.0, np.array([[0]]),
                          np.array([[1000000000000], [4000000000000]]))
    S.update_model(m2, cnt, 0.5)
    assert m2.phi[0, 0] == pytest.approx(0.4, rel=1e-12)
    for bad in (0.0, 1.5):
        with pytest.raises(S.ConfigError):
            S.update_model(m2, cnt, bad)


def test_phi_rows_stochastic_after_training(port):
    g = port.make_corpus(30, 8, 3, 6.0, 77)
    model, _ = S.train(g, S.SamplerConfig(n_topics=3, m=7.5, t_max=25, batch_fraction=0.2,
                                          seed=5))
    assert np.all(model.phi >= 0)
    np.testing.assert_allclose(model.phi.sum(1), 1.0, atol=1e-6)


def test_zero_periods_returns_init(port):
    g = port.make_corpus(10, 6, 2, 5.0, 12)
    model, trace = S.train(g, S.SamplerConfig(n_topics=2, t_max=0))
    assert trace == []
    np.testing.assert_allclose(model.phi, 1.0 / 6, rtol=1e-12)


def test_training_deterministic(port):
    g = port.make_corpus(60, 20, 3, 10.0, 44)
    tr, te = port.split_holdout(g, 0.2, 9)
    cfg = S.SamplerConfig(n_topics=3, m=20.0, t_max=12, batch_fraction=0.25, seed=31)
    a, ta = S.train(tr, cfg, te, 4)
    b, tb = S.train(tr, cfg, te, 4)
    assert [r["ll"] for r in ta] == [r["ll"] for r in tb]
    np.testing.assert_array_equal(a.phi, b.phi)


def test_config_validation():
    g = tiny(2, 2, [(0, 0, 1), (1, 1, 1)])
    for kw in [dict(n_topics=0), dict(m=-1.0), dict(tau0=0.5), dict(gamma=0.3),
               dict(batch_fraction=0.0), dict(t_max=-1), dict(inner_sweeps=0),
               dict(inner_sweeps=256), dict(alpha=0.0), dict(init_noise=-1.0)]:
        with pytest.raises(S.ConfigError):
            S.train(g, S.SamplerConfig(**{"n_topics": 2, "t_max": 1, **kw}))


# ------------------------------------------------ reference eval tests

def test_fold_in_known_answers():
    assert S.fold_in_theta(np.full((1, 4), 0.25), [0, 2], [3, 1], 0.1)[0] == pytest.approx(1.0)
    th = S.fold_in_theta(np.array([[1.0, 0.0], [0.0, 1.0]]), [0], [5], 1e-9)
    assert th[0] == pytest.approx(1.0, rel=1e-6) and abs(th[1]) < 1e-6
    np.testing.assert_allclose(S.fold_in_theta(np.full((4, 3), 1 / 3), [], [], 0.1), 0.25)


def test_uniform_model_scores_minus_log_w(port):
    g = port.make_corpus(15, 8, 2, 12.0, 71)
    assert S.perword_loglik(np.full((1, 8), 0.125), g, 0.1, 3) == pytest.approx(-math.log(8.0),
                                                                                  rel=1e-12)


def test_eval_errors(port):
    g = port.make_corpus(5, 8, 2, 12.0, 71)
    with pytest.raises(S.ConfigError):
        S.perword_loglik(np.full((1, 9), 1 / 9), g, 0.1, 3)
    with pytest.raises(S.NumericalError):
        S.perword_loglik(np.zeros((1, 8)), g, 0.1, 3)


def test_deferred_overflow_path_bit_exact(port, monkeypatch):
    """A full deferred-draw list makes records draw inline: results unchanged."""
    g = port.make_corpus(60, 50, 4, 60.0, 9)
    rng = np.random.default_rng(3)
    K = 64
    theta = rng.gamma(0.3, 1.0, size=(g.n_docs, K)) + 1e-3
    phi = rng.gamma(0.2, 1.0, size=(K, g.n_words)) + 1e-9
    phi /= phi.sum(1, keepdims=True)
    batch = all_docs(g)
    mu = port.sddmm(theta, phi, g, batch)
    otc, opc = port.sample_counts(theta, phi, mu, g, batch, 400.0, 5, 2, 1)  # many PTRS draws
    for cap in ("0", "7"):
        monkeypatch.setenv("SAMELDA_DRAW_CAP", cap)
        sc = S.sample_counts(theta, phi, mu, g, batch, 400.0, 5, 2, 1)
        np.testing.assert_array_equal(sc.theta_counts, otc)
        np.testing.assert_array_equal(sc.phi_counts, opc)


def test_trainer_reports_device_error_asynchronously(port):
    """A period that hits a non-finite rate raises NumericalError by the next
    synchronising call (periods are asynchronous)."""
    g = port.make_corpus(20, 15, 3, 10.0, 4)
    tr = S.Trainer(g, S.SamplerConfig(n_topics=3, m=5.0, t_max=4, batch_fraction=1.0, seed=2))
    model = tr.model()
    model.phi[:] = np.nan
    tr.ctx.check(tr.ctx.lib.samelda_cu_model_upload(tr.ctx.h, S._ptr(np.ascontiguousarray(model.phi)), None))
    tr.period(np.arange(g.n_docs, dtype=np.int32), 0, 5.0, 1.0)
    with pytest.raises(S.NumericalError):
        tr.ctx.synchronize()
    tr.ctx.synchronize()  # reported once, then cleared


@pytest.mark.parametrize("m,schedule", [(100.0, "constant"), (400.0, "linear")])
def test_train_k256_production_kernel_bit_exact(port, m, schedule):
    """The bench's kernel instantiation (K=256: 8 topics per lane, full slice,
    fused mu) on the period path, with high m so the search loop, the
    deferred PTRS draws and the band all occur."""
    g = port.make_corpus(120, 400, 12, 150.0, 29)
    tr, te = port.split_holdout(g, 0.1, 2)
    cfg = dict(n_topics=256, m=m, schedule=schedule, t_max=4, batch_fraction=0.5, seed=6)
    model, trace = S.train(tr, S.SamplerConfig(**cfg), te, 2)
    ophi, otheta, otrace = port.train(tr, TrainConfig(**cfg), te, 2)
    np.testing.assert_array_equal(model.phi, ophi)
    np.testing.assert_array_equal(model.theta, otheta)
    np.testing.assert_allclose([r["ll"] for r in trace], [r["ll"] for r in otrace], rtol=1e-12)


def test_long_run_bit_exact_through_the_regime_change():
    """40 periods (10 passes) at K = 256, m = 100 on a 1,500-document corpus:
    the run crosses from the early regime (~1% of nonzeros defer, mostly
    inversion draws inside their band) to ~29% by period 39 (mostly PTRS
    draws, decided from the fast path's lambda_f by ptrs_banded) and must stay
    bit-identical to the compiled reference's train() the whole way (phi,
    theta, the ll trace every 10 periods)."""
    from oracle import Ref
    ref = Ref()
    g = ref.make_corpus(1500, 1000, 16, 120.0, 5)
    tr, te = ref.split_holdout(g, 0.1, 4)
    cfg = dict(n_topics=256, m=100.0, t_max=40, batch_fraction=0.25, seed=8)
    model, trace = S.train(tr, S.SamplerConfig(**cfg), te, 10)
    rphi, rtheta, rtrace = ref.train(tr, TrainConfig(**cfg), te, 10)
    np.testing.assert_array_equal(model.phi, rphi)
    np.testing.assert_array_equal(model.theta, rtheta)
    np.testing.assert_allclose([r["ll"] for r in trace], [r["ll"] for r in rtrace], rtol=1e-12)
    # the same 40 periods through a Trainer: the deferral rate at the start and the end
    t = S.Trainer(tr, S.SamplerConfig(**cfg))
    stream = S.MinibatchStream(tr.n_docs, 0.25, 8)
    rates = []
    for p in range(40):
        probe = p in (0, 39)
        if probe:
            t.profile(True)
        t.period(stream.next(), p, 100.0, S.rho_schedule(p, 1.0, 0.5))
        if probe:
            prof = t.profile_read()
            t.profile(False)
            rates.append(prof["deferred"] / prof["nnz"])
    assert rates[0] < 0.05 and rates[1] > 0.25, rates
    np.testing.assert_array_equal(t.model().phi, rphi)


def test_converged_regime_banded_ptrs_bit_exact(port):
    """The converged-model path: once most nonzeros carry deferred (PTRS)
    draws, they are decided from the fast path's f32 rate with error bands
    (ptrs_banded) and only the undecided ones form the exact f64 mu (DESIGN.md
    4, "Two regimes").  m = 3000 puts a PTRS draw on nearly every nonzero from
    the first period; phi, theta and the ll trace must still equal the
    reference's bit for bit."""
    g = port.make_corpus(120, 400, 12, 150.0, 41)
    tr, te = port.split_holdout(g, 0.1, 3)
    cfg = dict(n_topics=256, m=3000.0, t_max=8, batch_fraction=0.5, seed=12)
    # the regime is really the converged one: the deferral rate per sweep
    t = S.Trainer(tr, S.SamplerConfig(**cfg))
    stream = S.MinibatchStream(tr.n_docs, 0.5, 12)
    t.profile(True)
    t.period(stream.next(), 0, 3000.0, S.rho_schedule(0, 1.0, 0.5))
    prof = t.profile_read()
    t.profile(False)
    assert prof["deferred"] > 0.5 * prof["nnz"], prof
    model, trace = S.train(tr, S.SamplerConfig(**cfg), te, 2)
    ophi, otheta, otrace = port.train(tr, TrainConfig(**cfg), te, 2)
    np.testing.assert_array_equal(model.phi, ophi)
    np.testing.assert_array_equal(model.theta, otheta)
    np.testing.assert_allclose([r["ll"] for r in trace], [r["ll"] for r in otrace], rtol=1e-12)


@pytest.mark.parametrize("m,K", [(2e4, 64), (2e5, 16), (5e3, 300)])
def test_large_rate_ptrs_bit_exact(port, m, K):
    """Rates of 1e3 .. 1e6 (m up to 2e5, counts up to ~40): the banded PTRS
    decisions (whose bands grow with lambda) and their exact fallbacks,
    including topic slices (K = 300), against the reference's train()."""
    g = port.make_corpus(60, 150, 6, 60.0, 23)
    tr, te = port.split_holdout(g, 0.2, 5)
    cfg = dict(n_topics=K, m=m, t_max=4, batch_fraction=0.5, seed=19)
    model, trace = S.train(tr, S.SamplerConfig(**cfg), te, 2)
    ophi, otheta, otrace = port.train(tr, TrainConfig(**cfg), te, 2)
    np.testing.assert_array_equal(model.phi, ophi)
    np.testing.assert_array_equal(model.theta, otheta)
    np.testing.assert_allclose([r["ll"] for r in trace], [r["ll"] for r in otrace], rtol=1e-12)


@pytest.mark.parametrize("K", [300, 520])
def test_train_sliced_k_bit_exact(port, K):
    """K > 256 on the period path: topic slices with the k_mu_f32 pre-pass."""
    g = port.make_corpus(50, 80, 5, 40.0, 17)
    tr, te = port.split_holdout(g, 0.2, 4)
    cfg = dict(n_topics=K, m=30.0, t_max=3, batch_fraction=0.5, seed=8)
    model, trace = S.train(tr, S.SamplerConfig(**cfg), te, 3)
    ophi, otheta, otrace = port.train(tr, TrainConfig(**cfg), te, 3)
    np.testing.assert_array_equal(model.phi, ophi)
    np.testing.assert_array_equal(model.theta, otheta)
    np.testing.assert_allclose([r["ll"] for r in trace], [r["ll"] for r in otrace], rtol=1e-12)


# ------------------- statistical / invariance cases (test_sampler.cpp, test_eval.cpp)

def _greedy_matched_mean_tv(phi, phi_true):
    """tests/support/oracles.cpp greedy_matched_mean_tv: rows paired greedily by
    smallest total-variation distance, mean over the pairs."""
    tv = 0.5 * np.abs(phi[:, None, :] - phi_true[None, :, :]).sum(-1)
    used_a, used_b, total = set(), set(), []
    for flat in np.argsort(tv, axis=None):
        a, b = divmod(int(flat), tv.shape[1])
        if a in used_a or b in used_b:
            continue
        used_a.add(a)
        used_b.add(b)
        total.append(tv[a, b])
    return float(np.mean(total))


def test_learned_topics_approach_generating_ones(port):
    """test_sampler.cpp:439-454 (10 passes, K=5, m=100, bf=0.05)."""
    g = port.make_corpus(2000, 100, 5, 50.0, 817)
    model, _ = S.train(g, S.SamplerConfig(n_topics=5, m=100.0, batch_fraction=0.05, t_max=200,
                                          seed=4))
    assert _greedy_matched_mean_tv(model.phi, g.phi_true) < 0.15


def test_larger_replica_counts_shrink_estimator_variance():
    """test_sampler.cpp:456-479: spread of phi(0,0) over 100 seeds falls as
    m rises 1 -> 10 -> 100."""
    c = S.Corpus(np.array([0, 2]), np.array([0, 1], np.int32), np.array([2, 1], np.int32), 2)
    spread = []
    for m in (1.0, 10.0, 100.0):
        est = [S.train(c, S.SamplerConfig(n_topics=2, m=m, t_max=1, batch_fraction=1.0,
                                          inner_sweeps=1, seed=run))[0].phi[0, 0]
               for run in range(100)]
        spread.append(np.var(est))
    assert spread[0] > spread[1] > spread[2]


def test_fold_in_fixed_point(port):
    """test_eval.cpp:41-50: 60 and 200 sweeps agree to 1e-10."""
    g = port.make_corpus(1, 10, 3, 40.0, 61)
    w = g.word_ids[g.doc_offsets[0]:g.doc_offsets[1]]
    c = g.counts[g.doc_offsets[0]:g.doc_offsets[1]]
    a = S.fold_in_theta(g.phi_true, w, c, 0.1, 60)
    b = S.fold_in_theta(g.phi_true, w, c, 0.1, 200)
    assert np.abs(a - b).max() < 1e-10
    want = port.fold_in_theta(g.phi_true, w, c, 0.1, 60)
    np.testing.assert_allclose(a, want, rtol=1e-12, atol=0)
    ctx = S.Context(0)
    ctx.set_eval_exact(True)  # the reference's summation order: bit-identical
    np.testing.assert_array_equal(S.fold_in_theta(g.phi_true, w, c, 0.1, 60, ctx=ctx), want)


def test_scaling_counts_leaves_the_score_unchanged(port):
    """test_eval.cpp:67-94."""
    g = port.make_corpus(10, 12, 3, 9.0, 72)
    doubled = S.Corpus(g.doc_offsets, g.word_ids, g.counts * 2, g.n_words)
    uniform = np.full((3, 12), 1.0 / 12)
    assert S.perword_loglik(uniform, g, 0.1, 5) == S.perword_loglik(uniform, doubled, 0.1, 5)
    big = port.make_corpus(100, 20, 3, 80.0, 72)
    big2 = S.Corpus(big.doc_offsets, big.word_ids, big.counts * 2, big.n_words)
    base = S.perword_loglik(big.phi_true, big, 0.1, 5)
    scaled = S.perword_loglik(big.phi_true, big2, 0.1, 5)
    assert abs(base - scaled) < 0.05 and base <= 0.0 and scaled <= 0.0
    assert base == pytest.approx(port.perword_loglik(big.phi_true, big, 0.1, 5), rel=1e-12)


def test_generating_model_beats_uniform(port):
    """test_eval.cpp:96-105."""
    g = port.make_corpus(200, 40, 4, 30.0, 73)
    _, te = port.split_holdout(g, 0.25, 7)
    ll_true = S.perword_loglik(g.phi_true, te, 0.1, 11)
    ll_uniform = S.perword_loglik(np.full((4, 40), 0.025), te, 0.1, 11)
    assert ll_true > ll_uniform and ll_true <= 0.0
    assert ll_uniform == pytest.approx(-math.log(40.0), rel=1e-9)


def test_evaluation_is_pure_and_repeatable(port):
    """test_eval.cpp:107-114 (n_threads cannot change the result; phi untouched)."""
    g = port.make_corpus(25, 10, 2, 8.0, 74)
    before = g.phi_true.copy()
    a = S.perword_loglik(g.phi_true, g, 0.1, 9, 1)
    b = S.perword_loglik(g.phi_true, g, 0.1, 9, 3)
    assert a == b
    np.testing.assert_array_equal(g.phi_true, before)


def test_eval_long_documents_multi_chunk(port):
    """k_eval_cta walks cells in chunks of 256 threads: documents with several
    hundred distinct words, K=256, against the oracle (eval.cpp:75-159)."""
    g = port.make_corpus(24, 3000, 6, 900.0, 5)
    assert np.diff(g.doc_offsets).max() > 512  # three 256-cell chunks
    rng = np.random.default_rng(8)
    phi = rng.gamma(0.3, 1.0, size=(256, g.n_words)) + 1e-12
    phi /= phi.sum(1, keepdims=True)
    ll = S.perword_loglik(phi, g, 0.1, 13)
    assert ll == pytest.approx(port.perword_loglik(phi, g, 0.1, 13), rel=1e-12, abs=0)


def test_reported_eval_error_does_not_leak_into_training(port):
    """A NumericalError raised by perword_loglik is reported once: the next
    training run on the same context starts with a clean device flag."""
    g = port.make_corpus(20, 8, 2, 12.0, 71)
    ctx = S.Context(0)
    with pytest.raises(S.NumericalError):
        S.perword_loglik(np.zeros((2, 8)), g, 0.1, 3, ctx=ctx)
    model, _ = S.train(g, S.SamplerConfig(n_topics=2, m=5.0, t_max=2, batch_fraction=1.0, seed=1),
                       ctx=ctx)
    ophi, _, _ = port.train(g, TrainConfig(n_topics=2, m=5.0, t_max=2, batch_fraction=1.0, seed=1))
    np.testing.assert_array_equal(model.phi, ophi)


# ------------------------------------------------ rate extremes on the K=256 period kernel

@pytest.mark.parametrize("m", [1e-3, 0.37, 1e4])
def test_train_rate_extremes_bit_exact(port, m):
    """Tiny rates (every draw decided at z = 0 or deferred as tiny), and huge
    rates (almost every draw in PTRS territory: deferred exact path, z far
    beyond the fast path's 40), K = 256, against the oracle."""
    g = port.make_corpus(60, 300, 10, 120.0, 44)
    kw = dict(n_topics=256, m=m, t_max=2, batch_fraction=0.6, seed=9)
    model, _ = S.train(g, S.SamplerConfig(**kw))
    ophi, otheta, _ = port.train(g, TrainConfig(**kw))
    np.testing.assert_array_equal(model.phi, ophi)
    np.testing.assert_array_equal(model.theta, otheta)


def test_large_counts_and_long_documents_bit_exact(port):
    """Cells with counts in the hundreds (lambda = m c w >> 10) and documents
    spanning many 128-nonzero warp chunks (the per-lane packed theta counts
    are flushed per chunk), K = 256."""
    rng = np.random.default_rng(17)
    D, W = 6, 900
    offsets, words, counts = [0], [], []
    for d in range(D):
        n = int(rng.integers(300, 700))
        ws = np.sort(rng.choice(W, size=n, replace=False)).astype(np.int32)
        cs = rng.integers(1, 400, size=n).astype(np.int32)
        words.append(ws)
        counts.append(cs)
        offsets.append(offsets[-1] + n)
    g = S.Corpus(np.array(offsets), np.concatenate(words), np.concatenate(counts), W)
    kw = dict(n_topics=256, m=5.0, t_max=2, batch_fraction=1.0, seed=2)
    model, _ = S.train(g, S.SamplerConfig(**kw))
    ophi, otheta, _ = port.train(g, TrainConfig(**kw))
    np.testing.assert_array_equal(model.phi, ophi)
    np.testing.assert_array_equal(model.theta, otheta)


# ------------------------------------------------ BASELINE size (NYTimes shape)

@pytest.mark.skipif(not __import__("oracle").have_ref(), reason="oracle/_ref not built")
def test_nytimes_scale_sweep_matches_compiled_reference():
    """One full-size sampling sweep at BASELINE configs[1] shape (NYTimes-shaped
    corpus, a 13,500-document minibatch, K=256, m=100) on a model trained for
    a few periods on the device: theta and phi counts bit-exact against the
    compiled reference's sample_counts (oracle/_ref, all host threads), and
    the sweep's mass balance."""
    import bench
    from oracle import Ref
    train, _ = bench.single_gpu_corpus("nytimes")
    cfg = S.SamplerConfig(n_topics=256, m=100.0, batch_fraction=0.05, t_max=4, seed=1)
    tr = S.Trainer(train, cfg)
    stream = S.MinibatchStream(train.n_docs, 0.05, 1)
    for t in range(3):
        tr.period(stream.next(), t, 100.0, S.rho_schedule(t, 1.0, 0.5))
    model = tr.model()
    batch = stream.next()
    tb = np.ascontiguousarray(model.theta[batch])
    ctx = tr.ctx
    mu = S.sddmm(tb, model.phi, train, batch, ctx=ctx)
    sc = S.sample_counts(tb, model.phi, mu, train, batch, 100.0, 1, 3, 1, ctx=ctx)
    ref = Ref()
    otc, opc = ref.sample_counts(tb, model.phi, mu, train, batch, 100.0, 1, 3, 1,
                                 n_threads=os.cpu_count() or 1)
    np.testing.assert_array_equal(sc.theta_counts, otc)
    np.testing.assert_array_equal(sc.phi_counts, opc)
    assert sc.theta_counts.sum() == sc.phi_counts.sum()


def test_eval_documents_beyond_one_fold_window(port):
    """k_eval_stage compacts fold cells per window of 1024 (cell order kept,
    lists rebuilt every sweep, staged rows only for window 0): documents with
    2,000-4,000 distinct words, K=64, against the oracle."""
    rng = np.random.default_rng(23)
    W = 6000
    offsets, words, counts = [0], [], []
    for n in (4000, 120, 2500, 1030, 3100):
        ws = np.sort(rng.choice(W, size=n, replace=False)).astype(np.int32)
        cs = rng.integers(1, 4, size=n).astype(np.int32)
        words.append(ws)
        counts.append(cs)
        offsets.append(offsets[-1] + n)
    g = S.Corpus(np.array(offsets), np.concatenate(words), np.concatenate(counts), W)
    phi = rng.gamma(0.5, 1.0, size=(64, W)) + 1e-12
    phi /= phi.sum(1, keepdims=True)
    ll = S.perword_loglik(phi, g, 0.1, 19)
    assert ll == pytest.approx(port.perword_loglik(phi, g, 0.1, 19), rel=1e-12, abs=0)


@pytest.mark.skipif(not __import__("oracle").have_ref(), reason="oracle/_ref not built")
def test_model_bin_and_metrics_csv_match_reference_training(port, tmp_path):
    """End to end through the output formats: a device
    training run written with save_checkpoint / write_metrics_csv against the
    compiled reference's own train() + save_checkpoint / write_metrics_csv:
    model.bin byte-equal, metrics.csv equal except the wall-clock column."""
    from oracle import Ref
    ref = Ref()
    g = port.make_corpus(150, 90, 5, 40.0, 77)
    tr, te = port.split_holdout(g, 0.2, 3)
    kw = dict(n_topics=16, m=30.0, t_max=6, batch_fraction=0.25, seed=11)
    ctx = S.Context(0)
    ctx.set_eval_exact(True)  # ll in the reference's summation order: identical csv text
    model, trace = S.train(tr, S.SamplerConfig(**kw), te, 2, ctx=ctx)
    rphi, _, rtrace = ref.train(tr, TrainConfig(**kw), te, 2)
    _, fast = S.train(tr, S.SamplerConfig(**kw), te, 2)  # default eval: 1e-12
    np.testing.assert_allclose([r["ll"] for r in fast], [r["ll"] for r in rtrace], rtol=1e-12, atol=0)
    ours, theirs = str(tmp_path / "ours.bin"), str(tmp_path / "ref.bin")
    S.save_checkpoint(model, ours)
    ref.save_checkpoint(theirs, rphi, model.alpha, model.beta)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    oc, rc = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    S.write_metrics_csv(trace, oc)
    ref.write_metrics_csv(rc, rtrace)
    drop_wall = lambda path: [ln.split(",")[:4] + ln.split(",")[5:]
                              for ln in open(path).read().splitlines()]
    assert drop_wall(oc) == drop_wall(rc)


def test_exact_kernel_cross_check(port, monkeypatch):
    """SAMELDA_SAMPLER=x: the all-f64 exact kernel (k_sample) on the per-call
    path gives the same counts as the fast-exact path and the oracle, K=256
    with PTRS-heavy rates."""
    g = port.make_corpus(80, 300, 8, 150.0, 31)
    rng = np.random.default_rng(2)
    K = 256
    theta = rng.gamma(0.3, 1.0, size=(g.n_docs, K)) + 1e-3
    phi = rng.gamma(0.2, 1.0, size=(K, g.n_words)) + 1e-9
    phi /= phi.sum(1, keepdims=True)
    batch = rng.permutation(g.n_docs)[:60].astype(np.int32)
    tb = theta[batch]
    mu = port.sddmm(tb, phi, g, batch)
    fast = S.sample_counts(tb, phi, mu, g, batch, 300.0, 5, 2, 1)
    monkeypatch.setenv("SAMELDA_SAMPLER", "x")
    exact = S.sample_counts(tb, phi, mu, g, batch, 300.0, 5, 2, 1)
    otc, opc = port.sample_counts(tb, phi, mu, g, batch, 300.0, 5, 2, 1)
    for sc in (fast, exact):
        np.testing.assert_array_equal(sc.theta_counts, otc)
        np.testing.assert_array_equal(sc.phi_counts, opc)
