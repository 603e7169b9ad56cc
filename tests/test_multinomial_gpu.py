"""Multinomial mode (SAMELDA_CU_MODE_MULTINOMIAL): north_star item 3's
multinomial(c m) replicas -- per batch nonzero, n = floor(c m_t) (+1 with
the fractional part's probability) categorical trials over the K topics with
probabilities theta phi / mu (sampler.cpp:150-185's responsibilities).  The
reference has no such mode, so parity is statistical against the oracle's
expected counts (the same mean as the Poisson replicas) plus the properties
the law fixes exactly:

  * sum_k z_k = n per nonzero: total counts = m_t x batch tokens exactly for
    integer m_t, and between the floor and ceiling sums otherwise;
  * the averaged counts match the expected counts with multinomial dispersion
    (var = n r (1 - r) <= the Poisson variance);
  * a full train() lands on the parity mode's held-out log-likelihood.
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_1409_5402_b200 import samelda
    return samelda


def _counts(S, port, g, K, m_t, seed, t, rng_seed=0):
    rng = np.random.default_rng(rng_seed)
    theta = rng.gamma(0.5, 1.0, size=(g.n_docs, K)) + 1e-4
    phi = rng.gamma(0.3, 1.0, size=(K, g.n_words)) + 1e-9
    phi /= phi.sum(1, keepdims=True)
    batch = np.arange(g.n_docs, dtype=np.int32)
    tb = theta[batch]
    mu = port.sddmm(tb, phi, g, batch)
    sc = S.sample_counts(tb, phi, mu, g, batch, m_t, seed, t, 0, mode=S.MODE_MULTINOMIAL)
    return sc, tb, phi, mu, batch


@pytest.mark.parametrize("K", [1, 7, 32, 64, 256, 300, 1000])
def test_trial_count_is_exact(S, port, K):
    g = port.make_corpus(40, 150, 4, 30.0, 5)
    tokens = int(g.counts.sum())
    sc, *_ = _counts(S, port, g, K, 7.0, 3, 1)
    assert sc.theta_total() == sc.phi_total() == 7 * tokens
    # fractional m_t: each nonzero draws floor(c m) or floor(c m) + 1 trials
    sc2, *_ = _counts(S, port, g, K, 2.37, 3, 1)
    cm = g.counts.astype(np.float64) * 2.37
    assert np.floor(cm).sum() <= sc2.phi_total() <= np.ceil(cm).sum()
    assert sc2.theta_total() == sc2.phi_total()
    assert abs(sc2.phi_total() - cm.sum()) < 6 * np.sqrt(len(cm) * 0.25) + 1


@pytest.mark.parametrize("K,m_t", [(64, 5.0), (256, 40.0), (300, 3.0)])
def test_mean_matches_expected_counts(S, port, K, m_t):
    """Mean over T seeds of the phi counts vs the oracle's expected counts
    (sampler.cpp:150-185 with z := E z): the dispersion sum((mean - e)^2 /
    (e / T)) / cells is <= ~1 (multinomial variance n r (1 - r) <= n r)."""
    g = port.make_corpus(50, 100, 5, 30.0, 17)
    T = 48
    acc = None
    for s in range(T):
        sc, tb, phi, mu, batch = _counts(S, port, g, K, m_t, 100 + s, 2)
        acc = sc.phi_counts.astype(np.float64) if acc is None else acc + sc.phi_counts
    _, pf = port.expected_counts(tb, phi, mu, g, batch, m_t)
    mean = acc / T
    pf_wk = pf.reshape(mean.shape)
    live = pf_wk > 1e-3
    disp = float(np.sum((mean[live] - pf_wk[live]) ** 2 / (pf_wk[live] / T)) / live.sum())
    assert disp < 1.0 + 6 * np.sqrt(2.0 / live.sum()) + 0.02, disp
    assert disp > 0.3, disp  # not degenerate
    assert np.all(acc[pf_wk == 0.0] == 0.0)


def test_deterministic_and_keyed(S, port):
    g = port.make_corpus(30, 80, 3, 25.0, 9)
    a, *_ = _counts(S, port, g, 128, 10.0, 5, 2)
    b, *_ = _counts(S, port, g, 128, 10.0, 5, 2)
    c, *_ = _counts(S, port, g, 128, 10.0, 5, 3)
    np.testing.assert_array_equal(a.phi_counts, b.phi_counts)
    np.testing.assert_array_equal(a.theta_counts, b.theta_counts)
    assert not np.array_equal(a.phi_counts, c.phi_counts)


def test_vanishing_mu_draws_uniformly(S, port):
    """A row without mass falls back to weight 1 / K (sampler.cpp:160-166)."""
    from oracle import CorpusArrays
    g = CorpusArrays(np.array([0, 1], np.int64), np.array([0], np.int32), np.array([1], np.int32), 2)
    K = 4
    theta = np.zeros((1, K))
    phi = np.full((K, 2), 0.5)
    tot = np.zeros(K)
    for s in range(200):
        sc = S.sample_counts(theta, phi, [0.0], g, [0], 50.0, s, 0, 0, mode=S.MODE_MULTINOMIAL)
        tot += sc.theta_counts.reshape(1, K)[0]
        assert sc.theta_total() == 50
    assert np.all(np.abs(tot / tot.sum() - 0.25) < 0.02), tot


def test_train_ll_matches_parity_mode(S, port):
    """The multinomial mode's held-out ll trajectory lies within max(0.01
    nats/token, 3 sigma of the parity mode's seed spread) of the parity mean."""
    g = port.make_corpus(400, 500, 8, 80.0, 31)
    tr, te = port.split_holdout(g, 0.1, 7)
    kw = dict(n_topics=64, m=100.0, t_max=120, batch_fraction=0.25)

    def trajectory(mode, seed):
        _, trace = S.train(tr, S.SamplerConfig(mode=mode, seed=seed, **kw), te, 30)
        return np.array([r["ll"] for r in trace])

    par = np.array([trajectory(S.MODE_PARITY, s) for s in range(9, 17)])
    multi = np.array([trajectory(S.MODE_MULTINOMIAL, s) for s in range(9, 13)])
    assert np.all(np.isfinite(multi))
    tol = np.maximum(0.01, 3 * par.std(0, ddof=1))
    assert np.all(np.abs(multi - par.mean(0)) <= tol), (par.mean(0), tol, multi)


def test_too_many_topics_rejected(S, port):
    g = port.make_corpus(10, 20, 2, 10.0, 1)
    with pytest.raises(S.ConfigError):
        S.Trainer(g, S.SamplerConfig(n_topics=1025, mode=S.MODE_MULTINOMIAL))
