"""Held-out evaluation on the device (perword_loglik / fold_in_theta,
eval.cpp:19-159) against the oracle on seeded inputs.

The default kernel (k_eval_fold) sums in tree order with FMA, so its bar is
SURVEY 8(d)'s tolerance: ll within 1e-12 relative of the reference's.  The
exact mode (Context.set_eval_exact) keeps the reference's summation order and
is checked at 1e-14 (libdevice vs glibc log).  Shapes cover every k_eval_fold instantiation
(K <= 64 ... <= 1024, odd K, K past 1024 falling back to the exact kernels),
documents whose fold rows overflow the register- and shared-memory-resident
sets (rows re-read from L2), empty documents and documents of one cell."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import CorpusArrays

pytestmark = pytest.mark.gpu

S = None


@pytest.fixture(scope="module", autouse=True)
def _samelda(cuda_ctx):
    global S
    from paper_1409_5402_b200 import samelda
    S = samelda
    yield


def random_corpus(rng, n_docs, n_words, len_lo, len_hi, empty_every=0):
    offs = [0]
    words, counts = [], []
    for d in range(n_docs):
        n = 0 if empty_every and d % empty_every == 0 else int(rng.integers(len_lo, len_hi + 1))
        n = min(n, n_words)
        w = np.sort(rng.choice(n_words, size=n, replace=False)).astype(np.int32)
        c = (1 + rng.geometric(0.6, size=n) - 1).astype(np.int32)
        words.append(w)
        counts.append(c)
        offs.append(offs[-1] + n)
    return CorpusArrays(np.array(offs, np.int64), np.concatenate(words).astype(np.int32),
                        np.concatenate(counts).astype(np.int32), n_words)


def random_phi(rng, K, W, conc=0.1):
    phi = rng.gamma(conc, size=(K, W)) + 1e-9
    return phi / phi.sum(1, keepdims=True)


@pytest.mark.parametrize("K", [1, 3, 16, 64, 65, 100, 128, 200, 256, 300, 512, 777, 1024, 1100])
def test_perword_loglik_within_1e12(port, K):
    rng = np.random.default_rng(1000 + K)
    W = 3000
    g = random_corpus(rng, 60, W, 1, 400, empty_every=17)
    phi = random_phi(rng, K, W)
    want = port.perword_loglik(phi, g, 0.1, 11)
    ctx = S.Context(0)
    got = S.perword_loglik(phi, g, 0.1, 11, ctx=ctx)
    assert got == pytest.approx(want, rel=1e-12, abs=0)
    ctx.set_eval_exact(True)
    # reference order (libdevice log vs glibc log may differ in the last ulp)
    assert S.perword_loglik(phi, g, 0.1, 11, ctx=ctx) == pytest.approx(want, rel=1e-14, abs=0)


@pytest.mark.parametrize("K", [32, 256, 1024])
def test_long_documents_overflow_on_chip_rows(port, K):
    """Fold lists longer than the register + shared-memory rows (~100 at K=256,
    ~25 at K=1024): the remainder is re-read from L2 every sweep."""
    rng = np.random.default_rng(7 + K)
    W = 6000
    g = random_corpus(rng, 6, W, 1500, 3000)
    phi = random_phi(rng, K, W, conc=0.05)
    want = port.perword_loglik(phi, g, 0.05, 3)
    assert S.perword_loglik(phi, g, 0.05, 3) == pytest.approx(want, rel=1e-12, abs=0)


@pytest.mark.parametrize("K", [1, 7, 64, 256, 513, 1024])
def test_fold_in_theta_within_1e12(port, K):
    rng = np.random.default_rng(50 + K)
    W = 900
    phi = random_phi(rng, K, W)
    for n in (0, 1, 5, 180, 700):
        words = rng.choice(W, size=n, replace=False).astype(np.int32)
        counts = rng.integers(0, 4, size=n).astype(np.int32)  # zero counts included
        for sweeps in (1, 7, 50):
            want = port.fold_in_theta(phi, words, counts, 0.1, sweeps)
            got = S.fold_in_theta(phi, words, counts, 0.1, sweeps)
            np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-15)
            assert got.sum() == pytest.approx(1.0, abs=1e-12)


def test_fold_in_zero_mu_cells_are_skipped(port):
    """eval.cpp:42-44: a word no topic can emit (mu = 0) cannot inform theta."""
    phi = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5]])
    phi[:, 2] = 0.0
    phi /= phi.sum(1, keepdims=True)
    words = np.array([0, 2, 1], np.int32)
    counts = np.array([3, 5, 1], np.int32)
    want = port.fold_in_theta(phi, words, counts, 0.2, 50)
    np.testing.assert_allclose(S.fold_in_theta(phi, words, counts, 0.2, 50), want, rtol=1e-12)


def test_fast_and_exact_modes_agree_on_trained_model(port, small_split):
    """A device-trained model (sharp topics) through both eval modes."""
    tr, te = small_split
    cfg = S.SamplerConfig(n_topics=24, m=20.0, t_max=12, batch_fraction=0.5, seed=4)
    ctx = S.Context(0)
    model, _ = S.train(tr, cfg, None, 0, ctx=ctx)
    fast = S.perword_loglik(model.phi, te, 0.1, 9, ctx=ctx)
    ctx.set_eval_exact(True)
    exact = S.perword_loglik(model.phi, te, 0.1, 9, ctx=ctx)
    assert exact == pytest.approx(port.perword_loglik(model.phi, te, 0.1, 9), rel=1e-14, abs=0)
    assert fast == pytest.approx(exact, rel=1e-12, abs=0)
