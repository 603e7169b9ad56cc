"""Parity AT the timed configuration (BASELINE.json configs[1], what bench.py times):
the NYTimes-shaped corpus, K=256, full 13,500-document minibatches, through the
period path the bench runs -- Trainer.period, i.e. k_sample_v2 with the fused f32 mu
(MUSRC = 0) in both PHI instantiations, the deferred exact passes, and the full
M-step over all 102,660 x 256 cells -- against the compiled reference
(oracle/_ref: its own sddmm -> sample_counts x 2 -> update_model on the same
MinibatchStream batches, sampler.cpp:307-333, all host threads).  Three periods:
the constant schedule at m = 100, then the linear schedule's extremes (config [2],
m_t = 2 m t / (T + 1) with m = 50, T = 99: m_t = 1 at t = 1 and 99 at t = 99).
phi and the batch's theta rows must be bit-identical after every period.  Also one
held-out evaluation at this shape against the reference's perword_loglik (1e-12)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import have_ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_ref(), reason="oracle/_ref (compiled reference) not built")]

ALPHA, BETA, SEED = 0.1, 0.01, 1


@pytest.fixture(scope="module")
def setup():
    import bench
    from oracle import Ref
    from paper_1409_5402_b200 import samelda as S
    train, heldout = bench.single_gpu_corpus("nytimes")
    cfg = S.SamplerConfig(n_topics=256, m=100.0, batch_fraction=0.05, t_max=100, seed=SEED)
    tr = S.Trainer(train, cfg)
    return S, Ref(), train, heldout, tr


def test_periods_bit_exact_at_the_timed_config(setup):
    S, ref, train, _, tr = setup
    nt = os.cpu_count() or 1
    m0 = tr.model()
    phi, theta = m0.phi.copy(), m0.theta.copy()
    stream = S.MinibatchStream(train.n_docs, 0.05, SEED)
    schedule = [(0, 100.0),
                (1, S.anneal_m("linear", 1, 99, 50.0)),
                (2, S.anneal_m("linear", 99, 99, 50.0))]
    assert schedule[1][1] == 1.0 and schedule[2][1] == 99.0
    for t, m_t in schedule:
        batch = stream.next()
        assert len(batch) == 13500
        rho = S.rho_schedule(t, 1.0, 0.5)
        tr.period(batch, t, m_t, rho)
        # the reference period (sampler.cpp:313-332) on the same batch
        tb = np.ascontiguousarray(theta[batch])
        for sweep in range(2):
            mu = ref.sddmm(tb, phi, train, batch, nt)
            tc, pc = ref.sample_counts(tb, phi, mu, train, batch, m_t, SEED, t, sweep, nt)
            if sweep == 0:
                tb = tc / m_t + ALPHA
        # the device's mass balance of the final sweep equals the reference's counts
        dt, dp = tr.count_totals()
        assert dt == int(tc.sum()) and dp == int(pc.sum()) and dt == dp
        theta, phi = ref.update_model(theta, phi, batch, tc, pc, m_t, rho, ALPHA, BETA)
        dev = tr.model()
        np.testing.assert_array_equal(dev.phi, phi, err_msg=f"phi after period {t} (m_t={m_t})")
        np.testing.assert_array_equal(dev.theta[batch], theta[batch],
                                      err_msg=f"theta rows after period {t}")


def test_heldout_eval_at_the_timed_config(setup):
    """perword_loglik (eval.cpp:75-159) on 4,000 held-out NYTimes-shape documents with the
    trained model, through the resident path (Trainer.evaluate) and the per-call path."""
    S, ref, _, heldout, tr = setup
    from paper_1409_5402_b200 import synth
    sub = synth.subset(heldout, np.arange(4000))
    phi = tr.model(with_theta=False).phi
    want = ref.perword_loglik(phi, sub, ALPHA, SEED, n_threads=os.cpu_count() or 1)
    tr.set_heldout(sub, seed=SEED)
    assert tr.evaluate() == pytest.approx(want, rel=1e-12, abs=0)
    assert S.perword_loglik(phi, sub, ALPHA, SEED, ctx=tr.ctx) == pytest.approx(want, rel=1e-12, abs=0)


def test_converged_period_bit_exact_at_the_timed_config():
    """The converged-model regime at the timed shape: after 80 untimed periods
    nearly every nonzero carries a deferred PTRS draw, decided from the fast
    path's lambda_f with error bands (ptrs_banded, "Two
    regimes"); one more period must equal the compiled reference's period on
    the downloaded model bit for bit."""
    import bench
    from oracle import Ref
    from paper_1409_5402_b200 import samelda as S
    ref = Ref()
    train, _ = bench.single_gpu_corpus("nytimes")
    cfg = S.SamplerConfig(n_topics=256, m=100.0, batch_fraction=0.05, t_max=100, seed=SEED)
    tr = S.Trainer(train, cfg)
    stream = S.MinibatchStream(train.n_docs, 0.05, SEED)
    for t in range(80):
        tr.period(stream.next(), t, 100.0, S.rho_schedule(t, 1.0, 0.5))
    m0 = tr.model()
    phi, theta = m0.phi.copy(), m0.theta.copy()
    t, m_t = 80, 100.0
    batch = stream.next()
    rho = S.rho_schedule(t, 1.0, 0.5)
    tr.profile(True)
    tr.period(batch, t, m_t, rho)
    prof = tr.profile_read()
    tr.profile(False)
    assert prof["deferred"] > 0.9 * prof["nnz"], prof  # the converged regime
    nt = os.cpu_count() or 1
    tb = np.ascontiguousarray(theta[batch])
    for sweep in range(2):
        mu = ref.sddmm(tb, phi, train, batch, nt)
        tc, pc = ref.sample_counts(tb, phi, mu, train, batch, m_t, SEED, t, sweep, nt)
        if sweep == 0:
            tb = tc / m_t + ALPHA
    theta, phi = ref.update_model(theta, phi, batch, tc, pc, m_t, rho, ALPHA, BETA)
    dev = tr.model()
    np.testing.assert_array_equal(dev.phi, phi)
    np.testing.assert_array_equal(dev.theta[batch], theta[batch])
