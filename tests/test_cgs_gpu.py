"""The collapsed Gibbs sampler baseline on the device (kernels_cgs.cu; SURVEY.md 8(f)
row 4) against the compiled reference (oracle/_ref: cgs.cpp's own cgs_init / cgs_sweep /
cgs_train): the chain is the reference's, draw for draw -- every token assignment z and
every count (doc-topic, word-topic, topic totals) after init and after N sweeps is
bit-identical; cgs_train's model (phi, theta) bit-identical and its held-out trace equal
to 1e-12 (the evaluation's reduction order); the reference's argument errors."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import have_ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not have_ref(), reason="oracle/_ref (compiled reference) not built")]


@pytest.fixture(scope="module")
def ref():
    from oracle import Ref
    return Ref()


@pytest.fixture(scope="module")
def S():
    from paper_1409_5402_b200 import samelda
    return samelda


CASES = [  # (docs, words, generating topics, mean length, corpus seed, K, alpha, beta, seed)
    (40, 30, 3, 20.0, 1, 1, 0.1, 0.01, 3),
    (60, 80, 4, 30.0, 2, 4, 0.1, 0.01, 11),
    (120, 200, 6, 50.0, 3, 33, 0.5, 0.05, 7),
    (50, 120, 5, 40.0, 4, 300, 0.1, 0.01, 5),
]


@pytest.mark.parametrize("case", CASES, ids=[f"K{c[5]}" for c in CASES])
@pytest.mark.parametrize("n_sweeps", [0, 1, 7])
def test_chain_bit_identical(S, ref, port, case, n_sweeps):
    D, W, KG, L, cs, K, alpha, beta, seed = case
    g = port.make_corpus(D, W, KG, L, cs)
    want = ref.cgs_run(g, K, alpha, beta, seed, n_sweeps)
    cgs = S.Cgs(g, K, alpha, beta, seed)
    for s in range(1, n_sweeps + 1):
        cgs.sweep(seed, s)
    got = cgs.state()
    for name, a, b in zip(("z", "doc_topic", "word_topic", "topic_total"), got, want):
        np.testing.assert_array_equal(a, b, err_msg=name)
    # mass balance (cgs.hpp:12-15)
    assert got[1].sum() == got[2].sum() == got[3].sum() == len(got[0])


@pytest.mark.parametrize("K,n_sweeps,eval_every", [(3, 12, 4), (20, 9, 3), (2, 0, 1)])
def test_cgs_train_matches_reference(S, ref, port, K, n_sweeps, eval_every):
    g = port.make_corpus(150, 100, 4, 40.0, 9)
    tr, te = port.split_holdout(g, 0.2, 5)
    model, trace = S.cgs_train(tr, K, 0.1, 0.01, n_sweeps, 17, eval_every, te)
    phi, theta, rtrace = ref.cgs_train(tr, K, 0.1, 0.01, n_sweeps, 17, eval_every, te)
    np.testing.assert_array_equal(model.phi, phi)
    np.testing.assert_array_equal(model.theta, theta)
    assert [r["t"] for r in trace] == [r["t"] for r in rtrace]
    assert [r["samples_per_word"] for r in trace] == [r["samples_per_word"] for r in rtrace]
    assert np.allclose([r["ll"] for r in trace], [r["ll"] for r in rtrace], rtol=1e-12, atol=0)


def test_cgs_argument_errors(S, port):
    g = port.make_corpus(10, 20, 2, 10.0, 1)
    for K, a, b in ((0, 0.1, 0.01), (2, -0.1, 0.01), (2, 0.1, 0.0)):
        with pytest.raises(S.ConfigError):
            S.Cgs(g, K, a, b, 1)
    with pytest.raises(S.ConfigError):
        S.cgs_train(g, 2, 0.1, 0.01, -1, 1)
