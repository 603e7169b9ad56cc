"""The C restatement (oracle/samelda_oracle.c) against the compiled reference's
golden fixtures (tests/golden/, made by make_golden.py from oracle/_ref) and
the SURVEY.md Appendix A known answers.  CPU only."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import TrainConfig

M0, M1 = 0xD2511F53, 0xCD9E8D57


def port_stream_words(port, seed, t, doc, word, tag, n):
    k0 = (seed & 0xFFFFFFFF) ^ ((tag * M0) & 0xFFFFFFFF)
    k1 = (seed >> 32) ^ ((tag * M1) & 0xFFFFFFFF)
    out = []
    for blk in range((n + 3) // 4):
        out.extend(port.philox_block([blk, word, doc, t], [k0, k1]).tolist())
    return np.array(out[:n], np.uint32)


def test_philox_known_answers(port):
    # seed 0 block 0 == ATen Philox4_32(0,0,0)
    assert [hex(x) for x in port.philox_block([0, 0, 0, 0], [0, 0])] == [
        "0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    w = port_stream_words(port, 0x0123456789ABCDEF, 7, 123456, 98765, 0, 4)
    assert [hex(x) for x in w] == ["0xe9cd43bb", "0xef191961", "0xa4ae72f3", "0x77ab4668"]
    assert port.make_tag(1, 1, 200) == 0x101000C8


def test_philox_stream_words_match_reference(port, golden):
    for key, words in zip(golden["philox_keys"], golden["philox_words"]):
        seed, t, doc, word, tag = (int(x) for x in key)
        np.testing.assert_array_equal(port_stream_words(port, seed, t, doc, word, tag, 16), words)


def test_poisson_table_appendix_a(port):
    table = {0.3: [0, 1, 1, 0], 4: [3, 7, 7, 4], 9.99: [8, 15, 14, 10], 10: [8, 16, 15, 10],
             57.5: [52, 72, 69, 58], 1234.5: [1211, 1302, 1288, 1236]}
    for lam, want in table.items():
        assert port.poisson_grid(lam, 1, 0, 5, 17, 0, 0, 4).tolist() == want


def test_poisson_grid_matches_reference(port, golden):
    for lam, draws, draws2 in zip(golden["poisson_lambdas"], golden["poisson_draws"],
                                  golden["poisson_draws_s2"]):
        np.testing.assert_array_equal(port.poisson_grid(float(lam), 1, 0, 5, 17, 0, 0, 256), draws)
        np.testing.assert_array_equal(
            port.poisson_grid(float(lam), 0xDEADBEEFCAFEF00D, 9, 77, 4242, 3, 1000, 256), draws2)


def test_make_corpus_matches_reference(port, golden, small):
    g = port.make_corpus(60, 40, 4, 25.0, 5)
    np.testing.assert_array_equal(g.doc_offsets, small.doc_offsets)
    np.testing.assert_array_equal(g.word_ids, small.word_ids)
    np.testing.assert_array_equal(g.counts, small.counts)
    np.testing.assert_array_equal(g.phi_true, golden["small_phi_true"])


def test_split_holdout_matches_reference(port, golden, small):
    tr, te = port.split_holdout(small, 0.2, 9)
    np.testing.assert_array_equal(tr.doc_offsets, golden["split_train_offsets"])
    np.testing.assert_array_equal(te.doc_offsets, golden["split_test_offsets"])
    np.testing.assert_array_equal(tr.word_ids, golden["split_train_words"])
    np.testing.assert_array_equal(te.word_ids, golden["split_test_words"])


def test_sddmm_sample_update_match_reference(port, golden, small):
    theta, phi, batch = golden["small_theta"], golden["small_phi"], golden["small_batch"]
    tb = theta[batch]
    mu = port.sddmm(tb, phi, small, batch)
    np.testing.assert_array_equal(mu, golden["small_mu"])
    for i, (m_t, seed, (t, sweep)) in enumerate(zip(golden["sample_m_t"], golden["sample_seed"],
                                                    golden["sample_t_sweep"])):
        tc, pc = port.sample_counts(tb, phi, mu, small, batch, m_t, int(seed), int(t), int(sweep))
        np.testing.assert_array_equal(tc, golden[f"small_tc{i}"])
        np.testing.assert_array_equal(pc, golden[f"small_pc{i}"])
        assert tc.sum() == pc.sum()  # mass balance, test_sampler.cpp:196-219
        th2, ph2 = port.update_model(theta, phi, batch, tc, pc, m_t, 0.37 + 0.2 * i, 0.1, 0.01)
        np.testing.assert_array_equal(th2, golden[f"small_upd_theta{i}"])
        np.testing.assert_array_equal(ph2, golden[f"small_upd_phi{i}"])
    big = tb * 50.0
    mu_big = port.sddmm(big, phi, small, batch)
    tc, pc = port.sample_counts(big, phi, mu_big, small, batch, 2000.0, 5, 1, 0)
    np.testing.assert_array_equal(tc, golden["small_big_tc"])
    np.testing.assert_array_equal(pc, golden["small_big_pc"])


def test_eval_matches_reference(port, golden, small):
    assert port.perword_loglik(small.phi_true, small, 0.1, 3) == golden["small_ll_true"][0]
    assert port.perword_loglik(golden["small_phi"], small, 0.1, 12345) == golden["small_ll_rand"][0]
    w0 = small.word_ids[small.doc_offsets[0]:small.doc_offsets[1]]
    c0 = small.counts[small.doc_offsets[0]:small.doc_offsets[1]]
    np.testing.assert_array_equal(port.fold_in_theta(small.phi_true, w0, c0, 0.1, 50),
                                  golden["small_fold_in"])
    np.testing.assert_array_equal(port.fold_in_theta(golden["small_phi"], w0, c0, 0.3, 5),
                                  golden["small_fold_in_5"])


def test_schedules_match_reference(port, golden):
    for s, t, tmax, v in golden["anneal_grid"]:
        assert port.anneal_m(int(s), int(t), int(tmax), 100.0) == v
    for t, tau, gm, v in golden["rho_grid"]:
        assert port.rho_schedule(int(t), tau, gm) == v


def _cfg_from(arr):
    n_topics, m, sched, t_max, bf, inner, seed, noise = arr
    return TrainConfig(n_topics=int(n_topics), m=float(m),
                       schedule=["constant", "linear", "log", "invlinear"][int(sched)],
                       t_max=int(t_max), batch_fraction=float(bf), inner_sweeps=int(inner),
                       seed=int(seed), init_noise=float(noise))


@pytest.mark.parametrize("name", ["train_a", "train_b", "train_c"])
def test_train_matches_reference(port, golden, small_split, name):
    tr, te = small_split
    phi, theta, trace = port.train(tr, _cfg_from(golden[f"{name}_cfg"]), te, 2)
    np.testing.assert_array_equal(phi, golden[f"{name}_phi"])
    np.testing.assert_array_equal(theta, golden[f"{name}_theta"])
    np.testing.assert_array_equal([r["ll"] for r in trace], golden[f"{name}_ll"])
    np.testing.assert_array_equal([r["samples_per_word"] for r in trace], golden[f"{name}_spw"])
    np.testing.assert_array_equal([r["passes"] for r in trace], golden[f"{name}_passes"])


def test_c1_corpus_matches_reference(port):
    rec = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c1_train.json")))
    c = rec["corpus"]
    g = port.make_corpus(c["n_docs"], c["n_words"], c["n_topics"], c["len_mean"], c["seed"])
    dig = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    assert dig(g.doc_offsets) == rec["corpus_digest"]["offsets"]
    assert dig(g.word_ids) == rec["corpus_digest"]["words"]
    assert dig(g.counts) == rec["corpus_digest"]["counts"]
    tr, _ = port.split_holdout(g, 0.1, 1)
    assert tr.nnz == rec["train_nnz"] and tr.n_tokens == rec["train_tokens"]


def test_expected_counts_formula(port):
    # test_sampler.cpp:221-260: E[theta_hat[d,k]] = sum_w c_dw lambda_dwk
    from oracle import CorpusArrays
    corpus = CorpusArrays(np.array([0, 3], np.int64), np.array([0, 1, 2], np.int32),
                          np.array([2, 1, 3], np.int32), 3)
    theta = np.array([[0.5, 1.5, 1.0]])
    phi = np.array([0.6, 0.3, 0.1, 0.2, 0.3, 0.5, 0.25, 0.5, 0.25]).reshape(3, 3)
    mu = port.sddmm(theta, phi, corpus, np.array([0], np.int32))
    tf, pf = port.expected_counts(theta, phi, mu, corpus, np.array([0], np.int32), 2.0)
    want = np.zeros(3)
    for i, (w, c) in enumerate(zip(corpus.word_ids, corpus.counts)):
        want += c * theta[0] * phi[:, w] / mu[i]
    np.testing.assert_allclose(tf[0] / 2.0, want, rtol=1e-14)
    np.testing.assert_allclose(pf.sum(), tf.sum(), rtol=1e-14)
