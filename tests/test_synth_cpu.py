"""Synthetic corpora (include/samelda_synth.h, host C++): the reference's own
generator restated for BASELINE.json configs[0] and split_holdout, checked
against the oracle port (pinned to the compiled reference in test_oracle.py)
and against the corpus totals SURVEY.md 8(d) measured with the reference;
the NYTimes-shape generator's shard property (strong-scaling shards)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import CorpusArrays
from paper_1409_5402_b200 import synth


def _arrays(c):
    return CorpusArrays(c.doc_offsets, c.word_ids, c.counts, c.n_words)


@pytest.mark.parametrize("n_docs,n_words,K,L,seed", [(300, 500, 8, 40.0, 3), (2000, 5000, 32, 100.0, 1),
                                                     (50, 97, 3, 5.0, 11)])
def test_make_corpus_ref_matches_oracle(port, n_docs, n_words, K, L, seed):
    c = synth.make_corpus_ref(n_docs, n_words, K, L, seed, n_threads=3)
    g = port.make_corpus(n_docs, n_words, K, L, seed)
    np.testing.assert_array_equal(c.doc_offsets, g.doc_offsets)
    np.testing.assert_array_equal(c.word_ids, g.word_ids)
    np.testing.assert_array_equal(c.counts, g.counts)


def test_c1_corpus_and_split_totals():
    """make_corpus(10000, 5000, 32, 100, 1) -> nnz 971,596, tokens 1,000,696;
    split_holdout(0.1, seed 1) train nnz 874,617, tokens 900,840 [measured with the reference]."""
    c = synth.make_corpus_ref(10000, 5000, 32, 100.0, 1)
    assert (c.nnz, c.n_tokens) == (971_596, 1_000_696)
    tr, te = synth.split_holdout(c, 0.1, 1)
    assert (tr.nnz, tr.n_tokens) == (874_617, 900_840)
    assert tr.n_docs + te.n_docs == 10000 and te.n_docs == 1000


@pytest.mark.parametrize("frac,seed", [(0.1, 1), (0.2, 9), (0.5, 4)])
def test_split_holdout_matches_oracle(port, frac, seed):
    c = synth.make_corpus_ref(400, 300, 4, 20.0, 5)
    tr, te = synth.split_holdout(c, frac, seed)
    otr, ote = port.split_holdout(_arrays(c), frac, seed)
    for a, b in ((tr, otr), (te, ote)):
        np.testing.assert_array_equal(a.doc_offsets, b.doc_offsets)
        np.testing.assert_array_equal(a.word_ids, b.word_ids)
        np.testing.assert_array_equal(a.counts, b.counts)


def test_generator_shards_are_slices_of_the_whole():
    """A strong-scaling rank generates only its documents: shard [lo, hi) equals rows
    lo..hi-1 of the whole corpus (one stream per global document)."""
    kw = dict(synth.PRESETS["nytimes"])
    kw["n_docs"] = 2000
    whole = synth.generate(seed=1, n_threads=4, **kw)
    kw["n_docs"] = 700
    part = synth.generate(seed=1, n_threads=2, first_doc=600, **kw)
    ref = synth.subset(whole, np.arange(600, 1300))
    np.testing.assert_array_equal(part.doc_offsets, ref.doc_offsets)
    np.testing.assert_array_equal(part.word_ids, ref.word_ids)
    np.testing.assert_array_equal(part.counts, ref.counts)
