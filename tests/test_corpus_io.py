"""Data formats either side of the hot path:
the parallel UCI docword loader, save_uci_bow, the binary CSR cache,
checkpoints and metrics CSVs -- each checked against the compiled reference
(oracle/_ref, test infrastructure) on the reference's own test cases
(test_corpus.cpp:48-122, test_model.cpp, test_eval.cpp) and on randomised
files.  Host code only: no GPU needed."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import OracleError, have_ref
from paper_1409_5402_b200 import samelda as S

pytestmark = pytest.mark.skipif(not have_ref(), reason="oracle/_ref (compiled reference) not built")


@pytest.fixture(scope="module")
def ref():
    from oracle import Ref
    return Ref()


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return str(p)


def same_as_reference(ref, docword, vocab, n_threads=0):
    c = S.load_uci_bow(docword, vocab, n_threads)
    off, wid, cnt, W, tok, voc = ref.load_uci_bow(docword, vocab)
    np.testing.assert_array_equal(c.doc_offsets, off)
    np.testing.assert_array_equal(c.word_ids, wid)
    np.testing.assert_array_equal(c.counts, cnt)
    assert c.n_words == W and c.n_tokens == tok and c.vocab == voc
    return c


def same_error(ref, docword, vocab):
    with pytest.raises(S.IoError) as ours:
        S.load_uci_bow(docword, vocab)
    with pytest.raises(OracleError) as theirs:
        ref.load_uci_bow(docword, vocab)
    assert theirs.value.code == 2  # IoError
    assert str(ours.value) == theirs.value.msg


# ------------------------------------------- reference cases (test_corpus.cpp)

def test_loads_the_documented_toy_file(ref, tmp_path):
    c = same_as_reference(ref, write(tmp_path, "docword.txt", "2\n3\n3\n1 1 2\n1 3 1\n2 2 4\n"),
                          write(tmp_path, "vocab.txt", "a\nb\nc\n"))
    assert c.n_docs == 2 and c.n_words == 3 and c.nnz == 3 and c.n_tokens == 7
    assert list(c.word_ids[:2]) == [0, 2] and c.counts[2] == 4
    assert c.vocab == ["a", "b", "c"]


def test_rejects_triplet_count_disagreeing_with_header(ref, tmp_path):
    v = write(tmp_path, "vocab.txt", "a\nb\nc\n")
    same_error(ref, write(tmp_path, "short.txt", "2\n3\n3\n1 1 2\n1 3 1\n"), v)
    same_error(ref, write(tmp_path, "long.txt", "2\n3\n2\n1 1 2\n1 3 1\n2 2 4\n"), v)


def test_merges_duplicates_by_summing(ref, tmp_path):
    c = same_as_reference(ref, write(tmp_path, "d.txt", "1\n2\n2\n1 1 1\n1 1 2\n"),
                          write(tmp_path, "v.txt", "a\nb\n"))
    assert c.nnz == 1 and c.counts[0] == 3 and c.n_tokens == 3


@pytest.mark.parametrize("text", ["2\n3\n", "nope\n3\n1\n1 1 1\n", "2\n3\n1\n3 1 1\n",
                                  "2\n3\n1\n1 4 1\n", "2\n3\n1\n1 1 0\n", "2\n3\n1\n1 1 -2\n",
                                  "0\n3\n1\n1 1 1\n", "2\n3\n-1\n", "2\n3\n2\n1 1 1\n1 2\n",
                                  "2\n3\n1\n1 1 1 junk\n", "2\n3\n2\n1 1 1\n2 x 1\n",
                                  "2\n3\n1\n1 1 99999999999999999999\n", "2\n3\n0\n"])
def test_malformed_files_fail_like_the_reference(ref, tmp_path, text):
    v = write(tmp_path, "vocab.txt", "a\nb\nc\n")
    d = write(tmp_path, "d.txt", text)
    try:
        ref.load_uci_bow(d, v)
    except OracleError:
        same_error(ref, d, v)
    else:
        same_as_reference(ref, d, v)


def test_vocab_length_mismatch(ref, tmp_path):
    d = write(tmp_path, "ok.txt", "1\n3\n1\n1 1 1\n")
    for vt in ["a\nb\n", "a\nb\nc\n\n", "a\nb\nc\nd"]:
        same_error(ref, d, write(tmp_path, "v2.txt", vt))
    c = same_as_reference(ref, d, write(tmp_path, "v3.txt", "a\r\nb\r\nc"))  # CRLF, no final \n
    assert c.vocab == ["a", "b", "c"]


def test_missing_files(ref, tmp_path):
    v = write(tmp_path, "vocab.txt", "a\n")
    same_error(ref, str(tmp_path / "absent.txt"), v)
    same_error(ref, write(tmp_path, "d.txt", "1\n1\n1\n1 1 1\n"), str(tmp_path / "absent_v.txt"))


def test_drops_documents_that_end_up_empty(ref, tmp_path):
    c = same_as_reference(ref, write(tmp_path, "d.txt", "3\n2\n2\n1 1 1\n3 2 5\n"),
                          write(tmp_path, "v.txt", "a\nb\n"))
    assert c.n_docs == 2 and c.n_tokens == 6


def random_docword(rng, D, W, nnz, dup=0.1, ws=False):
    docs = rng.integers(1, D + 1, nnz)
    words = rng.integers(1, W + 1, nnz)
    if dup:  # repeat some (doc, word) pairs
        k = int(dup * nnz)
        idx = rng.integers(0, nnz, k)
        docs[rng.integers(0, nnz, k)] = docs[idx]
    cnts = rng.integers(1, 50, nnz)
    seps = [" ", "\t", "  "] if ws else [" "]
    lines = [f"{d}{seps[i % len(seps)]}{w} {c}" for i, (d, w, c) in enumerate(zip(docs, words, cnts))]
    eol = "\r\n" if ws else "\n"
    return f"{D}\n{W}\n{nnz}\n" + eol.join(lines) + eol


@pytest.mark.parametrize("seed,ws", [(0, False), (1, True), (2, False)])
def test_random_files_match_the_reference(ref, tmp_path, seed, ws):
    rng = np.random.default_rng(seed)
    D, W, nnz = 400, 300, 20000
    d = write(tmp_path, "d.txt", random_docword(rng, D, W, nnz, ws=ws))
    v = write(tmp_path, "v.txt", "".join(f"w{i}\n" for i in range(W)))
    for threads in (1, 3, 0):
        same_as_reference(ref, d, v, threads)


def test_save_load_round_trip_and_bytes(ref, tmp_path, port):
    g = port.make_corpus(30, 12, 3, 9.0, 99)
    c = S.Corpus(g.doc_offsets, g.word_ids, g.counts, g.n_words, [f"t{i}" for i in range(12)])
    ours = (str(tmp_path / "o_doc.txt"), str(tmp_path / "o_voc.txt"))
    theirs = (str(tmp_path / "r_doc.txt"), str(tmp_path / "r_voc.txt"))
    S.save_uci_bow(c, *ours)
    ref.save_uci_bow(c, c.vocab, *theirs)
    for a, b in zip(ours, theirs):
        assert open(a, "rb").read() == open(b, "rb").read()
    back = same_as_reference(ref, *ours)
    np.testing.assert_array_equal(back.doc_offsets, c.doc_offsets)
    np.testing.assert_array_equal(back.word_ids, c.word_ids)
    np.testing.assert_array_equal(back.counts, c.counts)


def test_corpus_cache_round_trip(ref, tmp_path):
    rng = np.random.default_rng(7)
    d = write(tmp_path, "d.txt", random_docword(rng, 200, 90, 5000))
    v = write(tmp_path, "v.txt", "".join(f"w{i}\n" for i in range(90)))
    c = S.load_uci_bow(d, v)
    path = str(tmp_path / "c.csr")
    S.save_corpus_cache(c, path)
    back = S.load_corpus_cache(path)
    for f in ("doc_offsets", "word_ids", "counts"):
        np.testing.assert_array_equal(getattr(back, f), getattr(c, f))
    assert back.n_words == c.n_words and back.vocab == c.vocab
    # corruption is an IoError, never a silently different corpus
    raw = bytearray(open(path, "rb").read())
    raw[-len(c.vocab[-1]) - 30] ^= 0xFF
    open(path, "wb").write(bytes(raw))
    with pytest.raises(S.IoError):
        S.load_corpus_cache(path)
    open(path, "wb").write(bytes(raw[:100]))
    with pytest.raises(S.IoError):
        S.load_corpus_cache(path)


# ----------------------------------------------- checkpoint (model.cpp:54-111)

def test_checkpoint_bytes_and_round_trip(ref, tmp_path):
    rng = np.random.default_rng(3)
    phi = rng.random((7, 33))
    m = S.Model(7, 33, 0.1, 0.01, phi, None)
    a, b = str(tmp_path / "ours.bin"), str(tmp_path / "ref.bin")
    S.save_checkpoint(m, a)
    ref.save_checkpoint(b, phi, 0.1, 0.01)
    assert open(a, "rb").read() == open(b, "rb").read()
    back = S.load_checkpoint(b)
    np.testing.assert_array_equal(back.phi, phi)
    assert (back.alpha, back.beta, back.n_topics, back.n_words) == (0.1, 0.01, 7, 33)


@pytest.mark.parametrize("mutate", ["magic", "version", "truncate", "trailing", "k0"])
def test_checkpoint_errors_match_reference(ref, tmp_path, mutate):
    phi = np.ones((2, 3)) / 3
    path = str(tmp_path / "m.bin")
    ref.save_checkpoint(path, phi, 0.5, 0.25)
    raw = bytearray(open(path, "rb").read())
    if mutate == "magic":
        raw[0] = ord("X")
    elif mutate == "version":
        raw[8] = 2
    elif mutate == "truncate":
        raw = raw[:-5]
    elif mutate == "trailing":
        raw += b"\0"
    else:
        raw[12:20] = (0).to_bytes(8, "little")
    open(path, "wb").write(bytes(raw))
    with pytest.raises(S.IoError) as ours:
        S.load_checkpoint(path)
    with pytest.raises(OracleError) as theirs:
        ref.load_checkpoint(path)
    assert str(ours.value) == theirs.value.msg


# ----------------------------------------------- metrics csv (eval.cpp:161-210)

def test_metrics_csv_bytes_and_round_trip(ref, tmp_path):
    trace = [dict(t=t, passes=0.05 * (t + 1), samples_per_word=1e2 * (t + 1) / 3.0,
                  ll=-7.0 - 1.0 / (t + 3), wall_seconds=0.001 * t * t + 1e-9, m_t=100.0 / (t + 1))
             for t in range(9)]
    a, b = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    S.write_metrics_csv(trace, a)
    ref.write_metrics_csv(b, trace)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert S.read_metrics_csv(b) == ref.read_metrics_csv(b) == trace


def test_metrics_csv_malformed(ref, tmp_path):
    for text in ["t,passes\n", "t,passes,samples_per_word,ll,wall_seconds,m_t\n1,2,3\n",
                 "t,passes,samples_per_word,ll,wall_seconds,m_t\r\n"]:
        p = write(tmp_path, "bad.csv", text)
        with pytest.raises(S.IoError) as ours:
            S.read_metrics_csv(p)
        with pytest.raises(OracleError) as theirs:
            ref.read_metrics_csv(p)
        assert str(ours.value) == theirs.value.msg
