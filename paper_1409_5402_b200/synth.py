"""Synthetic corpora at the BASELINE.json shapes (include/samelda_synth.h).

NYTimes shape: D=300,000, W=102,660, ~100M tokens (~333/doc), nnz/token ~0.70.
PubMed shape:  D=8.2M,    W=141,043, ~730M tokens (~89/doc),  nnz/token ~0.66.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .samelda import Corpus

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsamelda_synth.so")
_lib = None


def load_library() -> C.CDLL:
    """libsamelda_synth.so: the generator alone (host C++), so a process that
    only needs corpora -- bench.py's reference arm -- never maps the CUDA
    product library."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_1409_5402_b200.build`")
        _lib = C.CDLL(_LIB_PATH)
    return _lib


class _Params(C.Structure):
    _fields_ = [("n_docs", C.c_int64), ("n_words", C.c_int64), ("n_topics_gen", C.c_int64),
                ("mean_len", C.c_double), ("len_shape", C.c_double), ("zipf_s", C.c_double),
                ("background", C.c_double), ("topics_per_doc", C.c_double),
                ("seed", C.c_uint64), ("first_doc", C.c_int64)]


PRESETS = {
    "nytimes": dict(n_docs=300_000, n_words=102_660, n_topics_gen=200, mean_len=333.0,
                    len_shape=2.0, zipf_s=1.06, background=0.3, topics_per_doc=2.0),
    "pubmed": dict(n_docs=8_200_000, n_words=141_043, n_topics_gen=200, mean_len=89.0,
                   len_shape=3.0, zipf_s=1.07, background=0.3, topics_per_doc=1.5),
}


def generate(n_docs, n_words, n_topics_gen=200, mean_len=333.0, len_shape=2.0, zipf_s=1.07,
             background=0.3, topics_per_doc=2.0, seed=1, n_threads=None,
             first_doc=0) -> Corpus:
    lib = load_library()
    lib.samelda_synth_generate.restype = C.c_int
    lib.samelda_synth_generate.argtypes = [C.POINTER(_Params), C.c_int, C.POINTER(C.c_void_p),
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.samelda_synth_copy.argtypes = [C.c_void_p] * 4
    lib.samelda_synth_free.argtypes = [C.c_void_p]
    p = _Params(n_docs, n_words, n_topics_gen, mean_len, len_shape, zipf_s, background,
                topics_per_doc, seed, first_doc)
    h, nnz, tok = C.c_void_p(), C.c_int64(), C.c_int64()
    rc = lib.samelda_synth_generate(C.byref(p), int(n_threads or os.cpu_count() or 1),
                                    C.byref(h), C.byref(nnz), C.byref(tok))
    if rc:
        raise ValueError("samelda_synth_generate: bad parameters")
    offs = np.empty(n_docs + 1, np.int64)
    words = np.empty(max(nnz.value, 1), np.int32)
    counts = np.empty(max(nnz.value, 1), np.int32)
    lib.samelda_synth_copy(h, offs.ctypes.data, words.ctypes.data, counts.ctypes.data)
    lib.samelda_synth_free(h)
    return Corpus(offs, words[:nnz.value], counts[:nnz.value], n_words)


def preset(name: str, seed: int = 1, scale: float = 1.0, n_threads=None, shard: int = 0) -> Corpus:
    """Preset corpus; `shard` s generates global docs [s*D, (s+1)*D) (weak-scaling shards)."""
    kw = dict(PRESETS[name])
    kw["n_docs"] = max(2, int(kw["n_docs"] * scale))
    return generate(seed=seed, n_threads=n_threads, first_doc=shard * kw["n_docs"], **kw)


def make_corpus_ref(n_docs: int, n_words: int, n_topics: int, len_mean: float, seed: int,
                    theta_conc: float = 0.2, phi_conc: float = 0.08, n_threads=None) -> Corpus:
    """The reference's synthetic::make_corpus (tests/support/synthetic.cpp:61-106), value for
    value; BASELINE.json configs[0] is make_corpus_ref(10000, 5000, 32, 100.0, 1)."""
    lib = load_library()
    fn = lib.samelda_synth_make_corpus_ref
    fn.restype = C.c_int
    fn.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_double,
                   C.c_double, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                   C.POINTER(C.c_int64)]
    lib.samelda_synth_copy.argtypes = [C.c_void_p] * 4
    lib.samelda_synth_free.argtypes = [C.c_void_p]
    h, nnz, tok = C.c_void_p(), C.c_int64(), C.c_int64()
    rc = fn(n_docs, n_words, n_topics, len_mean, seed, theta_conc, phi_conc,
            int(n_threads or os.cpu_count() or 1), C.byref(h), C.byref(nnz), C.byref(tok))
    if rc:
        raise ValueError("samelda_synth_make_corpus_ref: bad parameters")
    offs = np.empty(n_docs + 1, np.int64)
    words = np.empty(max(nnz.value, 1), np.int32)
    counts = np.empty(max(nnz.value, 1), np.int32)
    lib.samelda_synth_copy(h, offs.ctypes.data, words.ctypes.data, counts.ctypes.data)
    lib.samelda_synth_free(h)
    return Corpus(offs, words[:nnz.value], counts[:nnz.value], n_words)


def subset(corpus: Corpus, doc_ids) -> Corpus:
    """subset_corpus (corpus.cpp): the rows doc_ids, in that order."""
    ids = np.asarray(doc_ids, np.int64)
    o = corpus.doc_offsets
    lens = o[ids + 1] - o[ids]
    offs = np.zeros(len(ids) + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    if len(ids) and offs[-1]:
        starts = np.repeat(o[ids] - offs[:-1], lens)
        idx = starts + np.arange(offs[-1])
    else:
        idx = np.zeros(0, np.int64)
    return Corpus(offs, np.ascontiguousarray(corpus.word_ids[idx]),
                  np.ascontiguousarray(corpus.counts[idx]), corpus.n_words)


def split_holdout(corpus: Corpus, test_fraction: float, seed: int) -> tuple[Corpus, Corpus]:
    """split_holdout (corpus.cpp:231-250): (train, test), ids sorted within each."""
    lib = load_library()
    fn = lib.samelda_synth_split_holdout
    fn.restype = C.c_int
    fn.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.c_void_p, C.POINTER(C.c_int64),
                   C.c_void_p]
    D = corpus.n_docs
    test = np.empty(D, np.int32)
    train = np.empty(D, np.int32)
    nt = C.c_int64()
    if fn(D, test_fraction, seed, test.ctypes.data, C.byref(nt), train.ctypes.data):
        raise ValueError("split_holdout: test_fraction must be in (0,1) and n_docs >= 2")
    n = nt.value
    return subset(corpus, train[:D - n]), subset(corpus, test[:n])
