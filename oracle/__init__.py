"""Parity oracles for the SAME/LDA hot path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here, both CPU-only and both built by ``oracle/Makefile``:

* ``Port``  -- ``libsamelda_oracle.so``, the plain-C restatement of the
  reference hot path (``samelda_oracle.c``; every function cites the
  reference file:line it restates).
* ``Ref``   -- ``_ref/libsamelda_ref.so``, the reference library itself,
  compiled from ``/root/reference/proj`` sources (this container only; the
  built ``.so`` travels to the GPU box, the sources do not).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1409_5402_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "libsamelda_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libsamelda_ref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

ERRORS = {1: "ConfigError", 2: "IoError", 3: "NumericalError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg
        self.kind = ERRORS.get(code, "Error")


def _check(code: int, lib=None) -> None:
    if code:
        msg = ""
        if lib is not None and hasattr(lib, "ref_last_error"):
            msg = lib.ref_last_error().decode(errors="replace")
        raise OracleError(code, msg)


@dataclass
class CorpusArrays:
    """CSR corpus (corpus.hpp:15-32): int64 offsets, int32 word ids / counts."""

    doc_offsets: np.ndarray
    word_ids: np.ndarray
    counts: np.ndarray
    n_words: int
    phi_true: np.ndarray | None = None

    @property
    def n_docs(self) -> int:
        return len(self.doc_offsets) - 1

    @property
    def nnz(self) -> int:
        return int(self.doc_offsets[-1])

    @property
    def n_tokens(self) -> int:
        return int(self.counts.astype(np.int64).sum())

    def subset(self, ids: np.ndarray) -> "CorpusArrays":
        """corpus.cpp:214-229 subset_corpus."""
        ids = np.asarray(ids, dtype=np.int64)
        lens = self.doc_offsets[ids + 1] - self.doc_offsets[ids]
        offs = np.zeros(len(ids) + 1, dtype=np.int64)
        np.cumsum(lens, out=offs[1:])
        idx = np.concatenate([np.arange(self.doc_offsets[d], self.doc_offsets[d + 1]) for d in ids]) \
            if len(ids) else np.zeros(0, dtype=np.int64)
        return CorpusArrays(offs, np.ascontiguousarray(self.word_ids[idx]),
                            np.ascontiguousarray(self.counts[idx]), self.n_words)


class _ConfigStruct(C.Structure):
    _fields_ = [("n_topics", C.c_int64), ("m", C.c_double), ("schedule", C.c_int),
                ("tau0", C.c_double), ("gamma", C.c_double), ("batch_fraction", C.c_double),
                ("t_max", C.c_int64), ("inner_sweeps", C.c_int64), ("seed", C.c_uint64),
                ("alpha", C.c_double), ("beta", C.c_double), ("init_noise", C.c_double),
                ("expected", C.c_int)]


class _RefConfigStruct(C.Structure):
    _fields_ = [("n_topics", C.c_int64), ("m", C.c_double), ("schedule", C.c_int),
                ("tau0", C.c_double), ("gamma", C.c_double), ("batch_fraction", C.c_double),
                ("t_max", C.c_int64), ("inner_sweeps", C.c_int64), ("seed", C.c_uint64),
                ("alpha", C.c_double), ("beta", C.c_double), ("init_noise", C.c_double),
                ("n_threads", C.c_int)]


class _TraceRow(C.Structure):
    _fields_ = [("t", C.c_int64), ("passes", C.c_double), ("samples_per_word", C.c_double),
                ("ll", C.c_double), ("wall_seconds", C.c_double), ("m_t", C.c_double)]


SCHEDULES = {"constant": 0, "linear": 1, "log": 2, "invlinear": 3}


@dataclass
class TrainConfig:
    """sampler.hpp:23-42 SamplerConfig (defaults identical)."""

    n_topics: int = 16
    m: float = 100.0
    schedule: str = "constant"
    tau0: float = 1.0
    gamma: float = 0.5
    batch_fraction: float = 0.05
    t_max: int = 0
    inner_sweeps: int = 2
    seed: int = 0
    alpha: float = 0.1
    beta: float = 0.01
    init_noise: float = 0.1
    n_threads: int = 1


def _trace_to_list(rows, n):
    return [dict(t=rows[i].t, passes=rows[i].passes, samples_per_word=rows[i].samples_per_word,
                 ll=rows[i].ll, wall_seconds=rows[i].wall_seconds, m_t=rows[i].m_t)
            for i in range(n)]


def _batch_nnz(corpus: CorpusArrays, doc_ids: np.ndarray) -> int:
    d = np.asarray(doc_ids, dtype=np.int64)
    return int((corpus.doc_offsets[d + 1] - corpus.doc_offsets[d]).sum())


class Port:
    """ctypes view of the C restatement (samelda_oracle.c)."""

    def __init__(self, path: str = PORT_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.so_make_tag.restype = C.c_uint32
        L.so_make_tag.argtypes = [C.c_uint32] * 3
        L.so_philox_block.argtypes = [_u32p, _u32p, _u32p]
        L.so_poisson_grid.argtypes = [C.c_double, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_uint32, C.c_uint32, C.c_uint32, C.c_int64, _i64p]
        L.so_sddmm.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p, C.c_int64, _i64p, _i32p,
                               _i32p, _f64p]
        L.so_sample_counts.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p, C.c_int64, _f64p,
                                       C.c_int64, _i64p, _i32p, _i32p, _i32p, C.c_double,
                                       C.c_uint64, C.c_int64, C.c_int, _i64p, _i64p]
        L.so_expected_counts.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p, C.c_int64, _f64p,
                                         C.c_int64, _i64p, _i32p, _i32p, _i32p, C.c_double,
                                         _f64p, _f64p]
        L.so_update_model.argtypes = [_f64p, C.c_int64, _f64p, C.c_int64, C.c_int64, C.c_double,
                                      C.c_double, _i32p, C.c_int64, _i64p, _i64p, C.c_double,
                                      C.c_double]
        L.so_update_model_expected.argtypes = [_f64p, C.c_int64, _f64p, C.c_int64, C.c_int64,
                                               C.c_double, C.c_double, _i32p, C.c_int64, _f64p,
                                               _f64p, C.c_double, C.c_double]
        L.so_rho_schedule.argtypes = [C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.so_anneal_m.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double,
                                  C.POINTER(C.c_double)]
        L.so_fold_in_theta.argtypes = [_f64p, C.c_int64, C.c_int64, _i32p, _i32p, C.c_int64,
                                       C.c_double, C.c_int, _f64p]
        L.so_perword_loglik.argtypes = [_f64p, C.c_int64, C.c_int64, _i64p, _i32p, _i32p,
                                        C.c_int64, C.c_double, C.c_uint64,
                                        C.POINTER(C.c_double)]
        L.so_split_holdout_ids.argtypes = [C.c_int64, C.c_double, C.c_uint64, _i32p,
                                           C.POINTER(C.c_int64), _i32p, C.POINTER(C.c_int64)]
        L.so_make_corpus.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                                     C.c_double, C.c_double, C.POINTER(C.c_void_p)]
        L.so_generated_free.argtypes = [C.c_void_p]
        L.so_train.argtypes = [_i64p, _i32p, _i32p, C.c_int64, C.c_int64, C.c_void_p,
                               C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(_ConfigStruct),
                               C.c_int64, _f64p, _f64p, C.POINTER(_TraceRow),
                               C.POINTER(C.c_int64)]
        L.so_init_phi.argtypes = [_f64p, C.c_int64, C.c_int64, C.c_double, C.c_uint64]

    # -- rng
    def make_tag(self, purpose, sub=0, index=0):
        return int(self.lib.so_make_tag(purpose, sub, index))

    def philox_block(self, ctr, key):
        out = np.zeros(4, np.uint32)
        self.lib.so_philox_block(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
        return out

    def poisson_grid(self, lam, seed, t, doc, word, sweep, k0, n):
        out = np.zeros(n, np.int64)
        _check(self.lib.so_poisson_grid(lam, seed, t, doc, word, sweep, k0, n, out))
        return out

    # -- corpus
    def make_corpus(self, n_docs, n_words, n_topics, len_mean, seed, theta_conc=0.2,
                    phi_conc=0.08) -> CorpusArrays:
        """tests/support/synthetic.cpp:61-106 make_corpus."""

        class _Gen(C.Structure):
            _fields_ = [("n_docs", C.c_int64), ("n_words", C.c_int64), ("n_topics", C.c_int64),
                        ("nnz", C.c_int64), ("n_tokens", C.c_int64),
                        ("doc_offsets", C.POINTER(C.c_int64)),
                        ("word_ids", C.POINTER(C.c_int32)), ("counts", C.POINTER(C.c_int32)),
                        ("phi_true", C.POINTER(C.c_double))]

        h = C.c_void_p()
        _check(self.lib.so_make_corpus(n_docs, n_words, n_topics, len_mean, seed, theta_conc,
                                       phi_conc, C.byref(h)))
        g = C.cast(h, C.POINTER(_Gen)).contents
        nnz = g.nnz
        out = CorpusArrays(
            np.ctypeslib.as_array(g.doc_offsets, (n_docs + 1,)).copy(),
            np.ctypeslib.as_array(g.word_ids, (max(nnz, 1),))[:nnz].copy(),
            np.ctypeslib.as_array(g.counts, (max(nnz, 1),))[:nnz].copy(),
            n_words,
            np.ctypeslib.as_array(g.phi_true, (n_topics * n_words,)).copy().reshape(
                n_topics, n_words))
        self.lib.so_generated_free(h)
        return out

    def split_holdout(self, corpus: CorpusArrays, test_fraction: float, seed: int):
        D = corpus.n_docs
        tr = np.zeros(D, np.int32)
        te = np.zeros(D, np.int32)
        ntr, nte = C.c_int64(), C.c_int64()
        _check(self.lib.so_split_holdout_ids(D, test_fraction, seed, tr, C.byref(ntr), te,
                                             C.byref(nte)))
        return corpus.subset(tr[:ntr.value]), corpus.subset(te[:nte.value])

    # -- sampler
    def sddmm(self, theta_batch, phi, corpus: CorpusArrays, doc_ids):
        theta_batch = np.ascontiguousarray(theta_batch, np.float64)
        phi = np.ascontiguousarray(phi, np.float64)
        doc_ids = np.ascontiguousarray(doc_ids, np.int32)
        mu = np.zeros(max(_batch_nnz(corpus, doc_ids), 1))
        B, K = theta_batch.shape
        _check(self.lib.so_sddmm(theta_batch.reshape(-1) if theta_batch.size else np.zeros(1),
                                 B, K, phi, phi.shape[1], corpus.doc_offsets, corpus.word_ids,
                                 doc_ids if len(doc_ids) else np.zeros(1, np.int32), mu))
        return mu[:_batch_nnz(corpus, doc_ids)]

    def sample_counts(self, theta_batch, phi, mu, corpus, doc_ids, m_t, seed, t, sweep=0):
        theta_batch = np.ascontiguousarray(theta_batch, np.float64)
        phi = np.ascontiguousarray(phi, np.float64)
        doc_ids = np.ascontiguousarray(doc_ids, np.int32)
        B, K = theta_batch.shape
        W = phi.shape[1]
        tc = np.zeros(max(B * K, 1), np.int64)
        pc = np.zeros(W * K, np.int64)
        mu = np.ascontiguousarray(mu, np.float64)
        _check(self.lib.so_sample_counts(theta_batch.reshape(-1) if B else np.zeros(1), B, K,
                                         phi, W, mu if len(mu) else np.zeros(1), len(mu),
                                         corpus.doc_offsets, corpus.word_ids, corpus.counts,
                                         doc_ids if B else np.zeros(1, np.int32), m_t, seed, t,
                                         sweep, tc, pc))
        return tc[:B * K].reshape(B, K), pc.reshape(W, K)

    def expected_counts(self, theta_batch, phi, mu, corpus, doc_ids, m_t):
        theta_batch = np.ascontiguousarray(theta_batch, np.float64)
        phi = np.ascontiguousarray(phi, np.float64)
        doc_ids = np.ascontiguousarray(doc_ids, np.int32)
        B, K = theta_batch.shape
        W = phi.shape[1]
        tc = np.zeros(max(B * K, 1))
        pc = np.zeros(W * K)
        mu = np.ascontiguousarray(mu, np.float64)
        _check(self.lib.so_expected_counts(theta_batch.reshape(-1), B, K, phi, W, mu, len(mu),
                                           corpus.doc_offsets, corpus.word_ids, corpus.counts,
                                           doc_ids, m_t, tc, pc))
        return tc[:B * K].reshape(B, K), pc.reshape(W, K)

    def update_model(self, theta, phi, doc_ids, theta_counts, phi_counts, m_t, rho_t, alpha,
                     beta, expected=False):
        """Returns updated (theta, phi) copies."""
        theta = np.array(theta, np.float64, copy=True)
        phi = np.array(phi, np.float64, copy=True)
        K, W = phi.shape
        doc_ids = np.ascontiguousarray(doc_ids, np.int32)
        fn = self.lib.so_update_model_expected if expected else self.lib.so_update_model
        dt = np.float64 if expected else np.int64
        _check(fn(theta.reshape(-1), theta.shape[0], phi.reshape(-1), K, W, alpha, beta, doc_ids,
                  len(doc_ids), np.ascontiguousarray(theta_counts, dt).reshape(-1),
                  np.ascontiguousarray(phi_counts, dt).reshape(-1), m_t, rho_t))
        return theta, phi

    def rho_schedule(self, t, tau0, gamma):
        out = C.c_double()
        _check(self.lib.so_rho_schedule(t, tau0, gamma, C.byref(out)))
        return out.value

    def anneal_m(self, schedule, t, t_max, m):
        out = C.c_double()
        _check(self.lib.so_anneal_m(SCHEDULES.get(schedule, schedule), t, t_max, m,
                                    C.byref(out)))
        return out.value

    # -- eval
    def fold_in_theta(self, phi, words, counts, alpha, sweeps=50):
        phi = np.ascontiguousarray(phi, np.float64)
        K, W = phi.shape
        out = np.zeros(K)
        w = np.ascontiguousarray(words, np.int32)
        c = np.ascontiguousarray(counts, np.int32)
        self.lib.so_fold_in_theta(phi, K, W, w if len(w) else np.zeros(1, np.int32),
                                  c if len(c) else np.zeros(1, np.int32), len(w), alpha, sweeps,
                                  out)
        return out

    def perword_loglik(self, phi, corpus: CorpusArrays, alpha, seed):
        phi = np.ascontiguousarray(phi, np.float64)
        out = C.c_double()
        _check(self.lib.so_perword_loglik(phi, phi.shape[0], phi.shape[1], corpus.doc_offsets,
                                          corpus.word_ids, corpus.counts, corpus.n_docs, alpha,
                                          seed, C.byref(out)))
        return out.value

    def init_phi(self, K, W, init_noise, seed):
        phi = np.zeros(K * W)
        self.lib.so_init_phi(phi, K, W, init_noise, seed)
        return phi.reshape(K, W)

    def train(self, corpus: CorpusArrays, cfg: TrainConfig, heldout: CorpusArrays | None = None,
              eval_every: int = 0, expected: bool = False):
        s = _ConfigStruct(cfg.n_topics, cfg.m, SCHEDULES[cfg.schedule], cfg.tau0, cfg.gamma,
                          cfg.batch_fraction, cfg.t_max, cfg.inner_sweeps, cfg.seed, cfg.alpha,
                          cfg.beta, cfg.init_noise, 1 if expected else 0)
        K, W, D = cfg.n_topics, corpus.n_words, corpus.n_docs
        phi = np.zeros(K * W)
        theta = np.zeros(D * K)
        rows = (_TraceRow * max(cfg.t_max, 1))()
        n = C.c_int64()
        ho = (heldout.doc_offsets.ctypes.data, heldout.word_ids.ctypes.data,
              heldout.counts.ctypes.data, heldout.n_docs) if heldout is not None else (
            None, None, None, 0)
        _check(self.lib.so_train(corpus.doc_offsets, corpus.word_ids, corpus.counts, D, W, *ho,
                                 C.byref(s), eval_every, phi, theta, rows, C.byref(n)))
        return phi.reshape(K, W), theta.reshape(D, K), _trace_to_list(rows, n.value)


class Ref:
    """ctypes view of the compiled reference (oracle/_ref/libsamelda_ref.so)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_stream_u32.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_int64, _u32p]
        L.ref_stream_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_int64, C.c_int, _f64p]
        L.ref_stream_below.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint64, C.c_int64, _u64p]
        L.ref_poisson_grid.argtypes = [C.c_double, C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint32, C.c_uint32, C.c_int64, _i64p]
        L.ref_poisson_stream.argtypes = [C.c_double, C.c_uint64, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_uint32, C.c_int64, _i64p]
        L.ref_make_corpus.restype = C.c_void_p
        L.ref_make_corpus.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                                      C.c_double, C.c_double]
        L.ref_generated_sizes.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 3
        L.ref_generated_copy.argtypes = [C.c_void_p, _i64p, _i32p, _i32p, _f64p]
        L.ref_generated_free.argtypes = [C.c_void_p]
        L.ref_sddmm.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p, C.c_int64, C.c_int64,
                                _i64p, _i32p, _i32p, C.c_int64, _i32p, _f64p, C.c_int64,
                                C.POINTER(C.c_int64), C.c_int]
        L.ref_sample_counts.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p, C.c_int64, _f64p,
                                        C.c_int64, _i64p, _i32p, _i32p, C.c_int64, _i32p,
                                        C.c_double, C.c_uint64, C.c_int64, C.c_int, C.c_int,
                                        _i64p, _i64p]
        L.ref_update_model.argtypes = [_f64p, C.c_int64, _f64p, C.c_int64, C.c_int64,
                                       C.c_double, C.c_double, _i32p, C.c_int64, _i64p, _i64p,
                                       C.c_double, C.c_double]
        L.ref_rho_schedule.argtypes = [C.c_int64, C.c_double, C.c_double,
                                       C.POINTER(C.c_double)]
        L.ref_anneal_m.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double,
                                   C.POINTER(C.c_double)]
        L.ref_fold_in_theta.argtypes = [_f64p, C.c_int64, C.c_int64, _i32p, _i32p, C.c_int64,
                                        C.c_double, C.c_int, _f64p]
        L.ref_perword_loglik.argtypes = [_f64p, C.c_int64, C.c_int64, _i64p, _i32p, _i32p,
                                         C.c_int64, C.c_double, C.c_uint64, C.c_int,
                                         C.POINTER(C.c_double)]
        L.ref_minibatches.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.c_int64, _i32p,
                                      _i64p]
        L.ref_train.argtypes = [_i64p, _i32p, _i32p, C.c_int64, C.c_int64, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(_RefConfigStruct),
                                C.c_int64, _f64p, _f64p, C.POINTER(_TraceRow),
                                C.POINTER(C.c_int64)]
        L.ref_split_holdout_ids.argtypes = [_i64p, _i32p, _i32p, C.c_int64, C.c_int64,
                                            C.c_double, C.c_uint64, _i64p, _i32p, _i32p,
                                            C.POINTER(C.c_int64), _i64p, _i32p, _i32p,
                                            C.POINTER(C.c_int64)]

    def _chk(self, code):
        _check(code, self.lib)

    def stream_u32(self, seed, t, doc, word, tag, n):
        out = np.zeros(n, np.uint32)
        self._chk(self.lib.ref_stream_u32(seed, t, doc, word, tag, n, out))
        return out

    def stream_uniform(self, seed, t, doc, word, tag, n, oo=False):
        out = np.zeros(n)
        self._chk(self.lib.ref_stream_uniform(seed, t, doc, word, tag, n, int(oo), out))
        return out

    def stream_below(self, seed, t, doc, word, tag, bound, n):
        out = np.zeros(n, np.uint64)
        self._chk(self.lib.ref_stream_below(seed, t, doc, word, tag, bound, n, out))
        return out

    def poisson_grid(self, lam, seed, t, doc, word, sweep, k0, n):
        out = np.zeros(n, np.int64)
        self._chk(self.lib.ref_poisson_grid(lam, seed, t, doc, word, sweep, k0, n, out))
        return out

    def poisson_stream(self, lam, seed, t, doc, word, tag, n):
        out = np.zeros(n, np.int64)
        self._chk(self.lib.ref_poisson_stream(lam, seed, t, doc, word, tag, n, out))
        return out

    def make_corpus(self, n_docs, n_words, n_topics, len_mean, seed, theta_conc=0.2,
                    phi_conc=0.08) -> CorpusArrays:
        h = self.lib.ref_make_corpus(n_docs, n_words, n_topics, len_mean, seed, theta_conc,
                                     phi_conc)
        nd, nnz, nt = C.c_int64(), C.c_int64(), C.c_int64()
        self.lib.ref_generated_sizes(h, C.byref(nd), C.byref(nnz), C.byref(nt))
        offs = np.zeros(nd.value + 1, np.int64)
        words = np.zeros(max(nnz.value, 1), np.int32)
        counts = np.zeros(max(nnz.value, 1), np.int32)
        phi = np.zeros(n_topics * n_words)
        self.lib.ref_generated_copy(h, offs, words, counts, phi)
        self.lib.ref_generated_free(h)
        return CorpusArrays(offs, words[:nnz.value].copy(), counts[:nnz.value].copy(), n_words,
                            phi.reshape(n_topics, n_words))

    def split_holdout(self, corpus: CorpusArrays, test_fraction, seed):
        D, nnz = corpus.n_docs, corpus.nnz
        bufs = [np.zeros(D + 1, np.int64), np.zeros(max(nnz, 1), np.int32),
                np.zeros(max(nnz, 1), np.int32), np.zeros(D + 1, np.int64),
                np.zeros(max(nnz, 1), np.int32), np.zeros(max(nnz, 1), np.int32)]
        ntr, nte = C.c_int64(), C.c_int64()
        self._chk(self.lib.ref_split_holdout_ids(corpus.doc_offsets, corpus.word_ids,
                                                 corpus.counts, D, corpus.n_words,
                                                 test_fraction, seed, bufs[0], bufs[1], bufs[2],
                                                 C.byref(ntr), bufs[3], bufs[4], bufs[5],
                                                 C.byref(nte)))
        tr_off = bufs[0][:ntr.value + 1].copy()
        te_off = bufs[3][:nte.value + 1].copy()
        return (CorpusArrays(tr_off, bufs[1][:tr_off[-1]].copy(), bufs[2][:tr_off[-1]].copy(),
                             corpus.n_words),
                CorpusArrays(te_off, bufs[4][:te_off[-1]].copy(), bufs[5][:te_off[-1]].copy(),
                             corpus.n_words))

    def sddmm(self, theta_batch, phi, corpus: CorpusArrays, doc_ids, n_threads=1):
        theta_batch = np.ascontiguousarray(theta_batch, np.float64)
        phi = np.ascontiguousarray(phi, np.float64)
        doc_ids = np.ascontiguousarray(doc_ids, np.int32)
        n = _batch_nnz(corpus, doc_ids)
        mu = np.zeros(max(n, 1))
        ln = C.c_int64()
        B, Kt = theta_batch.shape if theta_batch.ndim == 2 else (0, phi.shape[0])
        self._chk(self.lib.ref_sddmm(theta_batch.reshape(-1) if theta_batch.size else np.zeros(1),
                                     B, Kt, phi, phi.shape[0], phi.shape[1], corpus.doc_offsets,
                                     corpus.word_ids, corpus.counts, corpus.n_docs,
                                     doc_ids if len(doc_ids) else np.zeros(1, np.int32), mu,
                                     len(mu), C.byref(ln), n_threads))
        return mu[:ln.value]

    def sample_counts(self, theta_batch, phi, mu, corpus, doc_ids, m_t, seed, t, sweep=0,
                      n_threads=1):
        theta_batch = np.ascontiguousarray(theta_batch, np.float64)
        phi = np.ascontiguousarray(phi, np.float64)
        doc_ids = np.ascontiguousarray(doc_ids, np.int32)
        B, K = theta_batch.shape
        W = phi.shape[1]
        tc = np.zeros(max(B * K, 1), np.int64)
        pc = np.zeros(W * K, np.int64)
        mu = np.ascontiguousarray(mu, np.float64)
        self._chk(self.lib.ref_sample_counts(theta_batch.reshape(-1) if B else np.zeros(1), B, K,
                                             phi, W, mu if len(mu) else np.zeros(1), len(mu),
                                             corpus.doc_offsets, corpus.word_ids, corpus.counts,
                                             corpus.n_docs,
                                             doc_ids if B else np.zeros(1, np.int32), m_t, seed,
                                             t, sweep, n_threads, tc, pc))
        return tc[:B * K].reshape(B, K), pc.reshape(W, K)

    def update_model(self, theta, phi, doc_ids, theta_counts, phi_counts, m_t, rho_t, alpha,
                     beta):
        theta = np.array(theta, np.float64, copy=True)
        phi = np.array(phi, np.float64, copy=True)
        K, W = phi.shape
        doc_ids = np.ascontiguousarray(doc_ids, np.int32)
        self._chk(self.lib.ref_update_model(theta.reshape(-1), theta.shape[0], phi.reshape(-1),
                                            K, W, alpha, beta, doc_ids, len(doc_ids),
                                            np.ascontiguousarray(theta_counts,
                                                                 np.int64).reshape(-1),
                                            np.ascontiguousarray(phi_counts,
                                                                 np.int64).reshape(-1),
                                            m_t, rho_t))
        return theta, phi

    def rho_schedule(self, t, tau0, gamma):
        out = C.c_double()
        self._chk(self.lib.ref_rho_schedule(t, tau0, gamma, C.byref(out)))
        return out.value

    def anneal_m(self, schedule, t, t_max, m):
        out = C.c_double()
        self._chk(self.lib.ref_anneal_m(SCHEDULES.get(schedule, schedule), t, t_max, m,
                                        C.byref(out)))
        return out.value

    def fold_in_theta(self, phi, words, counts, alpha, sweeps=50):
        phi = np.ascontiguousarray(phi, np.float64)
        out = np.zeros(phi.shape[0])
        w = np.ascontiguousarray(words, np.int32)
        c = np.ascontiguousarray(counts, np.int32)
        self._chk(self.lib.ref_fold_in_theta(phi, phi.shape[0], phi.shape[1],
                                             w if len(w) else np.zeros(1, np.int32),
                                             c if len(c) else np.zeros(1, np.int32), len(w),
                                             alpha, sweeps, out))
        return out

    def perword_loglik(self, phi, corpus: CorpusArrays, alpha, seed, n_threads=1):
        phi = np.ascontiguousarray(phi, np.float64)
        out = C.c_double()
        self._chk(self.lib.ref_perword_loglik(phi, phi.shape[0], phi.shape[1],
                                              corpus.doc_offsets, corpus.word_ids,
                                              corpus.counts, corpus.n_docs, alpha, seed,
                                              n_threads, C.byref(out)))
        return out.value

    def minibatches(self, n_docs, batch_fraction, seed, n_batches):
        bs = max(1, int(round(batch_fraction * n_docs)))
        out = np.zeros(bs * n_batches, np.int32)
        sizes = np.zeros(n_batches, np.int64)
        self._chk(self.lib.ref_minibatches(n_docs, batch_fraction, seed, n_batches, out, sizes))
        res, pos = [], 0
        for s in sizes:
            res.append(out[pos:pos + s].copy())
            pos += s
        return res

    def train(self, corpus: CorpusArrays, cfg: TrainConfig, heldout: CorpusArrays | None = None,
              eval_every: int = 0):
        s = _RefConfigStruct(cfg.n_topics, cfg.m, SCHEDULES[cfg.schedule], cfg.tau0, cfg.gamma,
                             cfg.batch_fraction, cfg.t_max, cfg.inner_sweeps, cfg.seed,
                             cfg.alpha, cfg.beta, cfg.init_noise, cfg.n_threads)
        K, W, D = cfg.n_topics, corpus.n_words, corpus.n_docs
        phi = np.zeros(K * W)
        theta = np.zeros(D * K)
        rows = (_TraceRow * max(cfg.t_max, 1))()
        n = C.c_int64()
        ho = (heldout.doc_offsets.ctypes.data, heldout.word_ids.ctypes.data,
              heldout.counts.ctypes.data, heldout.n_docs) if heldout is not None else (
            None, None, None, 0)
        self._chk(self.lib.ref_train(corpus.doc_offsets, corpus.word_ids, corpus.counts, D, W,
                                     *ho, C.byref(s), eval_every, phi, theta, rows, C.byref(n)))
        return phi.reshape(K, W), theta.reshape(D, K), _trace_to_list(rows, n.value)


    # ---- collapsed Gibbs baseline
    def cgs_run(self, corpus: CorpusArrays, K, alpha, beta, seed, n_sweeps):
        """cgs_init + cgs_sweep 1..n_sweeps (cgs.cpp:11-98): (z, doc_topic, word_topic,
        topic_total)."""
        L = self.lib
        L.ref_cgs_run.argtypes = [_i64p, _i32p, _i32p, C.c_int64, C.c_int64, C.c_int64,
                                  C.c_double, C.c_double, C.c_uint64, C.c_int64, _i32p, _i32p,
                                  _i32p, _i64p]
        n_tok = int(np.asarray(corpus.counts, np.int64).sum())
        z = np.zeros(max(n_tok, 1), np.int32)
        dt = np.zeros(max(corpus.n_docs * K, 1), np.int32)
        wt = np.zeros(max(corpus.n_words * K, 1), np.int32)
        tt = np.zeros(K, np.int64)
        self._chk(L.ref_cgs_run(corpus.doc_offsets, corpus.word_ids, corpus.counts,
                                corpus.n_docs, corpus.n_words, K, alpha, beta, seed, n_sweeps,
                                z, dt, wt, tt))
        return (z[:n_tok], dt[:corpus.n_docs * K].reshape(corpus.n_docs, K),
                wt[:corpus.n_words * K].reshape(corpus.n_words, K), tt)

    def cgs_train(self, corpus: CorpusArrays, K, alpha, beta, n_sweeps, seed, eval_every=0,
                  heldout: CorpusArrays | None = None, n_threads=1):
        L = self.lib
        L.ref_cgs_train.argtypes = [_i64p, _i32p, _i32p, C.c_int64, C.c_int64, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double,
                                    C.c_double, C.c_int64, C.c_uint64, C.c_int64, C.c_int,
                                    _f64p, _f64p, C.POINTER(_TraceRow), C.POINTER(C.c_int64)]
        W, D = corpus.n_words, corpus.n_docs
        phi = np.zeros(max(K * W, 1))
        theta = np.zeros(max(D * K, 1))
        rows = (_TraceRow * max(n_sweeps, 1))()
        n = C.c_int64()
        ho = (heldout.doc_offsets.ctypes.data, heldout.word_ids.ctypes.data,
              heldout.counts.ctypes.data, heldout.n_docs) if heldout is not None else (
            None, None, None, 0)
        self._chk(L.ref_cgs_train(corpus.doc_offsets, corpus.word_ids, corpus.counts, D, W, *ho,
                                  K, alpha, beta, n_sweeps, seed, eval_every, n_threads, phi,
                                  theta, rows, C.byref(n)))
        return phi[:K * W].reshape(K, W), theta[:D * K].reshape(D, K), _trace_to_list(rows, n.value)

    # ---- data formats: the reference's own load/save
    def _io_sigs(self):
        L = self.lib
        if getattr(self, "_io_ready", False):
            return L
        L.ref_load_uci.restype = C.c_void_p
        L.ref_load_uci.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_int)]
        L.ref_loaded_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 5
        L.ref_loaded_copy.argtypes = [C.c_void_p, _i64p, _i32p, _i32p, C.c_char_p]
        L.ref_loaded_free.argtypes = [C.c_void_p]
        L.ref_save_uci.argtypes = [_i64p, _i32p, _i32p, C.c_int64, C.c_int64, C.c_char_p,
                                   C.c_int64, C.c_char_p, C.c_char_p]
        L.ref_save_checkpoint.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_double,
                                          C.c_double, _f64p]
        L.ref_load_checkpoint.argtypes = [C.c_char_p] + [C.POINTER(C.c_int64)] * 2 + [
            C.POINTER(C.c_double)] * 2 + [C.c_void_p, C.c_int64]
        L.ref_write_metrics_csv.argtypes = [C.c_char_p, C.POINTER(_TraceRow), C.c_int64]
        L.ref_read_metrics_csv.argtypes = [C.c_char_p, C.POINTER(_TraceRow), C.c_int64,
                                           C.POINTER(C.c_int64)]
        self._io_ready = True
        return L

    def load_uci_bow(self, docword: str, vocab: str):
        """corpus.cpp:62-183 -> (offsets, words, counts, n_words, n_tokens, vocab list)."""
        L = self._io_sigs()
        rc = C.c_int()
        h = L.ref_load_uci(docword.encode(), vocab.encode(), C.byref(rc))
        self._chk(rc.value)
        try:
            d, w, nnz, tok, vb = (C.c_int64() for _ in range(5))
            L.ref_loaded_dims(h, C.byref(d), C.byref(w), C.byref(nnz), C.byref(tok), C.byref(vb))
            off = np.zeros(d.value + 1, np.int64)
            wid = np.zeros(nnz.value, np.int32)
            cnt = np.zeros(nnz.value, np.int32)
            buf = C.create_string_buffer(vb.value + 1)
            L.ref_loaded_copy(h, off, wid, cnt, buf)
            vocab_list = buf.raw[:vb.value].decode("utf-8", "surrogateescape").split("\n")[:-1]
            return off, wid, cnt, w.value, tok.value, vocab_list
        finally:
            L.ref_loaded_free(h)

    def save_uci_bow(self, corpus, vocab_list, docword: str, vocab: str):
        L = self._io_sigs()
        vb = "".join(v + "\n" for v in vocab_list).encode("utf-8", "surrogateescape")
        self._chk(L.ref_save_uci(np.ascontiguousarray(corpus.doc_offsets, np.int64),
                                 np.ascontiguousarray(corpus.word_ids, np.int32),
                                 np.ascontiguousarray(corpus.counts, np.int32),
                                 len(corpus.doc_offsets) - 1, int(corpus.n_words), vb, len(vb),
                                 docword.encode(), vocab.encode()))

    def save_checkpoint(self, path: str, phi: np.ndarray, alpha: float, beta: float):
        L = self._io_sigs()
        phi = np.ascontiguousarray(phi, np.float64)
        self._chk(L.ref_save_checkpoint(path.encode(), phi.shape[0], phi.shape[1], alpha, beta,
                                        phi))

    def load_checkpoint(self, path: str):
        L = self._io_sigs()
        k, w, a, b = C.c_int64(), C.c_int64(), C.c_double(), C.c_double()
        self._chk(L.ref_load_checkpoint(path.encode(), C.byref(k), C.byref(w), C.byref(a),
                                        C.byref(b), None, 0))
        phi = np.zeros((k.value, w.value))
        self._chk(L.ref_load_checkpoint(path.encode(), C.byref(k), C.byref(w), C.byref(a),
                                        C.byref(b), phi.ctypes.data, phi.size))
        return phi, a.value, b.value

    def write_metrics_csv(self, path: str, trace):
        L = self._io_sigs()
        rows = (_TraceRow * max(len(trace), 1))()
        for i, r in enumerate(trace):
            rows[i] = _TraceRow(int(r["t"]), r["passes"], r["samples_per_word"], r["ll"],
                                r["wall_seconds"], r["m_t"])
        self._chk(L.ref_write_metrics_csv(path.encode(), rows, len(trace)))

    def read_metrics_csv(self, path: str):
        L = self._io_sigs()
        n = C.c_int64()
        self._chk(L.ref_read_metrics_csv(path.encode(), None, 0, C.byref(n)))
        rows = (_TraceRow * max(n.value, 1))()
        self._chk(L.ref_read_metrics_csv(path.encode(), rows, n.value, C.byref(n)))
        return _trace_to_list(rows, n.value)


def have_ref() -> bool:
    return os.path.exists(REF_PATH)
