"""Python mirror of the reference `samelda` sampler/eval interface over the C ABI.

Same names, argument meaning and error behaviour as the reference's
``sampler.hpp`` / ``eval.hpp`` (proj/include/samelda/), so the parity tests
read like the reference's own tests:

    sddmm(theta_batch, phi, corpus, doc_ids)                    sampler.hpp:74-81
    sample_counts(theta_batch, phi, mu, corpus, doc_ids, m_t,
                  seed, t, sweep)                               sampler.hpp:83-91
    update_model(model, counts, rho_t)                          sampler.hpp:93-97
    rho_schedule(t, tau0, gamma), anneal_m(schedule, t, t_max, m)
    train(corpus, config, heldout, eval_every)                  sampler.hpp:105-110
    fold_in_theta(phi, words, counts, alpha, sweeps)            eval.hpp:32-36
    perword_loglik(phi, test, alpha, seed)                      eval.hpp:38-43

Every call goes through ``libsamelda_cuda.so`` (include/samelda_cu.h).  There
is no CPU fallback: importing this module without the built library, or
calling it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsamelda_cuda.so")

MODE_PARITY = 0
MODE_EXPECTED = 1
MODE_THROUGHPUT = 2  # own f32 random streams: statistical (not bit) parity
MODE_MULTINOMIAL = 3  # multinomial(c m) replicas on own streams (no reference counterpart)
SCHEDULES = {"constant": 0, "linear": 1, "log": 2, "invlinear": 3}


class SameldaError(RuntimeError):
    """Base of the reference's error classes (errors.hpp:7-20)."""


class ConfigError(SameldaError):
    pass


class IoError(SameldaError):
    pass


class NumericalError(SameldaError):
    pass


class CudaError(SameldaError):
    pass


_CODES = {1: ConfigError, 2: IoError, 3: NumericalError, 4: CudaError}


class _Corpus(C.Structure):
    _fields_ = [("doc_offsets", C.c_void_p), ("word_ids", C.c_void_p), ("counts", C.c_void_p),
                ("n_docs", C.c_int64), ("n_words", C.c_int64)]


class _Config(C.Structure):
    _fields_ = [("n_topics", C.c_int64), ("m", C.c_double), ("schedule", C.c_int32),
                ("tau0", C.c_double), ("gamma", C.c_double), ("batch_fraction", C.c_double),
                ("t_max", C.c_int64), ("inner_sweeps", C.c_int64), ("seed", C.c_uint64),
                ("alpha", C.c_double), ("beta", C.c_double), ("init_noise", C.c_double),
                ("mode", C.c_int32)]


class _TraceRow(C.Structure):
    _fields_ = [("t", C.c_int64), ("passes", C.c_double), ("samples_per_word", C.c_double),
                ("ll", C.c_double), ("wall_seconds", C.c_double), ("m_t", C.c_double)]


# (name, restype, argtypes) of every entry point in include/samelda_cu.h
_P, _I64, _I32, _D, _U64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_uint64
_CP = C.POINTER(_Corpus)
SIGNATURES = [
    ("samelda_cu_version", C.c_int, []),
    ("samelda_cu_device_count", C.c_int, []),
    ("samelda_cu_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("samelda_cu_destroy", None, [_P]),
    ("samelda_cu_last_error", C.c_char_p, [_P]),
    ("samelda_cu_set_stream", C.c_int, [_P, _P]),
    ("samelda_cu_use_own_stream", C.c_int, [_P]),
    ("samelda_cu_synchronize", C.c_int, [_P]),
    ("samelda_cu_launch_count", _I64, [_P]),
    ("samelda_cu_sddmm", C.c_int, [_P, _CP, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _I64,
                                   C.POINTER(_I64)]),
    ("samelda_cu_sample_counts", C.c_int, [_P, _CP, _P, _I64, _I64, _P, _I64, _I64, _P, _I64,
                                           _P, _D, _U64, _I64, _I32, _P, _P]),
    ("samelda_cu_sample_counts_fast", C.c_int, [_P, _CP, _P, _I64, _I64, _P, _I64, _I64, _P, _I64,
                                           _P, _D, _U64, _I64, _I32, _P, _P]),
    ("samelda_cu_sample_theta_counts_fast", C.c_int, [_P, _CP, _P, _I64, _I64, _P, _I64, _I64, _P,
                                                      _D, _U64, _I64, _I32, _P]),
    ("samelda_cu_sample_counts_multinomial", C.c_int, [_P, _CP, _P, _I64, _I64, _P, _I64, _I64, _P, _I64,
                                           _P, _D, _U64, _I64, _I32, _P, _P]),
    ("samelda_cu_expected_counts", C.c_int, [_P, _CP, _P, _I64, _I64, _P, _I64, _I64, _P, _I64,
                                             _P, _D, _P, _P]),
    ("samelda_cu_update_model", C.c_int, [_P, _P, _I64, _P, _I64, _I64, _D, _D, _P, _I64, _P,
                                          _P, _D, _D]),
    ("samelda_cu_update_model_expected", C.c_int, [_P, _P, _I64, _P, _I64, _I64, _D, _D, _P,
                                                   _I64, _P, _P, _D, _D]),
    ("samelda_cu_rho_schedule", C.c_int, [_I64, _D, _D, C.POINTER(_D)]),
    ("samelda_cu_anneal_m", C.c_int, [_I32, _I64, _I64, _D, C.POINTER(_D)]),
    ("samelda_cu_fold_in_theta", C.c_int, [_P, _P, _I64, _I64, _P, _P, _I64, _D, _I32, _P]),
    ("samelda_cu_set_eval_exact", C.c_int, [_P, _I32]),
    ("samelda_cu_perword_loglik", C.c_int, [_P, _P, _I64, _I64, _CP, _D, _U64, C.POINTER(_D)]),
    ("samelda_cu_batches_create", C.c_int, [_I64, _D, _U64, C.POINTER(C.c_void_p)]),
    ("samelda_cu_batches_size", _I64, [_P]),
    ("samelda_cu_batches_per_pass", _I64, [_P]),
    ("samelda_cu_batches_next", _I64, [_P, _P]),
    ("samelda_cu_batches_destroy", None, [_P]),
    ("samelda_cu_train_begin", C.c_int, [_P, _CP, C.POINTER(_Config)]),
    ("samelda_cu_heldout", C.c_int, [_P, _CP, _U64]),
    ("samelda_cu_period", C.c_int, [_P, _P, _I64, _I64, _D, _D]),
    ("samelda_cu_period_sample", C.c_int, [_P, _P, _I64, _I64, _D]),
    ("samelda_cu_period_update", C.c_int, [_P, _D]),
    ("samelda_cu_phi_counts_pack32", C.c_int, [_P, C.c_void_p, _I64, _I32, C.c_void_p]),
    ("samelda_cu_phi_counts_unpack32", C.c_int, [_P, C.c_void_p, _I64]),
    ("samelda_cu_phi_counts_device", C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(_I64),
                                               C.POINTER(_I32), C.POINTER(_I32)]),
    ("samelda_cu_batch_theta", C.c_int, [_P, _P, _I64]),
    ("samelda_cu_batch_theta_async", C.c_int, [_P, _P, _I64]),
    ("samelda_cu_set_doc_base", C.c_int, [_P, _I64]),
    ("samelda_cu_profile", C.c_int, [_P, _I32]),
    ("samelda_cu_profile_read", C.c_int, [_P, _P, _P, C.POINTER(_I64), C.POINTER(_I64),
                                          C.POINTER(_I64)]),
    ("samelda_cu_count_totals", C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I64)]),
    ("samelda_cu_evaluate", C.c_int, [_P, C.POINTER(_D)]),
    ("samelda_cu_model_download", C.c_int, [_P, _P, _P]),
    ("samelda_cu_model_upload", C.c_int, [_P, _P, _P]),
    ("samelda_cu_train", C.c_int, [_P, _CP, C.POINTER(_Config), _CP, _I64, _P, _P,
                                   C.POINTER(_TraceRow), _I64, C.POINTER(_I64)]),
    # collapsed Gibbs sampler baseline
    ("samelda_cu_cgs_init", C.c_int, [_P, _CP, _I64, _D, _D, _U64]),
    ("samelda_cu_cgs_sweep", C.c_int, [_P, _U64, _I64]),
    ("samelda_cu_cgs_state", C.c_int, [_P, _P, _P, _P, _P]),
    ("samelda_cu_cgs_set_state", C.c_int, [_P, _P, _P, _P, _P]),
    ("samelda_cu_cgs_model", C.c_int, [_P, _P, _P]),
    ("samelda_cu_cgs_train", C.c_int, [_P, _CP, _I64, _D, _D, _I64, _U64, _I64, _CP, _P, _P,
                                       C.POINTER(_TraceRow), _I64, C.POINTER(_I64)]),
    # multi-GPU group (one process, N devices)
    ("samelda_cu_group_create", C.c_int, [_P, C.c_int, C.POINTER(C.c_void_p)]),
    ("samelda_cu_group_destroy", None, [_P]),
    ("samelda_cu_group_last_error", C.c_char_p, [_P]),
    ("samelda_cu_group_size", C.c_int, [_P]),
    ("samelda_cu_group_uses_nccl", C.c_int, [_P]),
    ("samelda_cu_group_train_begin", C.c_int, [_P, _CP, C.POINTER(_Config)]),
    ("samelda_cu_group_heldout", C.c_int, [_P, _CP, _U64]),
    ("samelda_cu_group_period", C.c_int, [_P, _P, _I64, _I64, _D, _D]),
    ("samelda_cu_group_synchronize", C.c_int, [_P]),
    ("samelda_cu_group_evaluate", C.c_int, [_P, C.POINTER(_D)]),
    ("samelda_cu_group_model_download", C.c_int, [_P, _P, _P]),
    ("samelda_cu_group_train", C.c_int, [_P, _CP, C.POINTER(_Config), _CP, _I64, _P, _P,
                                         C.POINTER(_TraceRow), _I64, C.POINTER(_I64)]),
    # data formats (include/samelda_io.h)
    ("samelda_io_last_error", C.c_char_p, []),
    ("samelda_io_load_uci", C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    ("samelda_io_save_csr", C.c_int, [C.c_char_p, _CP, C.c_char_p, _I64]),
    ("samelda_io_load_csr", C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    ("samelda_io_corpus_dims", None, [_P] + [C.POINTER(_I64)] * 6),
    ("samelda_io_corpus_view", None, [_P, _CP, C.POINTER(C.c_void_p)]),
    ("samelda_io_corpus_free", None, [_P]),
    ("samelda_io_save_uci", C.c_int, [_CP, C.c_char_p, _I64, C.c_char_p, C.c_char_p]),
    ("samelda_io_save_checkpoint", C.c_int, [C.c_char_p, _I64, _I64, _D, _D, _P]),
    ("samelda_io_checkpoint_header", C.c_int, [C.c_char_p, C.POINTER(_I64), C.POINTER(_I64),
                                               C.POINTER(_D), C.POINTER(_D)]),
    ("samelda_io_load_checkpoint", C.c_int, [C.c_char_p, _P, _I64]),
    ("samelda_io_write_metrics_csv", C.c_int, [C.c_char_p, C.POINTER(_TraceRow), _I64]),
    ("samelda_io_read_metrics_csv", C.c_int, [C.c_char_p, C.POINTER(_TraceRow), _I64,
                                              C.POINTER(_I64)]),
]

_lib = None


def load_library(path: str | None = None) -> C.CDLL:
    """Load libsamelda_cuda.so (raises if it was not built -- no fallback).

    SAMELDA_CUDA_LIB overrides the path (profiling of alternative builds)."""
    global _lib
    path = path or os.environ.get("SAMELDA_CUDA_LIB") or _LIB_PATH
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -m paper_1409_5402_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Corpus:
    """CSR corpus (corpus.hpp:15-32)."""

    doc_offsets: np.ndarray
    word_ids: np.ndarray
    counts: np.ndarray
    n_words: int
    vocab: list | None = None  # n_words tokens (corpus.hpp:23), when loaded from files

    def __post_init__(self):
        self.doc_offsets = np.ascontiguousarray(self.doc_offsets, np.int64)
        self.word_ids = np.ascontiguousarray(self.word_ids, np.int32)
        self.counts = np.ascontiguousarray(self.counts, np.int32)
        if len(self.word_ids) == 0:  # keep valid pointers for empty corpora
            self._w_keep = np.zeros(1, np.int32)
            self._c_keep = np.zeros(1, np.int32)

    @classmethod
    def of(cls, c) -> "Corpus":
        return c if isinstance(c, Corpus) else cls(c.doc_offsets, c.word_ids, c.counts,
                                                   int(c.n_words), getattr(c, "vocab", None))

    @property
    def n_docs(self) -> int:
        return len(self.doc_offsets) - 1

    @property
    def nnz(self) -> int:
        return int(self.doc_offsets[-1])

    @property
    def n_tokens(self) -> int:
        return int(self.counts.astype(np.int64).sum())

    def doc_tokens(self) -> np.ndarray:
        return np.add.reduceat(self.counts.astype(np.int64), self.doc_offsets[:-1]) * (
            np.diff(self.doc_offsets) > 0) if self.nnz else np.zeros(self.n_docs, np.int64)

    def _struct(self) -> _Corpus:
        w = self.word_ids if len(self.word_ids) else self._w_keep
        c = self.counts if len(self.counts) else self._c_keep
        return _Corpus(self.doc_offsets.ctypes.data, w.ctypes.data, c.ctypes.data, self.n_docs,
                       int(self.n_words))


@dataclass
class SamplerConfig:
    """sampler.hpp:23-42 (same defaults); `mode` selects parity / expected counts."""

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
    n_threads: int = 1
    init_noise: float = 0.1
    mode: int = MODE_PARITY

    def _struct(self) -> _Config:
        if self.schedule not in SCHEDULES:
            raise ConfigError(f"unknown schedule '{self.schedule}' "
                              "(expected constant|linear|log|invlinear)")
        return _Config(int(self.n_topics), float(self.m), SCHEDULES[self.schedule],
                       float(self.tau0), float(self.gamma), float(self.batch_fraction),
                       int(self.t_max), int(self.inner_sweeps), int(self.seed), float(self.alpha),
                       float(self.beta), float(self.init_noise), int(self.mode))


@dataclass
class SampledCounts:
    """sampler.hpp:50-68: theta B x K and phi W x K integer counts."""

    doc_ids: np.ndarray
    n_topics: int
    n_words: int
    m_t: float
    theta_counts: np.ndarray
    phi_counts: np.ndarray

    def theta_hat(self, b, k):
        return float(self.theta_counts[b, k]) / self.m_t

    def phi_hat(self, k, w):
        return float(self.phi_counts[w, k]) / self.m_t

    def theta_total(self) -> int:
        return int(self.theta_counts.sum())

    def phi_total(self) -> int:
        return int(self.phi_counts.sum())


@dataclass
class Model:
    """model.hpp:40-47: phi K x W, theta D x K."""

    n_topics: int
    n_words: int
    alpha: float
    beta: float
    phi: np.ndarray
    theta: np.ndarray


def init_model(n_topics, n_words, n_docs, alpha, beta) -> Model:
    """model.cpp:41-52 (host fill; not on the hot path)."""
    return Model(n_topics, n_words, alpha, beta,
                 np.full((n_topics, n_words), 1.0 / n_words),
                 np.full((n_docs, n_topics), alpha + 1.0 / n_topics))


class Context:
    """Owns one device context (streams, resident corpus/model, scratch)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.samelda_cu_create(device, C.byref(h))
        if rc:
            raise CudaError(f"samelda_cu_create(device={device}) failed with code {rc}: "
                            "no usable CUDA device (there is no CPU fallback)")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.samelda_cu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc:
            msg = self.lib.samelda_cu_last_error(self.h).decode(errors="replace")
            raise _CODES.get(rc, SameldaError)(msg)

    def set_stream(self, stream_handle: int):
        """Run on a caller's cudaStream_t handle (0 = the legacy default stream,
        which is torch's default stream)."""
        self.check(self.lib.samelda_cu_set_stream(self.h, C.c_void_p(int(stream_handle))))

    def set_eval_exact(self, exact: bool = True):
        """Held-out evaluation in the reference's summation order (bit-identical
        ll, ~10x slower) instead of the default tree-ordered fold-in (1e-12)."""
        self.check(self.lib.samelda_cu_set_eval_exact(self.h, int(bool(exact))))

    def use_own_stream(self):
        self.check(self.lib.samelda_cu_use_own_stream(self.h))

    def synchronize(self):
        self.check(self.lib.samelda_cu_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(self.lib.samelda_cu_launch_count(self.h))


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _f64(a):
    return np.ascontiguousarray(a, np.float64)


def _ids(doc_ids):
    ids = np.ascontiguousarray(doc_ids, np.int32)
    return ids if len(ids) else np.zeros(1, np.int32), len(ids)


# --------------------------------------------------------------- per-call API

def sddmm(theta_batch, phi, corpus, doc_ids, n_threads: int = 1, ctx: Context | None = None):
    """sampler.cpp:88-123 on the device; returns mu aligned with the batch nonzeros."""
    ctx = ctx or default_context()
    ctx._train_token = None  # per-call use replaces a Trainer's device state
    corpus = Corpus.of(corpus)
    theta_batch = _f64(theta_batch)
    phi = _f64(phi)
    ids, B = _ids(doc_ids)
    K, W = phi.shape
    Kt = theta_batch.shape[1] if theta_batch.ndim == 2 else K
    if theta_batch.shape[0] != B if theta_batch.ndim == 2 else B != 0:
        raise ConfigError("sddmm: theta rows must match the batch size")
    nnz = int((corpus.doc_offsets[ids[:B].astype(np.int64) + 1] -
               corpus.doc_offsets[ids[:B].astype(np.int64)]).sum()) if B else 0
    mu = np.zeros(max(nnz, 1))
    n = C.c_int64()
    cs = corpus._struct()
    tb = theta_batch if theta_batch.size else np.zeros(1)
    ctx.check(ctx.lib.samelda_cu_sddmm(ctx.h, C.byref(cs), _ptr(tb), B, Kt, _ptr(phi), K, W,
                                       _ptr(ids), _ptr(mu), len(mu), C.byref(n)))
    return mu[:n.value]


def sample_counts(theta_batch, phi, mu, corpus, doc_ids, m_t, seed, t, sweep=0, n_threads=1,
                  ctx: Context | None = None, mode: int = MODE_PARITY) -> SampledCounts:
    """sampler.cpp:125-195 on the device: reference-identical Poisson replicas
    (MODE_PARITY), or the same law on this library's own f32 streams
    (MODE_THROUGHPUT), or the c m_t replicas of each nonzero drawn jointly as
    a multinomial (MODE_MULTINOMIAL); mu is then only checked for alignment."""
    if mode not in (MODE_PARITY, MODE_THROUGHPUT, MODE_MULTINOMIAL):
        raise ConfigError("sample_counts: mode must be MODE_PARITY, MODE_THROUGHPUT or MODE_MULTINOMIAL")
    ctx = ctx or default_context()
    ctx._train_token = None  # per-call use replaces a Trainer's device state
    corpus = Corpus.of(corpus)
    theta_batch = _f64(theta_batch)
    phi = _f64(phi)
    mu = _f64(mu)
    ids, B = _ids(doc_ids)
    K, W = phi.shape
    Kt = theta_batch.shape[1] if theta_batch.ndim == 2 and theta_batch.size else K
    tc = np.zeros(max(B * K, 1), np.int64)
    pc = np.zeros(max(W * K, 1), np.int64)
    cs = corpus._struct()
    fn = {MODE_PARITY: ctx.lib.samelda_cu_sample_counts,
          MODE_THROUGHPUT: ctx.lib.samelda_cu_sample_counts_fast,
          MODE_MULTINOMIAL: ctx.lib.samelda_cu_sample_counts_multinomial}[mode]
    ctx.check(fn(
        ctx.h, C.byref(cs), _ptr(theta_batch if theta_batch.size else np.zeros(1)), B, Kt,
        _ptr(phi), K, W, _ptr(mu if len(mu) else np.zeros(1)), len(mu), _ptr(ids), float(m_t),
        int(seed) & (2**64 - 1), int(t), int(sweep), _ptr(tc), _ptr(pc)))
    return SampledCounts(ids[:B].copy(), K, W, float(m_t), tc[:B * K].reshape(B, K),
                         pc[:W * K].reshape(W, K))


def sample_theta_counts_fast(theta_batch, phi, corpus, doc_ids, m_t, seed, t, sweep,
                             ctx: Context | None = None):
    """The throughput mode's non-final inner sweep (theta counts only, B x K
    int64): one Poisson draw per (document, topic) of the summed rate
    theta_bk sum_w (m_t c_w / mu_w) phi_wk -- the law of the sum of the
    per-(nonzero, topic) draws (samelda_cu_sample_theta_counts_fast)."""
    ctx = ctx or default_context()
    ctx._train_token = None  # per-call use replaces a Trainer's device state
    corpus = Corpus.of(corpus)
    theta_batch = _f64(theta_batch)
    phi = _f64(phi)
    ids, B = _ids(doc_ids)
    K, W = phi.shape
    Kt = theta_batch.shape[1] if theta_batch.ndim == 2 and theta_batch.size else K
    tc = np.zeros(max(B * K, 1), np.int64)
    cs = corpus._struct()
    ctx.check(ctx.lib.samelda_cu_sample_theta_counts_fast(
        ctx.h, C.byref(cs), _ptr(theta_batch if theta_batch.size else np.zeros(1)), B, Kt,
        _ptr(phi), K, W, _ptr(ids), float(m_t), int(seed) & (2**64 - 1), int(t), int(sweep),
        _ptr(tc)))
    return tc[:B * K].reshape(B, K)


def expected_counts(theta_batch, phi, mu, corpus, doc_ids, m_t, ctx: Context | None = None):
    """Deterministic factored path: (theta_expected B x K, phi_expected W x K), f64."""
    ctx = ctx or default_context()
    ctx._train_token = None  # per-call use replaces a Trainer's device state
    corpus = Corpus.of(corpus)
    theta_batch = _f64(theta_batch)
    phi = _f64(phi)
    mu = _f64(mu)
    ids, B = _ids(doc_ids)
    K, W = phi.shape
    tf = np.zeros(max(B * K, 1))
    pf = np.zeros(max(W * K, 1))
    cs = corpus._struct()
    ctx.check(ctx.lib.samelda_cu_expected_counts(
        ctx.h, C.byref(cs), _ptr(theta_batch if theta_batch.size else np.zeros(1)), B,
        theta_batch.shape[1] if theta_batch.size else K, _ptr(phi), K, W,
        _ptr(mu if len(mu) else np.zeros(1)), len(mu), _ptr(ids), float(m_t), _ptr(tf),
        _ptr(pf)))
    return tf[:B * K].reshape(B, K), pf[:W * K].reshape(W, K)


def update_model(model: Model, counts, rho_t: float, ctx: Context | None = None,
                 expected: bool = False) -> None:
    """sampler.cpp:197-229 on the device; updates model.theta / model.phi in place."""
    ctx = ctx or default_context()
    ctx._train_token = None  # per-call use replaces a Trainer's device state
    if counts.n_topics != model.n_topics or counts.n_words != model.n_words:
        raise ConfigError("update_model: counts are not shaped for this model")
    model.theta = _f64(model.theta)
    model.phi = _f64(model.phi)
    ids, B = _ids(counts.doc_ids)
    fn = ctx.lib.samelda_cu_update_model_expected if expected else ctx.lib.samelda_cu_update_model
    dt = np.float64 if expected else np.int64
    tc = np.ascontiguousarray(counts.theta_counts, dt).reshape(-1)
    pc = np.ascontiguousarray(counts.phi_counts, dt).reshape(-1)
    ctx.check(fn(ctx.h, _ptr(model.theta), model.theta.shape[0], _ptr(model.phi),
                 model.n_topics, model.n_words, float(model.alpha), float(model.beta), _ptr(ids),
                 B, _ptr(tc if len(tc) else np.zeros(1, dt)), _ptr(pc if len(pc) else
                                                                    np.zeros(1, dt)),
                 float(counts.m_t), float(rho_t)))


def rho_schedule(t: int, tau0: float, gamma: float) -> float:
    out = C.c_double()
    rc = load_library().samelda_cu_rho_schedule(int(t), float(tau0), float(gamma), C.byref(out))
    if rc:
        raise _CODES[rc]("rho_schedule: argument out of range")
    return out.value


def anneal_m(schedule, t: int, t_max: int, m: float) -> float:
    s = SCHEDULES[schedule] if isinstance(schedule, str) else int(schedule)
    out = C.c_double()
    rc = load_library().samelda_cu_anneal_m(s, int(t), int(t_max), float(m), C.byref(out))
    if rc:
        raise _CODES[rc]("anneal_m: t must be in [1, t_max]")
    return out.value


def parse_schedule(name: str) -> str:
    if name not in SCHEDULES:
        raise ConfigError(f"unknown schedule '{name}' (expected constant|linear|log|invlinear)")
    return name


def fold_in_theta(phi, words, counts, alpha, sweeps=50, ctx: Context | None = None):
    """eval.cpp:19-73 on the device."""
    ctx = ctx or default_context()
    ctx._train_token = None  # per-call use replaces a Trainer's device state
    phi = _f64(phi)
    K, W = phi.shape
    w = np.ascontiguousarray(words, np.int32)
    c = np.ascontiguousarray(counts, np.int32)
    out = np.zeros(K)
    ctx.check(ctx.lib.samelda_cu_fold_in_theta(
        ctx.h, _ptr(phi), K, W, _ptr(w if len(w) else np.zeros(1, np.int32)),
        _ptr(c if len(c) else np.zeros(1, np.int32)), len(w), float(alpha), int(sweeps),
        _ptr(out)))
    return out


def perword_loglik(phi, test_corpus, alpha, seed, n_threads=1, ctx: Context | None = None):
    """eval.cpp:75-159 on the device: held-out per-word log-likelihood (nats)."""
    ctx = ctx or default_context()
    ctx._train_token = None  # per-call use replaces a Trainer's device state
    phi = _f64(phi)
    K, W = phi.shape
    test = Corpus.of(test_corpus)
    out = C.c_double()
    cs = test._struct()
    ctx.check(ctx.lib.samelda_cu_perword_loglik(ctx.h, _ptr(phi), K, W, C.byref(cs),
                                                float(alpha), int(seed) & (2**64 - 1),
                                                C.byref(out)))
    return out.value


# ----------------------------------------------------------------- trainer

class MinibatchStream:
    """corpus.cpp:252-285 (host, same Philox streams as the reference)."""

    def __init__(self, n_docs: int, batch_fraction: float, seed: int):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.samelda_cu_batches_create(int(n_docs), float(batch_fraction),
                                                int(seed) & (2**64 - 1), C.byref(h))
        if rc:
            raise ConfigError("minibatch_stream: batch_fraction must be in (0,1]")
        self.h = h
        self.batch_size = int(self.lib.samelda_cu_batches_size(h))
        self._buf = np.zeros(max(self.batch_size, 1), np.int32)

    def batches_per_pass(self) -> int:
        return int(self.lib.samelda_cu_batches_per_pass(self.h))

    def next(self) -> np.ndarray:
        n = self.lib.samelda_cu_batches_next(self.h, _ptr(self._buf))
        return self._buf[:n].copy()

    def __del__(self):
        try:
            self.lib.samelda_cu_batches_destroy(self.h)
        except Exception:
            pass


class Trainer:
    """Device-resident train() split at the period (sampler.cpp:269-353)."""

    def __init__(self, corpus, config: SamplerConfig, ctx: Context | None = None):
        # The training state (model, batch, counts) lives in the device
        # context, so a Trainer gets a context of its own unless one is passed;
        # a context re-initialised by another Trainer or train() makes this
        # Trainer's calls raise instead of silently using the other's state.
        self.ctx = ctx if ctx is not None else Context(0)
        self.corpus = Corpus.of(corpus)
        self.config = config
        self._cs = self.corpus._struct()
        self._cfg = config._struct()
        self._token = object()
        self.ctx._train_token = self._token
        self.ctx.check(self.ctx.lib.samelda_cu_train_begin(self.ctx.h, C.byref(self._cs),
                                                           C.byref(self._cfg)))

    def _live(self) -> Context:
        if getattr(self.ctx, "_train_token", None) is not self._token:
            raise ConfigError("Trainer: its context was re-initialised by another Trainer or "
                              "train(); use one Trainer per Context")
        return self.ctx

    def set_heldout(self, heldout, seed: int | None = None):
        self.heldout = Corpus.of(heldout)
        self._hs = self.heldout._struct()
        c = self._live()
        c.check(c.lib.samelda_cu_heldout(
            c.h, C.byref(self._hs),
            int(self.config.seed if seed is None else seed) & (2**64 - 1)))

    def period(self, doc_ids, t, m_t, rho_t):
        ids, B = _ids(doc_ids)
        c = self._live()
        c.check(c.lib.samelda_cu_period(c.h, _ptr(ids), B, int(t), float(m_t), float(rho_t)))

    def period_sample(self, doc_ids, t, m_t):
        ids, B = _ids(doc_ids)
        c = self._live()
        c.check(c.lib.samelda_cu_period_sample(c.h, _ptr(ids), B, int(t), float(m_t)))

    def period_update(self, rho_t):
        c = self._live()
        c.check(c.lib.samelda_cu_period_update(c.h, float(rho_t)))

    def phi_counts_device(self):
        """(device pointer, n elements, element bytes, is_float) of the phi count buffer."""
        p, n, eb, fl = C.c_void_p(), C.c_int64(), C.c_int32(), C.c_int32()
        c = self._live()
        c.check(c.lib.samelda_cu_phi_counts_device(
            c.h, C.byref(p), C.byref(n), C.byref(eb), C.byref(fl)))
        return p.value, n.value, eb.value, bool(fl.value)

    def phi_counts_pack32(self, lo_ptr: int, n: int, world_size: int, n_over_ptr: int):
        """Pack the u64 phi counts into the int32 device buffer at lo_ptr (exact
        below (2^31 - 1) / world_size; the count of cells at or above it goes to
        the u64 device word at n_over_ptr), on the context's stream."""
        c = self._live()
        c.check(c.lib.samelda_cu_phi_counts_pack32(c.h, C.c_void_p(lo_ptr), int(n), int(world_size),
                                                   C.c_void_p(n_over_ptr)))

    def phi_counts_unpack32(self, lo_ptr: int, n: int):
        """Write the (all-reduced) int32 counts at lo_ptr back into the u64 phi counts."""
        c = self._live()
        c.check(c.lib.samelda_cu_phi_counts_unpack32(c.h, C.c_void_p(lo_ptr), int(n)))

    def set_doc_base(self, base: int):
        c = self._live()
        c.check(c.lib.samelda_cu_set_doc_base(c.h, int(base)))

    def profile(self, enable: bool = True):
        c = self._live()
        c.check(c.lib.samelda_cu_profile(c.h, 1 if enable else 0))

    def profile_read(self) -> dict:
        ms = np.zeros(4)
        n = np.zeros(4, np.int64)
        nnz, docs, dfr = C.c_int64(), C.c_int64(), C.c_int64()
        c = self._live()
        c.check(c.lib.samelda_cu_profile_read(c.h, _ptr(ms), _ptr(n), C.byref(nnz),
                                              C.byref(docs), C.byref(dfr)))
        # nnz / docs count every timed sampling launch (both kinds)
        return dict(sample_ms=ms[0] + ms[3], sddmm_ms=ms[1], mstep_ms=ms[2],
                    sample_launches=int(n[0] + n[3]), sddmm_launches=int(n[1]),
                    mstep_launches=int(n[2]), sample_first_ms=ms[0], sample_first_launches=int(n[0]),
                    sample_last_ms=ms[3], sample_last_launches=int(n[3]), nnz=nnz.value,
                    docs=docs.value, deferred=dfr.value)

    def count_totals(self):
        a, b = C.c_int64(), C.c_int64()
        c = self._live()
        c.check(c.lib.samelda_cu_count_totals(c.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def batch_theta(self, B: int) -> np.ndarray:
        out = np.zeros(max(B * self.config.n_topics, 1))
        c = self._live()
        c.check(c.lib.samelda_cu_batch_theta(c.h, _ptr(out), len(out)))
        return out[:B * self.config.n_topics].reshape(B, self.config.n_topics)

    def batch_theta_async(self, B: int, out: np.ndarray) -> np.ndarray:
        """Enqueue the copy of the batch theta rows into `out` (float64,
        >= B * K elements, page-locked to overlap later periods) without a
        host wait; the rows are there after ctx.synchronize()."""
        if out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("batch_theta_async: out must be a contiguous float64 array")
        c = self._live()
        c.check(c.lib.samelda_cu_batch_theta_async(c.h, _ptr(out), out.size))
        return out[:B * self.config.n_topics].reshape(B, self.config.n_topics)

    def evaluate(self) -> float:
        out = C.c_double()
        c = self._live()
        c.check(c.lib.samelda_cu_evaluate(c.h, C.byref(out)))
        return out.value

    def model(self, with_theta: bool = True) -> Model:
        K, W, D = self.config.n_topics, self.corpus.n_words, self.corpus.n_docs
        phi = np.zeros(K * W)
        theta = np.zeros(D * K) if with_theta else None
        c = self._live()
        c.check(c.lib.samelda_cu_model_download(c.h, _ptr(phi), _ptr(theta)))
        return Model(K, W, self.config.alpha, self.config.beta, phi.reshape(K, W),
                     theta.reshape(D, K) if theta is not None else None)


def train(corpus, config: SamplerConfig, heldout=None, eval_every: int = 0,
          ctx: Context | None = None):
    """sampler.cpp:269-353 end to end on the device -> (Model, trace rows)."""
    ctx = ctx or default_context()
    ctx._train_token = None  # per-call use replaces a Trainer's device state
    corpus = Corpus.of(corpus)
    cs = corpus._struct()
    cfg = config._struct()
    hs = Corpus.of(heldout)._struct() if heldout is not None else None
    K, W, D = config.n_topics, corpus.n_words, corpus.n_docs
    phi = np.zeros(max(K * W, 1))
    theta = np.zeros(max(D * K, 1))
    cap = max(int(config.t_max), 1)
    rows = (_TraceRow * cap)()
    n = C.c_int64()
    ctx.check(ctx.lib.samelda_cu_train(ctx.h, C.byref(cs), C.byref(cfg),
                                       C.byref(hs) if hs is not None else None, int(eval_every),
                                       _ptr(phi), _ptr(theta), rows, cap, C.byref(n)))
    trace = [dict(t=rows[i].t, passes=rows[i].passes, samples_per_word=rows[i].samples_per_word,
                  ll=rows[i].ll, wall_seconds=rows[i].wall_seconds, m_t=rows[i].m_t)
             for i in range(n.value)]
    return Model(K, W, config.alpha, config.beta, phi[:K * W].reshape(K, W),
                 theta[:D * K].reshape(D, K)), trace


class Cgs:
    """The collapsed Gibbs sampler baseline (cgs.hpp:17-49) on the device: the
    reference's chain, draw for draw.  State lives in the
    context; `state()` returns CgsState's arrays."""

    def __init__(self, corpus, n_topics: int, alpha: float, beta: float, seed: int,
                 ctx: Context | None = None):
        self.ctx = ctx if ctx is not None else Context(0)
        self.corpus = Corpus.of(corpus)
        self.K = int(n_topics)
        self._cs = self.corpus._struct()
        self.ctx.check(self.ctx.lib.samelda_cu_cgs_init(self.ctx.h, C.byref(self._cs), self.K,
                                                        float(alpha), float(beta), int(seed)))

    def sweep(self, seed: int, sweep_index: int):
        self.ctx.check(self.ctx.lib.samelda_cu_cgs_sweep(self.ctx.h, int(seed), int(sweep_index)))

    def state(self):
        """(z, doc_topic D x K, word_topic W x K, topic_total K)"""
        c, K = self.corpus, self.K
        z = np.zeros(max(c.n_tokens, 1), np.int32)
        dt = np.zeros(max(c.n_docs * K, 1), np.int32)
        wt = np.zeros(max(c.n_words * K, 1), np.int32)
        tt = np.zeros(K, np.int64)
        self.ctx.check(self.ctx.lib.samelda_cu_cgs_state(self.ctx.h, _ptr(z), _ptr(dt), _ptr(wt),
                                                         _ptr(tt)))
        return (z[:c.n_tokens], dt[:c.n_docs * K].reshape(c.n_docs, K),
                wt[:c.n_words * K].reshape(c.n_words, K), tt)

    def model(self):
        """cgs_model (cgs.cpp:100-129) -> (phi K x W, theta D x K)"""
        c, K = self.corpus, self.K
        phi = np.zeros(max(K * c.n_words, 1))
        theta = np.zeros(max(c.n_docs * K, 1))
        self.ctx.check(self.ctx.lib.samelda_cu_cgs_model(self.ctx.h, _ptr(phi), _ptr(theta)))
        return phi[:K * c.n_words].reshape(K, c.n_words), theta[:c.n_docs * K].reshape(c.n_docs, K)


def cgs_train(corpus, n_topics: int, alpha: float, beta: float, n_sweeps: int, seed: int,
              eval_every: int = 0, heldout=None, ctx: Context | None = None):
    """cgs.cpp:131-157 on the device -> (Model, trace rows)."""
    ctx = ctx or default_context()
    ctx._train_token = None
    corpus = Corpus.of(corpus)
    cs = corpus._struct()
    hs = Corpus.of(heldout)._struct() if heldout is not None else None
    K, W, D = int(n_topics), corpus.n_words, corpus.n_docs
    phi = np.zeros(max(K * W, 1))
    theta = np.zeros(max(D * K, 1))
    cap = max(int(n_sweeps), 1)
    rows = (_TraceRow * cap)()
    n = C.c_int64()
    ctx.check(ctx.lib.samelda_cu_cgs_train(ctx.h, C.byref(cs), K, float(alpha), float(beta),
                                           int(n_sweeps), int(seed), int(eval_every),
                                           C.byref(hs) if hs is not None else None, _ptr(phi),
                                           _ptr(theta), rows, cap, C.byref(n)))
    trace = [dict(t=rows[i].t, passes=rows[i].passes, samples_per_word=rows[i].samples_per_word,
                  ll=rows[i].ll, wall_seconds=rows[i].wall_seconds, m_t=rows[i].m_t)
             for i in range(n.value)]
    return Model(K, W, alpha, beta, phi[:K * W].reshape(K, W), theta[:D * K].reshape(D, K)), trace


class Group:
    """One process driving several GPUs (samelda_cu_group_*): documents sharded in
    contiguous nnz-balanced ranges, the W x K counts summed over the devices with
    NCCL once per period, the M-step replicated.  A list repeating one device is the
    one-GPU test mode (device-side sum instead of NCCL)."""

    def __init__(self, devices):
        self.lib = load_library()
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        rc = self.lib.samelda_cu_group_create(devs, len(devices), C.byref(h))
        if rc:
            raise _CODES.get(rc, SameldaError)(f"samelda_cu_group_create({list(devices)}) failed "
                                               f"with code {rc}")
        self.h = h
        self.devices = list(devices)

    def close(self):
        if getattr(self, "h", None):
            self.lib.samelda_cu_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc:
            msg = self.lib.samelda_cu_group_last_error(self.h).decode(errors="replace")
            raise _CODES.get(rc, SameldaError)(msg)

    @property
    def uses_nccl(self) -> bool:
        return bool(self.lib.samelda_cu_group_uses_nccl(self.h))

    def train(self, corpus, config: SamplerConfig, heldout=None, eval_every: int = 0):
        """sampler.cpp:269-353 over the group -> (Model, trace rows)."""
        corpus = Corpus.of(corpus)
        cs, cfg = corpus._struct(), config._struct()
        hs = Corpus.of(heldout)._struct() if heldout is not None else None
        K, W, D = config.n_topics, corpus.n_words, corpus.n_docs
        phi = np.zeros(max(K * W, 1))
        theta = np.zeros(max(D * K, 1))
        cap = max(int(config.t_max), 1)
        rows = (_TraceRow * cap)()
        n = C.c_int64()
        self.check(self.lib.samelda_cu_group_train(self.h, C.byref(cs), C.byref(cfg),
                                                   C.byref(hs) if hs is not None else None,
                                                   int(eval_every), _ptr(phi), _ptr(theta), rows,
                                                   cap, C.byref(n)))
        trace = [dict(t=rows[i].t, passes=rows[i].passes,
                      samples_per_word=rows[i].samples_per_word, ll=rows[i].ll,
                      wall_seconds=rows[i].wall_seconds, m_t=rows[i].m_t) for i in range(n.value)]
        return Model(K, W, config.alpha, config.beta, phi[:K * W].reshape(K, W),
                     theta[:D * K].reshape(D, K)), trace


# ------------------------------------------------------------ data formats
# corpus ingest, binary CSR cache, checkpoint and metrics files
# (include/samelda_io.h)

def _io_check(rc: int):
    if rc:
        lib = load_library()
        msg = (lib.samelda_io_last_error() or b"").decode(errors="replace")
        raise _CODES.get(rc, SameldaError)(msg)


def _enc(path) -> bytes:
    return os.fsencode(os.fspath(path))


def _vocab_bytes(vocab, n_words: int) -> bytes:
    if vocab is None:
        vocab = [str(i) for i in range(n_words)]
    return "".join(v + "\n" for v in vocab).encode("utf-8", "surrogateescape")


def _take_io_corpus(h) -> Corpus:
    lib = load_library()
    try:
        d, w, nnz, tok, vb, dropped = (C.c_int64() for _ in range(6))
        lib.samelda_io_corpus_dims(h, C.byref(d), C.byref(w), C.byref(nnz), C.byref(tok),
                                   C.byref(vb), C.byref(dropped))
        view = _Corpus()
        vptr = C.c_void_p()
        lib.samelda_io_corpus_view(h, C.byref(view), C.byref(vptr))
        off = np.ctypeslib.as_array(C.cast(view.doc_offsets, C.POINTER(C.c_int64)),
                                    (d.value + 1,)).copy()
        if nnz.value:
            wid = np.ctypeslib.as_array(C.cast(view.word_ids, C.POINTER(C.c_int32)),
                                        (nnz.value,)).copy()
            cnt = np.ctypeslib.as_array(C.cast(view.counts, C.POINTER(C.c_int32)),
                                        (nnz.value,)).copy()
        else:
            wid = np.zeros(0, np.int32)
            cnt = np.zeros(0, np.int32)
        raw = C.string_at(vptr, vb.value) if vb.value else b""
        vocab = raw.decode("utf-8", "surrogateescape").split("\n")[:-1]
        return Corpus(off, wid, cnt, int(w.value), vocab)
    finally:
        lib.samelda_io_corpus_free(h)


def load_uci_bow(docword_path, vocab_path, n_threads: int = 0) -> Corpus:
    """corpus.cpp:62-183 (parallel mmap parser; same result and IoErrors)."""
    h = C.c_void_p()
    _io_check(load_library().samelda_io_load_uci(_enc(docword_path), _enc(vocab_path),
                                                 int(n_threads), C.byref(h)))
    return _take_io_corpus(h)


def save_uci_bow(corpus, docword_path, vocab_path) -> None:
    """corpus.cpp:186-213 (same bytes)."""
    c = Corpus.of(corpus)
    vb = _vocab_bytes(c.vocab, c.n_words)
    s = c._struct()
    _io_check(load_library().samelda_io_save_uci(C.byref(s), vb, len(vb), _enc(docword_path),
                                                 _enc(vocab_path)))


def save_corpus_cache(corpus, path) -> None:
    """Binary CSR cache (header + offsets + word ids + counts + vocab)."""
    c = Corpus.of(corpus)
    vb = _vocab_bytes(c.vocab, c.n_words)
    s = c._struct()
    _io_check(load_library().samelda_io_save_csr(_enc(path), C.byref(s), vb, len(vb)))


def load_corpus_cache(path, n_threads: int = 0) -> Corpus:
    h = C.c_void_p()
    _io_check(load_library().samelda_io_load_csr(_enc(path), int(n_threads), C.byref(h)))
    return _take_io_corpus(h)


def save_checkpoint(model: Model, path) -> None:
    """model.cpp:54-69 (same bytes; phi K x W)."""
    phi = np.ascontiguousarray(model.phi, np.float64)
    _io_check(load_library().samelda_io_save_checkpoint(
        _enc(path), int(model.n_topics), int(model.n_words), float(model.alpha),
        float(model.beta), _ptr(phi)))


def load_checkpoint(path) -> Model:
    """model.cpp:71-111 (same checks and IoErrors); theta is not stored."""
    lib = load_library()
    k, w, a, b = C.c_int64(), C.c_int64(), C.c_double(), C.c_double()
    _io_check(lib.samelda_io_checkpoint_header(_enc(path), C.byref(k), C.byref(w), C.byref(a),
                                               C.byref(b)))
    phi = np.zeros((k.value, w.value))
    _io_check(lib.samelda_io_load_checkpoint(_enc(path), _ptr(phi), phi.size))
    return Model(int(k.value), int(w.value), a.value, b.value, phi, None)


def write_metrics_csv(trace, path) -> None:
    """eval.cpp:161-177 (same bytes)."""
    rows = (_TraceRow * max(len(trace), 1))()
    for i, r in enumerate(trace):
        rows[i] = _TraceRow(int(r["t"]), float(r["passes"]), float(r["samples_per_word"]),
                            float(r["ll"]), float(r["wall_seconds"]), float(r["m_t"]))
    _io_check(load_library().samelda_io_write_metrics_csv(_enc(path), rows, len(trace)))


def read_metrics_csv(path) -> list:
    """eval.cpp:179-208."""
    lib = load_library()
    n = C.c_int64()
    _io_check(lib.samelda_io_read_metrics_csv(_enc(path), None, 0, C.byref(n)))
    rows = (_TraceRow * max(n.value, 1))()
    _io_check(lib.samelda_io_read_metrics_csv(_enc(path), rows, n.value, C.byref(n)))
    return [dict(t=rows[i].t, passes=rows[i].passes, samples_per_word=rows[i].samples_per_word,
                 ll=rows[i].ll, wall_seconds=rows[i].wall_seconds, m_t=rows[i].m_t)
            for i in range(n.value)]
