// capi.cu -- libsamelda_cuda.so: device context and the C ABI of include/samelda_cu.h.
//
// Host-side logic here mirrors the reference's host code exactly where it
// feeds the hot path (MinibatchStream corpus.cpp:252-285, anneal_m /
// rho_schedule sampler.cpp:231-267, the train() period loop and its trace
// bookkeeping sampler.cpp:269-353); every arithmetic step of the hot path
// itself runs in the kernels of kernels_{sample,mstep,eval}.cu.  There is no CPU fallback: a
// missing device is an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler attaches

#include "../../include/samelda_cu.h"
#include "kernels.cuh"
#include "philox.cuh"

namespace {

constexpr int kVersion = 1;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw Fail{code, buf};
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(SAMELDA_CU_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

template <class T>
T* ensure(DevBuf& b, int64_t n) {
  const size_t need = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T);
  if (b.bytes < need) {
    if (b.p) ck(cudaFree(b.p), "cudaFree");
    b.p = nullptr;
    b.bytes = 0;
    ck(cudaMalloc(&b.p, need), "cudaMalloc");
    b.bytes = need;
  }
  return static_cast<T*>(b.p);
}

// Resident CSR corpus with a cheap identity check: the per-call API receives
// an arbitrary corpus every call (sampler.hpp:74-91), so the slot re-uploads
// only when pointers, sizes or a content fingerprint change.
struct CorpusSlot {
  bool valid = false;
  uint64_t fp = 0;
  int64_t n_docs = 0, n_words = 0, nnz = 0, n_tokens = 0;
  std::vector<int64_t> offsets;     // host copy (batch prefixes)
  std::vector<int64_t> doc_tokens;  // Corpus::doc_tokens (corpus.cpp:16-23)
  DevBuf offs, words, counts;
};

// Content hash of a byte range: four independent 64-bit multiply-xor lanes
// over 32-byte strides (several GB/s per thread), folded at the end.
uint64_t hash_range(const void* data, size_t bytes, uint64_t seed) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h[4] = {seed ^ 0x9E3779B97F4A7C15ull, seed ^ 0xC2B2AE3D27D4EB4Full,
                   seed ^ 0x165667B19E3779F9ull, seed ^ 0x27D4EB2F165667C5ull};
  auto mix = [](uint64_t a, uint64_t v) {
    a ^= v * 0x9FB21C651E98DF25ull;
    a = (a << 29) | (a >> 35);
    return a * 0xC2B2AE3D27D4EB4Full;
  };
  size_t i = 0;
  for (; i + 32 <= bytes; i += 32) {
    uint64_t v[4];
    std::memcpy(v, p + i, 32);
    for (int j = 0; j < 4; ++j) h[j] = mix(h[j], v[j]);
  }
  uint64_t tail = bytes;
  for (; i < bytes; ++i) tail = (tail << 8 | p[i]) * 0x100000001B3ull;
  uint64_t r = mix(mix(mix(mix(h[0], h[1]), h[2]), h[3]), tail);
  r ^= r >> 31;
  return r * 0x9E3779B97F4A7C15ull;
}

// Hash of the whole byte range, split over host threads for large inputs
// (a corpus at NYTimes shape is ~0.5 GB: ~20 ms on 16 cores).
uint64_t hash_bytes(const void* data, size_t bytes, uint64_t seed) {
  constexpr size_t kPiece = size_t{32} << 20;
  const size_t pieces = (bytes + kPiece - 1) / kPiece;
  if (pieces <= 1) return hash_range(data, bytes, seed);
  std::vector<uint64_t> part(pieces);
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  std::atomic<size_t> next{0};
  for (unsigned t = 0; t < std::min<size_t>(hw, pieces); ++t)
    pool.emplace_back([&] {
      for (size_t i = next++; i < pieces; i = next++) {
        const size_t off = i * kPiece;
        part[i] = hash_range(static_cast<const unsigned char*>(data) + off,
                             std::min(kPiece, bytes - off), seed + i);
      }
    });
  for (auto& th : pool) th.join();
  return hash_range(part.data(), sizeof(uint64_t) * pieces, seed);
}

// Identity of a corpus: pointers, dimensions and a hash of ALL of its
// content (offsets, word ids, counts), so a corpus changed in place or a new
// one at reused addresses is re-uploaded like the reference re-reads it.
uint64_t fingerprint(const samelda_cu_corpus* c) {
  const int64_t nnz = c->doc_offsets[c->n_docs];
  const uint64_t head[6] = {reinterpret_cast<uintptr_t>(c->doc_offsets),
                            reinterpret_cast<uintptr_t>(c->word_ids),
                            reinterpret_cast<uintptr_t>(c->counts),
                            static_cast<uint64_t>(c->n_docs), static_cast<uint64_t>(c->n_words),
                            static_cast<uint64_t>(nnz)};
  uint64_t h = hash_range(head, sizeof(head), 1469598103934665603ull);
  h = hash_bytes(c->doc_offsets, sizeof(int64_t) * (c->n_docs + 1), h);
  if (nnz > 0) {
    h = hash_bytes(c->word_ids, sizeof(int32_t) * nnz, h);
    h = hash_bytes(c->counts, sizeof(int32_t) * nnz, h);
  }
  return h;
}

void validate_corpus(const samelda_cu_corpus* c) {
  if (c == nullptr || c->doc_offsets == nullptr) fail(SAMELDA_CU_CONFIG, "corpus is null");
  if (c->n_docs < 0 || c->n_words < 0) fail(SAMELDA_CU_CONFIG, "corpus dimensions negative");
  if (c->doc_offsets[0] != 0) fail(SAMELDA_CU_CONFIG, "corpus doc_offsets[0] != 0");
}

// Large copies between device memory and caller-owned (pageable) host
// buffers -- the corpus upload, the model download -- staged through two
// pinned 32 MB chunks: the DMA of one chunk overlaps the multi-threaded host
// memcpy of the other.  A pageable cudaMemcpy runs at ~5 GB/s on the B200
// boxes (the drop-in train()'s 824 MB model download took 160 ms).
struct PinnedStage {
  static constexpr size_t kChunk = size_t{32} << 20;
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool pending[2] = {false, false};
  void init() {
    if (buf[0]) return;
    for (int i = 0; i < 2; ++i) {
      ck(cudaHostAlloc(reinterpret_cast<void**>(&buf[i]), kChunk, cudaHostAllocDefault), "pinned stage");
      ck(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "stage event");
    }
  }
  ~PinnedStage() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) {
        cudaEventSynchronize(ev[i]);
        cudaEventDestroy(ev[i]);
      }
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
};

void par_memcpy(void* dst, const void* src, size_t n) {
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  if (n < (size_t{4} << 20) || hw == 1) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t per = (n + hw - 1) / hw;
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < hw; ++t) {
    const size_t off = per * t;
    if (off >= n) break;
    pool.emplace_back([=] {
      std::memcpy(static_cast<unsigned char*>(dst) + off, static_cast<const unsigned char*>(src) + off,
                  std::min(per, n - off));
    });
  }
  std::memcpy(dst, src, std::min(per, n));
  for (auto& th : pool) th.join();
}

constexpr size_t kStageMin = size_t{16} << 20;  // smaller copies go direct

// device -> pageable host; returns with the data in dst
void copy_d2h(PinnedStage* ps, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!ps || bytes < kStageMin) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "download");
    ck(cudaStreamSynchronize(st), "download");
    return;
  }
  ps->init();
  auto* d = static_cast<unsigned char*>(dst);
  const auto* sp = static_cast<const unsigned char*>(src);
  int prev = -1;
  size_t prev_off = 0, prev_n = 0;
  for (size_t off = 0, i = 0; off < bytes; off += PinnedStage::kChunk, ++i) {
    const int slot = static_cast<int>(i & 1);
    const size_t n = std::min(PinnedStage::kChunk, bytes - off);
    ck(cudaMemcpyAsync(ps->buf[slot], sp + off, n, cudaMemcpyDeviceToHost, st), "download");
    ck(cudaEventRecord(ps->ev[slot], st), "stage event");
    ps->pending[slot] = true;
    if (prev >= 0) {
      ck(cudaEventSynchronize(ps->ev[prev]), "download");
      par_memcpy(d + prev_off, ps->buf[prev], prev_n);
    }
    prev = slot;
    prev_off = off;
    prev_n = n;
  }
  ck(cudaEventSynchronize(ps->ev[prev]), "download");
  par_memcpy(d + prev_off, ps->buf[prev], prev_n);
}

// pageable host -> device, enqueued on st (the source may be reused on return)
void copy_h2d(PinnedStage* ps, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!ps || bytes < kStageMin) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "upload");
    return;
  }
  ps->init();
  auto* d = static_cast<unsigned char*>(dst);
  const auto* sp = static_cast<const unsigned char*>(src);
  for (size_t off = 0, i = 0; off < bytes; off += PinnedStage::kChunk, ++i) {
    const int slot = static_cast<int>(i & 1);
    const size_t n = std::min(PinnedStage::kChunk, bytes - off);
    if (ps->pending[slot]) ck(cudaEventSynchronize(ps->ev[slot]), "upload");
    par_memcpy(ps->buf[slot], sp + off, n);
    ck(cudaMemcpyAsync(d + off, ps->buf[slot], n, cudaMemcpyHostToDevice, st), "upload");
    ck(cudaEventRecord(ps->ev[slot], st), "stage event");
    ps->pending[slot] = true;
  }
}

void upload_corpus(CorpusSlot& s, const samelda_cu_corpus* c, cudaStream_t st,
                   PinnedStage* ps = nullptr) {
  validate_corpus(c);
  const int64_t nnz = c->doc_offsets[c->n_docs];
  const bool same_shape = s.valid && s.n_docs == c->n_docs && s.nnz == nnz && s.n_words == c->n_words;
  uint64_t fp = 0;
  std::thread fp_thread;
  if (same_shape) {
    fp = fingerprint(c);
    if (s.fp == fp) return;
  } else {
    // a new corpus: its identity hash runs beside the upload
    fp_thread = std::thread([&] { fp = fingerprint(c); });
  }
  struct Join {
    std::thread& t;
    ~Join() {
      if (t.joinable()) t.join();
    }
  } join{fp_thread};
  s.valid = false;
  s.n_docs = c->n_docs;
  s.n_words = c->n_words;
  s.nnz = nnz;
  s.offsets.assign(c->doc_offsets, c->doc_offsets + c->n_docs + 1);
  s.doc_tokens.assign(static_cast<size_t>(c->n_docs), 0);
  s.n_tokens = 0;
  {
    // per-document token totals, documents split over host threads
    const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const int64_t nt = nnz > (int64_t{1} << 22) ? hw : 1;
    std::vector<int64_t> part(static_cast<size_t>(nt), 0);
    auto run = [&](int64_t t) {
      const int64_t d0 = c->n_docs * t / nt, d1 = c->n_docs * (t + 1) / nt;
      int64_t sum = 0;
      for (int64_t d = d0; d < d1; ++d) {
        int64_t tok = 0;
        for (int64_t i = c->doc_offsets[d]; i < c->doc_offsets[d + 1]; ++i) tok += c->counts[i];
        s.doc_tokens[static_cast<size_t>(d)] = tok;
        sum += tok;
      }
      part[static_cast<size_t>(t)] = sum;
    };
    std::vector<std::thread> pool;
    for (int64_t t = 1; t < nt; ++t) pool.emplace_back(run, t);
    run(0);
    for (auto& th : pool) th.join();
    for (int64_t v : part) s.n_tokens += v;
  }
  copy_h2d(ps, ensure<int64_t>(s.offs, c->n_docs + 1), c->doc_offsets,
           sizeof(int64_t) * (c->n_docs + 1), st);
  if (nnz > 0) {
    copy_h2d(ps, ensure<int32_t>(s.words, nnz), c->word_ids, sizeof(int32_t) * nnz, st);
    copy_h2d(ps, ensure<int32_t>(s.counts, nnz), c->counts, sizeof(int32_t) * nnz, st);
  } else {
    ensure<int32_t>(s.words, 1);
    ensure<int32_t>(s.counts, 1);
  }
  ck(cudaStreamSynchronize(st), "corpus upload");
  if (fp_thread.joinable()) fp_thread.join();
  s.fp = fp;
  s.valid = true;
}

// Host MinibatchStream (corpus.cpp:252-285) on the same Philox streams.
struct Batches {
  int64_t n_docs = 0;
  uint64_t seed = 0;
  int64_t batch_size = 1;
  uint32_t pass = 0;
  int64_t cursor = 0;
  std::vector<int32_t> order;

  void start_pass() {
    scu::Stream s;
    s.init(seed, pass, 0, 0, scu::make_tag(scu::kBatchShuffle, 0, 0));
    order.resize(static_cast<size_t>(n_docs));
    for (int64_t i = 0; i < n_docs; ++i) order[static_cast<size_t>(i)] = static_cast<int32_t>(i);
    for (int64_t i = n_docs - 1; i > 0; --i) {
      const int64_t j = static_cast<int64_t>(s.uniform_below(static_cast<uint64_t>(i) + 1));
      std::swap(order[static_cast<size_t>(i)], order[static_cast<size_t>(j)]);
    }
    cursor = 0;
  }
  int64_t next(int32_t* out) {
    if (cursor >= n_docs) {
      ++pass;
      start_pass();
    }
    const int64_t take = std::min<int64_t>(batch_size, n_docs - cursor);
    std::memcpy(out, order.data() + cursor, sizeof(int32_t) * static_cast<size_t>(take));
    cursor += take;
    return take;
  }
  int64_t per_pass() const { return (n_docs + batch_size - 1) / batch_size; }
};

void validate_config(const samelda_cu_config* c) {
  // sampler.cpp:47-78
  if (c == nullptr) fail(SAMELDA_CU_CONFIG, "config is null");
  if (c->n_topics < 1 || c->n_topics >= (1 << 20)) fail(SAMELDA_CU_CONFIG, "n_topics must be in [1, 2^20)");
  if (!(c->m > 0.0) || !std::isfinite(c->m)) fail(SAMELDA_CU_CONFIG, "m must be positive and finite");
  if (!(c->tau0 >= 1.0)) fail(SAMELDA_CU_CONFIG, "tau0 must be >= 1");
  if (!(c->gamma >= 0.5 && c->gamma <= 1.0)) fail(SAMELDA_CU_CONFIG, "gamma must be in [0.5, 1]");
  if (!(c->batch_fraction > 0.0 && c->batch_fraction <= 1.0))
    fail(SAMELDA_CU_CONFIG, "batch_fraction must be in (0, 1]");
  if (c->t_max < 0) fail(SAMELDA_CU_CONFIG, "t_max must be >= 0");
  if (c->inner_sweeps < 1 || c->inner_sweeps > 255) fail(SAMELDA_CU_CONFIG, "inner_sweeps must be in [1, 255]");
  if (!(c->alpha > 0.0) || !(c->beta > 0.0)) fail(SAMELDA_CU_CONFIG, "alpha and beta must be positive");
  if (!(c->init_noise >= 0.0) || !std::isfinite(c->init_noise))
    fail(SAMELDA_CU_CONFIG, "init_noise must be finite and >= 0");
  if (c->mode != SAMELDA_CU_MODE_PARITY && c->mode != SAMELDA_CU_MODE_EXPECTED &&
      c->mode != SAMELDA_CU_MODE_THROUGHPUT && c->mode != SAMELDA_CU_MODE_MULTINOMIAL)
    fail(SAMELDA_CU_CONFIG, "unknown sampling mode %d", c->mode);
  if (c->mode == SAMELDA_CU_MODE_MULTINOMIAL && c->n_topics > 1024)
    fail(SAMELDA_CU_CONFIG, "multinomial mode supports n_topics <= 1024");
  if (c->schedule < 0 || c->schedule > 3) fail(SAMELDA_CU_CONFIG, "unknown schedule %d", c->schedule);
}

double rho_schedule_host(int64_t t, double tau0, double gamma) {
  // sampler.cpp:231-242
  if (t < 0) fail(SAMELDA_CU_CONFIG, "rho_schedule: t must be >= 0");
  if (!(tau0 >= 1.0)) fail(SAMELDA_CU_CONFIG, "rho_schedule: tau0 must be >= 1");
  if (!(gamma >= 0.5 && gamma <= 1.0)) fail(SAMELDA_CU_CONFIG, "rho_schedule: gamma must be in [0.5, 1]");
  return std::pow(tau0 + static_cast<double>(t), -gamma);
}

double anneal_m_host(int schedule, int64_t t, int64_t t_max, double m) {
  // sampler.cpp:244-267
  if (t < 1 || t > t_max) fail(SAMELDA_CU_CONFIG, "anneal_m: t must be in [1, t_max]");
  const double td = static_cast<double>(t);
  const double nd = static_cast<double>(t_max);
  switch (schedule) {
    case SAMELDA_CU_SCHEDULE_CONSTANT: return m;
    case SAMELDA_CU_SCHEDULE_LINEAR: return 2.0 * m * td / (nd + 1.0);
    case SAMELDA_CU_SCHEDULE_INVLINEAR: return 2.0 * m * (nd + 1.0 - td) / (nd + 1.0);
    case SAMELDA_CU_SCHEDULE_LOG: {
      if (t_max == 1) return m;
      const double value = m * nd * std::log(td) / std::lgamma(nd + 1.0);
      return std::max(value, 0.01);
    }
    default: fail(SAMELDA_CU_CONFIG, "anneal_m: unknown schedule");
  }
}

}  // namespace

namespace scu {
const Tuning& tuning() {
  static const Tuning t = [] {
    Tuning v;
    auto env = [](const char* n) { return std::getenv(n); };
    if (const char* e = env("SAMELDA_SAMPLER")) v.sampler_exact = e[0] == 'x';
    if (const char* e = env("SAMELDA_COLSUM")) v.colsum_chain = e[0] == 'c';
    if (const char* e = env("SAMELDA_DRAW_CAP")) v.draw_cap = std::atoll(e);
    if (const char* e = env("SAMELDA_EVAL")) v.eval_variant = e[0];
    if (env("SAMELDA_EVAL_WARP")) v.eval_variant = 'w';
    if (const char* e = env("SAMELDA_EVAL_CTAS_PER_SM")) v.eval_ctas_per_sm = std::atoi(e);

    if (const char* e = env("SAMELDA_MINB")) v.minb = std::atoi(e);
    if (const char* e = env("SAMELDA_DEC")) v.dec = std::atoi(e);
    if (const char* e = env("SAMELDA_TAIL")) v.tail = std::atoi(e);
    if (const char* e = env("SAMELDA_FAST_PTRS")) v.fast_ptrs = e[0] != '0';
    return v;
  }();
  return t;
}
}  // namespace scu

struct samelda_cu_ctx {
  int device = 0;
  PinnedStage pstage;  // staged copies of large caller buffers (destroyed last)
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string error;
  int64_t launches = 0;

  CorpusSlot train;    // corpus of the per-call API and of the resident trainer
  CorpusSlot heldout;  // test corpus of perword_loglik / evaluate
  uint64_t split_seed = 0;
  bool split_ready = false;
  DevBuf tok_offsets, slots, fold_counts, score_counts, doc_logp, doc_scored;
  // compacted fold / score cell lists of the split (k_eval_fold's input)
  DevBuf n_fold, fold_l, n_score, score_l;
  // held-out evaluation: false = k_eval_fold (ll within 1e-12
  // relative, tree-ordered sums); true = the reference's summation order bit
  // for bit (k_eval_stage / k_eval_cta / k_eval_docs, ~10x slower)
  bool eval_exact = false;

  // resident model (train_begin)
  bool model_ready = false;
  samelda_cu_config cfg{};
  int K = 0;
  int64_t W = 0, D = 0;
  DevBuf theta, phi;  // D x K, W x K (f64)
  DevBuf phi32;       // W x K f32 shadow of phi (sampler fast path)
  DevBuf colsum;      // exact parallel column-sum scan (partials, segment items)

  // doc-sharded runs: global id of local doc 0 (Philox keys use global ids)
  int64_t doc_base = 0;

  // collapsed Gibbs sampler state (cgs_* entry points; corpus in `train`)
  bool cgs_ready = false;
  int cgs_K = 0;
  double cgs_alpha = 0.0, cgs_beta = 0.0;
  int64_t cgs_tokens = 0;
  DevBuf cgs_tok, cgs_z, cgs_dt, cgs_wt, cgs_tt, cgs_phi;

  // optional per-kernel CUDA-event timing (bench roofline)
  bool profile = false;
  enum { kSample = 0, kSddmm = 1, kMstep = 2, kSampleLast = 3, kKinds = 4 };
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events[kKinds];
  size_t events_used[kKinds] = {0, 0, 0, 0};
  int64_t prof_nnz = 0, prof_docs = 0, prof_deferred = 0;

  // NVTX ranges around the sampling sweeps, the SDDMM and the M-step (every
  // call; the profiler timeline shows where each period's launches come from),
  // CUDA events only when profiling
  void tick(int kind, bool start) {
    static const char* const kNames[kKinds] = {"samelda:sample_sweep", "samelda:sddmm",
                                               "samelda:update_model", "samelda:sample_sweep_last"};
    if (start) nvtxRangePushA(kNames[kind]);
    else nvtxRangePop();
    if (!profile) return;
    auto& v = events[kind];
    size_t& used = events_used[kind];
    if (start) {
      if (used == v.size()) {
        cudaEvent_t a, b;
        ck(cudaEventCreate(&a), "event");
        ck(cudaEventCreate(&b), "event");
        v.emplace_back(a, b);
      }
      ck(cudaEventRecord(v[used].first, stream), "event record");
    } else {
      ck(cudaEventRecord(v[used].second, stream), "event record");
      ++used;
    }
  }

  // per-period state
  int64_t B = 0, nnzB = 0;
  double m_t = 1.0;
  bool counts_ready = false;
  bool counts_float = false;

  // scratch
  DevBuf batch, prefix, theta_batch, theta_batch32, mu, tc, pc, tf, pf, totals, err, ll,
      phi_call, phi_call_wk, phi_call32, theta_call, theta_call32, eval_scratch, theta_rows,
      deferred, n_deferred, cand, deferred_aux, mu_f32, rates32;
  // double-buffered pinned staging of batch ids / prefixes: the host may run
  // periods ahead of the device; a buffer is reused only after the copies of
  // two periods ago have executed (event)
  struct Staging {
    int32_t* batch = nullptr;
    int64_t* prefix = nullptr;
    int64_t cap = 0;
    cudaEvent_t done = nullptr;
  };
  Staging stg[2];
  int stg_next = 0;
  // batch-theta read-back (samelda_cu_batch_theta_async): the D2H copy runs
  // on its own stream so it overlaps the next period's kernels; two row
  // buffers, each reused only after its previous copy has finished
  // exact f64 mu on a side stream, concurrent with the fast sampler, once most
  // nonzeros carry deferred draws (a converged model: PTRS at every dominant
  // topic); the deferral rate is read back asynchronously, a sweep or more late
  cudaStream_t mu_stream = nullptr;
  cudaEvent_t mu_theta_ready = nullptr, mu_done = nullptr, defer_read = nullptr;
  unsigned long long* h_deferred = nullptr;
  int64_t defer_read_nnz = 0;
  bool defer_read_pending = false;
  double defer_frac = 0.0;
  static constexpr double kManyDeferred = 0.25;
  cudaStream_t copy_stream = nullptr;
  DevBuf rows2[2];
  cudaEvent_t rows_ready[2] = {nullptr, nullptr};
  cudaEvent_t rows_copied[2] = {nullptr, nullptr};
  int rows_next = 0;
  // sticky device error flag, read back asynchronously after each period
  int* h_err = nullptr;
  cudaEvent_t err_event = nullptr;
  bool err_pending = false;

  ~samelda_cu_ctx() {
    for (auto& v : events)
      for (auto& e : v) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
      }
    for (auto& sb : stg) {
      if (sb.batch) cudaFreeHost(sb.batch);
      if (sb.prefix) cudaFreeHost(sb.prefix);
      if (sb.done) cudaEventDestroy(sb.done);
    }
    if (h_err) cudaFreeHost(h_err);
    if (err_event) cudaEventDestroy(err_event);
    for (int i = 0; i < 2; ++i) {
      if (rows_ready[i]) cudaEventDestroy(rows_ready[i]);
      if (rows_copied[i]) cudaEventDestroy(rows_copied[i]);
    }
    if (copy_stream) {
      cudaStreamSynchronize(copy_stream);
      cudaStreamDestroy(copy_stream);
    }
    if (mu_stream) {
      cudaStreamSynchronize(mu_stream);
      cudaStreamDestroy(mu_stream);
      cudaEventDestroy(mu_theta_ready);
      cudaEventDestroy(mu_done);
    }
    if (h_deferred) {
      cudaEventSynchronize(defer_read);
      cudaEventDestroy(defer_read);
      cudaFreeHost(h_deferred);
    }
    if (own_stream) cudaStreamDestroy(own_stream);
  }

  int* d_err() {
    if (err.p == nullptr) {
      ensure<int>(err, 1);
      ck(cudaMemsetAsync(err.p, 0, sizeof(int), stream), "zero error flag");
    }
    return err.as<int>();
  }

  // enqueue the read-back of the sticky error flag (no host wait)
  void post_err_check() {
    if (h_err == nullptr) ck(cudaHostAlloc(&h_err, sizeof(int), cudaHostAllocDefault), "pinned err");
    if (err_event == nullptr) ck(cudaEventCreateWithFlags(&err_event, cudaEventDisableTiming), "err event");
    ck(cudaMemcpyAsync(h_err, d_err(), sizeof(int), cudaMemcpyDeviceToHost, stream), "read error flag");
    ck(cudaEventRecord(err_event, stream), "err event");
    err_pending = true;
  }

  // report a pending device error (NumericalError) once its read-back landed;
  // wait == true blocks for it
  void poll_err(bool wait, const char* what) {
    if (!err_pending) return;
    if (wait) {
      ck(cudaEventSynchronize(err_event), what);
    } else if (cudaEventQuery(err_event) == cudaErrorNotReady) {
      cudaGetLastError();
      return;
    }
    err_pending = false;
    if (*h_err & scu::kErrNumerical) {
      *h_err = 0;
      ck(cudaMemsetAsync(d_err(), 0, sizeof(int), stream), "reset error flag");
      fail(SAMELDA_CU_NUMERICAL, "%s: nonfinite or negative value (NumericalError)", what);
    }
  }

  void reset_err() {
    poll_err(true, "previous period");  // never clear an unreported device error
    ck(cudaMemsetAsync(d_err(), 0, sizeof(int), stream), "reset error flag");
  }

  void check_err(const char* what) {
    int h = 0;
    ck(cudaMemcpyAsync(&h, err.p, sizeof(int), cudaMemcpyDeviceToHost, stream), "read error flag");
    ck(cudaStreamSynchronize(stream), what);
    ck(cudaGetLastError(), what);
    if (h & scu::kErrNumerical) {
      // reported here, once: a stale flag must not surface as a later
      // period's error (the period path reads the same sticky flag)
      ck(cudaMemsetAsync(err.p, 0, sizeof(int), stream), "reset error flag");
      ck(cudaStreamSynchronize(stream), what);
      fail(SAMELDA_CU_NUMERICAL, "%s: nonfinite or negative value", what);
    }
  }

  Staging& stage(int64_t B_) {
    Staging& sb = stg[stg_next];
    stg_next ^= 1;
    if (sb.done) ck(cudaEventSynchronize(sb.done), "batch staging");
    else ck(cudaEventCreateWithFlags(&sb.done, cudaEventDisableTiming), "staging event");
    if (sb.cap < B_ + 1) {
      if (sb.batch) cudaFreeHost(sb.batch);
      if (sb.prefix) cudaFreeHost(sb.prefix);
      sb.cap = std::max<int64_t>(B_ + 1, 1024);
      ck(cudaHostAlloc(&sb.batch, sizeof(int32_t) * sb.cap, cudaHostAllocDefault), "pinned batch");
      ck(cudaHostAlloc(&sb.prefix, sizeof(int64_t) * sb.cap, cudaHostAllocDefault), "pinned prefix");
    }
    return sb;
  }

  // Upload a batch of doc ids of `slot` and its nonzero prefix (sampler.cpp:18-24).
  scu::BatchView upload_batch(const CorpusSlot& slot, const int32_t* doc_ids, int64_t B_) {
    Staging& sb = stage(B_);
    int32_t* h_batch = sb.batch;
    int64_t* h_prefix = sb.prefix;
    h_prefix[0] = 0;
    for (int64_t b = 0; b < B_; ++b) {
      const int32_t d = doc_ids[b];
      if (d < 0 || d >= slot.n_docs) fail(SAMELDA_CU_CONFIG, "batch doc id %d out of range", d);
      h_batch[b] = d;
      h_prefix[b + 1] = h_prefix[b] + (slot.offsets[static_cast<size_t>(d) + 1] -
                                       slot.offsets[static_cast<size_t>(d)]);
    }
    int32_t* db = ensure<int32_t>(batch, B_);
    int64_t* dp = ensure<int64_t>(prefix, B_ + 1);
    if (B_ > 0)
      ck(cudaMemcpyAsync(db, h_batch, sizeof(int32_t) * B_, cudaMemcpyHostToDevice, stream),
         "upload batch");
    ck(cudaMemcpyAsync(dp, h_prefix, sizeof(int64_t) * (B_ + 1), cudaMemcpyHostToDevice, stream),
       "upload prefix");
    ck(cudaEventRecord(sb.done, stream), "staging event");
    scu::BatchView bv;
    bv.doc_offsets = slot.offs.as<int64_t>();
    bv.word_ids = slot.words.as<int32_t>();
    bv.counts = slot.counts.as<int32_t>();
    bv.batch_docs = db;
    bv.batch_prefix = dp;
    bv.B = B_;
    bv.nnz = h_prefix[B_];
    bv.doc_base = 0;
    return bv;
  }

  // phi K x W host -> W x K device (per-call boundary), plus its f32 shadow
  double* upload_phi(const double* phi_kw, int64_t K_, int64_t W_, float** out32 = nullptr) {
    double* tmp = ensure<double>(phi_call, K_ * W_);
    double* out = ensure<double>(phi_call_wk, K_ * W_);
    if (K_ * W_ > 0) {
      ck(cudaMemcpyAsync(tmp, phi_kw, sizeof(double) * K_ * W_, cudaMemcpyHostToDevice, stream),
         "upload phi");
      launches += scu::launch_transpose(tmp, K_, W_, out, stream);
    }
    if (out32) {
      *out32 = ensure<float>(phi_call32, K_ * W_);
      launches += scu::launch_to_f32(out, K_ * W_, *out32, stream);
    }
    return out;
  }

  // flat deferred-draw list: 32 per possible record, at most 64 Mi entries
  static int64_t draw_cap_for(int64_t records) {
    if (scu::tuning().draw_cap >= 0) return scu::tuning().draw_cap;  // tests
    return std::min<int64_t>(records * 32, int64_t{1} << 26);
  }

  // the materialised M-step candidate (count / m_t + beta): needed by the
  // sequential-chain column sums (SAMELDA_COLSUM=chain), expected counts and
  // an m_t outside the reciprocal path's range; otherwise the scan recomputes
  // it from the u64 counts and no W x K candidate exists
  double* cand_scratch(int64_t n, bool expected, double m_t_) {
    const bool need = scu::tuning().colsum_chain || expected || !(m_t_ >= 0x1p-900 && m_t_ <= 0x1p900);
    return need ? ensure<double>(cand, n) : nullptr;
  }

  // scratch of the exact parallel column-sum scan (grown at train_begin /
  // the first per-call M-step, never inside a period)
  void* colsum_scratch(int64_t W_, int64_t K_) {
    return ensure<unsigned char>(colsum, scu::colsum_scratch_bytes(W_, static_cast<int>(K_)));
  }

  // Size every per-batch device buffer (and both pinned staging buffers) for
  // batches of up to B_ documents and nnz_ nonzeros, so that no period has to
  // grow one: a grow is a cudaFree (device-wide sync) plus a fresh allocation
  // of up to ~1 GB for the deferred queues, milliseconds inside a period.
  void reserve_batches(int64_t B_, int64_t nnz_, int K_, int64_t W_, int mode) {
    ensure<int32_t>(batch, B_);
    ensure<int64_t>(prefix, B_ + 1);
    ensure<double>(theta_batch, B_ * K_);
    ensure<float>(theta_batch32, B_ * K_);
    ensure<double>(theta_rows, B_ * K_);
    cand_scratch(W_ * K_, mode == SAMELDA_CU_MODE_EXPECTED, 1.0);
    ensure<double>(totals, K_);
    if (mode == SAMELDA_CU_MODE_EXPECTED) {
      ensure<double>(mu, nnz_);
      ensure<double>(tf, B_ * K_);
      ensure<double>(pf, W_ * K_);
    } else {
      ensure<unsigned long long>(tc, B_ * K_);
      ensure<unsigned long long>(pc, W_ * K_);
      if (K_ > 256) ensure<float>(mu_f32, nnz_);
      if (mode == SAMELDA_CU_MODE_THROUGHPUT || mode == SAMELDA_CU_MODE_MULTINOMIAL) {
        if (mode == SAMELDA_CU_MODE_THROUGHPUT) ensure<float>(rates32, B_ * K_);
        for (int i = 0; i < 2; ++i) stage(B_);
        return;
      }
      const int64_t records = scu::deferred_max_records(nnz_, K_);
      ensure<unsigned char>(deferred, scu::deferred_buffer_bytes(nnz_, K_));
      ensure<unsigned char>(deferred_aux, scu::deferred_aux_bytes(records, draw_cap_for(records)));
      ensure<unsigned long long>(n_deferred, 1);
    }
    for (int i = 0; i < 2; ++i) stage(B_);
  }

  // one sweep's sampling into tc/pc (or tf/pf): zeroes the count buffers first
  // mu_d: the caller's mu (per-call API) or nullptr (the kernel forms mu)
  void sample_sweep(const scu::BatchView& bv, const double* theta_b, const float* theta_b32,
                    const double* phi_wk, const float* phi_wk32, const double* mu_d, int K_,
                    int64_t W_, double m_t_, uint64_t seed, int64_t t, int sweep, int mode,
                    bool need_phi = true) {
    if (profile) {
      prof_nnz += bv.nnz;
      prof_docs += bv.B;
    }
    if (mode == SAMELDA_CU_MODE_EXPECTED) {
      double* tf_ = ensure<double>(tf, bv.B * K_);
      double* pf_ = ensure<double>(pf, W_ * K_);
      if (!need_phi && mu_d == nullptr && K_ <= 256) {
        // a non-final inner sweep: the expected theta counts only (k_theta_rates)
        tick(kSample, true);
        launches += scu::launch_expected_theta(bv, theta_b, phi_wk, K_, m_t_, tf_, stream);
        tick(kSample, false);
        return;
      }
      ck(cudaMemsetAsync(tf_, 0, sizeof(double) * std::max<int64_t>(bv.B * K_, 1), stream), "zero tf");
      ck(cudaMemsetAsync(pf_, 0, sizeof(double) * std::max<int64_t>(W_ * K_, 1), stream), "zero pf");
      tick(need_phi ? kSampleLast : kSample, true);
      launches += scu::launch_sample(bv, theta_b, phi_wk, mu_d, K_, m_t_, seed,
                                     static_cast<uint32_t>(t), static_cast<uint32_t>(sweep), mode,
                                     nullptr, nullptr, tf_, pf_, d_err(), stream);
      tick(need_phi ? kSampleLast : kSample, false);
    } else {
      auto* tc_ = ensure<unsigned long long>(tc, bv.B * K_);
      auto* pc_ = ensure<unsigned long long>(pc, W_ * K_);
      ck(cudaMemsetAsync(tc_, 0, sizeof(unsigned long long) * std::max<int64_t>(bv.B * K_, 1), stream), "zero tc");
      // a non-final inner sweep of the K = 256 period kernel skips the phi-count
      // scatter (only the last sweep's phi counts feed update_model)
      const bool skip_phi =
          !need_phi && mu_d == nullptr &&
          (K_ == 256 || mode == SAMELDA_CU_MODE_THROUGHPUT || mode == SAMELDA_CU_MODE_MULTINOMIAL);
      if (skip_phi) pc_ = nullptr;
      else ck(cudaMemsetAsync(pc_, 0, sizeof(unsigned long long) * std::max<int64_t>(W_ * K_, 1), stream), "zero pc");
      tick(need_phi ? kSampleLast : kSample, true);
      if (mode == SAMELDA_CU_MODE_MULTINOMIAL) {
        const int r = scu::launch_sample_multinomial(bv, theta_b32, phi_wk32, K_, m_t_, seed,
                                                     static_cast<uint32_t>(t), static_cast<uint32_t>(sweep),
                                                     tc_, pc_, d_err(), stream);
        if (r < 0) fail(SAMELDA_CU_CONFIG, "multinomial mode supports n_topics <= 1024");
        launches += r;
        tick(need_phi ? kSampleLast : kSample, false);
        return;
      }
      if (mode == SAMELDA_CU_MODE_THROUGHPUT) {
        launches += scu::launch_sample_throughput(
            bv, theta_b32, phi_wk32, K_, m_t_, seed, static_cast<uint32_t>(t), static_cast<uint32_t>(sweep),
            tc_, pc_, K_ > 256 ? ensure<float>(mu_f32, bv.nnz) : nullptr,
            pc_ ? nullptr : ensure<float>(rates32, bv.B * K_), stream);
        tick(need_phi ? kSampleLast : kSample, false);
        return;
      }
      const int64_t records = scu::deferred_max_records(bv.nnz, K_);
      const int64_t draw_cap = draw_cap_for(records);
      void* rec = ensure<unsigned char>(deferred, scu::deferred_buffer_bytes(bv.nnz, K_));
      void* aux = ensure<unsigned char>(deferred_aux, scu::deferred_aux_bytes(records, draw_cap));
      // the last readback of the deferral rate, if it has landed
      if (defer_read_pending && cudaEventQuery(defer_read) == cudaSuccess) {
        defer_frac = static_cast<double>(*h_deferred) / static_cast<double>(std::max<int64_t>(defer_read_nnz, 1));
        defer_read_pending = false;
      }
      // once most nonzeros defer (a PTRS draw each, late in training) the
      // deferred draws are decided from the fast path's rate (ptrs_banded);
      // SAMELDA_FAST_PTRS=0 keeps the exact mu from a concurrent SDDMM instead
      const bool fast_ptrs_now = defer_frac > kManyDeferred && scu::tuning().fast_ptrs;
      const double* mu_ex = nullptr;
      if (mu_d == nullptr && defer_frac > kManyDeferred && !scu::tuning().fast_ptrs) {
        if (!mu_stream) {
          ck(cudaStreamCreateWithFlags(&mu_stream, cudaStreamNonBlocking), "mu stream");
          ck(cudaEventCreateWithFlags(&mu_theta_ready, cudaEventDisableTiming), "event");
          ck(cudaEventCreateWithFlags(&mu_done, cudaEventDisableTiming), "event");
        }
        double* m = ensure<double>(mu, bv.nnz);
        ck(cudaEventRecord(mu_theta_ready, stream), "event record");
        ck(cudaStreamWaitEvent(mu_stream, mu_theta_ready, 0), "wait theta");
        launches += scu::launch_sddmm(bv, theta_b, phi_wk, K_, m, mu_stream);
        ck(cudaEventRecord(mu_done, mu_stream), "event record");
        mu_ex = m;
      }
      unsigned long long* nd_ = ensure<unsigned long long>(n_deferred, 1);
      launches += scu::launch_sample_fast(bv, theta_b, theta_b32, phi_wk, phi_wk32, mu_d, K_,
                                          m_t_, seed, static_cast<uint32_t>(t),
                                          static_cast<uint32_t>(sweep), tc_, pc_, rec, nd_, aux, draw_cap,
                                          K_ > 256 ? ensure<float>(mu_f32, bv.nnz) : nullptr, d_err(),
                                          stream, mu_ex, mu_ex ? mu_done : nullptr,
                                          mu_d == nullptr && fast_ptrs_now);
      if (!defer_read_pending && mu_d == nullptr) {
        if (!h_deferred) {
          ck(cudaMallocHost(&h_deferred, sizeof(unsigned long long)), "pinned");
          ck(cudaEventCreateWithFlags(&defer_read, cudaEventDisableTiming), "event");
        }
        ck(cudaMemcpyAsync(h_deferred, nd_, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream),
           "defer readback");
        ck(cudaEventRecord(defer_read, stream), "event record");
        defer_read_nnz = bv.nnz;
        defer_read_pending = true;
      }
      tick(need_phi ? kSampleLast : kSample, false);
      if (profile) {
        unsigned long long nd = 0;
        ck(cudaMemcpyAsync(&nd, n_deferred.p, sizeof(nd), cudaMemcpyDeviceToHost, stream), "n_deferred");
        ck(cudaStreamSynchronize(stream), "n_deferred");
        prof_deferred += static_cast<int64_t>(nd);
      }
    }
  }

  // eval split for the heldout slot (eval.cpp:99-121), cached per (corpus, seed)
  void prepare_split(uint64_t seed) {
    if (split_ready && split_seed == seed) return;
    const int64_t nd = heldout.n_docs;
    std::vector<int64_t> tok(static_cast<size_t>(nd) + 1, 0);
    for (int64_t d = 0; d < nd; ++d) tok[d + 1] = tok[d] + heldout.doc_tokens[static_cast<size_t>(d)];
    int64_t* dtok = ensure<int64_t>(tok_offsets, nd + 1);
    ck(cudaMemcpyAsync(dtok, tok.data(), sizeof(int64_t) * (nd + 1), cudaMemcpyHostToDevice, stream),
       "upload token offsets");
    launches += scu::launch_eval_split(heldout.offs.as<int64_t>(), heldout.words.as<int32_t>(),
                                       heldout.counts.as<int32_t>(), dtok, nd, seed,
                                       ensure<int32_t>(slots, tok[nd]),
                                       ensure<int32_t>(fold_counts, heldout.nnz),
                                       ensure<int32_t>(score_counts, heldout.nnz),
                                       eval_lists(nd, heldout.nnz), stream);
    ck(cudaStreamSynchronize(stream), "eval split");
    split_seed = seed;
    split_ready = true;
  }

  scu::EvalLists eval_lists(int64_t nd, int64_t nnz) {
    const int64_t n = std::max<int64_t>(nnz, 1), m = std::max<int64_t>(nd, 1);
    return scu::EvalLists{ensure<int32_t>(n_fold, m), ensure<int2>(fold_l, n), ensure<int32_t>(n_score, m),
                          ensure<int2>(score_l, n)};
  }

  // fold-in + scoring of every document of the split (eval.cpp:19-145);
  // per-doc results into doc_logp / doc_scored (+ theta rows when asked)
  int eval_docs(const CorpusSlot& c, const int32_t* fcounts, const int32_t* scounts,
                const scu::EvalLists& L, const double* phi_wk, int K_, double alpha, int sweeps,
                double* lp, int64_t* sc, double* theta_out) {
    if (!eval_exact) {
      const int r = scu::launch_eval_fold(c.offs.as<int64_t>(), L, c.n_docs, phi_wk, K_, alpha,
                                          sweeps, lp, sc, theta_out, d_err(), stream);
      if (r >= 0) return r;
    }
    const int64_t need = scu::eval_scratch_doubles(K_);
    double* scratch = need > 0 ? ensure<double>(eval_scratch, need) : nullptr;
    return scu::launch_eval_docs(c.offs.as<int64_t>(), c.words.as<int32_t>(), fcounts, scounts,
                                 c.n_docs, phi_wk, K_, alpha, sweeps, lp, sc, theta_out, scratch,
                                 need, d_err(), stream);
  }

  double eval_ll(const double* phi_wk, int K_, double alpha) {
    struct Range {
      Range() { nvtxRangePushA("samelda:perword_loglik"); }
      ~Range() { nvtxRangePop(); }
    } range;
    const int64_t nd = heldout.n_docs;
    double* lp = ensure<double>(doc_logp, nd);
    int64_t* sc = ensure<int64_t>(doc_scored, nd + 1);  // + the eval kernel's work counter
    reset_err();
    launches += eval_docs(heldout, fold_counts.as<int32_t>(), score_counts.as<int32_t>(),
                          eval_lists(nd, heldout.nnz), phi_wk, K_, alpha, 50, lp, sc, nullptr);
    double* dll = ensure<double>(ll, 1);
    launches += scu::launch_ordered_ll(lp, sc, nd, dll, d_err(), stream);
    double out = 0.0;
    ck(cudaMemcpyAsync(&out, dll, sizeof(double), cudaMemcpyDeviceToHost, stream), "read ll");
    check_err("perword_loglik");
    return out;
  }
};

namespace {

template <class F>
int guarded(samelda_cu_ctx* ctx, F&& fn) {
  if (ctx == nullptr) return SAMELDA_CU_CONFIG;
  try {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    fn();
    ctx->error.clear();
    return SAMELDA_CU_OK;
  } catch (const Fail& f) {
    ctx->error = f.msg;
    if (f.code == SAMELDA_CU_CUDA) cudaGetLastError();
    return f.code;
  } catch (const std::exception& e) {
    ctx->error = e.what();
    return SAMELDA_CU_CUDA;
  }
}

int64_t batch_nnz_host(const CorpusSlot& s, const int32_t* doc_ids, int64_t B) {
  int64_t n = 0;
  for (int64_t b = 0; b < B; ++b) {
    const int32_t d = doc_ids[b];
    if (d < 0 || d >= s.n_docs) fail(SAMELDA_CU_CONFIG, "batch doc id %d out of range", d);
    n += s.offsets[static_cast<size_t>(d) + 1] - s.offsets[static_cast<size_t>(d)];
  }
  return n;
}

}  // namespace

extern "C" {

int samelda_cu_version(void) { return kVersion; }

int samelda_cu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int samelda_cu_create(int device, samelda_cu_ctx** out) {
  if (out == nullptr) return SAMELDA_CU_CONFIG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) {
    cudaGetLastError();
    return SAMELDA_CU_CUDA;
  }
  (void)scu::tuning();  // the environment is read here, once per process
  auto* ctx = new samelda_cu_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      scu::init_lgamma_table() != 0) {
    delete ctx;
    return SAMELDA_CU_CUDA;
  }
  ctx->stream = ctx->own_stream;
  const char ev = scu::tuning().eval_variant;  // SAMELDA_EVAL=x (or c / w): exact order
  ctx->eval_exact = ev == 'x' || ev == 'c' || ev == 'w';
  *out = ctx;
  return SAMELDA_CU_OK;
}

int samelda_cu_set_eval_exact(samelda_cu_ctx* ctx, int exact) {
  if (ctx == nullptr) return SAMELDA_CU_CONFIG;
  ctx->eval_exact = exact != 0;
  return SAMELDA_CU_OK;
}

void samelda_cu_destroy(samelda_cu_ctx* ctx) {
  if (ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete ctx;
  }
}

const char* samelda_cu_last_error(const samelda_cu_ctx* ctx) {
  return ctx ? ctx->error.c_str() : "null context";
}

int samelda_cu_set_stream(samelda_cu_ctx* ctx, void* cuda_stream) {
  return guarded(ctx, [&] {
    ck(cudaStreamSynchronize(ctx->stream), "sync old stream");
    // NULL is the legacy default stream (e.g. torch's default stream), not "own"
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  });
}

int samelda_cu_use_own_stream(samelda_cu_ctx* ctx) {
  return guarded(ctx, [&] {
    ck(cudaStreamSynchronize(ctx->stream), "sync old stream");
    ctx->stream = ctx->own_stream;
  });
}

int samelda_cu_synchronize(samelda_cu_ctx* ctx) {
  return guarded(ctx, [&] {
    ck(cudaStreamSynchronize(ctx->stream), "synchronize");
    if (ctx->copy_stream) ck(cudaStreamSynchronize(ctx->copy_stream), "synchronize copies");
    ctx->poll_err(true, "period");
  });
}

int64_t samelda_cu_launch_count(const samelda_cu_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ------------------------------------------------------------ per-call API

int samelda_cu_sddmm(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                     const double* theta_batch, int64_t B, int64_t K_theta, const double* phi,
                     int64_t K, int64_t W, const int32_t* doc_ids, double* mu_out,
                     int64_t mu_cap, int64_t* mu_len) {
  return guarded(ctx, [&] {
    // sampler.cpp:90-98
    if (K_theta != K) fail(SAMELDA_CU_CONFIG, "sddmm: theta columns must match phi rows");
    validate_corpus(corpus);
    if (W != corpus->n_words) fail(SAMELDA_CU_CONFIG, "sddmm: phi columns must match the vocabulary size");
    if (K < 1 || K >= (1 << 20)) fail(SAMELDA_CU_CONFIG, "sddmm: K out of range");
    *mu_len = 0;
    if (B == 0) return;
    upload_corpus(ctx->train, corpus, ctx->stream, &ctx->pstage);
    const scu::BatchView bv = ctx->upload_batch(ctx->train, doc_ids, B);
    if (bv.nnz > mu_cap) fail(SAMELDA_CU_CONFIG, "sddmm: mu buffer too small");
    double* th = ensure<double>(ctx->theta_call, B * K);
    ck(cudaMemcpyAsync(th, theta_batch, sizeof(double) * B * K, cudaMemcpyHostToDevice, ctx->stream), "upload theta");
    const double* phi_wk = ctx->upload_phi(phi, K, W);
    double* mu = ensure<double>(ctx->mu, bv.nnz);
    ctx->launches += scu::launch_sddmm(bv, th, phi_wk, static_cast<int>(K), mu, ctx->stream);
    if (bv.nnz > 0)
      ck(cudaMemcpyAsync(mu_out, mu, sizeof(double) * bv.nnz, cudaMemcpyDeviceToHost, ctx->stream), "download mu");
    ck(cudaStreamSynchronize(ctx->stream), "sddmm");
    ck(cudaGetLastError(), "sddmm");
    *mu_len = bv.nnz;
  });
}

static void sample_call(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                        const double* theta_batch, int64_t B, int64_t K_theta,
                        const double* phi, int64_t K, int64_t W, const double* mu,
                        int64_t mu_len, const int32_t* doc_ids, double m_t, uint64_t seed,
                        int64_t t, int32_t sweep, int mode, void* theta_out, void* phi_out,
                        bool theta_only = false) {
  // sampler.cpp:130-140
  if (!(m_t > 0.0) || !std::isfinite(m_t)) fail(SAMELDA_CU_CONFIG, "sample_counts: m_t must be positive and finite");
  if (K_theta != K) fail(SAMELDA_CU_CONFIG, "sample_counts: theta columns must match phi rows");
  if (K < 1 || K >= (1 << 20)) fail(SAMELDA_CU_CONFIG, "sample_counts: K out of range");
  validate_corpus(corpus);
  if (W != corpus->n_words) fail(SAMELDA_CU_CONFIG, "sample_counts: phi columns must match the vocabulary size");
  if (sweep < 0 || sweep > 255) fail(SAMELDA_CU_CONFIG, "sample_counts: sweep out of range");
  upload_corpus(ctx->train, corpus, ctx->stream, &ctx->pstage);
  const int64_t nnz = batch_nnz_host(ctx->train, doc_ids, B);
  if (!theta_only && mu_len != nnz) fail(SAMELDA_CU_CONFIG, "sample_counts: mu is not aligned with the batch nonzeros");
  const size_t elem = 8;
  if (B == 0) {
    if (!theta_only) std::memset(phi_out, 0, elem * W * K);
    return;
  }
  const scu::BatchView bv = ctx->upload_batch(ctx->train, doc_ids, B);
  double* th = ensure<double>(ctx->theta_call, B * K);
  ck(cudaMemcpyAsync(th, theta_batch, sizeof(double) * B * K, cudaMemcpyHostToDevice, ctx->stream), "upload theta");
  float* th32 = ensure<float>(ctx->theta_call32, B * K);
  ctx->launches += scu::launch_to_f32(th, B * K, th32, ctx->stream);
  float* phi32 = nullptr;
  const double* phi_wk = ctx->upload_phi(phi, K, W, &phi32);
  double* mu_d = theta_only ? nullptr : ensure<double>(ctx->mu, nnz);
  if (nnz > 0 && !theta_only)
    ck(cudaMemcpyAsync(mu_d, mu, sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx->stream), "upload mu");
  ctx->reset_err();
  ctx->sample_sweep(bv, th, th32, phi_wk, phi32, mu_d, static_cast<int>(K), W, m_t, seed, t, sweep, mode,
                    !theta_only);
  ctx->check_err("sample_counts");
  if (theta_only) {
    ck(cudaMemcpyAsync(theta_out, ctx->tc.p, elem * B * K, cudaMemcpyDeviceToHost, ctx->stream), "download theta counts");
    ck(cudaStreamSynchronize(ctx->stream), "sample_counts");
    return;
  }
  const void* tsrc = mode == SAMELDA_CU_MODE_EXPECTED ? ctx->tf.p : ctx->tc.p;
  const void* psrc = mode == SAMELDA_CU_MODE_EXPECTED ? ctx->pf.p : ctx->pc.p;
  ck(cudaMemcpyAsync(theta_out, tsrc, elem * B * K, cudaMemcpyDeviceToHost, ctx->stream), "download theta counts");
  ck(cudaMemcpyAsync(phi_out, psrc, elem * W * K, cudaMemcpyDeviceToHost, ctx->stream), "download phi counts");
  ck(cudaStreamSynchronize(ctx->stream), "sample_counts");
}

int samelda_cu_sample_counts(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                             const double* theta_batch, int64_t B, int64_t K_theta,
                             const double* phi, int64_t K, int64_t W, const double* mu,
                             int64_t mu_len, const int32_t* doc_ids, double m_t, uint64_t seed,
                             int64_t t, int32_t sweep, int64_t* theta_counts,
                             int64_t* phi_counts) {
  return guarded(ctx, [&] {
    sample_call(ctx, corpus, theta_batch, B, K_theta, phi, K, W, mu, mu_len, doc_ids, m_t, seed,
                t, sweep, SAMELDA_CU_MODE_PARITY, theta_counts, phi_counts);
  });
}

int samelda_cu_sample_counts_fast(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                                  const double* theta_batch, int64_t B, int64_t K_theta,
                                  const double* phi, int64_t K, int64_t W, const double* mu,
                                  int64_t mu_len, const int32_t* doc_ids, double m_t,
                                  uint64_t seed, int64_t t, int32_t sweep, int64_t* theta_counts,
                                  int64_t* phi_counts) {
  return guarded(ctx, [&] {
    sample_call(ctx, corpus, theta_batch, B, K_theta, phi, K, W, mu, mu_len, doc_ids, m_t, seed,
                t, sweep, SAMELDA_CU_MODE_THROUGHPUT, theta_counts, phi_counts);
  });
}

int samelda_cu_sample_theta_counts_fast(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                                        const double* theta_batch, int64_t B, int64_t K_theta,
                                        const double* phi, int64_t K, int64_t W, const int32_t* doc_ids,
                                        double m_t, uint64_t seed, int64_t t, int32_t sweep,
                                        int64_t* theta_counts) {
  return guarded(ctx, [&] {
    sample_call(ctx, corpus, theta_batch, B, K_theta, phi, K, W, nullptr, 0, doc_ids, m_t, seed, t,
                sweep, SAMELDA_CU_MODE_THROUGHPUT, theta_counts, nullptr, true);
  });
}

int samelda_cu_sample_counts_multinomial(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                                         const double* theta_batch, int64_t B, int64_t K_theta,
                                         const double* phi, int64_t K, int64_t W, const double* mu,
                                         int64_t mu_len, const int32_t* doc_ids, double m_t,
                                         uint64_t seed, int64_t t, int32_t sweep,
                                         int64_t* theta_counts, int64_t* phi_counts) {
  return guarded(ctx, [&] {
    sample_call(ctx, corpus, theta_batch, B, K_theta, phi, K, W, mu, mu_len, doc_ids, m_t, seed,
                t, sweep, SAMELDA_CU_MODE_MULTINOMIAL, theta_counts, phi_counts);
  });
}

int samelda_cu_expected_counts(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                               const double* theta_batch, int64_t B, int64_t K_theta,
                               const double* phi, int64_t K, int64_t W, const double* mu,
                               int64_t mu_len, const int32_t* doc_ids, double m_t,
                               double* theta_expected, double* phi_expected) {
  return guarded(ctx, [&] {
    sample_call(ctx, corpus, theta_batch, B, K_theta, phi, K, W, mu, mu_len, doc_ids, m_t, 0, 0,
                0, SAMELDA_CU_MODE_EXPECTED, theta_expected, phi_expected);
  });
}

static void update_call(samelda_cu_ctx* ctx, double* theta, int64_t D, double* phi, int64_t K,
                        int64_t W, double alpha, double beta, const int32_t* doc_ids, int64_t B,
                        const void* tcounts, const void* pcounts, bool expected, double m_t,
                        double rho_t) {
  // sampler.cpp:197-229
  if (!(rho_t > 0.0 && rho_t <= 1.0)) fail(SAMELDA_CU_CONFIG, "update_model: rho_t must be in (0, 1]");
  if (K < 1 || W < 0 || D < 0) fail(SAMELDA_CU_CONFIG, "update_model: counts are not shaped for this model");
  for (int64_t b = 0; b < B; ++b)
    if (doc_ids[b] < 0 || doc_ids[b] >= D) fail(SAMELDA_CU_CONFIG, "update_model: doc id out of range");
  cudaStream_t st = ctx->stream;
  const int Ki = static_cast<int>(K);
  ctx->reset_err();
  // theta rows: computed on the device for the batch, placed into the host rows
  if (B > 0) {
    int32_t* db = ensure<int32_t>(ctx->batch, B);
    ck(cudaMemcpyAsync(db, doc_ids, sizeof(int32_t) * B, cudaMemcpyHostToDevice, st), "upload ids");
    double* rows = ensure<double>(ctx->theta_rows, B * K);
    if (expected) {
      double* tf = ensure<double>(ctx->tf, B * K);
      ck(cudaMemcpyAsync(tf, tcounts, sizeof(double) * B * K, cudaMemcpyHostToDevice, st), "upload tf");
      ctx->launches += scu::launch_theta_from_counts(nullptr, tf, B * K, m_t, alpha, rows, nullptr, st);
    } else {
      auto* tc = ensure<unsigned long long>(ctx->tc, B * K);
      ck(cudaMemcpyAsync(tc, tcounts, sizeof(int64_t) * B * K, cudaMemcpyHostToDevice, st), "upload tc");
      ctx->launches += scu::launch_theta_from_counts(tc, nullptr, B * K, m_t, alpha, rows, nullptr, st);
    }
    std::vector<double> h(static_cast<size_t>(B * K));
    ck(cudaMemcpyAsync(h.data(), rows, sizeof(double) * B * K, cudaMemcpyDeviceToHost, st), "download rows");
    ck(cudaStreamSynchronize(st), "theta rows");
    for (int64_t b = 0; b < B; ++b)
      std::memcpy(theta + static_cast<int64_t>(doc_ids[b]) * K, h.data() + b * K, sizeof(double) * K);
  }
  if (W * K == 0) return;
  double* phi_wk = ctx->upload_phi(phi, K, W);
  double* totals = ensure<double>(ctx->totals, K);
  if (expected) {
    double* pf = ensure<double>(ctx->pf, W * K);
    ck(cudaMemcpyAsync(pf, pcounts, sizeof(double) * W * K, cudaMemcpyHostToDevice, st), "upload pf");
    ctx->launches += scu::launch_phi_mstep(nullptr, pf, W, Ki, m_t, beta, rho_t, phi_wk, nullptr,
                                           ctx->cand_scratch(W * K, true, m_t), totals,
                                           ctx->colsum_scratch(W, Ki), ctx->d_err(), st);
  } else {
    auto* pc = ensure<unsigned long long>(ctx->pc, W * K);
    ck(cudaMemcpyAsync(pc, pcounts, sizeof(int64_t) * W * K, cudaMemcpyHostToDevice, st), "upload pc");
    ctx->launches += scu::launch_phi_mstep(pc, nullptr, W, Ki, m_t, beta, rho_t, phi_wk, nullptr,
                                           ctx->cand_scratch(W * K, false, m_t), totals,
                                           ctx->colsum_scratch(W, Ki), ctx->d_err(), st);
  }
  double* back = ensure<double>(ctx->phi_call, K * W);
  ctx->launches += scu::launch_transpose(phi_wk, W, K, back, st);
  ctx->check_err("update_model: phi row mass is not positive and finite");
  ck(cudaMemcpyAsync(phi, back, sizeof(double) * K * W, cudaMemcpyDeviceToHost, st), "download phi");
  ck(cudaStreamSynchronize(st), "update_model");
}

int samelda_cu_update_model(samelda_cu_ctx* ctx, double* theta, int64_t D, double* phi,
                            int64_t K, int64_t W, double alpha, double beta,
                            const int32_t* doc_ids, int64_t B, const int64_t* theta_counts,
                            const int64_t* phi_counts, double m_t, double rho_t) {
  return guarded(ctx, [&] {
    update_call(ctx, theta, D, phi, K, W, alpha, beta, doc_ids, B, theta_counts, phi_counts,
                false, m_t, rho_t);
  });
}

int samelda_cu_update_model_expected(samelda_cu_ctx* ctx, double* theta, int64_t D,
                                     double* phi, int64_t K, int64_t W, double alpha,
                                     double beta, const int32_t* doc_ids, int64_t B,
                                     const double* theta_expected, const double* phi_expected,
                                     double m_t, double rho_t) {
  return guarded(ctx, [&] {
    update_call(ctx, theta, D, phi, K, W, alpha, beta, doc_ids, B, theta_expected, phi_expected,
                true, m_t, rho_t);
  });
}

int samelda_cu_rho_schedule(int64_t t, double tau0, double gamma, double* out) {
  try {
    *out = rho_schedule_host(t, tau0, gamma);
    return SAMELDA_CU_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

int samelda_cu_anneal_m(int32_t schedule, int64_t t, int64_t t_max, double m, double* out) {
  try {
    *out = anneal_m_host(schedule, t, t_max, m);
    return SAMELDA_CU_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

int samelda_cu_fold_in_theta(samelda_cu_ctx* ctx, const double* phi, int64_t K, int64_t W,
                             const int32_t* words, const int32_t* counts, int64_t n,
                             double alpha, int32_t sweeps, double* theta_out) {
  return guarded(ctx, [&] {
    if (K < 1) fail(SAMELDA_CU_CONFIG, "fold_in_theta: K must be >= 1");
    for (int64_t i = 0; i < n; ++i)
      if (words[i] < 0 || words[i] >= W) fail(SAMELDA_CU_CONFIG, "fold_in_theta: word id out of range");
    // one-document corpus: the fold counts are the given counts
    const int64_t offs[2] = {0, n};
    std::vector<int32_t> zeros(static_cast<size_t>(std::max<int64_t>(n, 1)), 0);
    samelda_cu_corpus c{offs, n ? words : zeros.data(), n ? counts : zeros.data(), 1, W};
    CorpusSlot one;
    upload_corpus(one, &c, ctx->stream);
    const double* phi_wk = ctx->upload_phi(phi, K, W);
    int32_t* fc = ensure<int32_t>(ctx->fold_counts, std::max<int64_t>(n, 1));
    int32_t* sc = ensure<int32_t>(ctx->score_counts, std::max<int64_t>(n, 1));
    if (n > 0) {
      ck(cudaMemcpyAsync(fc, counts, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream), "upload counts");
      ck(cudaMemsetAsync(sc, 0, sizeof(int32_t) * n, ctx->stream), "zero score");
    }
    ctx->split_ready = false;  // fold/score buffers now hold this call's counts
    double* lp = ensure<double>(ctx->doc_logp, 1);
    int64_t* scd = ensure<int64_t>(ctx->doc_scored, 2);  // + the eval kernel's work counter
    double* th = ensure<double>(ctx->theta_rows, K);
    // the document's fold list: its nonzero-count cells in cell order (a
    // zero count adds exactly +0 in eval.cpp:45-49); no score cells
    std::vector<int2> lf;
    for (int64_t i = 0; i < n; ++i)
      if (counts[i] != 0) lf.push_back(make_int2(words[i], counts[i]));
    const int32_t meta[2] = {static_cast<int32_t>(lf.size()), 0};
    scu::EvalLists L = ctx->eval_lists(1, n);
    ck(cudaMemcpyAsync(L.n_fold, &meta[0], sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream), "upload list");
    ck(cudaMemcpyAsync(L.n_score, &meta[1], sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream), "upload list");
    if (!lf.empty())
      ck(cudaMemcpyAsync(L.fold, lf.data(), sizeof(int2) * lf.size(), cudaMemcpyHostToDevice, ctx->stream),
         "upload list");
    ctx->reset_err();
    ctx->launches += ctx->eval_docs(one, fc, sc, L, phi_wk, static_cast<int>(K), alpha, sweeps, lp, scd, th);
    ck(cudaMemcpyAsync(theta_out, th, sizeof(double) * K, cudaMemcpyDeviceToHost, ctx->stream), "download theta");
    ck(cudaStreamSynchronize(ctx->stream), "fold_in_theta");
    ck(cudaGetLastError(), "fold_in_theta");
  });
}

int samelda_cu_perword_loglik(samelda_cu_ctx* ctx, const double* phi, int64_t K, int64_t W,
                              const samelda_cu_corpus* test, double alpha, uint64_t seed,
                              double* ll_out) {
  return guarded(ctx, [&] {
    validate_corpus(test);
    if (test->n_docs < 1) fail(SAMELDA_CU_CONFIG, "perword_loglik: test corpus is empty");
    if (W != test->n_words) fail(SAMELDA_CU_CONFIG, "perword_loglik: phi width disagrees with corpus vocabulary");
    if (K < 1) fail(SAMELDA_CU_CONFIG, "perword_loglik: K must be >= 1");
    const uint64_t before = ctx->heldout.fp;
    const bool was_valid = ctx->heldout.valid;
    upload_corpus(ctx->heldout, test, ctx->stream, &ctx->pstage);
    if (!was_valid || before != ctx->heldout.fp) ctx->split_ready = false;
    ctx->prepare_split(seed);
    const double* phi_wk = ctx->upload_phi(phi, K, W);
    *ll_out = ctx->eval_ll(phi_wk, static_cast<int>(K), alpha);
  });
}

// ------------------------------------------------------------ CGS baseline

static void cgs_require(samelda_cu_ctx* ctx) {
  if (!ctx->cgs_ready) fail(SAMELDA_CU_CONFIG, "cgs: call samelda_cu_cgs_init first");
}

int samelda_cu_cgs_init(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus, int64_t n_topics,
                        double alpha, double beta, uint64_t seed) {
  return guarded(ctx, [&] {
    // cgs.cpp:13-18
    if (n_topics < 1 || n_topics > (1 << 20)) fail(SAMELDA_CU_CONFIG, "cgs_init: n_topics must be >= 1");
    if (!(alpha > 0.0) || !(beta > 0.0)) fail(SAMELDA_CU_CONFIG, "cgs_init: alpha and beta must be positive");
    if (n_topics > 1024) fail(SAMELDA_CU_CONFIG, "cgs_init: the device sampler supports n_topics <= 1024");
    validate_corpus(corpus);
    upload_corpus(ctx->train, corpus, ctx->stream, &ctx->pstage);
    const CorpusSlot& s = ctx->train;
    const int K = static_cast<int>(n_topics);
    std::vector<int64_t> tok(static_cast<size_t>(s.nnz) + 1, 0);
    for (int64_t i = 0; i < s.nnz; ++i) tok[i + 1] = tok[i] + corpus->counts[i];
    ctx->cgs_tokens = tok[s.nnz];
    int64_t* dtok = ensure<int64_t>(ctx->cgs_tok, s.nnz + 1);
    ck(cudaMemcpyAsync(dtok, tok.data(), sizeof(int64_t) * (s.nnz + 1), cudaMemcpyHostToDevice, ctx->stream),
       "upload token offsets");
    int32_t* z = ensure<int32_t>(ctx->cgs_z, ctx->cgs_tokens);
    int32_t* dt = ensure<int32_t>(ctx->cgs_dt, s.n_docs * K);
    int32_t* wt = ensure<int32_t>(ctx->cgs_wt, s.n_words * K);
    auto* tt = ensure<unsigned long long>(ctx->cgs_tt, K);
    ck(cudaMemsetAsync(dt, 0, sizeof(int32_t) * std::max<int64_t>(s.n_docs * K, 1), ctx->stream), "zero dt");
    ck(cudaMemsetAsync(wt, 0, sizeof(int32_t) * std::max<int64_t>(s.n_words * K, 1), ctx->stream), "zero wt");
    ck(cudaMemsetAsync(tt, 0, sizeof(unsigned long long) * K, ctx->stream), "zero tt");
    ctx->launches += scu::launch_cgs_init(s.offs.as<int64_t>(), s.words.as<int32_t>(), s.counts.as<int32_t>(),
                                          dtok, s.n_docs, K, seed, z, dt, wt, tt, ctx->stream);
    ck(cudaStreamSynchronize(ctx->stream), "cgs_init");
    ck(cudaGetLastError(), "cgs_init");
    ctx->cgs_K = K;
    ctx->cgs_alpha = alpha;
    ctx->cgs_beta = beta;
    ctx->cgs_ready = true;
  });
}

int samelda_cu_cgs_sweep(samelda_cu_ctx* ctx, uint64_t seed, int64_t sweep_index) {
  return guarded(ctx, [&] {
    cgs_require(ctx);
    const CorpusSlot& s = ctx->train;
    ctx->poll_err(false, "cgs_sweep");
    ctx->launches += scu::launch_cgs_sweep(
        s.offs.as<int64_t>(), s.words.as<int32_t>(), s.counts.as<int32_t>(), ctx->cgs_tok.as<int64_t>(),
        s.n_docs, ctx->cgs_K, s.n_words, ctx->cgs_alpha, ctx->cgs_beta, seed,
        static_cast<uint32_t>(sweep_index), ctx->cgs_z.as<int32_t>(), ctx->cgs_dt.as<int32_t>(),
        ctx->cgs_wt.as<int32_t>(), ctx->cgs_tt.as<unsigned long long>(), ctx->d_err(), ctx->stream);
    ck(cudaGetLastError(), "cgs_sweep launch");
    ctx->post_err_check();
  });
}

int samelda_cu_cgs_state(samelda_cu_ctx* ctx, int32_t* z, int32_t* doc_topic, int32_t* word_topic,
                         int64_t* topic_total) {
  return guarded(ctx, [&] {
    cgs_require(ctx);
    ctx->poll_err(true, "cgs_sweep");
    const CorpusSlot& s = ctx->train;
    const int64_t K = ctx->cgs_K;
    cudaStream_t st = ctx->stream;
    if (z && ctx->cgs_tokens)
      ck(cudaMemcpyAsync(z, ctx->cgs_z.p, sizeof(int32_t) * ctx->cgs_tokens, cudaMemcpyDeviceToHost, st), "z");
    if (doc_topic && s.n_docs * K)
      ck(cudaMemcpyAsync(doc_topic, ctx->cgs_dt.p, sizeof(int32_t) * s.n_docs * K, cudaMemcpyDeviceToHost, st), "dt");
    if (word_topic && s.n_words * K)
      ck(cudaMemcpyAsync(word_topic, ctx->cgs_wt.p, sizeof(int32_t) * s.n_words * K, cudaMemcpyDeviceToHost, st), "wt");
    if (topic_total)
      ck(cudaMemcpyAsync(topic_total, ctx->cgs_tt.p, sizeof(int64_t) * K, cudaMemcpyDeviceToHost, st), "tt");
    ck(cudaStreamSynchronize(st), "cgs_state");
  });
}

int samelda_cu_cgs_set_state(samelda_cu_ctx* ctx, const int32_t* z, const int32_t* doc_topic,
                             const int32_t* word_topic, const int64_t* topic_total) {
  return guarded(ctx, [&] {
    cgs_require(ctx);
    const CorpusSlot& s = ctx->train;
    const int64_t K = ctx->cgs_K;
    cudaStream_t st = ctx->stream;
    if (z && ctx->cgs_tokens)
      ck(cudaMemcpyAsync(ctx->cgs_z.p, z, sizeof(int32_t) * ctx->cgs_tokens, cudaMemcpyHostToDevice, st), "z");
    if (doc_topic && s.n_docs * K)
      ck(cudaMemcpyAsync(ctx->cgs_dt.p, doc_topic, sizeof(int32_t) * s.n_docs * K, cudaMemcpyHostToDevice, st), "dt");
    if (word_topic && s.n_words * K)
      ck(cudaMemcpyAsync(ctx->cgs_wt.p, word_topic, sizeof(int32_t) * s.n_words * K, cudaMemcpyHostToDevice, st), "wt");
    if (topic_total)
      ck(cudaMemcpyAsync(ctx->cgs_tt.p, topic_total, sizeof(int64_t) * K, cudaMemcpyHostToDevice, st), "tt");
    ck(cudaStreamSynchronize(st), "cgs_set_state");
  });
}

int samelda_cu_cgs_model(samelda_cu_ctx* ctx, double* phi, double* theta) {
  return guarded(ctx, [&] {
    cgs_require(ctx);
    ctx->poll_err(true, "cgs_sweep");
    const CorpusSlot& s = ctx->train;
    const int K = ctx->cgs_K;
    double* pw = ensure<double>(ctx->cgs_phi, s.n_words * K);
    double* th = theta ? ensure<double>(ctx->theta_rows, s.n_docs * K) : nullptr;
    ctx->launches += scu::launch_cgs_model(ctx->cgs_dt.as<int32_t>(), ctx->cgs_wt.as<int32_t>(),
                                           ctx->cgs_tt.as<unsigned long long>(), s.n_docs, s.n_words, K,
                                           ctx->cgs_alpha, ctx->cgs_beta, pw, th, ctx->stream);
    if (phi && s.n_words * K) {
      double* tmp = ensure<double>(ctx->phi_call, K * s.n_words);
      ctx->launches += scu::launch_transpose(pw, s.n_words, K, tmp, ctx->stream);
      ck(cudaMemcpyAsync(phi, tmp, sizeof(double) * K * s.n_words, cudaMemcpyDeviceToHost, ctx->stream), "phi");
    }
    if (theta && s.n_docs * K)
      ck(cudaMemcpyAsync(theta, th, sizeof(double) * s.n_docs * K, cudaMemcpyDeviceToHost, ctx->stream), "theta");
    ck(cudaStreamSynchronize(ctx->stream), "cgs_model");
  });
}

int samelda_cu_cgs_train(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus, int64_t n_topics,
                         double alpha, double beta, int64_t n_sweeps, uint64_t seed,
                         int64_t eval_every, const samelda_cu_corpus* heldout, double* phi_out,
                         double* theta_out, samelda_cu_trace_row* trace, int64_t trace_cap,
                         int64_t* n_trace) {
  // cgs.cpp:131-157
  if (ctx == nullptr) return SAMELDA_CU_CONFIG;
  if (n_sweeps < 0) {
    ctx->error = "cgs_train: n_sweeps must be >= 0";
    return SAMELDA_CU_CONFIG;
  }
  *n_trace = 0;
  int rc = samelda_cu_cgs_init(ctx, corpus, n_topics, alpha, beta, seed);
  if (rc) return rc;
  const bool do_eval = heldout != nullptr && eval_every > 0;
  if (do_eval && n_sweeps > 0) {
    rc = samelda_cu_heldout(ctx, heldout, seed);
    if (rc) return rc;
  }
  return guarded(ctx, [&] {
    const auto t_start = std::chrono::steady_clock::now();
    const int K = ctx->cgs_K;
    for (int64_t sweep = 1; sweep <= n_sweeps; ++sweep) {
      int r = samelda_cu_cgs_sweep(ctx, seed, sweep);
      if (r) throw Fail{r, ctx->error};
      if (do_eval && (sweep % eval_every == 0 || sweep == n_sweeps)) {
        if (ctx->heldout.n_words != ctx->train.n_words)
          fail(SAMELDA_CU_CONFIG, "perword_loglik: phi width disagrees with corpus vocabulary");
        double* pw = ensure<double>(ctx->cgs_phi, ctx->train.n_words * K);
        ctx->launches += scu::launch_cgs_model(ctx->cgs_dt.as<int32_t>(), ctx->cgs_wt.as<int32_t>(),
                                               ctx->cgs_tt.as<unsigned long long>(), ctx->train.n_docs,
                                               ctx->train.n_words, K, alpha, beta, pw, nullptr, ctx->stream);
        const double ll = ctx->eval_ll(pw, K, alpha);
        const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t_start;
        if (*n_trace >= trace_cap) fail(SAMELDA_CU_CONFIG, "trace buffer too small");
        // one sample per token per sweep: samples/word == sweep (cgs.cpp:149-151)
        trace[(*n_trace)++] = {sweep, static_cast<double>(sweep), static_cast<double>(sweep), ll, el.count(), 1.0};
      }
    }
    const int r = samelda_cu_cgs_model(ctx, phi_out, theta_out);
    if (r) throw Fail{r, ctx->error};
  });
}

// ------------------------------------------------------------ trainer

int samelda_cu_batches_create(int64_t n_docs, double batch_fraction, uint64_t seed,
                              samelda_cu_batches** out) {
  if (!(batch_fraction > 0.0 && batch_fraction <= 1.0)) return SAMELDA_CU_CONFIG;
  if (n_docs < 0 || out == nullptr) return SAMELDA_CU_CONFIG;
  auto* b = new Batches();
  b->n_docs = n_docs;
  b->seed = seed;
  b->batch_size = std::max<int64_t>(
      1, static_cast<int64_t>(std::llround(batch_fraction * static_cast<double>(n_docs))));
  b->start_pass();
  *out = reinterpret_cast<samelda_cu_batches*>(b);
  return SAMELDA_CU_OK;
}

int64_t samelda_cu_batches_size(const samelda_cu_batches* s) {
  return reinterpret_cast<const Batches*>(s)->batch_size;
}

int64_t samelda_cu_batches_per_pass(const samelda_cu_batches* s) {
  return reinterpret_cast<const Batches*>(s)->per_pass();
}

int64_t samelda_cu_batches_next(samelda_cu_batches* s, int32_t* out) {
  return reinterpret_cast<Batches*>(s)->next(out);
}

void samelda_cu_batches_destroy(samelda_cu_batches* s) { delete reinterpret_cast<Batches*>(s); }

int samelda_cu_train_begin(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                           const samelda_cu_config* config) {
  return guarded(ctx, [&] {
    validate_config(config);
    validate_corpus(corpus);
    if (corpus->n_docs < 1) fail(SAMELDA_CU_CONFIG, "train: corpus is empty");
    upload_corpus(ctx->train, corpus, ctx->stream, &ctx->pstage);
    ctx->cfg = *config;
    ctx->K = static_cast<int>(config->n_topics);
    ctx->W = corpus->n_words;
    ctx->D = corpus->n_docs;
    const int64_t K = ctx->K;
    double* th = ensure<double>(ctx->theta, ctx->D * K);
    double* ph = ensure<double>(ctx->phi, ctx->W * K);
    // init_model (model.cpp:41-52) then the seeded perturbation
    // (sampler.cpp:285-298), which only applies when t_max > 0
    ctx->launches += scu::launch_fill(th, ctx->D * K, config->alpha + 1.0 / static_cast<double>(K), ctx->stream);
    ctx->launches += scu::launch_phi_init(ph, ctx->W, ctx->K, config->t_max > 0 ? config->init_noise : 0.0,
                                          config->seed, ensure<double>(ctx->totals, K),
                                          ctx->colsum_scratch(ctx->W, ctx->K), ctx->stream);
    ctx->launches += scu::launch_to_f32(ph, ctx->W * K, ensure<float>(ctx->phi32, ctx->W * K), ctx->stream);
    // per-batch buffers for the largest batch the minibatch stream can draw:
    // its size (samelda_cu_batches_create) times the longest documents
    {
      const int64_t bsz = std::min<int64_t>(
          ctx->D, std::max<int64_t>(1, static_cast<int64_t>(std::llround(
                                             config->batch_fraction * static_cast<double>(ctx->D)))));
      std::vector<int64_t> len(static_cast<size_t>(ctx->D));
      for (int64_t d = 0; d < ctx->D; ++d)
        len[static_cast<size_t>(d)] = corpus->doc_offsets[d + 1] - corpus->doc_offsets[d];
      std::nth_element(len.begin(), len.begin() + (bsz - 1), len.end(), std::greater<int64_t>());
      int64_t nnz_max = 0;
      for (int64_t i = 0; i < bsz; ++i) nnz_max += len[static_cast<size_t>(i)];
      ctx->reserve_batches(bsz, nnz_max, ctx->K, ctx->W, config->mode);
    }
    ck(cudaStreamSynchronize(ctx->stream), "train_begin");
    ck(cudaGetLastError(), "train_begin");
    ctx->model_ready = true;
    ctx->counts_ready = false;
  });
}

int samelda_cu_heldout(samelda_cu_ctx* ctx, const samelda_cu_corpus* test, uint64_t seed) {
  return guarded(ctx, [&] {
    validate_corpus(test);
    if (test->n_docs < 1) fail(SAMELDA_CU_CONFIG, "perword_loglik: test corpus is empty");
    const uint64_t before = ctx->heldout.fp;
    const bool was_valid = ctx->heldout.valid;
    upload_corpus(ctx->heldout, test, ctx->stream, &ctx->pstage);
    if (!was_valid || before != ctx->heldout.fp) ctx->split_ready = false;
    ctx->prepare_split(seed);
  });
}

int samelda_cu_period_sample(samelda_cu_ctx* ctx, const int32_t* doc_ids, int64_t B, int64_t t,
                             double m_t) {
  return guarded(ctx, [&] {
    struct Range {
      Range() { nvtxRangePushA("samelda:period"); }
      ~Range() { nvtxRangePop(); }
    } range;
    if (!ctx->model_ready) fail(SAMELDA_CU_CONFIG, "period: call samelda_cu_train_begin first");
    if (!(m_t > 0.0) || !std::isfinite(m_t)) fail(SAMELDA_CU_CONFIG, "sample_counts: m_t must be positive and finite");
    const samelda_cu_config& c = ctx->cfg;
    const int K = ctx->K;
    cudaStream_t st = ctx->stream;
    ctx->poll_err(false, "period");
    scu::BatchView bv = ctx->upload_batch(ctx->train, doc_ids, B);
    bv.doc_base = ctx->doc_base;
    ctx->B = B;
    ctx->nnzB = bv.nnz;
    ctx->m_t = m_t;
    double* thb = ensure<double>(ctx->theta_batch, B * K);
    float* thb32 = ensure<float>(ctx->theta_batch32, B * K);
    const bool expected = c.mode == SAMELDA_CU_MODE_EXPECTED;
    double* mu = expected ? ensure<double>(ctx->mu, bv.nnz) : nullptr;
    ctx->launches += scu::launch_gather_theta(ctx->theta.as<double>(), bv.batch_docs, B, K, thb, thb32, st);
    for (int64_t sweep = 0; sweep < c.inner_sweeps; ++sweep) {
      if (expected && K > 256) {
        // K <= 256: the expected-count kernel forms mu itself (f64 tree);
        // wider K takes an explicit mu (sampler.cpp:321)
        ctx->tick(samelda_cu_ctx::kSddmm, true);
        ctx->launches += scu::launch_sddmm(bv, thb, ctx->phi.as<double>(), K, mu, st);
        ctx->tick(samelda_cu_ctx::kSddmm, false);
      }
      // parity mode: the SDDMM is fused into the sampling kernel (mu == nullptr)
      ctx->sample_sweep(bv, thb, thb32, ctx->phi.as<double>(), ctx->phi32.as<float>(),
                        expected && K <= 256 ? nullptr : mu, K, ctx->W,
                        m_t, c.seed, t, static_cast<int>(sweep), c.mode,
                        /*need_phi=*/sweep + 1 == c.inner_sweeps);
      if (sweep + 1 < c.inner_sweeps) {
        if (expected)
          ctx->launches += scu::launch_theta_from_counts(nullptr, ctx->tf.as<double>(), B * K, m_t, c.alpha, thb,
                                                         thb32, st);
        else
          ctx->launches += scu::launch_theta_from_counts(ctx->tc.as<unsigned long long>(), nullptr, B * K, m_t,
                                                         c.alpha, thb, thb32, st);
      }
    }
    ck(cudaGetLastError(), "period sample launch");
    ctx->counts_ready = true;
    ctx->counts_float = c.mode == SAMELDA_CU_MODE_EXPECTED;
  });
}

int samelda_cu_period_update(samelda_cu_ctx* ctx, double rho_t) {
  return guarded(ctx, [&] {
    if (!ctx->counts_ready) fail(SAMELDA_CU_CONFIG, "period_update without period_sample");
    if (!(rho_t > 0.0 && rho_t <= 1.0)) fail(SAMELDA_CU_CONFIG, "update_model: rho_t must be in (0, 1]");
    const samelda_cu_config& c = ctx->cfg;
    const int K = ctx->K;
    cudaStream_t st = ctx->stream;
    const bool f = ctx->counts_float;
    const auto* tcu = f ? nullptr : ctx->tc.as<unsigned long long>();
    const auto* pcu = f ? nullptr : ctx->pc.as<unsigned long long>();
    const double* tcf = f ? ctx->tf.as<double>() : nullptr;
    const double* pcf = f ? ctx->pf.as<double>() : nullptr;
    ctx->tick(samelda_cu_ctx::kMstep, true);
    ctx->launches += scu::launch_theta_persist(tcu, tcf, ctx->batch.as<int32_t>(), ctx->B, K, ctx->m_t, c.alpha,
                                               ctx->theta.as<double>(), st);
    ctx->launches += scu::launch_phi_mstep(pcu, pcf, ctx->W, K, ctx->m_t, c.beta, rho_t, ctx->phi.as<double>(),
                                           ctx->phi32.as<float>(), ctx->cand_scratch(ctx->W * K, f, ctx->m_t),
                                           ensure<double>(ctx->totals, K), ctx->colsum_scratch(ctx->W, K),
                                           ctx->d_err(), st);
    ctx->tick(samelda_cu_ctx::kMstep, false);
    ck(cudaGetLastError(), "period launch");
    // no host wait: the flag is read back asynchronously and reported by the
    // next call (NumericalError), or at the next synchronising call
    ctx->post_err_check();
  });
}

int samelda_cu_period(samelda_cu_ctx* ctx, const int32_t* doc_ids, int64_t B, int64_t t,
                      double m_t, double rho_t) {
  int rc = samelda_cu_period_sample(ctx, doc_ids, B, t, m_t);
  if (rc) return rc;
  return samelda_cu_period_update(ctx, rho_t);
}

int samelda_cu_set_doc_base(samelda_cu_ctx* ctx, int64_t doc_base) {
  return guarded(ctx, [&] {
    if (doc_base < 0) fail(SAMELDA_CU_CONFIG, "doc_base must be >= 0");
    ctx->doc_base = doc_base;
  });
}

int samelda_cu_profile(samelda_cu_ctx* ctx, int32_t enable) {
  return guarded(ctx, [&] {
    ctx->profile = enable != 0;
    for (auto& u : ctx->events_used) u = 0;
    ctx->prof_nnz = ctx->prof_docs = ctx->prof_deferred = 0;
  });
}

int samelda_cu_profile_read(samelda_cu_ctx* ctx, double* ms_out, int64_t* launches_out,
                            int64_t* nnz_sampled, int64_t* docs_sampled, int64_t* deferred) {
  return guarded(ctx, [&] {
    ck(cudaStreamSynchronize(ctx->stream), "profile sync");
    for (int k = 0; k < samelda_cu_ctx::kKinds; ++k) {
      double total = 0.0;
      for (size_t i = 0; i < ctx->events_used[k]; ++i) {
        float ms = 0.0f;
        ck(cudaEventElapsedTime(&ms, ctx->events[k][i].first, ctx->events[k][i].second), "elapsed");
        total += ms;
      }
      ms_out[k] = total;
      launches_out[k] = static_cast<int64_t>(ctx->events_used[k]);
      ctx->events_used[k] = 0;
    }
    *nnz_sampled = ctx->prof_nnz;
    *docs_sampled = ctx->prof_docs;
    if (deferred) *deferred = ctx->prof_deferred;
    ctx->prof_nnz = ctx->prof_docs = ctx->prof_deferred = 0;
  });
}

int samelda_cu_phi_counts_device(samelda_cu_ctx* ctx, void** ptr, int64_t* n_elems,
                                 int32_t* elem_bytes, int32_t* is_float) {
  return guarded(ctx, [&] {
    if (!ctx->counts_ready) fail(SAMELDA_CU_CONFIG, "no sampled counts yet");
    *ptr = ctx->counts_float ? ctx->pf.p : ctx->pc.p;
    *n_elems = ctx->W * ctx->K;
    *elem_bytes = 8;
    *is_float = ctx->counts_float ? 1 : 0;
  });
}

int samelda_cu_phi_counts_pack32(samelda_cu_ctx* ctx, void* lo, int64_t n_elems, int32_t world_size,
                                 void* n_over) {
  return guarded(ctx, [&] {
    if (!ctx->counts_ready) fail(SAMELDA_CU_CONFIG, "no sampled counts yet");
    if (ctx->counts_float) fail(SAMELDA_CU_CONFIG, "pack32: the expected-count mode exchanges f64 counts");
    if (n_elems != ctx->W * ctx->K) fail(SAMELDA_CU_CONFIG, "pack32: n_elems must be W x K");
    if (world_size < 1) fail(SAMELDA_CU_CONFIG, "pack32: world_size must be >= 1");
    // world_size x (bound - 1) < 2^31: the int32 sum of packed cells never wraps
    const unsigned long long bound = (0x7fffffffull / static_cast<unsigned long long>(world_size));
    ctx->launches += scu::launch_pack_counts(ctx->pc.as<unsigned long long>(), n_elems, bound,
                                             static_cast<int32_t*>(lo), static_cast<unsigned long long*>(n_over),
                                             ctx->stream);
  });
}

int samelda_cu_phi_counts_unpack32(samelda_cu_ctx* ctx, const void* lo, int64_t n_elems) {
  return guarded(ctx, [&] {
    if (!ctx->counts_ready || ctx->counts_float) fail(SAMELDA_CU_CONFIG, "unpack32: no integer counts");
    if (n_elems != ctx->W * ctx->K) fail(SAMELDA_CU_CONFIG, "unpack32: n_elems must be W x K");
    ctx->launches += scu::launch_unpack_counts(static_cast<const int32_t*>(lo), n_elems,
                                               ctx->pc.as<unsigned long long>(), ctx->stream);
  });
}

int samelda_cu_batch_theta(samelda_cu_ctx* ctx, double* out, int64_t cap) {
  return guarded(ctx, [&] {
    ctx->poll_err(true, "period");
    if (!ctx->model_ready) fail(SAMELDA_CU_CONFIG, "no model");
    const int64_t n = ctx->B * ctx->K;
    if (cap < n) fail(SAMELDA_CU_CONFIG, "batch_theta: buffer too small");
    double* rows = ensure<double>(ctx->theta_rows, n);
    ctx->launches += scu::launch_gather_theta(ctx->theta.as<double>(), ctx->batch.as<int32_t>(), ctx->B, ctx->K,
                                              rows, nullptr, ctx->stream);
    if (n > 0)
      ck(cudaMemcpyAsync(out, rows, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "download rows");
    ck(cudaStreamSynchronize(ctx->stream), "batch_theta");
  });
}

int samelda_cu_batch_theta_async(samelda_cu_ctx* ctx, double* out, int64_t cap) {
  return guarded(ctx, [&] {
    ctx->poll_err(false, "period");
    if (!ctx->model_ready) fail(SAMELDA_CU_CONFIG, "no model");
    const int64_t n = ctx->B * ctx->K;
    if (cap < n) fail(SAMELDA_CU_CONFIG, "batch_theta: buffer too small");
    if (n == 0) return;
    if (!ctx->copy_stream) {
      ck(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
      for (int i = 0; i < 2; ++i) {
        ck(cudaEventCreateWithFlags(&ctx->rows_ready[i], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&ctx->rows_copied[i], cudaEventDisableTiming), "event");
        ck(cudaEventRecord(ctx->rows_copied[i], ctx->copy_stream), "event");
      }
    }
    const int i = ctx->rows_next;
    ctx->rows_next ^= 1;
    // rows2[i] may still be the source of the copy two calls ago
    ck(cudaStreamWaitEvent(ctx->stream, ctx->rows_copied[i], 0), "wait copy");
    double* rows = ensure<double>(ctx->rows2[i], n);
    ctx->launches += scu::launch_gather_theta(ctx->theta.as<double>(), ctx->batch.as<int32_t>(), ctx->B, ctx->K,
                                              rows, nullptr, ctx->stream);
    ck(cudaEventRecord(ctx->rows_ready[i], ctx->stream), "rows ready");
    ck(cudaStreamWaitEvent(ctx->copy_stream, ctx->rows_ready[i], 0), "wait rows");
    ck(cudaMemcpyAsync(out, rows, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->copy_stream),
       "download rows");
    ck(cudaEventRecord(ctx->rows_copied[i], ctx->copy_stream), "rows copied");
  });
}

int samelda_cu_count_totals(samelda_cu_ctx* ctx, int64_t* theta_total, int64_t* phi_total) {
  return guarded(ctx, [&] {
    ctx->poll_err(true, "period");
    if (!ctx->counts_ready || ctx->counts_float) fail(SAMELDA_CU_CONFIG, "no integer counts");
    std::vector<int64_t> a(static_cast<size_t>(std::max<int64_t>(ctx->B * ctx->K, 1)));
    std::vector<int64_t> b(static_cast<size_t>(std::max<int64_t>(ctx->W * ctx->K, 1)));
    ck(cudaMemcpyAsync(a.data(), ctx->tc.p, sizeof(int64_t) * ctx->B * ctx->K, cudaMemcpyDeviceToHost, ctx->stream), "tc");
    ck(cudaMemcpyAsync(b.data(), ctx->pc.p, sizeof(int64_t) * ctx->W * ctx->K, cudaMemcpyDeviceToHost, ctx->stream), "pc");
    ck(cudaStreamSynchronize(ctx->stream), "count totals");
    int64_t s0 = 0, s1 = 0;
    for (int64_t i = 0; i < ctx->B * ctx->K; ++i) s0 += a[static_cast<size_t>(i)];
    for (int64_t i = 0; i < ctx->W * ctx->K; ++i) s1 += b[static_cast<size_t>(i)];
    *theta_total = s0;
    *phi_total = s1;
  });
}

int samelda_cu_evaluate(samelda_cu_ctx* ctx, double* ll_out) {
  return guarded(ctx, [&] {
    if (!ctx->model_ready) fail(SAMELDA_CU_CONFIG, "evaluate: no model");
    if (!ctx->heldout.valid || !ctx->split_ready) fail(SAMELDA_CU_CONFIG, "evaluate: call samelda_cu_heldout first");
    if (ctx->heldout.n_words != ctx->W) fail(SAMELDA_CU_CONFIG, "perword_loglik: phi width disagrees with corpus vocabulary");
    *ll_out = ctx->eval_ll(ctx->phi.as<double>(), ctx->K, ctx->cfg.alpha);
  });
}

int samelda_cu_model_download(samelda_cu_ctx* ctx, double* phi, double* theta) {
  return guarded(ctx, [&] {
    ctx->poll_err(true, "period");
    if (!ctx->model_ready) fail(SAMELDA_CU_CONFIG, "no model");
    const int64_t K = ctx->K;
    if (phi) {
      double* tmp = ensure<double>(ctx->phi_call, K * ctx->W);
      ctx->launches += scu::launch_transpose(ctx->phi.as<double>(), ctx->W, K, tmp, ctx->stream);
      copy_d2h(&ctx->pstage, phi, tmp, sizeof(double) * K * ctx->W, ctx->stream);
    }
    if (theta) copy_d2h(&ctx->pstage, theta, ctx->theta.p, sizeof(double) * ctx->D * K, ctx->stream);
    ck(cudaStreamSynchronize(ctx->stream), "model_download");
  });
}

int samelda_cu_model_upload(samelda_cu_ctx* ctx, const double* phi, const double* theta) {
  return guarded(ctx, [&] {
    if (!ctx->model_ready) fail(SAMELDA_CU_CONFIG, "no model");
    const int64_t K = ctx->K;
    if (phi) {
      const double* wk = ctx->upload_phi(phi, K, ctx->W);
      ck(cudaMemcpyAsync(ctx->phi.p, wk, sizeof(double) * K * ctx->W, cudaMemcpyDeviceToDevice, ctx->stream), "phi");
      ctx->launches += scu::launch_to_f32(ctx->phi.as<double>(), K * ctx->W, ctx->phi32.as<float>(), ctx->stream);
    }
    if (theta)
      ck(cudaMemcpyAsync(ctx->theta.p, theta, sizeof(double) * ctx->D * K, cudaMemcpyHostToDevice, ctx->stream), "theta");
    ck(cudaStreamSynchronize(ctx->stream), "model_upload");
  });
}

int samelda_cu_train(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                     const samelda_cu_config* config, const samelda_cu_corpus* heldout,
                     int64_t eval_every, double* phi_out, double* theta_out,
                     samelda_cu_trace_row* trace, int64_t trace_cap, int64_t* n_trace) {
  // sampler.cpp:269-353
  int rc = samelda_cu_train_begin(ctx, corpus, config);
  if (rc) return rc;
  *n_trace = 0;
  const bool do_eval = heldout != nullptr && eval_every > 0;
  if (do_eval && config->t_max > 0) {
    rc = samelda_cu_heldout(ctx, heldout, config->seed);
    if (rc) return rc;
  }
  return guarded(ctx, [&] {
    if (config->t_max > 0) {
      Batches batches;
      batches.n_docs = corpus->n_docs;
      batches.seed = config->seed;
      batches.batch_size = std::max<int64_t>(
          1, static_cast<int64_t>(std::llround(config->batch_fraction * static_cast<double>(corpus->n_docs))));
      batches.start_pass();
      const auto t_start = std::chrono::steady_clock::now();
      double tokens_seen = 0.0;
      double samples_per_word = 0.0;
      const double corpus_tokens = static_cast<double>(ctx->train.n_tokens);
      std::vector<int32_t> batch(static_cast<size_t>(batches.batch_size));
      for (int64_t t = 0; t < config->t_max; ++t) {
        const int64_t B = batches.next(batch.data());
        const double m_t = anneal_m_host(config->schedule, t + 1, config->t_max, config->m);
        const double rho_t = rho_schedule_host(t, config->tau0, config->gamma);
        int r = samelda_cu_period(ctx, batch.data(), B, t, m_t, rho_t);
        if (r) throw Fail{r, ctx->error};
        double batch_tokens = 0.0;
        for (int64_t b = 0; b < B; ++b)
          batch_tokens += static_cast<double>(ctx->train.doc_tokens[static_cast<size_t>(batch[b])]);
        tokens_seen += batch_tokens;
        samples_per_word += m_t * batch_tokens / corpus_tokens;
        if (do_eval && ((t + 1) % eval_every == 0 || t + 1 == config->t_max)) {
          double ll = 0.0;
          r = samelda_cu_evaluate(ctx, &ll);
          if (r) throw Fail{r, ctx->error};
          const std::chrono::duration<double> el = std::chrono::steady_clock::now() - t_start;
          if (*n_trace >= trace_cap) fail(SAMELDA_CU_CONFIG, "trace buffer too small");
          trace[(*n_trace)++] = {t, tokens_seen / corpus_tokens, samples_per_word, ll, el.count(), m_t};
        }
      }
    }
    int r = samelda_cu_model_download(ctx, phi_out, theta_out);
    if (r) throw Fail{r, ctx->error};
  });
}

}  // extern "C"
