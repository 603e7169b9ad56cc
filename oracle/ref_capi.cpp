// ref_capi.cpp -- extern "C" wrapper over the COMPILED REFERENCE library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources, where they lie under /root/reference/proj
// (src/{rng,corpus,model,eval,sampler}.cpp and tests/support/*.cpp), into
// oracle/_ref/libsamelda_ref.so.  No reference source is copied into this
// repository.  The wrapper only converts plain pointers to the reference's
// value types and exceptions to return codes (errors.hpp:7-20).
//
// Uses: the golden-fixture generator (tests/golden/make_golden.py), the
// parity tests, and bench.py's cpu_baseline / --impl reference legs
// (kind "reference": the reference's multi-threaded CPU sampler).

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "samelda/cgs.hpp"
#include "samelda/corpus.hpp"
#include "samelda/errors.hpp"
#include "samelda/eval.hpp"
#include "samelda/model.hpp"
#include "samelda/rng.hpp"
#include "samelda/sampler.hpp"
#include "support/synthetic.hpp"

using namespace samelda;

namespace {

thread_local char g_error[512];

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const ConfigError& e) {
    std::snprintf(g_error, sizeof(g_error), "%s", e.what());
    return 1;
  } catch (const IoError& e) {
    std::snprintf(g_error, sizeof(g_error), "%s", e.what());
    return 2;
  } catch (const NumericalError& e) {
    std::snprintf(g_error, sizeof(g_error), "%s", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::snprintf(g_error, sizeof(g_error), "%s", e.what());
    return 9;
  }
}

Corpus make_corpus(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                   int64_t n_docs, int64_t n_words) {
  Corpus c;
  c.n_docs = n_docs;
  c.n_words = n_words;
  c.doc_offsets.assign(offsets, offsets + n_docs + 1);
  const int64_t nnz = offsets[n_docs];
  c.word_ids.assign(words, words + nnz);
  c.counts.assign(counts, counts + nnz);
  for (int64_t i = 0; i < nnz; ++i) c.n_tokens += counts[i];
  return c;
}

DenseMatrix make_matrix(const double* data, int64_t rows, int64_t cols) {
  DenseMatrix m(rows, cols);
  if (rows * cols > 0) std::memcpy(m.data.data(), data, sizeof(double) * rows * cols);
  return m;
}

struct Generated {
  synthetic::GeneratedCorpus g;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error; }

int ref_stream_u32(uint64_t seed, uint32_t t, uint32_t doc, uint32_t word, uint32_t tag,
                   int64_t n, uint32_t* out) {
  return guarded([&] {
    auto s = stream_for(seed, {t, doc, word, tag});
    for (int64_t i = 0; i < n; ++i) out[i] = s.next_u32();
  });
}

int ref_stream_uniform(uint64_t seed, uint32_t t, uint32_t doc, uint32_t word, uint32_t tag,
                       int64_t n, int oo, double* out) {
  return guarded([&] {
    auto s = stream_for(seed, {t, doc, word, tag});
    for (int64_t i = 0; i < n; ++i) out[i] = oo ? s.uniform_oo() : s.uniform();
  });
}

int ref_stream_below(uint64_t seed, uint32_t t, uint32_t doc, uint32_t word, uint32_t tag,
                     uint64_t bound, int64_t n, uint64_t* out) {
  return guarded([&] {
    auto s = stream_for(seed, {t, doc, word, tag});
    for (int64_t i = 0; i < n; ++i) out[i] = s.uniform_below(bound);
  });
}

// Draw i from a fresh stream keyed like sample_counts (sampler.cpp:176-181).
int ref_poisson_grid(double lambda, uint64_t seed, uint32_t t, uint32_t doc, uint32_t word,
                     uint32_t sweep, uint32_t k0, int64_t n, int64_t* out) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      auto s = stream_for(seed, {t, doc, word,
                                 make_tag(StreamPurpose::poisson_counts, sweep,
                                          k0 + static_cast<uint32_t>(i))});
      out[i] = poisson_sample(lambda, s);
    }
  });
}

// n sequential draws from one stream (moments / chi-square tests).
int ref_poisson_stream(double lambda, uint64_t seed, uint32_t t, uint32_t doc, uint32_t word,
                       uint32_t tag, int64_t n, int64_t* out) {
  return guarded([&] {
    auto s = stream_for(seed, {t, doc, word, tag});
    for (int64_t i = 0; i < n; ++i) out[i] = poisson_sample(lambda, s);
  });
}

void* ref_make_corpus(int64_t n_docs, int64_t n_words, int64_t n_topics, double len_mean,
                      uint64_t seed, double theta_conc, double phi_conc) {
  auto* g = new Generated{synthetic::make_corpus(n_docs, n_words, n_topics, len_mean, seed,
                                                 theta_conc, phi_conc)};
  return g;
}

void ref_generated_sizes(void* h, int64_t* n_docs, int64_t* nnz, int64_t* n_tokens) {
  auto* g = static_cast<Generated*>(h);
  *n_docs = g->g.corpus.n_docs;
  *nnz = g->g.corpus.nnz();
  *n_tokens = g->g.corpus.n_tokens;
}

void ref_generated_copy(void* h, int64_t* offsets, int32_t* words, int32_t* counts,
                        double* phi_true) {
  auto* g = static_cast<Generated*>(h);
  const auto& c = g->g.corpus;
  std::memcpy(offsets, c.doc_offsets.data(), sizeof(int64_t) * c.doc_offsets.size());
  std::memcpy(words, c.word_ids.data(), sizeof(int32_t) * c.word_ids.size());
  std::memcpy(counts, c.counts.data(), sizeof(int32_t) * c.counts.size());
  std::memcpy(phi_true, g->g.phi_true.data.data(), sizeof(double) * g->g.phi_true.data.size());
}

void ref_generated_free(void* h) { delete static_cast<Generated*>(h); }

int ref_sddmm(const double* theta_batch, int64_t B, int64_t K_theta, const double* phi,
              int64_t K, int64_t W, const int64_t* offsets, const int32_t* words,
              const int32_t* counts, int64_t n_docs, const int32_t* doc_ids, double* mu_out,
              int64_t mu_cap, int64_t* mu_len, int n_threads) {
  return guarded([&] {
    const Corpus corpus = make_corpus(offsets, words, counts, n_docs, W);
    MiniBatch batch;
    batch.doc_ids.assign(doc_ids, doc_ids + B);
    const auto mu = sddmm(make_matrix(theta_batch, B, K_theta), make_matrix(phi, K, W),
                          corpus, batch, n_threads);
    *mu_len = static_cast<int64_t>(mu.size());
    if (*mu_len > mu_cap) throw ConfigError("mu buffer too small");
    std::memcpy(mu_out, mu.data(), sizeof(double) * mu.size());
  });
}

int ref_sample_counts(const double* theta_batch, int64_t B, int64_t K, const double* phi,
                      int64_t W, const double* mu, int64_t mu_len, const int64_t* offsets,
                      const int32_t* words, const int32_t* counts, int64_t n_docs,
                      const int32_t* doc_ids, double m_t, uint64_t seed, int64_t t, int sweep,
                      int n_threads, int64_t* theta_counts, int64_t* phi_counts) {
  return guarded([&] {
    const Corpus corpus = make_corpus(offsets, words, counts, n_docs, W);
    MiniBatch batch;
    batch.doc_ids.assign(doc_ids, doc_ids + B);
    const auto sc = sample_counts(make_matrix(theta_batch, B, K), make_matrix(phi, K, W),
                                  std::span<const double>(mu, static_cast<size_t>(mu_len)),
                                  corpus, batch, m_t, seed, t, sweep, n_threads);
    std::memcpy(theta_counts, sc.theta_counts.data(), sizeof(int64_t) * sc.theta_counts.size());
    std::memcpy(phi_counts, sc.phi_counts.data(), sizeof(int64_t) * sc.phi_counts.size());
  });
}

int ref_update_model(double* theta, int64_t D, double* phi, int64_t K, int64_t W, double alpha,
                     double beta, const int32_t* doc_ids, int64_t B,
                     const int64_t* theta_counts, const int64_t* phi_counts, double m_t,
                     double rho_t) {
  return guarded([&] {
    Model model;
    model.n_topics = K;
    model.n_words = W;
    model.alpha = alpha;
    model.beta = beta;
    model.phi = make_matrix(phi, K, W);
    model.theta = make_matrix(theta, D, K);
    SampledCounts c;
    c.doc_ids.assign(doc_ids, doc_ids + B);
    c.n_topics = K;
    c.n_words = W;
    c.m_t = m_t;
    c.theta_counts.assign(theta_counts, theta_counts + B * K);
    c.phi_counts.assign(phi_counts, phi_counts + W * K);
    update_model(model, c, rho_t);
    std::memcpy(phi, model.phi.data.data(), sizeof(double) * K * W);
    std::memcpy(theta, model.theta.data.data(), sizeof(double) * D * K);
  });
}

int ref_rho_schedule(int64_t t, double tau0, double gamma, double* out) {
  return guarded([&] { *out = rho_schedule(t, tau0, gamma); });
}

int ref_anneal_m(int schedule, int64_t t, int64_t t_max, double m, double* out) {
  static const AnnealSchedule kinds[4] = {AnnealSchedule::constant, AnnealSchedule::linear,
                                          AnnealSchedule::logarithmic,
                                          AnnealSchedule::invlinear};
  return guarded([&] { *out = anneal_m(kinds[schedule & 3], t, t_max, m); });
}

int ref_fold_in_theta(const double* phi, int64_t K, int64_t W, const int32_t* words,
                      const int32_t* counts, int64_t n, double alpha, int sweeps,
                      double* theta_out) {
  return guarded([&] {
    const auto theta = fold_in_theta(make_matrix(phi, K, W),
                                     std::span<const int32_t>(words, static_cast<size_t>(n)),
                                     std::span<const int32_t>(counts, static_cast<size_t>(n)),
                                     alpha, sweeps);
    std::memcpy(theta_out, theta.data(), sizeof(double) * theta.size());
  });
}

int ref_perword_loglik(const double* phi, int64_t K, int64_t W, const int64_t* offsets,
                       const int32_t* words, const int32_t* counts, int64_t n_docs,
                       double alpha, uint64_t seed, int n_threads, double* ll_out) {
  return guarded([&] {
    const Corpus corpus = make_corpus(offsets, words, counts, n_docs, W);
    *ll_out = perword_loglik(make_matrix(phi, K, W), corpus, alpha, seed, n_threads);
  });
}

int ref_split_holdout_ids(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                          int64_t n_docs, int64_t n_words, double test_fraction, uint64_t seed,
                          int64_t* train_offsets, int32_t* train_words, int32_t* train_counts,
                          int64_t* n_train, int64_t* test_offsets, int32_t* test_words,
                          int32_t* test_counts, int64_t* n_test) {
  return guarded([&] {
    const Corpus corpus = make_corpus(offsets, words, counts, n_docs, n_words);
    const auto [tr, te] = split_holdout(corpus, test_fraction, seed);
    *n_train = tr.n_docs;
    *n_test = te.n_docs;
    std::memcpy(train_offsets, tr.doc_offsets.data(), sizeof(int64_t) * tr.doc_offsets.size());
    std::memcpy(train_words, tr.word_ids.data(), sizeof(int32_t) * tr.word_ids.size());
    std::memcpy(train_counts, tr.counts.data(), sizeof(int32_t) * tr.counts.size());
    std::memcpy(test_offsets, te.doc_offsets.data(), sizeof(int64_t) * te.doc_offsets.size());
    std::memcpy(test_words, te.word_ids.data(), sizeof(int32_t) * te.word_ids.size());
    std::memcpy(test_counts, te.counts.data(), sizeof(int32_t) * te.counts.size());
  });
}

// First n_batches batches of MinibatchStream(corpus of n_docs docs).
int ref_minibatches(int64_t n_docs, double batch_fraction, uint64_t seed, int64_t n_batches,
                    int32_t* out, int64_t* sizes) {
  return guarded([&] {
    Corpus corpus;
    corpus.n_docs = n_docs;
    MinibatchStream stream(corpus, batch_fraction, seed);
    int64_t pos = 0;
    for (int64_t i = 0; i < n_batches; ++i) {
      const auto b = stream.next();
      sizes[i] = static_cast<int64_t>(b.doc_ids.size());
      std::memcpy(out + pos, b.doc_ids.data(), sizeof(int32_t) * b.doc_ids.size());
      pos += sizes[i];
    }
  });
}

struct ref_config {
  int64_t n_topics;
  double m;
  int schedule;
  double tau0, gamma, batch_fraction;
  int64_t t_max, inner_sweeps;
  uint64_t seed;
  double alpha, beta, init_noise;
  int n_threads;
};

struct ref_trace_row {
  int64_t t;
  double passes, samples_per_word, ll, wall_seconds, m_t;
};

int ref_train(const int64_t* offsets, const int32_t* words, const int32_t* counts,
              int64_t n_docs, int64_t n_words, const int64_t* ho_offsets,
              const int32_t* ho_words, const int32_t* ho_counts, int64_t ho_docs,
              const ref_config* cfg, int64_t eval_every, double* phi_out, double* theta_out,
              ref_trace_row* trace_out, int64_t* n_trace) {
  static const AnnealSchedule kinds[4] = {AnnealSchedule::constant, AnnealSchedule::linear,
                                          AnnealSchedule::logarithmic,
                                          AnnealSchedule::invlinear};
  return guarded([&] {
    const Corpus corpus = make_corpus(offsets, words, counts, n_docs, n_words);
    Corpus heldout;
    const Corpus* ho = nullptr;
    if (ho_offsets != nullptr) {
      heldout = make_corpus(ho_offsets, ho_words, ho_counts, ho_docs, n_words);
      ho = &heldout;
    }
    SamplerConfig config;
    config.n_topics = cfg->n_topics;
    config.m = cfg->m;
    config.schedule = kinds[cfg->schedule & 3];
    config.tau0 = cfg->tau0;
    config.gamma = cfg->gamma;
    config.batch_fraction = cfg->batch_fraction;
    config.t_max = cfg->t_max;
    config.inner_sweeps = cfg->inner_sweeps;
    config.seed = cfg->seed;
    config.alpha = cfg->alpha;
    config.beta = cfg->beta;
    config.init_noise = cfg->init_noise;
    config.n_threads = cfg->n_threads;
    auto [model, trace] = train(corpus, config, ho, eval_every);
    std::memcpy(phi_out, model.phi.data.data(), sizeof(double) * model.phi.data.size());
    std::memcpy(theta_out, model.theta.data.data(), sizeof(double) * model.theta.data.size());
    *n_trace = static_cast<int64_t>(trace.size());
    for (size_t i = 0; i < trace.size(); ++i) {
      trace_out[i] = {trace[i].t, trace[i].passes, trace[i].samples_per_word, trace[i].ll,
                      trace[i].wall_seconds, trace[i].m_t};
    }
  });
}

// ---- collapsed Gibbs baseline: cgs_init + sweeps 1..n
// (cgs.cpp:11-98), the state after them; and cgs_train (cgs.cpp:131-157)
int ref_cgs_run(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                int64_t n_docs, int64_t n_words, int64_t K, double alpha, double beta,
                uint64_t seed, int64_t n_sweeps, int32_t* z, int32_t* doc_topic,
                int32_t* word_topic, int64_t* topic_total) {
  return guarded([&] {
    const Corpus corpus = make_corpus(offsets, words, counts, n_docs, n_words);
    CgsState st = cgs_init(corpus, K, alpha, beta, seed);
    for (int64_t s = 1; s <= n_sweeps; ++s) cgs_sweep(st, corpus, seed, s);
    std::memcpy(z, st.z.data(), sizeof(int32_t) * st.z.size());
    std::memcpy(doc_topic, st.doc_topic.data(), sizeof(int32_t) * st.doc_topic.size());
    std::memcpy(word_topic, st.word_topic.data(), sizeof(int32_t) * st.word_topic.size());
    std::memcpy(topic_total, st.topic_total.data(), sizeof(int64_t) * st.topic_total.size());
  });
}

int ref_cgs_train(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                  int64_t n_docs, int64_t n_words, const int64_t* ho_offsets,
                  const int32_t* ho_words, const int32_t* ho_counts, int64_t ho_docs, int64_t K,
                  double alpha, double beta, int64_t n_sweeps, uint64_t seed, int64_t eval_every,
                  int n_threads, double* phi_out, double* theta_out, ref_trace_row* trace_out,
                  int64_t* n_trace) {
  return guarded([&] {
    const Corpus corpus = make_corpus(offsets, words, counts, n_docs, n_words);
    Corpus heldout;
    const Corpus* ho = nullptr;
    if (ho_offsets != nullptr) {
      heldout = make_corpus(ho_offsets, ho_words, ho_counts, ho_docs, n_words);
      ho = &heldout;
    }
    auto [model, trace] = cgs_train(corpus, K, alpha, beta, n_sweeps, seed, eval_every, ho, n_threads);
    std::memcpy(phi_out, model.phi.data.data(), sizeof(double) * model.phi.data.size());
    std::memcpy(theta_out, model.theta.data.data(), sizeof(double) * model.theta.data.size());
    *n_trace = static_cast<int64_t>(trace.size());
    for (size_t i = 0; i < trace.size(); ++i)
      trace_out[i] = {trace[i].t, trace[i].passes, trace[i].samples_per_word, trace[i].ll,
                      trace[i].wall_seconds, trace[i].m_t};
  });
}

// ---- data formats: the reference's own I/O
struct LoadedCorpus {
  Corpus c;
  std::string vocab;  // '\n'-terminated lines
};

void* ref_load_uci(const char* docword, const char* vocab, int* rc) {
  LoadedCorpus* out = nullptr;
  *rc = guarded([&] {
    auto* l = new LoadedCorpus{load_uci_bow(docword, vocab), {}};
    for (const auto& v : l->c.vocab) {
      l->vocab += v;
      l->vocab.push_back('\n');
    }
    out = l;
  });
  return out;
}

void ref_loaded_dims(void* h, int64_t* n_docs, int64_t* n_words, int64_t* nnz, int64_t* n_tokens,
                     int64_t* vocab_bytes) {
  auto* l = static_cast<LoadedCorpus*>(h);
  *n_docs = l->c.n_docs;
  *n_words = l->c.n_words;
  *nnz = l->c.nnz();
  *n_tokens = l->c.n_tokens;
  *vocab_bytes = static_cast<int64_t>(l->vocab.size());
}

void ref_loaded_copy(void* h, int64_t* offsets, int32_t* words, int32_t* counts, char* vocab) {
  auto* l = static_cast<LoadedCorpus*>(h);
  std::memcpy(offsets, l->c.doc_offsets.data(), sizeof(int64_t) * l->c.doc_offsets.size());
  std::memcpy(words, l->c.word_ids.data(), sizeof(int32_t) * l->c.word_ids.size());
  std::memcpy(counts, l->c.counts.data(), sizeof(int32_t) * l->c.counts.size());
  std::memcpy(vocab, l->vocab.data(), l->vocab.size());
}

void ref_loaded_free(void* h) { delete static_cast<LoadedCorpus*>(h); }

int ref_save_uci(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                 int64_t n_docs, int64_t n_words, const char* vocab, int64_t vocab_bytes,
                 const char* docword, const char* vocab_path) {
  return guarded([&] {
    Corpus c = make_corpus(offsets, words, counts, n_docs, n_words);
    std::string cur;
    for (int64_t i = 0; i < vocab_bytes; ++i) {
      if (vocab[i] == '\n') {
        c.vocab.push_back(cur);
        cur.clear();
      } else {
        cur.push_back(vocab[i]);
      }
    }
    save_uci_bow(c, docword, vocab_path);
  });
}

int ref_save_checkpoint(const char* path, int64_t K, int64_t W, double alpha, double beta,
                        const double* phi) {
  return guarded([&] {
    Model m;
    m.n_topics = K;
    m.n_words = W;
    m.alpha = alpha;
    m.beta = beta;
    m.phi = DenseMatrix(K, W);
    std::memcpy(m.phi.data.data(), phi, sizeof(double) * K * W);
    save_checkpoint(m, path);
  });
}

int ref_load_checkpoint(const char* path, int64_t* K, int64_t* W, double* alpha, double* beta,
                        double* phi, int64_t cap) {
  return guarded([&] {
    const Model m = load_checkpoint(path);
    *K = m.n_topics;
    *W = m.n_words;
    *alpha = m.alpha;
    *beta = m.beta;
    if (phi && cap >= m.n_topics * m.n_words)
      std::memcpy(phi, m.phi.data.data(), sizeof(double) * m.phi.data.size());
  });
}

struct RefTraceRow {
  int64_t t;
  double passes, samples_per_word, ll, wall_seconds, m_t;
};

int ref_write_metrics_csv(const char* path, const RefTraceRow* rows, int64_t n) {
  return guarded([&] {
    MetricsTrace tr;
    for (int64_t i = 0; i < n; ++i)
      tr.push_back(TraceRow{rows[i].t, rows[i].passes, rows[i].samples_per_word, rows[i].ll,
                            rows[i].wall_seconds, rows[i].m_t});
    write_metrics_csv(tr, path);
  });
}

int ref_read_metrics_csv(const char* path, RefTraceRow* rows, int64_t cap, int64_t* n) {
  return guarded([&] {
    const MetricsTrace tr = read_metrics_csv(path);
    *n = static_cast<int64_t>(tr.size());
    for (int64_t i = 0; i < *n && i < cap; ++i)
      rows[i] = RefTraceRow{tr[i].t, tr[i].passes, tr[i].samples_per_word, tr[i].ll,
                            tr[i].wall_seconds, tr[i].m_t};
  });
}

}  // extern "C"
