// cgs_cuda.cpp -- drop-in replacement for the reference's src/cgs.cpp.
//
// Compiled against the reference's unchanged cgs.hpp: the collapsed Gibbs
// baseline (cgs_init / cgs_sweep / cgs_model / cgs_train) runs on the device
// through the C ABI (include/samelda_cu.h, samelda_cu_cgs_*), with the
// reference's draws and its ConfigError behaviour.  CgsState stays the
// reference's host value type: a per-call cgs_sweep / cgs_model uploads the
// state, runs on the device and writes it back; cgs_train keeps the chain
// device-resident for all its sweeps.  The device sampler supports
// n_topics <= 1024.
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "samelda/cgs.hpp"
#include "samelda/errors.hpp"
#include "samelda_cu.h"

namespace samelda {
namespace cuda_shim {
samelda_cu_ctx* context();
std::mutex& lock();
void check(int rc, const char* what);
samelda_cu_corpus view(const Corpus& c);
}  // namespace cuda_shim

namespace {

void validate(std::int64_t n_topics, double alpha, double beta) {
  // cgs.cpp:13-18
  if (n_topics < 1) throw ConfigError("cgs_init: n_topics must be >= 1");
  if (!(alpha > 0.0) || !(beta > 0.0)) throw ConfigError("cgs_init: alpha and beta must be positive");
}

void download(CgsState& st) {
  cuda_shim::check(samelda_cu_cgs_state(cuda_shim::context(), st.z.data(), st.doc_topic.data(),
                                        st.word_topic.data(), st.topic_total.data()),
                   "cgs state");
}

// the device chain at `st` (the corpus and K, alpha, beta are re-bound; the
// seed of the init draw is irrelevant: the state overwrites it)
void upload(const CgsState& st, const Corpus& corpus) {
  const samelda_cu_corpus cv = cuda_shim::view(corpus);
  cuda_shim::check(samelda_cu_cgs_init(cuda_shim::context(), &cv, st.n_topics, st.alpha, st.beta, 0),
                   "cgs state");
  cuda_shim::check(samelda_cu_cgs_set_state(cuda_shim::context(), st.z.data(), st.doc_topic.data(),
                                            st.word_topic.data(), st.topic_total.data()),
                   "cgs state");
}

}  // namespace

CgsState cgs_init(const Corpus& corpus, std::int64_t n_topics, double alpha, double beta,
                  std::uint64_t seed) {
  validate(n_topics, alpha, beta);
  CgsState state;
  state.n_topics = n_topics;
  state.n_docs = corpus.n_docs;
  state.n_words = corpus.n_words;
  state.alpha = alpha;
  state.beta = beta;
  state.token_offsets.assign(1, 0);
  for (const auto c : corpus.counts) state.token_offsets.push_back(state.token_offsets.back() + c);
  state.z.assign(static_cast<std::size_t>(state.token_offsets.back()), 0);
  state.doc_topic.assign(static_cast<std::size_t>(corpus.n_docs * n_topics), 0);
  state.word_topic.assign(static_cast<std::size_t>(corpus.n_words * n_topics), 0);
  state.topic_total.assign(static_cast<std::size_t>(n_topics), 0);
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  const samelda_cu_corpus cv = cuda_shim::view(corpus);
  cuda_shim::check(samelda_cu_cgs_init(cuda_shim::context(), &cv, n_topics, alpha, beta, seed),
                   "cgs_init");
  download(state);
  return state;
}

void cgs_sweep(CgsState& state, const Corpus& corpus, std::uint64_t master_seed,
               std::int64_t sweep_index) {
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  upload(state, corpus);
  cuda_shim::check(samelda_cu_cgs_sweep(cuda_shim::context(), master_seed, sweep_index), "cgs_sweep");
  download(state);
}

Model cgs_model(const CgsState& state) {
  Model model;
  model.n_topics = state.n_topics;
  model.n_words = state.n_words;
  model.alpha = state.alpha;
  model.beta = state.beta;
  model.phi = DenseMatrix(state.n_topics, state.n_words);
  model.theta = DenseMatrix(state.n_docs, state.n_topics);
  // a corpus view with the state's shape (the model needs only the counts)
  Corpus shape;
  shape.n_docs = state.n_docs;
  shape.n_words = state.n_words;
  shape.doc_offsets.assign(static_cast<std::size_t>(state.n_docs) + 1, 0);
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  const samelda_cu_corpus cv = cuda_shim::view(shape);
  cuda_shim::check(samelda_cu_cgs_init(cuda_shim::context(), &cv, state.n_topics, state.alpha,
                                       state.beta, 0),
                   "cgs_model");
  cuda_shim::check(samelda_cu_cgs_set_state(cuda_shim::context(), nullptr, state.doc_topic.data(),
                                            state.word_topic.data(), state.topic_total.data()),
                   "cgs_model");
  cuda_shim::check(samelda_cu_cgs_model(cuda_shim::context(), model.phi.data.data(),
                                        model.theta.data.data()),
                   "cgs_model");
  return model;
}

std::pair<Model, MetricsTrace> cgs_train(const Corpus& corpus, std::int64_t n_topics, double alpha,
                                         double beta, std::int64_t n_sweeps, std::uint64_t seed,
                                         std::int64_t eval_every, const Corpus* heldout,
                                         int /*n_threads_eval*/) {
  if (n_sweeps < 0) throw ConfigError("cgs_train: n_sweeps must be >= 0");
  validate(n_topics, alpha, beta);
  Model model;
  model.n_topics = n_topics;
  model.n_words = corpus.n_words;
  model.alpha = alpha;
  model.beta = beta;
  model.phi = DenseMatrix(n_topics, corpus.n_words);
  model.theta = DenseMatrix(corpus.n_docs, n_topics);
  std::vector<samelda_cu_trace_row> rows(static_cast<std::size_t>(std::max<std::int64_t>(n_sweeps, 1)));
  std::int64_t n_rows = 0;
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  const samelda_cu_corpus cv = cuda_shim::view(corpus);
  samelda_cu_corpus hv{};
  if (heldout != nullptr) hv = cuda_shim::view(*heldout);
  cuda_shim::check(samelda_cu_cgs_train(cuda_shim::context(), &cv, n_topics, alpha, beta, n_sweeps,
                                        seed, eval_every, heldout != nullptr ? &hv : nullptr,
                                        model.phi.data.data(), model.theta.data.data(), rows.data(),
                                        static_cast<std::int64_t>(rows.size()), &n_rows),
                   "cgs_train");
  MetricsTrace trace;
  for (std::int64_t i = 0; i < n_rows; ++i) {
    const auto& r = rows[static_cast<std::size_t>(i)];
    trace.push_back({r.t, r.passes, r.samples_per_word, r.ll, r.wall_seconds, r.m_t});
  }
  return {std::move(model), std::move(trace)};
}

}  // namespace samelda
