// sampler_cuda.cpp -- drop-in replacement for the reference's src/sampler.cpp.
//
// Compiled against the reference's own, unchanged headers
// (proj/include/samelda/sampler.hpp et al.); every function keeps its
// signature and error behaviour and forwards to libsamelda_cuda.so through
// the C ABI in include/samelda_cu.h.  Link this file (and eval_cuda.cpp) in
// place of sampler.cpp / eval.cpp; the rest of the reference library (corpus,
// model, rng, cgs, commands) and its CLI link unchanged.  See INTEGRATION.md.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "samelda/errors.hpp"
#include "samelda/sampler.hpp"
#include "samelda_cu.h"

namespace samelda {
namespace cuda_shim {

// One device context per process (the reference API carries no handle).
samelda_cu_ctx* context() {
  static std::once_flag once;
  static samelda_cu_ctx* ctx = nullptr;
  std::call_once(once, [] {
    if (samelda_cu_create(0, &ctx) != SAMELDA_CU_OK) ctx = nullptr;
  });
  if (ctx == nullptr) throw std::runtime_error("samelda_cu: no usable CUDA device");
  return ctx;
}

// The devices train() shards over: SAMELDA_CU_DEVICES as a
// comma-separated list of device ids ("0,1,2,3"; repeating one device, e.g.
// "0,0", is the one-GPU test mode of the group), else every visible device.
// One device -> the single context above; more -> a samelda_cu_group.  The
// result does not depend on the choice (global Philox doc ids, integer
// counts), as the reference's n_threads never changes results.
samelda_cu_group* group() {
  static std::once_flag once;
  static samelda_cu_group* grp = nullptr;
  static bool single = false;
  std::call_once(once, [] {
    std::vector<int> devs;
    if (const char* e = std::getenv("SAMELDA_CU_DEVICES")) {
      std::string s(e);
      size_t pos = 0;
      while (pos < s.size()) {
        const size_t comma = s.find(',', pos);
        const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        if (!tok.empty()) devs.push_back(std::atoi(tok.c_str()));
        if (comma == std::string::npos) break;
        pos = comma + 1;
      }
    } else {
      const int n = samelda_cu_device_count();
      for (int d = 0; d < n; ++d) devs.push_back(d);
    }
    if (devs.size() <= 1) {
      single = true;
      return;
    }
    if (samelda_cu_group_create(devs.data(), static_cast<int>(devs.size()), &grp) != SAMELDA_CU_OK)
      grp = nullptr;
  });
  if (grp == nullptr && !single) throw std::runtime_error("samelda_cu: cannot form the device group (SAMELDA_CU_DEVICES / NCCL)");
  return grp;
}

std::mutex& lock() {
  static std::mutex m;
  return m;
}

// return code -> the reference's exception classes (errors.hpp:7-20)
void check(int rc, const char* what) {
  if (rc == SAMELDA_CU_OK) return;
  const std::string msg = std::string(what) + ": " + samelda_cu_last_error(context());
  switch (rc) {
    case SAMELDA_CU_CONFIG: throw ConfigError(msg);
    case SAMELDA_CU_IO: throw IoError(msg);
    case SAMELDA_CU_NUMERICAL: throw NumericalError(msg);
    default: throw std::runtime_error(msg);
  }
}

samelda_cu_corpus view(const Corpus& c) {
  static const int32_t empty = 0;
  return samelda_cu_corpus{c.doc_offsets.data(), c.word_ids.empty() ? &empty : c.word_ids.data(),
                           c.counts.empty() ? &empty : c.counts.data(), c.n_docs, c.n_words};
}

int32_t schedule_code(AnnealSchedule s) {
  switch (s) {
    case AnnealSchedule::constant: return SAMELDA_CU_SCHEDULE_CONSTANT;
    case AnnealSchedule::linear: return SAMELDA_CU_SCHEDULE_LINEAR;
    case AnnealSchedule::logarithmic: return SAMELDA_CU_SCHEDULE_LOG;
    case AnnealSchedule::invlinear: return SAMELDA_CU_SCHEDULE_INVLINEAR;
  }
  return SAMELDA_CU_SCHEDULE_CONSTANT;
}

}  // namespace cuda_shim

using cuda_shim::check;
using cuda_shim::context;

AnnealSchedule parse_schedule(std::string_view name) {
  if (name == "constant") return AnnealSchedule::constant;
  if (name == "linear") return AnnealSchedule::linear;
  if (name == "log") return AnnealSchedule::logarithmic;
  if (name == "invlinear") return AnnealSchedule::invlinear;
  throw ConfigError("unknown schedule '" + std::string(name) +
                    "' (expected constant|linear|log|invlinear)");
}

std::string schedule_name(AnnealSchedule schedule) {
  switch (schedule) {
    case AnnealSchedule::constant: return "constant";
    case AnnealSchedule::linear: return "linear";
    case AnnealSchedule::logarithmic: return "log";
    case AnnealSchedule::invlinear: return "invlinear";
  }
  return "constant";
}

void validate(const SamplerConfig& c) {
  // the same domain checks as the reference (sampler.cpp:47-78)
  if (c.n_topics < 1 || c.n_topics >= (1 << 20)) throw ConfigError("n_topics must be in [1, 2^20)");
  if (!(c.m > 0.0) || !std::isfinite(c.m)) throw ConfigError("m must be positive and finite");
  if (!(c.tau0 >= 1.0)) throw ConfigError("tau0 must be >= 1");
  if (!(c.gamma >= 0.5 && c.gamma <= 1.0)) throw ConfigError("gamma must be in [0.5, 1]");
  if (!(c.batch_fraction > 0.0 && c.batch_fraction <= 1.0))
    throw ConfigError("batch_fraction must be in (0, 1]");
  if (c.t_max < 0) throw ConfigError("t_max must be >= 0");
  if (c.inner_sweeps < 1 || c.inner_sweeps > 255) throw ConfigError("inner_sweeps must be in [1, 255]");
  if (!(c.alpha > 0.0) || !(c.beta > 0.0)) throw ConfigError("alpha and beta must be positive");
  if (c.n_threads < 1) throw ConfigError("n_threads must be >= 1");
  if (!(c.init_noise >= 0.0) || !std::isfinite(c.init_noise))
    throw ConfigError("init_noise must be finite and >= 0");
}

std::int64_t SampledCounts::theta_total() const {
  return std::accumulate(theta_counts.begin(), theta_counts.end(), std::int64_t{0});
}

std::int64_t SampledCounts::phi_total() const {
  return std::accumulate(phi_counts.begin(), phi_counts.end(), std::int64_t{0});
}

std::vector<double> sddmm(const DenseMatrix& theta_batch, const DenseMatrix& phi,
                          const Corpus& corpus, const MiniBatch& batch, int /*n_threads*/) {
  if (theta_batch.cols != phi.rows) throw ConfigError("sddmm: theta columns must match phi rows");
  if (theta_batch.rows != static_cast<std::int64_t>(batch.doc_ids.size()))
    throw ConfigError("sddmm: theta rows must match the batch size");
  if (phi.cols != corpus.n_words) throw ConfigError("sddmm: phi columns must match the vocabulary size");
  std::int64_t nnz = 0;
  for (const auto d : batch.doc_ids) nnz += corpus.doc_nnz(d);
  std::vector<double> mu(static_cast<std::size_t>(nnz));
  if (batch.doc_ids.empty()) return mu;
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  const samelda_cu_corpus cv = cuda_shim::view(corpus);
  std::int64_t len = 0;
  check(samelda_cu_sddmm(context(), &cv, theta_batch.data.data(), theta_batch.rows, theta_batch.cols,
                         phi.data.data(), phi.rows, phi.cols, batch.doc_ids.data(),
                         mu.data(), nnz, &len),
        "sddmm");
  return mu;
}

SampledCounts sample_counts(const DenseMatrix& theta_batch, const DenseMatrix& phi,
                            std::span<const double> mu, const Corpus& corpus,
                            const MiniBatch& batch, double m_t, std::uint64_t master_seed,
                            std::int64_t t, int sweep, int /*n_threads*/) {
  SampledCounts counts;
  counts.doc_ids = batch.doc_ids;
  counts.n_topics = phi.rows;
  counts.n_words = phi.cols;
  counts.m_t = m_t;
  const auto B = static_cast<std::int64_t>(batch.doc_ids.size());
  counts.theta_counts.assign(static_cast<std::size_t>(B * phi.rows), 0);
  counts.phi_counts.assign(static_cast<std::size_t>(phi.cols * phi.rows), 0);
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  const samelda_cu_corpus cv = cuda_shim::view(corpus);
  static const double no_mu = 0.0;
  static const std::int32_t no_ids = 0;
  check(samelda_cu_sample_counts(context(), &cv, theta_batch.data.empty() ? &no_mu : theta_batch.data.data(),
                                 B, B ? theta_batch.cols : phi.rows, phi.data.data(), phi.rows,
                                 phi.cols, mu.empty() ? &no_mu : mu.data(),
                                 static_cast<std::int64_t>(mu.size()),
                                 B ? batch.doc_ids.data() : &no_ids, m_t, master_seed, t, sweep,
                                 counts.theta_counts.data(), counts.phi_counts.data()),
        "sample_counts");
  return counts;
}

void update_model(Model& model, const SampledCounts& counts, double rho_t) {
  if (!(rho_t > 0.0 && rho_t <= 1.0)) throw ConfigError("update_model: rho_t must be in (0, 1]");
  if (counts.n_topics != model.n_topics || counts.n_words != model.n_words)
    throw ConfigError("update_model: counts are not shaped for this model");
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  check(samelda_cu_update_model(context(), model.theta.data.data(), model.theta.rows,
                                model.phi.data.data(), model.n_topics, model.n_words, model.alpha,
                                model.beta, counts.doc_ids.data(),
                                static_cast<std::int64_t>(counts.doc_ids.size()),
                                counts.theta_counts.data(), counts.phi_counts.data(), counts.m_t,
                                rho_t),
        "update_model");
}

double rho_schedule(std::int64_t t, double tau0, double gamma) {
  double out = 0.0;
  const int rc = samelda_cu_rho_schedule(t, tau0, gamma, &out);
  if (rc) throw ConfigError("rho_schedule: argument out of range");
  return out;
}

double anneal_m(AnnealSchedule schedule, std::int64_t t, std::int64_t t_max, double m) {
  double out = 0.0;
  const int rc = samelda_cu_anneal_m(cuda_shim::schedule_code(schedule), t, t_max, m, &out);
  if (rc) throw ConfigError("anneal_m: t must be in [1, t_max]");
  return out;
}

std::pair<Model, MetricsTrace> train(const Corpus& corpus, const SamplerConfig& config,
                                     const Corpus* heldout, std::int64_t eval_every) {
  validate(config);
  if (corpus.n_docs < 1) throw ConfigError("train: corpus is empty");
  samelda_cu_config c{};
  c.n_topics = config.n_topics;
  c.m = config.m;
  c.schedule = cuda_shim::schedule_code(config.schedule);
  c.tau0 = config.tau0;
  c.gamma = config.gamma;
  c.batch_fraction = config.batch_fraction;
  c.t_max = config.t_max;
  c.inner_sweeps = config.inner_sweeps;
  c.seed = config.seed;
  c.alpha = config.alpha;
  c.beta = config.beta;
  c.init_noise = config.init_noise;
  c.mode = SAMELDA_CU_MODE_PARITY;
  Model model;
  model.n_topics = config.n_topics;
  model.n_words = corpus.n_words;
  model.alpha = config.alpha;
  model.beta = config.beta;
  model.phi = DenseMatrix(config.n_topics, corpus.n_words);
  model.theta = DenseMatrix(corpus.n_docs, config.n_topics);
  std::vector<samelda_cu_trace_row> rows(static_cast<std::size_t>(std::max<std::int64_t>(config.t_max, 1)));
  std::int64_t n_rows = 0;
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  const samelda_cu_corpus cv = cuda_shim::view(corpus);
  samelda_cu_corpus hv{};
  if (heldout != nullptr) hv = cuda_shim::view(*heldout);
  if (samelda_cu_group* grp = cuda_shim::group()) {
    const int rc = samelda_cu_group_train(grp, &cv, &c, heldout != nullptr ? &hv : nullptr, eval_every,
                                          model.phi.data.data(), model.theta.data.data(), rows.data(),
                                          static_cast<std::int64_t>(rows.size()), &n_rows);
    if (rc != SAMELDA_CU_OK) {
      const std::string msg = std::string("train: ") + samelda_cu_group_last_error(grp);
      if (rc == SAMELDA_CU_CONFIG) throw ConfigError(msg);
      if (rc == SAMELDA_CU_NUMERICAL) throw NumericalError(msg);
      throw std::runtime_error(msg);
    }
  } else {
    check(samelda_cu_train(context(), &cv, &c, heldout != nullptr ? &hv : nullptr, eval_every,
                           model.phi.data.data(), model.theta.data.data(), rows.data(),
                           static_cast<std::int64_t>(rows.size()), &n_rows),
          "train");
  }
  MetricsTrace trace;
  for (std::int64_t i = 0; i < n_rows; ++i) {
    const auto& r = rows[static_cast<std::size_t>(i)];
    trace.push_back({r.t, r.passes, r.samples_per_word, r.ll, r.wall_seconds, r.m_t});
  }
  return {std::move(model), std::move(trace)};
}

}  // namespace samelda
