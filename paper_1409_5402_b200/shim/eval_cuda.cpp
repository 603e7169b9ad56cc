// eval_cuda.cpp -- drop-in replacement for the reference's src/eval.cpp.
//
// fold_in_theta and perword_loglik run on the device through the C ABI
// (include/samelda_cu.h); the metrics-CSV pair (eval.hpp:45-49) goes through
// the library's host formats (include/samelda_io.h), since this translation
// unit replaces eval.cpp as a whole.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <mutex>
#include <string>
#include <vector>

#include "samelda/errors.hpp"
#include "samelda/eval.hpp"
#include "samelda_cu.h"
#include "samelda_io.h"

namespace samelda {
namespace cuda_shim {
samelda_cu_ctx* context();
std::mutex& lock();
void check(int rc, const char* what);
samelda_cu_corpus view(const Corpus& c);
}  // namespace cuda_shim

std::vector<double> fold_in_theta(const DenseMatrix& phi, std::span<const std::int32_t> words,
                                  std::span<const std::int32_t> counts, double alpha,
                                  int sweeps) {
  std::vector<double> theta(static_cast<std::size_t>(phi.rows));
  static const std::int32_t none = 0;
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  cuda_shim::check(samelda_cu_fold_in_theta(cuda_shim::context(), phi.data.data(), phi.rows, phi.cols,
                                            words.empty() ? &none : words.data(),
                                            counts.empty() ? &none : counts.data(),
                                            static_cast<std::int64_t>(words.size()), alpha, sweeps,
                                            theta.data()),
                   "fold_in_theta");
  return theta;
}

double perword_loglik(const DenseMatrix& phi, const Corpus& test_corpus, double alpha,
                      std::uint64_t seed, int /*n_threads*/) {
  if (test_corpus.n_docs < 1) throw ConfigError("perword_loglik: test corpus is empty");
  if (phi.cols != test_corpus.n_words)
    throw ConfigError("perword_loglik: phi width disagrees with corpus vocabulary");
  double ll = 0.0;
  const std::lock_guard<std::mutex> g(cuda_shim::lock());
  const samelda_cu_corpus cv = cuda_shim::view(test_corpus);
  cuda_shim::check(samelda_cu_perword_loglik(cuda_shim::context(), phi.data.data(), phi.rows,
                                             phi.cols, &cv, alpha, seed, &ll),
                   "perword_loglik");
  return ll;
}

// eval.cpp:161-210 -- the metrics-CSV pair through include/samelda_io.h
// (byte-identical files, same IoErrors)
void write_metrics_csv(const MetricsTrace& trace, const std::string& path) {
  std::vector<samelda_cu_trace_row> rows(trace.size());
  for (std::size_t i = 0; i < trace.size(); ++i)
    rows[i] = {trace[i].t, trace[i].passes, trace[i].samples_per_word, trace[i].ll,
               trace[i].wall_seconds, trace[i].m_t};
  if (samelda_io_write_metrics_csv(path.c_str(), rows.data(), static_cast<int64_t>(rows.size())))
    throw IoError(samelda_io_last_error());
}

MetricsTrace read_metrics_csv(const std::string& path) {
  int64_t n = 0;
  if (samelda_io_read_metrics_csv(path.c_str(), nullptr, 0, &n)) throw IoError(samelda_io_last_error());
  std::vector<samelda_cu_trace_row> rows(static_cast<std::size_t>(n));
  if (samelda_io_read_metrics_csv(path.c_str(), rows.data(), n, &n))
    throw IoError(samelda_io_last_error());
  MetricsTrace trace;
  for (const auto& r : rows)
    trace.push_back(TraceRow{r.t, r.passes, r.samples_per_word, r.ll, r.wall_seconds, r.m_t});
  return trace;
}

}  // namespace samelda
