// eval_cuda.cpp -- drop-in replacement for the reference's src/eval.cpp.
//
// fold_in_theta and perword_loglik run on the device through the C ABI
// (include/samelda_cu.h); the metrics-CSV pair is the reference's host file
// format (eval.hpp:45-49: header "t,passes,samples_per_word,ll,wall_seconds,m_t",
// %.17g fields) restated here because this translation unit replaces eval.cpp
// as a whole.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <mutex>
#include <string>
#include <vector>

#include "samelda/errors.hpp"
#include "samelda/eval.hpp"
#include "samelda_cu.h"

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

void write_metrics_csv(const MetricsTrace& trace, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot write metrics csv: " + path);
  out << "t,passes,samples_per_word,ll,wall_seconds,m_t\n";
  char line[256];
  for (const auto& row : trace) {
    std::snprintf(line, sizeof(line), "%lld,%.17g,%.17g,%.17g,%.17g,%.17g\n",
                  static_cast<long long>(row.t), row.passes, row.samples_per_word, row.ll,
                  row.wall_seconds, row.m_t);
    out << line;
  }
  if (!out) throw IoError("write failed: " + path);
}

MetricsTrace read_metrics_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open metrics csv: " + path);
  std::string header;
  if (!std::getline(in, header) || header != "t,passes,samples_per_word,ll,wall_seconds,m_t")
    throw IoError("unexpected metrics csv header in " + path);
  MetricsTrace trace;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    TraceRow row;
    char* end = nullptr;
    row.t = std::strtoll(line.c_str(), &end, 10);
    double* fields[] = {&row.passes, &row.samples_per_word, &row.ll, &row.wall_seconds, &row.m_t};
    for (double* f : fields) {
      if (*end != ',') throw IoError("malformed metrics csv row in " + path);
      *f = std::strtod(end + 1, &end);
    }
    trace.push_back(row);
  }
  return trace;
}

}  // namespace samelda
