// synth.cpp -- fast synthetic LDA corpora of NYTimes / PubMed shape (host C++).
//
// The reference's generator (tests/support/synthetic.cpp:61-106) draws every
// token with a linear categorical scan over W words: ~10 h for a NYTimes-sized
// corpus.  This one keeps the LDA generative story but
// is O(1) per token (Walker alias tables), threaded over documents, and
// deterministic for any thread count (one Philox stream per document).
//
//   topic k:  phi_k = (1 - bg) * Zipf(s) over a topic-specific permutation of
//             the vocabulary + bg * a shared Zipf(s) background
//   doc d:    length ~ 1 + round(L * Gamma(a)/a) (broad, NYTimes-like),
//             T_d ~ 1 + Geometric topics drawn uniformly, Exp(1) weights,
//             tokens: topic by weight, word from the topic's alias table
//
// (zipf_s, background) are tuned so nnz/token ~ 0.70 at NYTimes shape
// (real NYTimes: 69.7M nonzeros / 99.5M tokens).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/samelda_synth.h"
#include "philox.cuh"

namespace {

struct Alias {
  std::vector<float> prob;
  std::vector<int32_t> alias;
};

Alias build_alias(const std::vector<double>& p) {
  const int64_t n = static_cast<int64_t>(p.size());
  Alias a;
  a.prob.resize(n);
  a.alias.resize(n);
  std::vector<double> q(n);
  std::vector<int64_t> small, large;
  for (int64_t i = 0; i < n; ++i) {
    q[i] = p[i] * static_cast<double>(n);
    (q[i] < 1.0 ? small : large).push_back(i);
  }
  while (!small.empty() && !large.empty()) {
    const int64_t s = small.back(), l = large.back();
    small.pop_back();
    a.prob[s] = static_cast<float>(q[s]);
    a.alias[s] = static_cast<int32_t>(l);
    q[l] = (q[l] + q[s]) - 1.0;
    if (q[l] < 1.0) {
      large.pop_back();
      small.push_back(l);
    }
  }
  for (int64_t i : large) {
    a.prob[i] = 1.0f;
    a.alias[i] = static_cast<int32_t>(i);
  }
  for (int64_t i : small) {
    a.prob[i] = 1.0f;
    a.alias[i] = static_cast<int32_t>(i);
  }
  return a;
}

struct Rng {
  scu::Stream s;
  double u() { return s.uniform_oo(); }
  uint32_t u32() { return s.next_u32(); }
  double normal() {
    const double u1 = u(), u2 = u();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  double gamma(double a) {  // Marsaglia-Tsang
    if (a < 1.0) return gamma(a + 1.0) * std::pow(u(), 1.0 / a);
    const double d = a - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * d);
    for (;;) {
      const double x = normal(), t = 1.0 + c * x;
      if (t <= 0.0) continue;
      const double v = t * t * t;
      if (std::log(u()) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v;
    }
  }
};

struct Generated {
  std::vector<int64_t> offsets;
  std::vector<int32_t> words;
  std::vector<int32_t> counts;
};

}  // namespace

// ------------------------------------------------------------------------
// The reference's own generator, value for value: synthetic::make_corpus
// (tests/support/synthetic.cpp:61-106) on the reference's streams
// (rng.cpp:90-137: phi rows from one stream keyed (0,0,0,tag(synthetic,1)),
// document d from (0,d,0,tag(synthetic,2))), with poisson_sample and
// categorical_sample (rng.cpp:139-179) restated.  BASELINE.json configs[0]
// is this corpus at (10000, 5000, 32, 100, seed 1).  Two changes of method,
// not of result: documents are generated in parallel (each has its own
// stream), and a token's categorical scan over a phi row is a binary search
// over that row's running sums, which are the scan's own partial sums
// (same order, same rounding; they are non-decreasing, so the first index
// with u < cum is the same).
namespace refgen {

constexpr uint32_t kSynthetic = 7;

double normal_variate(scu::Stream& s) {  // synthetic.cpp:17-22
  const double u1 = s.uniform_oo();
  const double u2 = s.uniform_oo();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
}

double gamma_variate(double shape, scu::Stream& s) {  // synthetic.cpp:38-58
  if (shape < 1.0) {
    const double u = s.uniform_oo();  // drawn BEFORE the recursive variate
    const double g = gamma_variate(shape + 1.0, s);
    return g * std::pow(u, 1.0 / shape);
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / std::sqrt(9.0 * d);
  for (;;) {
    const double x = normal_variate(s);
    const double t = 1.0 + c * x;
    if (t <= 0.0) continue;
    const double v = t * t * t;
    const double u = s.uniform_oo();
    if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v;
  }
}

void dirichlet_variate(int64_t k, double conc, scu::Stream& s, double* out) {  // :24-35
  double total = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    out[i] = gamma_variate(conc, s);
    total += out[i];
  }
  for (int64_t i = 0; i < k; ++i) out[i] /= total;
}

int64_t poisson_sample(double lambda, scu::Stream& s) {  // rng.cpp:39-86,139-150
  if (lambda == 0.0) return 0;
  if (lambda < 10.0) {
    const double u = s.uniform();
    double pmf = std::exp(-lambda), cdf = pmf;
    int64_t k = 0;
    while (u > cdf && k < 1000) {
      ++k;
      pmf *= lambda / static_cast<double>(k);
      cdf += pmf;
    }
    return k;
  }
  const double log_lambda = std::log(lambda);
  const double b = 0.931 + 2.53 * std::sqrt(lambda);
  const double a = -0.059 + 0.02483 * b;
  const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4);
  const double v_r = 0.9277 - 3.6224 / (b - 2.0);
  for (;;) {
    const double u = s.uniform_oo() - 0.5;
    const double v = s.uniform_oo();
    const double us = 0.5 - std::abs(u);
    const double g = (2.0 * a / us + b) * u + lambda + 0.43;
    if (us >= 0.07 && v <= v_r) return static_cast<int64_t>(g);
    if (g < 0.0 || g > 9.0e18 || (us < 0.013 && v > us)) continue;
    const int64_t k = static_cast<int64_t>(g);
    const double lhs = std::log(v * inv_alpha / (a / (us * us) + b));
    const double rhs = -lambda + static_cast<double>(k) * log_lambda -
                       std::lgamma(static_cast<double>(k) + 1.0);
    if (lhs <= rhs) return k;
  }
}

// categorical_sample (rng.cpp:152-179) given the weights' running sums
// cum[0..n-1] (cum[n-1] = the total, summed in the same order)
int categorical(const double* w, const double* cum, int64_t n, scu::Stream& s) {
  const double u = s.uniform() * cum[n - 1];
  // first k < n - 1 with u < cum[k]
  int64_t lo = 0, hi = n - 1;  // answer in [lo, hi]; hi = n - 1 means "none"
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (u < cum[mid]) hi = mid; else lo = mid + 1;
  }
  if (lo < n - 1) return static_cast<int>(lo);
  for (int64_t k = n; k-- > 0;)
    if (w[k] > 0.0) return static_cast<int>(k);
  return 0;
}

}  // namespace refgen

extern "C" {

int samelda_synth_generate(const samelda_synth_params* p, int n_threads, void** handle,
                           int64_t* nnz, int64_t* n_tokens) {
  if (!p || p->n_docs < 1 || p->n_words < 1 || p->n_topics_gen < 1 || !(p->mean_len >= 1.0) ||
      !(p->len_shape > 0.0) || !(p->zipf_s > 0.0) || p->background < 0.0 ||
      p->background > 1.0 || handle == nullptr)
    return 1;
  const int64_t W = p->n_words, KG = p->n_topics_gen, D = p->n_docs;
  // Zipf base weights over ranks
  std::vector<double> zipf(W);
  double zs = 0.0;
  for (int64_t r = 0; r < W; ++r) zs += (zipf[r] = std::pow(static_cast<double>(r + 1), -p->zipf_s));
  for (auto& z : zipf) z /= zs;
  // background ranks: a fixed permutation
  auto permutation = [&](uint32_t key) {
    std::vector<int32_t> perm(W);
    for (int64_t i = 0; i < W; ++i) perm[i] = static_cast<int32_t>(i);
    scu::Stream s;
    s.init(p->seed, key, 0, 0, scu::make_tag(7, 4, 0));
    for (int64_t i = W - 1; i > 0; --i) {
      const int64_t j = static_cast<int64_t>(s.next_u64() % static_cast<uint64_t>(i + 1));
      std::swap(perm[i], perm[j]);
    }
    return perm;
  };
  const std::vector<int32_t> bg_perm = permutation(0xffffffffu);
  std::vector<double> bg(W, 0.0);
  for (int64_t r = 0; r < W; ++r) bg[bg_perm[r]] = zipf[r];
  std::vector<Alias> tables(static_cast<size_t>(KG));
  {
    std::vector<std::thread> th;
    const int nt = std::max(1, n_threads);
    for (int w = 0; w < nt; ++w) {
      th.emplace_back([&, w] {
        for (int64_t k = w; k < KG; k += nt) {
          const std::vector<int32_t> perm = permutation(static_cast<uint32_t>(k));
          std::vector<double> phi(W);
          for (int64_t i = 0; i < W; ++i) phi[i] = p->background * bg[i];
          for (int64_t r = 0; r < W; ++r) phi[perm[r]] += (1.0 - p->background) * zipf[r];
          tables[static_cast<size_t>(k)] = build_alias(phi);
        }
      });
    }
    for (auto& t : th) t.join();
  }
  // documents, in contiguous per-thread ranges (output independent of nt)
  const int nt = std::max(1, n_threads);
  std::vector<Generated> parts(static_cast<size_t>(nt));
  std::vector<std::thread> th;
  for (int w = 0; w < nt; ++w) {
    th.emplace_back([&, w] {
      const int64_t lo = D * w / nt, hi = D * (w + 1) / nt;
      Generated& g = parts[static_cast<size_t>(w)];
      g.offsets.reserve(static_cast<size_t>(hi - lo));
      std::vector<int32_t> toks;
      std::vector<int64_t> topics;
      std::vector<double> cdf;
      int64_t pos = 0;
      for (int64_t d = lo; d < hi; ++d) {
        Rng r;
        r.s.init(p->seed, 0, static_cast<uint32_t>(p->first_doc + d), 0, scu::make_tag(7, 3, 0));
        const double lam = p->mean_len * r.gamma(p->len_shape) / p->len_shape;
        int64_t len = static_cast<int64_t>(std::llround(lam + std::sqrt(lam) * r.normal()));
        len = std::max<int64_t>(1, len);
        int64_t nt_d = 1;
        while (nt_d < 16 && r.u() < p->topics_per_doc / (1.0 + p->topics_per_doc)) ++nt_d;
        topics.resize(static_cast<size_t>(nt_d));
        cdf.resize(static_cast<size_t>(nt_d));
        double acc = 0.0;
        for (int64_t i = 0; i < nt_d; ++i) {
          topics[i] = static_cast<int64_t>(r.u32() % static_cast<uint32_t>(KG));
          acc += -std::log(r.u());
          cdf[i] = acc;
        }
        toks.resize(static_cast<size_t>(len));
        for (int64_t i = 0; i < len; ++i) {
          const double x = r.u() * acc;
          int64_t z = 0;
          while (z + 1 < nt_d && x >= cdf[z]) ++z;
          const Alias& a = tables[static_cast<size_t>(topics[z])];
          const uint64_t bits = r.s.next_u64();
          const int64_t col = static_cast<int64_t>((bits >> 32) % static_cast<uint64_t>(W));
          const float f = static_cast<float>(bits & 0xffffffu) * (1.0f / 16777216.0f);
          toks[i] = f < a.prob[col] ? static_cast<int32_t>(col) : a.alias[col];
        }
        std::sort(toks.begin(), toks.end());
        for (int64_t i = 0; i < len;) {
          int64_t j = i;
          while (j < len && toks[j] == toks[i]) ++j;
          g.words.push_back(toks[i]);
          g.counts.push_back(static_cast<int32_t>(j - i));
          ++pos;
          i = j;
        }
        g.offsets.push_back(pos);
      }
    });
  }
  for (auto& t : th) t.join();
  auto* out = new Generated();
  out->offsets.reserve(static_cast<size_t>(D + 1));
  out->offsets.push_back(0);
  int64_t base = 0, tok = 0;
  size_t total = 0;
  for (auto& g : parts) total += g.words.size();
  out->words.reserve(total);
  out->counts.reserve(total);
  for (auto& g : parts) {
    for (int64_t o : g.offsets) out->offsets.push_back(base + o);
    base += static_cast<int64_t>(g.words.size());
    out->words.insert(out->words.end(), g.words.begin(), g.words.end());
    out->counts.insert(out->counts.end(), g.counts.begin(), g.counts.end());
    for (int32_t c : g.counts) tok += c;
    g = Generated();
  }
  *nnz = base;
  *n_tokens = tok;
  *handle = out;
  return 0;
}

int samelda_synth_make_corpus_ref(int64_t n_docs, int64_t n_words, int64_t n_topics,
                                  double len_mean, uint64_t seed, double theta_conc,
                                  double phi_conc, int n_threads, void** handle, int64_t* nnz,
                                  int64_t* n_tokens) {
  if (n_docs < 1 || n_words < 1 || n_topics < 1 || !(len_mean >= 1.0) || !(theta_conc > 0.0) ||
      !(phi_conc > 0.0) || handle == nullptr)
    return 1;
  const int64_t W = n_words, K = n_topics, D = n_docs;
  std::vector<double> phi(static_cast<size_t>(K * W)), cum(static_cast<size_t>(K * W));
  {
    scu::Stream s;
    s.init(seed, 0, 0, 0, scu::make_tag(refgen::kSynthetic, 1, 0));
    for (int64_t k = 0; k < K; ++k) refgen::dirichlet_variate(W, phi_conc, s, phi.data() + k * W);
  }
  for (int64_t k = 0; k < K; ++k) {
    double c = 0.0;
    for (int64_t w = 0; w < W; ++w) cum[k * W + w] = (c += phi[k * W + w]);
  }
  const int nt = std::max(1, n_threads);
  std::vector<Generated> parts(static_cast<size_t>(nt));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    th.emplace_back([&, t] {
      const int64_t lo = D * t / nt, hi = D * (t + 1) / nt;
      Generated& g = parts[static_cast<size_t>(t)];
      std::vector<int32_t> word_count(static_cast<size_t>(W));
      std::vector<double> theta(static_cast<size_t>(K)), tcum(static_cast<size_t>(K));
      int64_t pos = 0;
      for (int64_t d = lo; d < hi; ++d) {
        scu::Stream s;
        s.init(seed, 0, static_cast<uint32_t>(d), 0, scu::make_tag(refgen::kSynthetic, 2, 0));
        refgen::dirichlet_variate(K, theta_conc, s, theta.data());
        double c = 0.0;
        for (int64_t k = 0; k < K; ++k) tcum[k] = (c += theta[k]);
        const int64_t length = 1 + refgen::poisson_sample(len_mean - 1.0, s);
        std::fill(word_count.begin(), word_count.end(), 0);
        for (int64_t i = 0; i < length; ++i) {
          const int k = refgen::categorical(theta.data(), tcum.data(), K, s);
          const int w = refgen::categorical(phi.data() + k * W, cum.data() + k * W, W, s);
          ++word_count[static_cast<size_t>(w)];
        }
        for (int64_t w = 0; w < W; ++w)
          if (word_count[static_cast<size_t>(w)] > 0) {
            g.words.push_back(static_cast<int32_t>(w));
            g.counts.push_back(word_count[static_cast<size_t>(w)]);
            ++pos;
          }
        g.offsets.push_back(pos);
      }
    });
  }
  for (auto& x : th) x.join();
  auto* out = new Generated();
  out->offsets.push_back(0);
  int64_t base = 0, tok = 0;
  for (auto& g : parts) {
    for (int64_t o : g.offsets) out->offsets.push_back(base + o);
    base += static_cast<int64_t>(g.words.size());
    out->words.insert(out->words.end(), g.words.begin(), g.words.end());
    out->counts.insert(out->counts.end(), g.counts.begin(), g.counts.end());
    for (int32_t c : g.counts) tok += c;
  }
  *nnz = base;
  *n_tokens = tok;
  *handle = out;
  return 0;
}

int samelda_synth_split_holdout(int64_t n_docs, double test_fraction, uint64_t seed,
                                int32_t* test_ids, int64_t* n_test, int32_t* train_ids) {
  // corpus.cpp:231-250 (ids only; the caller subsets the CSR)
  if (!(test_fraction > 0.0 && test_fraction < 1.0) || n_docs < 2) return 1;
  scu::Stream s;
  s.init(seed, 0, 0, 0, scu::make_tag(scu::kHoldoutSplit, 0, 0));
  std::vector<int32_t> order(static_cast<size_t>(n_docs));
  for (int64_t i = 0; i < n_docs; ++i) order[static_cast<size_t>(i)] = static_cast<int32_t>(i);
  for (int64_t i = n_docs - 1; i > 0; --i) {  // shuffled_indices, rng.cpp:181-192
    const int64_t j = static_cast<int64_t>(s.uniform_below(static_cast<uint64_t>(i) + 1));
    std::swap(order[static_cast<size_t>(i)], order[static_cast<size_t>(j)]);
  }
  int64_t nt = static_cast<int64_t>(std::llround(test_fraction * static_cast<double>(n_docs)));
  nt = std::clamp<int64_t>(nt, 1, n_docs - 1);
  std::sort(order.begin(), order.begin() + nt);
  std::sort(order.begin() + nt, order.end());
  std::memcpy(test_ids, order.data(), sizeof(int32_t) * static_cast<size_t>(nt));
  std::memcpy(train_ids, order.data() + nt, sizeof(int32_t) * static_cast<size_t>(n_docs - nt));
  *n_test = nt;
  return 0;
}

void samelda_synth_copy(void* handle, int64_t* offsets, int32_t* words, int32_t* counts) {
  auto* g = static_cast<Generated*>(handle);
  std::memcpy(offsets, g->offsets.data(), sizeof(int64_t) * g->offsets.size());
  std::memcpy(words, g->words.data(), sizeof(int32_t) * g->words.size());
  std::memcpy(counts, g->counts.data(), sizeof(int32_t) * g->counts.size());
}

void samelda_synth_free(void* handle) { delete static_cast<Generated*>(handle); }

}  // extern "C"
