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

void samelda_synth_copy(void* handle, int64_t* offsets, int32_t* words, int32_t* counts) {
  auto* g = static_cast<Generated*>(handle);
  std::memcpy(offsets, g->offsets.data(), sizeof(int64_t) * g->offsets.size());
  std::memcpy(words, g->words.data(), sizeof(int32_t) * g->words.size());
  std::memcpy(counts, g->counts.data(), sizeof(int32_t) * g->counts.size());
}

void samelda_synth_free(void* handle) { delete static_cast<Generated*>(handle); }

}  // extern "C"
