/*
 * samelda_oracle.c -- CPU restatement of the reference SAME/LDA hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see samelda_oracle.h).  Single-threaded, plain
 * C11, compiled without -march and with -ffp-contract=off so every f64
 * operation rounds exactly like the reference's x86-64 Release build.
 * Each function cites the reference function it restates (proj/ paths).
 */
#include "samelda_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* rng.cpp:12-15 */
#define PHILOX_W32A 0x9E3779B9u
#define PHILOX_W32B 0xBB67AE85u
#define PHILOX_M4x32A 0xD2511F53u
#define PHILOX_M4x32B 0xCD9E8D57u

uint32_t so_make_tag(uint32_t purpose, uint32_t sub, uint32_t index) {
  /* rng.hpp:35-39: [purpose:4][sub:8][index:20] */
  return (purpose << 28) | ((sub & 0xffu) << 20) | (index & 0xfffffu);
}

void so_philox_block(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  /* rng.cpp:24-35: ten Philox4x32 rounds, key bumped after every round */
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)PHILOX_M4x32A * c0;
    const uint64_t p1 = (uint64_t)PHILOX_M4x32B * c2;
    const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
    const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += PHILOX_W32A;
    k1 += PHILOX_W32B;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

void so_stream_init(so_stream* s, uint64_t seed, uint32_t t, uint32_t doc, uint32_t word,
                    uint32_t tag) {
  /* rng.cpp:90-94: counter {block, word, doc, t}; key = seed halves ^ tag*M */
  s->base[0] = 0;
  s->base[1] = word;
  s->base[2] = doc;
  s->base[3] = t;
  s->key[0] = (uint32_t)seed ^ (uint32_t)(tag * PHILOX_M4x32A);
  s->key[1] = (uint32_t)(seed >> 32) ^ (uint32_t)(tag * PHILOX_M4x32B);
  s->block = 0;
  s->pos = 4;
}

static void so_refill(so_stream* s) {
  /* rng.cpp:96-101 */
  uint32_t ctr[4] = {s->block, s->base[1], s->base[2], s->base[3]};
  s->block += 1u;
  so_philox_block(ctr, s->key, s->buf);
  s->pos = 0;
}

uint32_t so_next_u32(so_stream* s) {
  /* rng.cpp:103-108 */
  if (s->pos == 4) so_refill(s);
  return s->buf[s->pos++];
}

uint64_t so_next_u64(so_stream* s) {
  /* rng.cpp:110-114: first word is the low half */
  const uint64_t lo = so_next_u32(s);
  const uint64_t hi = so_next_u32(s);
  return (hi << 32) | lo;
}

double so_uniform(so_stream* s) {
  /* rng.cpp:116-118 */
  return (double)(so_next_u64(s) >> 11) * 0x1.0p-53;
}

double so_uniform_oo(so_stream* s) {
  /* rng.cpp:120-122 */
  return ((double)(so_next_u64(s) >> 11) + 0.5) * 0x1.0p-53;
}

uint64_t so_uniform_below(so_stream* s, uint64_t n) {
  /* rng.cpp:124-133 */
  const uint64_t rem = (0 - n) % n;
  for (;;) {
    const uint64_t x = so_next_u64(s);
    if (x >= rem) return (x - rem) % n;
  }
}

static int64_t so_poisson_inversion(double lambda, so_stream* s) {
  /* rng.cpp:39-52 */
  const double u = so_uniform(s);
  double pmf = exp(-lambda);
  double cdf = pmf;
  int64_t k = 0;
  while (u > cdf && k < 1000) {
    ++k;
    pmf *= lambda / (double)k;
    cdf += pmf;
  }
  return k;
}

static int64_t so_poisson_ptrs(double lambda, so_stream* s) {
  /* rng.cpp:57-86 (Hormann 1993 PTRS) */
  const double log_lambda = log(lambda);
  const double b = 0.931 + 2.53 * sqrt(lambda);
  const double a = -0.059 + 0.02483 * b;
  const double inv_alpha = 1.1239 + 1.1328 / (b - 3.4);
  const double v_r = 0.9277 - 3.6224 / (b - 2.0);
  for (;;) {
    const double u = so_uniform_oo(s) - 0.5;
    const double v = so_uniform_oo(s);
    const double u_shifted = 0.5 - fabs(u);
    const double g = (2.0 * a / u_shifted + b) * u + lambda + 0.43;
    if (u_shifted >= 0.07 && v <= v_r) return (int64_t)g;
    if (g < 0.0 || g > 9.0e18 || (u_shifted < 0.013 && v > u_shifted)) continue;
    const int64_t k = (int64_t)g;
    const double lhs = log(v * inv_alpha / (a / (u_shifted * u_shifted) + b));
    const double rhs = -lambda + (double)k * log_lambda - lgamma((double)k + 1.0);
    if (lhs <= rhs) return k;
  }
}

int64_t so_poisson_sample(double lambda, so_stream* s, int* err) {
  /* rng.cpp:139-150 */
  if (isnan(lambda) || lambda < 0.0 || !isfinite(lambda)) {
    *err = SO_NUMERICAL;
    return 0;
  }
  if (lambda == 0.0) return 0;
  if (lambda < 10.0) return so_poisson_inversion(lambda, s);
  return so_poisson_ptrs(lambda, s);
}

int so_poisson_grid(double lambda, uint64_t seed, uint32_t t, uint32_t doc, uint32_t word,
                    uint32_t sweep, uint32_t k0, int64_t n, int64_t* out) {
  int err = SO_OK;
  for (int64_t i = 0; i < n; ++i) {
    so_stream s;
    so_stream_init(&s, seed, t, doc, word,
                   so_make_tag(SO_POISSON_COUNTS, sweep, k0 + (uint32_t)i));
    out[i] = so_poisson_sample(lambda, &s, &err);
    if (err) return err;
  }
  return SO_OK;
}

int so_categorical_sample(const double* weights, int64_t n, so_stream* s, int* err) {
  /* rng.cpp:152-179 */
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (isnan(weights[i]) || weights[i] < 0.0) {
      *err = SO_NUMERICAL;
      return 0;
    }
    total += weights[i];
  }
  if (!(total > 0.0) || !isfinite(total)) {
    *err = SO_NUMERICAL;
    return 0;
  }
  const double u = so_uniform(s) * total;
  double cum = 0.0;
  for (int64_t k = 0; k + 1 < n; ++k) {
    cum += weights[k];
    if (u < cum) return (int)k;
  }
  for (int64_t k = n; k-- > 0;) {
    if (weights[k] > 0.0) return (int)k;
  }
  return 0;
}

/* Same result as so_categorical_sample, by binary search over the prefix sums
 * cum[k] = w[0] + ... + w[k] accumulated in the reference's order (the first
 * k with u < cum[k] is unique because cum is nondecreasing). */
static int so_categorical_prefix(const double* weights, const double* cum, int64_t n,
                                 so_stream* s) {
  const double total = cum[n - 1];
  const double u = so_uniform(s) * total;
  int64_t lo = 0, hi = n - 1; /* search k in [0, n-2] */
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (u < cum[mid]) hi = mid; else lo = mid + 1;
  }
  if (lo < n - 1) return (int)lo;
  for (int64_t k = n; k-- > 0;) {
    if (weights[k] > 0.0) return (int)k;
  }
  return 0;
}

void so_shuffled_indices(int64_t n, so_stream* s, int32_t* order) {
  /* rng.cpp:181-192 */
  for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)i;
  for (int64_t i = n - 1; i > 0; --i) {
    const int64_t j = (int64_t)so_uniform_below(s, (uint64_t)i + 1);
    const int32_t tmp = order[i];
    order[i] = order[j];
    order[j] = tmp;
  }
}

/* ------------------------------------------------------------------ sampler */

static int64_t* so_batch_prefix(const int64_t* doc_offsets, const int32_t* doc_ids,
                                int64_t B) {
  /* sampler.cpp:18-24 */
  int64_t* prefix = (int64_t*)malloc(sizeof(int64_t) * (size_t)(B + 1));
  prefix[0] = 0;
  for (int64_t b = 0; b < B; ++b) {
    const int32_t d = doc_ids[b];
    prefix[b + 1] = prefix[b] + (doc_offsets[d + 1] - doc_offsets[d]);
  }
  return prefix;
}

int so_sddmm(const double* theta_batch, int64_t B, int64_t K, const double* phi, int64_t W,
             const int64_t* doc_offsets, const int32_t* word_ids, const int32_t* doc_ids,
             double* mu_out) {
  /* sampler.cpp:88-123; sequential k order, product then add (no FMA) */
  (void)W;
  int64_t out = 0;
  for (int64_t b = 0; b < B; ++b) {
    const int32_t d = doc_ids[b];
    const double* theta_row = theta_batch + b * K;
    for (int64_t p = doc_offsets[d]; p < doc_offsets[d + 1]; ++p) {
      const int32_t w = word_ids[p];
      double dot = 0.0;
      for (int64_t k = 0; k < K; ++k) dot += theta_row[k] * phi[k * W + w];
      mu_out[out++] = dot;
    }
  }
  return SO_OK;
}

int so_sample_counts(const double* theta_batch, int64_t B, int64_t K, const double* phi,
                     int64_t W, const double* mu, int64_t mu_len, const int64_t* doc_offsets,
                     const int32_t* word_ids, const int32_t* counts, const int32_t* doc_ids,
                     double m_t, uint64_t seed, int64_t t, int sweep, int64_t* theta_counts,
                     int64_t* phi_counts) {
  /* sampler.cpp:125-195 */
  if (!(m_t > 0.0) || !isfinite(m_t)) return SO_CONFIG;
  int64_t* prefix = so_batch_prefix(doc_offsets, doc_ids, B);
  if (mu_len != prefix[B]) {
    free(prefix);
    return SO_CONFIG;
  }
  memset(theta_counts, 0, sizeof(int64_t) * (size_t)(B * K));
  memset(phi_counts, 0, sizeof(int64_t) * (size_t)(W * K));
  const double uniform_weight = 1.0 / (double)K;
  int err = SO_OK;
  for (int64_t b = 0; b < B && !err; ++b) {
    const int32_t d = doc_ids[b];
    const double* theta_row = theta_batch + b * K;
    int64_t* theta_out = theta_counts + b * K;
    const int64_t begin = doc_offsets[d];
    const int64_t n = doc_offsets[d + 1] - begin;
    for (int64_t i = 0; i < n && !err; ++i) {
      const int32_t w = word_ids[begin + i];
      const double cell_scale = m_t * (double)counts[begin + i];
      const double mu_dw = mu[prefix[b] + i];
      const int degenerate = mu_dw < 1e-30;
      int64_t* phi_out = phi_counts + (int64_t)w * K;
      for (int64_t k = 0; k < K; ++k) {
        const double weight =
            degenerate ? uniform_weight : theta_row[k] * phi[k * W + w] / mu_dw;
        const double rate = weight * cell_scale;
        if (!isfinite(rate)) {
          err = SO_NUMERICAL;
          break;
        }
        so_stream s;
        so_stream_init(&s, seed, (uint32_t)t, (uint32_t)d, (uint32_t)w,
                       so_make_tag(SO_POISSON_COUNTS, (uint32_t)sweep, (uint32_t)k));
        const int64_t z = so_poisson_sample(rate, &s, &err);
        if (err) break;
        if (z != 0) {
          theta_out[k] += z;
          phi_out[k] += z;
        }
      }
    }
  }
  free(prefix);
  return err;
}

int so_expected_counts(const double* theta_batch, int64_t B, int64_t K, const double* phi,
                       int64_t W, const double* mu, int64_t mu_len,
                       const int64_t* doc_offsets, const int32_t* word_ids,
                       const int32_t* counts, const int32_t* doc_ids, double m_t,
                       double* theta_expected, double* phi_expected) {
  /* sampler.cpp:151-193 with z := rate (the Poisson mean) */
  if (!(m_t > 0.0) || !isfinite(m_t)) return SO_CONFIG;
  int64_t* prefix = so_batch_prefix(doc_offsets, doc_ids, B);
  if (mu_len != prefix[B]) {
    free(prefix);
    return SO_CONFIG;
  }
  memset(theta_expected, 0, sizeof(double) * (size_t)(B * K));
  memset(phi_expected, 0, sizeof(double) * (size_t)(W * K));
  const double uniform_weight = 1.0 / (double)K;
  int err = SO_OK;
  for (int64_t b = 0; b < B && !err; ++b) {
    const int32_t d = doc_ids[b];
    const double* theta_row = theta_batch + b * K;
    const int64_t begin = doc_offsets[d];
    const int64_t n = doc_offsets[d + 1] - begin;
    for (int64_t i = 0; i < n; ++i) {
      const int32_t w = word_ids[begin + i];
      const double cell_scale = m_t * (double)counts[begin + i];
      const double mu_dw = mu[prefix[b] + i];
      const int degenerate = mu_dw < 1e-30;
      for (int64_t k = 0; k < K; ++k) {
        const double weight =
            degenerate ? uniform_weight : theta_row[k] * phi[k * W + w] / mu_dw;
        const double rate = weight * cell_scale;
        if (!isfinite(rate) || rate < 0.0) {
          err = SO_NUMERICAL;
          break;
        }
        theta_expected[b * K + k] += rate;
        phi_expected[(int64_t)w * K + k] += rate;
      }
    }
  }
  free(prefix);
  return err;
}

static int so_update_model_impl(double* theta, int64_t K_theta, double* phi, int64_t K,
                                int64_t W, double alpha, double beta, const int32_t* doc_ids,
                                int64_t B, const int64_t* tc_i, const int64_t* pc_i,
                                const double* tc_f, const double* pc_f, double m_t,
                                double rho_t) {
  /* sampler.cpp:197-229 */
  (void)K_theta;
  if (!(rho_t > 0.0 && rho_t <= 1.0)) return SO_CONFIG;
  for (int64_t b = 0; b < B; ++b) {
    const int32_t d = doc_ids[b];
    for (int64_t k = 0; k < K; ++k) {
      const double hat = tc_i ? (double)tc_i[b * K + k] / m_t : tc_f[b * K + k] / m_t;
      theta[(int64_t)d * K + k] = hat + alpha;
    }
  }
  double* candidate = (double*)malloc(sizeof(double) * (size_t)W);
  for (int64_t k = 0; k < K; ++k) {
    double total = 0.0;
    for (int64_t w = 0; w < W; ++w) {
      const double hat = pc_i ? (double)pc_i[w * K + k] / m_t : pc_f[w * K + k] / m_t;
      const double value = hat + beta;
      candidate[w] = value;
      total += value;
    }
    if (!(total > 0.0) || !isfinite(total)) {
      free(candidate);
      return SO_NUMERICAL;
    }
    double* row = phi + k * W;
    for (int64_t w = 0; w < W; ++w) {
      row[w] = (1.0 - rho_t) * row[w] + rho_t * candidate[w] / total;
    }
  }
  free(candidate);
  return SO_OK;
}

int so_update_model(double* theta, int64_t D, double* phi, int64_t K, int64_t W,
                    double alpha, double beta, const int32_t* doc_ids, int64_t B,
                    const int64_t* theta_counts, const int64_t* phi_counts, double m_t,
                    double rho_t) {
  (void)D;
  return so_update_model_impl(theta, K, phi, K, W, alpha, beta, doc_ids, B, theta_counts,
                              phi_counts, NULL, NULL, m_t, rho_t);
}

int so_update_model_expected(double* theta, int64_t D, double* phi, int64_t K, int64_t W,
                             double alpha, double beta, const int32_t* doc_ids, int64_t B,
                             const double* theta_expected, const double* phi_expected,
                             double m_t, double rho_t) {
  (void)D;
  return so_update_model_impl(theta, K, phi, K, W, alpha, beta, doc_ids, B, NULL, NULL,
                              theta_expected, phi_expected, m_t, rho_t);
}

int so_rho_schedule(int64_t t, double tau0, double gamma, double* out) {
  /* sampler.cpp:231-242 */
  if (t < 0) return SO_CONFIG;
  if (!(tau0 >= 1.0)) return SO_CONFIG;
  if (!(gamma >= 0.5 && gamma <= 1.0)) return SO_CONFIG;
  *out = pow(tau0 + (double)t, -gamma);
  return SO_OK;
}

int so_anneal_m(int schedule, int64_t t, int64_t t_max, double m, double* out) {
  /* sampler.cpp:244-267 */
  if (t < 1 || t > t_max) return SO_CONFIG;
  const double td = (double)t;
  const double nd = (double)t_max;
  switch (schedule) {
    case 0: *out = m; return SO_OK;
    case 1: *out = 2.0 * m * td / (nd + 1.0); return SO_OK;
    case 3: *out = 2.0 * m * (nd + 1.0 - td) / (nd + 1.0); return SO_OK;
    case 2: {
      if (t_max == 1) {
        *out = m;
        return SO_OK;
      }
      const double value = m * nd * log(td) / lgamma(nd + 1.0);
      *out = (value < 0.01) ? 0.01 : value; /* std::max(value, 0.01) */
      return SO_OK;
    }
    default: return SO_CONFIG;
  }
}

/* --------------------------------------------------------------------- eval */

void so_fold_in_theta(const double* phi, int64_t K, int64_t W, const int32_t* words,
                      const int32_t* counts, int64_t n, double alpha, int sweeps,
                      double* theta) {
  /* eval.cpp:19-64 (phi indexed K x W instead of through the transpose) */
  for (int64_t k = 0; k < K; ++k) theta[k] = 1.0 / (double)K;
  if (n == 0) return;
  double* next = (double*)malloc(sizeof(double) * (size_t)K);
  for (int sweep = 0; sweep < sweeps; ++sweep) {
    for (int64_t k = 0; k < K; ++k) next[k] = alpha;
    for (int64_t i = 0; i < n; ++i) {
      const int32_t w = words[i];
      double mu = 0.0;
      for (int64_t k = 0; k < K; ++k) mu += theta[k] * phi[k * W + w];
      if (!(mu > 0.0)) continue;
      const double scale = (double)counts[i] / mu;
      for (int64_t k = 0; k < K; ++k) next[k] += scale * theta[k] * phi[k * W + w];
    }
    double total = 0.0;
    for (int64_t k = 0; k < K; ++k) total += next[k];
    double delta = 0.0;
    for (int64_t k = 0; k < K; ++k) {
      const double value = next[k] / total;
      const double diff = fabs(value - theta[k]);
      if (delta < diff) delta = diff; /* std::max(delta, diff) */
      theta[k] = value;
    }
    if (delta < 1e-12) break;
  }
  free(next);
}

int so_perword_loglik(const double* phi, int64_t K, int64_t W, const int64_t* doc_offsets,
                      const int32_t* word_ids, const int32_t* counts, int64_t n_docs,
                      double alpha, uint64_t seed, double* ll_out) {
  /* eval.cpp:75-159 */
  if (n_docs < 1) return SO_CONFIG;
  double* doc_logp = (double*)calloc((size_t)n_docs, sizeof(double));
  int64_t* doc_scored = (int64_t*)calloc((size_t)n_docs, sizeof(int64_t));
  double* theta = (double*)malloc(sizeof(double) * (size_t)K);
  int err = SO_OK;
  for (int64_t d = 0; d < n_docs && !err; ++d) {
    const int64_t begin = doc_offsets[d];
    const int64_t n_cells = doc_offsets[d + 1] - begin;
    const int32_t* words = word_ids + begin;
    const int32_t* cnts = counts + begin;
    int64_t n_tokens = 0;
    for (int64_t i = 0; i < n_cells; ++i) n_tokens += cnts[i];
    /* eval.cpp:99-121: expand, seeded Fisher-Yates, first ceil(N/2) fold in */
    int32_t* slots = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_tokens + 1));
    int64_t pos = 0;
    for (int64_t i = 0; i < n_cells; ++i)
      for (int32_t rep = 0; rep < cnts[i]; ++rep) slots[pos++] = (int32_t)i;
    so_stream s;
    so_stream_init(&s, seed, 0, (uint32_t)d, 0, so_make_tag(SO_EVAL_SPLIT, 0, 0));
    for (int64_t i = n_tokens - 1; i > 0; --i) {
      const int64_t j = (int64_t)so_uniform_below(&s, (uint64_t)i + 1);
      const int32_t tmp = slots[i];
      slots[i] = slots[j];
      slots[j] = tmp;
    }
    const int64_t n_fold = (n_tokens + 1) / 2;
    int32_t* fold = (int32_t*)calloc((size_t)(n_cells + 1), sizeof(int32_t));
    int32_t* score = (int32_t*)calloc((size_t)(n_cells + 1), sizeof(int32_t));
    for (int64_t i = 0; i < n_tokens; ++i) {
      if (i < n_fold) ++fold[slots[i]]; else ++score[slots[i]];
    }
    so_fold_in_theta(phi, K, W, words, fold, n_cells, alpha, 50, theta);
    double logp = 0.0;
    int64_t scored = 0;
    for (int64_t i = 0; i < n_cells; ++i) {
      const int32_t c = score[i];
      if (c == 0) continue;
      double p = 0.0;
      for (int64_t k = 0; k < K; ++k) p += theta[k] * phi[k * W + words[i]];
      if (!(p > 0.0)) {
        err = SO_NUMERICAL;
        break;
      }
      logp += (double)c * log(p);
      scored += c;
    }
    doc_logp[d] = logp;
    doc_scored[d] = scored;
    free(slots);
    free(fold);
    free(score);
  }
  double total_logp = 0.0;
  int64_t total_scored = 0;
  for (int64_t d = 0; d < n_docs; ++d) {
    total_logp += doc_logp[d];
    total_scored += doc_scored[d];
  }
  free(doc_logp);
  free(doc_scored);
  free(theta);
  if (err) return err;
  if (total_scored == 0) return SO_NUMERICAL;
  *ll_out = total_logp / (double)total_scored;
  return SO_OK;
}

/* ------------------------------------------------------------------- corpus */

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int so_split_holdout_ids(int64_t n_docs, double test_fraction, uint64_t seed,
                         int32_t* train_ids, int64_t* n_train, int32_t* test_ids,
                         int64_t* n_test) {
  /* corpus.cpp:231-250 */
  if (!(test_fraction > 0.0 && test_fraction < 1.0)) return SO_CONFIG;
  if (n_docs < 2) return SO_CONFIG;
  so_stream s;
  so_stream_init(&s, seed, 0, 0, 0, so_make_tag(SO_HOLDOUT_SPLIT, 0, 0));
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_docs);
  so_shuffled_indices(n_docs, &s, order);
  int64_t nt = (int64_t)llround(test_fraction * (double)n_docs);
  if (nt < 1) nt = 1;
  if (nt > n_docs - 1) nt = n_docs - 1;
  memcpy(test_ids, order, sizeof(int32_t) * (size_t)nt);
  memcpy(train_ids, order + nt, sizeof(int32_t) * (size_t)(n_docs - nt));
  qsort(test_ids, (size_t)nt, sizeof(int32_t), cmp_i32);
  qsort(train_ids, (size_t)(n_docs - nt), sizeof(int32_t), cmp_i32);
  *n_test = nt;
  *n_train = n_docs - nt;
  free(order);
  return SO_OK;
}

static void so_minibatch_start_pass(so_minibatch_stream* s) {
  /* corpus.cpp:268-273 */
  so_stream st;
  so_stream_init(&st, s->seed, s->pass, 0, 0, so_make_tag(SO_BATCH_SHUFFLE, 0, 0));
  so_shuffled_indices(s->n_docs, &st, s->order);
  s->cursor = 0;
}

int so_minibatch_init(so_minibatch_stream* s, int64_t n_docs, double batch_fraction,
                      uint64_t seed) {
  /* corpus.cpp:252-262 */
  if (!(batch_fraction > 0.0 && batch_fraction <= 1.0)) return SO_CONFIG;
  s->n_docs = n_docs;
  s->seed = seed;
  int64_t bs = (int64_t)llround(batch_fraction * (double)n_docs);
  s->batch_size = bs < 1 ? 1 : bs;
  s->pass = 0;
  s->order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_docs > 0 ? n_docs : 1));
  so_minibatch_start_pass(s);
  return SO_OK;
}

int64_t so_minibatch_next(so_minibatch_stream* s, int32_t* out) {
  /* corpus.cpp:275-285 */
  if (s->cursor >= s->n_docs) {
    s->pass += 1u;
    so_minibatch_start_pass(s);
  }
  int64_t take = s->n_docs - s->cursor;
  if (s->batch_size < take) take = s->batch_size;
  memcpy(out, s->order + s->cursor, sizeof(int32_t) * (size_t)take);
  s->cursor += take;
  return take;
}

void so_minibatch_free(so_minibatch_stream* s) {
  free(s->order);
  s->order = NULL;
}

/* ------------------------------------------------- synthetic corpus generator */

static double so_normal_variate(so_stream* s) {
  /* tests/support/synthetic.cpp:16-21 */
  const double u1 = so_uniform_oo(s);
  const double u2 = so_uniform_oo(s);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}

static double so_gamma_variate(double shape, so_stream* s) {
  /* tests/support/synthetic.cpp:39-59 (Marsaglia-Tsang) */
  if (shape < 1.0) {
    const double u = so_uniform_oo(s);
    return so_gamma_variate(shape + 1.0, s) * pow(u, 1.0 / shape);
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    const double x = so_normal_variate(s);
    const double t = 1.0 + c * x;
    if (t <= 0.0) continue;
    const double v = t * t * t;
    const double u = so_uniform_oo(s);
    if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) return d * v;
  }
}

static void so_dirichlet_variate(int64_t k, double conc, so_stream* s, double* out) {
  /* tests/support/synthetic.cpp:23-35 */
  double total = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    out[i] = so_gamma_variate(conc, s);
    total += out[i];
  }
  for (int64_t i = 0; i < k; ++i) out[i] /= total;
}

int so_make_corpus(int64_t n_docs, int64_t n_words, int64_t n_topics, double len_mean,
                   uint64_t seed, double theta_conc, double phi_conc, so_generated** out) {
  /* tests/support/synthetic.cpp:61-106; categorical draws by prefix binary
   * search, which returns the same index as the linear scan (rng.cpp:163-170). */
  so_generated* g = (so_generated*)calloc(1, sizeof(so_generated));
  g->n_docs = n_docs;
  g->n_words = n_words;
  g->n_topics = n_topics;
  g->phi_true = (double*)malloc(sizeof(double) * (size_t)(n_topics * n_words));
  double* cum = (double*)malloc(sizeof(double) * (size_t)(n_topics * n_words));
  {
    so_stream s;
    so_stream_init(&s, seed, 0, 0, 0, so_make_tag(SO_SYNTHETIC, 1, 0));
    for (int64_t k = 0; k < n_topics; ++k) {
      double* row = g->phi_true + k * n_words;
      so_dirichlet_variate(n_words, phi_conc, &s, row);
      double acc = 0.0;
      for (int64_t w = 0; w < n_words; ++w) {
        acc += row[w];
        cum[k * n_words + w] = acc;
      }
    }
  }
  int64_t cap = 1024;
  g->doc_offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_docs + 1));
  g->word_ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  g->counts = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  int32_t* word_count = (int32_t*)calloc((size_t)n_words, sizeof(int32_t));
  double* theta = (double*)malloc(sizeof(double) * (size_t)n_topics);
  int err = SO_OK;
  g->doc_offsets[0] = 0;
  for (int64_t d = 0; d < n_docs; ++d) {
    so_stream s;
    so_stream_init(&s, seed, 0, (uint32_t)d, 0, so_make_tag(SO_SYNTHETIC, 2, 0));
    so_dirichlet_variate(n_topics, theta_conc, &s, theta);
    const int64_t length = 1 + so_poisson_sample(len_mean - 1.0, &s, &err);
    memset(word_count, 0, sizeof(int32_t) * (size_t)n_words);
    for (int64_t i = 0; i < length; ++i) {
      const int k = so_categorical_sample(theta, n_topics, &s, &err);
      const int w = so_categorical_prefix(g->phi_true + (int64_t)k * n_words,
                                          cum + (int64_t)k * n_words, n_words, &s);
      ++word_count[w];
    }
    for (int64_t w = 0; w < n_words; ++w) {
      if (word_count[w] > 0) {
        if (g->nnz == cap) {
          cap *= 2;
          g->word_ids = (int32_t*)realloc(g->word_ids, sizeof(int32_t) * (size_t)cap);
          g->counts = (int32_t*)realloc(g->counts, sizeof(int32_t) * (size_t)cap);
        }
        g->word_ids[g->nnz] = (int32_t)w;
        g->counts[g->nnz] = word_count[w];
        g->nnz += 1;
        g->n_tokens += word_count[w];
      }
    }
    g->doc_offsets[d + 1] = g->nnz;
  }
  free(word_count);
  free(theta);
  free(cum);
  *out = g;
  return err;
}

void so_generated_free(so_generated* g) {
  if (!g) return;
  free(g->doc_offsets);
  free(g->word_ids);
  free(g->counts);
  free(g->phi_true);
  free(g);
}

/* -------------------------------------------------------------------- train */

void so_init_phi(double* phi, int64_t K, int64_t W, double init_noise, uint64_t seed) {
  /* model.cpp:41-52 then sampler.cpp:285-298 */
  for (int64_t i = 0; i < K * W; ++i) phi[i] = 1.0 / (double)W;
  if (!(init_noise > 0.0)) return;
  so_stream s;
  so_stream_init(&s, seed, 0, 0, 0, so_make_tag(SO_PHI_INIT, 0, 0));
  for (int64_t k = 0; k < K; ++k) {
    double* row = phi + k * W;
    double total = 0.0;
    for (int64_t w = 0; w < W; ++w) {
      row[w] = 1.0 + init_noise * so_uniform(&s);
      total += row[w];
    }
    for (int64_t w = 0; w < W; ++w) row[w] /= total;
  }
}

static int so_validate(const so_config* c) {
  /* sampler.cpp:47-78 */
  if (c->n_topics < 1 || c->n_topics >= (1 << 20)) return SO_CONFIG;
  if (!(c->m > 0.0) || !isfinite(c->m)) return SO_CONFIG;
  if (!(c->tau0 >= 1.0)) return SO_CONFIG;
  if (!(c->gamma >= 0.5 && c->gamma <= 1.0)) return SO_CONFIG;
  if (!(c->batch_fraction > 0.0 && c->batch_fraction <= 1.0)) return SO_CONFIG;
  if (c->t_max < 0) return SO_CONFIG;
  if (c->inner_sweeps < 1 || c->inner_sweeps > 255) return SO_CONFIG;
  if (!(c->alpha > 0.0) || !(c->beta > 0.0)) return SO_CONFIG;
  if (!(c->init_noise >= 0.0) || !isfinite(c->init_noise)) return SO_CONFIG;
  return SO_OK;
}

int so_train(const int64_t* doc_offsets, const int32_t* word_ids, const int32_t* counts,
             int64_t n_docs, int64_t n_words, const int64_t* ho_offsets,
             const int32_t* ho_words, const int32_t* ho_counts, int64_t ho_docs,
             const so_config* config, int64_t eval_every, double* phi, double* theta,
             so_trace_row* trace, int64_t* n_trace) {
  /* sampler.cpp:269-353 */
  int err = so_validate(config);
  if (err) return err;
  if (n_docs < 1) return SO_CONFIG;
  const int64_t K = config->n_topics, W = n_words;
  *n_trace = 0;
  for (int64_t i = 0; i < K * W; ++i) phi[i] = 1.0 / (double)W;
  for (int64_t i = 0; i < n_docs * K; ++i) theta[i] = config->alpha + 1.0 / (double)K;
  if (config->t_max == 0) return SO_OK;
  so_init_phi(phi, K, W, config->init_noise, config->seed);

  so_minibatch_stream batches;
  err = so_minibatch_init(&batches, n_docs, config->batch_fraction, config->seed);
  if (err) return err;
  int64_t corpus_tokens_i = 0;
  for (int64_t p = 0; p < doc_offsets[n_docs]; ++p) corpus_tokens_i += counts[p];
  const double corpus_tokens = (double)corpus_tokens_i;
  double tokens_seen = 0.0, samples_per_word = 0.0;

  const int64_t bs = batches.batch_size;
  int32_t* batch = (int32_t*)malloc(sizeof(int32_t) * (size_t)bs);
  double* theta_batch = (double*)malloc(sizeof(double) * (size_t)(bs * K));
  int64_t max_nnz = 0;
  for (int64_t d = 0; d < n_docs; ++d) max_nnz += doc_offsets[d + 1] - doc_offsets[d];
  double* mu = (double*)malloc(sizeof(double) * (size_t)(max_nnz + 1));
  int64_t* tc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(bs * K));
  int64_t* pc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(W * K));
  double* tcf = config->expected ? (double*)malloc(sizeof(double) * (size_t)(bs * K)) : NULL;
  double* pcf = config->expected ? (double*)malloc(sizeof(double) * (size_t)(W * K)) : NULL;

  for (int64_t t = 0; t < config->t_max && !err; ++t) {
    const int64_t B = so_minibatch_next(&batches, batch);
    double m_t = 0.0, rho_t = 0.0;
    err = so_anneal_m(config->schedule, t + 1, config->t_max, config->m, &m_t);
    if (!err) err = so_rho_schedule(t, config->tau0, config->gamma, &rho_t);
    if (err) break;
    for (int64_t b = 0; b < B; ++b)
      memcpy(theta_batch + b * K, theta + (int64_t)batch[b] * K, sizeof(double) * (size_t)K);
    int64_t nnz_b = 0;
    for (int64_t b = 0; b < B; ++b) nnz_b += doc_offsets[batch[b] + 1] - doc_offsets[batch[b]];
    for (int64_t sweep = 0; sweep < config->inner_sweeps && !err; ++sweep) {
      so_sddmm(theta_batch, B, K, phi, W, doc_offsets, word_ids, batch, mu);
      if (config->expected) {
        err = so_expected_counts(theta_batch, B, K, phi, W, mu, nnz_b, doc_offsets, word_ids,
                                 counts, batch, m_t, tcf, pcf);
      } else {
        err = so_sample_counts(theta_batch, B, K, phi, W, mu, nnz_b, doc_offsets, word_ids,
                               counts, batch, m_t, config->seed, t, (int)sweep, tc, pc);
      }
      if (!err && sweep + 1 < config->inner_sweeps) {
        for (int64_t i = 0; i < B * K; ++i)
          theta_batch[i] =
              (config->expected ? tcf[i] / m_t : (double)tc[i] / m_t) + config->alpha;
      }
    }
    if (err) break;
    if (config->expected) {
      err = so_update_model_expected(theta, n_docs, phi, K, W, config->alpha, config->beta,
                                     batch, B, tcf, pcf, m_t, rho_t);
    } else {
      err = so_update_model(theta, n_docs, phi, K, W, config->alpha, config->beta, batch, B,
                            tc, pc, m_t, rho_t);
    }
    if (err) break;
    double batch_tokens = 0.0;
    for (int64_t b = 0; b < B; ++b) {
      int64_t toks = 0;
      for (int64_t p = doc_offsets[batch[b]]; p < doc_offsets[batch[b] + 1]; ++p)
        toks += counts[p];
      batch_tokens += (double)toks;
    }
    tokens_seen += batch_tokens;
    samples_per_word += m_t * batch_tokens / corpus_tokens;
    if (ho_offsets != NULL && eval_every > 0 &&
        ((t + 1) % eval_every == 0 || t + 1 == config->t_max)) {
      double ll = 0.0;
      err = so_perword_loglik(phi, K, W, ho_offsets, ho_words, ho_counts, ho_docs,
                              config->alpha, config->seed, &ll);
      if (err) break;
      so_trace_row row = {t, tokens_seen / corpus_tokens, samples_per_word, ll, 0.0, m_t};
      trace[(*n_trace)++] = row;
    }
  }
  free(batch);
  free(theta_batch);
  free(mu);
  free(tc);
  free(pc);
  free(tcf);
  free(pcf);
  so_minibatch_free(&batches);
  return err;
}
