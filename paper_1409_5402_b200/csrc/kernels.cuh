// kernels.cuh -- launchers for the sm_100a SAME/LDA kernels (internal API).
//
// Device data model:
//   corpus   CSR, doc-major: doc_offsets i64[D+1], word_ids i32[nnz], counts i32[nnz]
//            (corpus.hpp:15-32), uploaded once and kept resident
//   theta    D x K f64, row-major (model.hpp:40-47)
//   phi      W x K f64, WORD-major (the reference stores K x W and transposes
//            twice per sweep, sampler.cpp:100,140; we never transpose on the
//            hot path)
//   counts   theta B x K and phi W x K, u64 (SampledCounts, sampler.hpp:50-68)
//   batch    doc ids i32[B] in MinibatchStream order + nnz prefix i64[B+1]
//            (batch_nnz_prefix, sampler.cpp:18-24)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace scu {

enum Mode : int { kModeParity = 0, kModeExpected = 1, kModeFast = 2 };

enum ErrBits : int { kErrNumerical = 1 };

// Process-wide tuning switches, read from the environment ONCE (forced at
// samelda_cu_create), never per launch.  All of them select bit-identical
// alternatives or test-only limits:
//   SAMELDA_SAMPLER=x      per-call sample_counts on the all-f64 exact kernel
//                          (device-side cross-check of the fast-exact path)
//   SAMELDA_COLSUM=chain   sequential TMA-chain column sums instead of the scan
//   SAMELDA_DRAW_CAP=n     deferred-draw list capacity (tests: overflow path)
//   SAMELDA_EVAL=...       held-out evaluation kernel variant (A/B)
//   SAMELDA_MINB/DEC/TAIL  k_sample_v2 A/B variants; only in a library built
//                          with -DSAMELDA_AB_VARIANTS (tools/), else ignored
struct Tuning {
  bool sampler_exact = false;
  bool colsum_chain = false;
  long long draw_cap = -1;  // < 0: default
  char eval_variant = 0;    // 0 default, 'c' cta, 'w' warp
  int eval_ctas_per_sm = 0;
  int minb = 4, dec = 1, tail = 0;
  bool fast_ptrs = true;  // deferred PTRS draws decided from the fast path's rate
};
const Tuning& tuning();

struct BatchView {
  const int64_t* doc_offsets;
  const int32_t* word_ids;
  const int32_t* counts;
  const int32_t* batch_docs;
  const int64_t* batch_prefix;
  int64_t B;
  int64_t nnz;       // batch_prefix[B]
  int64_t doc_base;  // global id of local doc 0 (doc-sharded runs): Philox keys use global ids
};

// theta_batch[b,:] = theta[batch_docs[b],:]            (sampler.cpp:313-317)
int launch_gather_theta(const double* theta, const int32_t* batch_docs, int64_t B, int K,
                        double* theta_batch, float* theta_batch32, cudaStream_t st);

// mu[p] = sum_k theta_batch[b,k] * phi[w,k], sequential k  (sampler.cpp:88-123)
int launch_sddmm(const BatchView& bv, const double* theta_batch, const double* phi_wk, int K,
                  double* mu, cudaStream_t st);

// Poisson replica sampling + count scatter                (sampler.cpp:125-195)
// mode kModeParity: reference-identical draws into u64 counts;
// mode kModeExpected: z := rate into f64 counts (deterministic factored path).
int launch_sample(const BatchView& bv, const double* theta_batch, const double* phi_wk,
                   const double* mu, int K, double m_t, uint64_t seed, uint32_t t,
                   uint32_t sweep, int mode, unsigned long long* theta_counts,
                   unsigned long long* phi_counts, double* theta_exp, double* phi_exp,
                   int* err, cudaStream_t st);

// The expected-count mode's non-final inner sweep: theta_exp[b,k] only
// (= theta_bk sum_w (m_t c_w / mu_w) phi_wk, written, f64; k_theta_rates).
// Returns -1 for K > 256 (the caller runs launch_sample).
int launch_expected_theta(const BatchView& bv, const double* theta_batch, const double* phi_wk, int K,
                          double m_t, double* theta_exp, cudaStream_t st);

// Same draws, bit for bit, through an f32 fast path with exact f64 fallback
// (see kernels_sample.cu).  mu == nullptr: the kernel forms mu itself (period path).
// mu_f_scratch: nnz floats (used when K > 256).
// `deferred` holds deferred_buffer_bytes(nnz, K) (fixed record slots per work
// item + a record count per item); n_deferred is one u64 (the records of the
// sweep, for profiling); `aux` holds deferred_aux_bytes(deferred_max_records(
// nnz, K), draw_cap) (per-record mu + a flat list of up to draw_cap deferred
// draws; overflow is drawn inline, never dropped).
int launch_sample_fast(const BatchView& bv, const double* theta_b64, const float* theta_b32,
                       const double* phi64, const float* phi32, const double* mu, int K,
                       double m_t, uint64_t seed, uint32_t t, uint32_t sweep,
                       unsigned long long* theta_counts, unsigned long long* phi_counts,
                       void* deferred, unsigned long long* n_deferred, void* aux,
                       int64_t draw_cap, float* mu_f_scratch, int* err, cudaStream_t st,
                       const double* mu_exact = nullptr, cudaEvent_t mu_ready = nullptr,
                       bool fast_ptrs = false);
// Throughput mode: the same sampler on its own random
// streams in f32, four draws per Philox block, no deferral -- statistically,
// not bit-for-bit, the reference's.  mu_f_scratch: nnz floats when K > 256.
// phi_counts == nullptr (a non-final inner sweep): theta counts only, drawn
// once per (document, topic) from the summed rate (k_theta_rates /
// k_theta_draws); rate_scratch: B x K floats.
int launch_sample_throughput(const BatchView& bv, const float* theta_b32, const float* phi32, int K,
                             double m_t, uint64_t seed, uint32_t t, uint32_t sweep,
                             unsigned long long* theta_counts, unsigned long long* phi_counts,
                             float* mu_f_scratch, float* rate_scratch, cudaStream_t st);
// Multinomial mode: per nonzero, floor(c m_t) (+1 with the fractional
// part's probability) categorical trials over the K topics (K <= 1024;
// returns -1 above), on this library's own streams.
int launch_sample_multinomial(const BatchView& bv, const float* theta_b32, const float* phi32, int K,
                              double m_t, uint64_t seed, uint32_t t, uint32_t sweep,
                              unsigned long long* theta_counts, unsigned long long* phi_counts,
                              int* err, cudaStream_t st);
int64_t deferred_max_records(int64_t nnz, int K);
int64_t deferred_buffer_bytes(int64_t nnz, int K);
// fills the device's glibc lgamma table (call once per device, after cudaSetDevice)
int init_lgamma_table();
int64_t deferred_aux_bytes(int64_t max_records, int64_t draw_cap);

// out[i] = counts[i] / m_t + alpha over n entries       (sampler.cpp:324-330)
int launch_theta_from_counts(const unsigned long long* counts_u, const double* counts_f,
                             int64_t n, double m_t, double alpha, double* out, float* out32,
                             cudaStream_t st);

// theta[batch_docs[b],k] = counts[b,k] / m_t + alpha     (sampler.cpp:204-210)
int launch_theta_persist(const unsigned long long* counts_u, const double* counts_f,
                          const int32_t* batch_docs, int64_t B, int K, double m_t,
                          double alpha, double* theta, cudaStream_t st);

// M-step for phi (sampler.cpp:211-228):
//   cand[w,k] = counts[w,k]/m_t + beta; total[k] = sum_w cand (sequential w, warp per topic);
//   phi = (1-rho) phi + rho cand / total
//   colsum_scratch (colsum_scratch_bytes(W, K) bytes): the exact parallel
//   column-sum scan; nullptr runs the sequential chain kernel
int launch_phi_mstep(const unsigned long long* counts_u, const double* counts_f, int64_t W,
                     int K, double m_t, double beta, double rho, double* phi_wk, float* phi32,
                     double* cand_scratch, double* totals, void* colsum_scratch, int* err,
                     cudaStream_t st);
int64_t colsum_scratch_bytes(int64_t W, int K);
// totals[k] = the reference's sequential sum over w of x[w,k], bit for bit
int launch_col_sums(const double* x, int64_t W, int K, double* totals, void* colsum_scratch,
                    int* err, cudaStream_t st);

// f32 shadow copy (the sampler's fast path reads f32 theta / phi)
// the count exchange in 32-bit words: lo[i] = c[i] (exact below bound),
// *n_over = number of cells >= bound (zeroed first)
int launch_pack_counts(const unsigned long long* c, int64_t n, unsigned long long bound, int32_t* lo,
                       unsigned long long* n_over, cudaStream_t st);
int launch_unpack_counts(const int32_t* lo, int64_t n, unsigned long long* c, cudaStream_t st);
int launch_to_f32(const double* x, int64_t n, float* y, cudaStream_t st);

// phi init with seeded perturbation (model.cpp:41-52, sampler.cpp:285-298)
int launch_phi_init(double* phi_wk, int64_t W, int K, double init_noise, uint64_t seed,
                     double* totals, void* colsum_scratch, cudaStream_t st);

// theta init alpha + 1/K (model.cpp:41-52)
int launch_fill(double* p, int64_t n, double v, cudaStream_t st);

// K x W <-> W x K transposes for the per-call boundary (model.cpp:31-39)
int launch_transpose(const double* in, int64_t rows, int64_t cols, double* out,
                      cudaStream_t st);

// per test document: the cells with a nonzero fold (score) half, compacted in
// cell order at the document's CSR offset, and their number
struct EvalLists {
  int32_t* n_fold;  // [n_docs]
  int2* fold;       // [nnz] (word id, fold count)
  int32_t* n_score; // [n_docs]
  int2* score;      // [nnz] (word id, score count)
};

// eval.cpp:99-121: per-doc seeded token split -> fold / score counts per cell
// (+ the compacted lists when lists.fold != nullptr)
int launch_eval_split(const int64_t* doc_offsets, const int32_t* word_ids, const int32_t* counts,
                       const int64_t* token_offsets, int64_t n_docs, uint64_t seed,
                       int32_t* slots, int32_t* fold_counts, int32_t* score_counts,
                       const EvalLists& lists, cudaStream_t st);

// eval.cpp:19-159 at 1e-12 relative (tree-ordered f64 sums, FMA; see
// kernels_eval.cu k_eval_fold): per-doc fold-in over the compacted lists,
// scoring, per-doc log p / scored.  Returns -1 when K > 1024 (use
// launch_eval_docs).
int launch_eval_fold(const int64_t* doc_offsets, const EvalLists& lists, int64_t n_docs,
                      const double* phi_wk, int K, double alpha, int sweeps, double* doc_logp,
                      int64_t* doc_scored, double* theta_out, int* err, cudaStream_t st);

// eval.cpp:19-64 + 125-145: per-doc fold-in then scoring.  theta_out (optional) n_docs x K.
int launch_eval_docs(const int64_t* doc_offsets, const int32_t* word_ids,
                      const int32_t* fold_counts, const int32_t* score_counts, int64_t n_docs,
                      const double* phi_wk, int K, double alpha, int sweeps, double* doc_logp,
                      int64_t* doc_scored, double* theta_out, double* scratch,
                      int64_t scratch_doubles, int* err, cudaStream_t st);

// eval.cpp:148-158: doc-order reduction -> ll
int launch_ordered_ll(const double* doc_logp, const int64_t* doc_scored, int64_t n_docs,
                       double* ll_out, int* err, cudaStream_t st);

// scratch doubles launch_eval_docs needs when K is too large for shared memory
int64_t eval_scratch_doubles(int K);

// collapsed Gibbs sampler baseline (cgs.cpp:11-157): state z (tokens), dt
// (D x K), wt (W x K) int32, tt (K) u64; tok_off = nnz + 1 token offsets
int launch_cgs_init(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                    const int64_t* tok_off, int64_t D, int K, uint64_t seed, int32_t* z, int32_t* dt,
                    int32_t* wt, unsigned long long* tt, cudaStream_t st);
int launch_cgs_sweep(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                     const int64_t* tok_off, int64_t D, int K, int64_t W, double alpha, double beta,
                     uint64_t seed, uint32_t sweep, int32_t* z, int32_t* dt, int32_t* wt,
                     unsigned long long* tt, int* err, cudaStream_t st);
// phi_wk W x K (eval layout); theta D x K (optional)
int launch_cgs_model(const int32_t* dt, const int32_t* wt, const unsigned long long* tt, int64_t D,
                     int64_t W, int K, double alpha, double beta, double* phi_wk, double* theta,
                     cudaStream_t st);

}  // namespace scu
