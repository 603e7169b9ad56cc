/*
 * samelda_cu.h -- C ABI of libsamelda_cuda.so, the B200 (sm_100a) drop-in for
 * the SAME factored Gibbs sampler hot path of the reference library
 * `samelda` (arXiv 1409.5402; reference sources under proj/).
 *
 * Plain pointers and sizes only: no CUDA, torch or C++ types cross this
 * boundary.  All host buffers are caller-owned (the reference passes values
 * and const references and returns by value, sampler.hpp / eval.hpp).
 *
 * Return codes map onto the reference's exception classes (errors.hpp:7-20):
 *   0 ok, 1 ConfigError, 2 IoError, 3 NumericalError, 4 CUDA runtime failure.
 * samelda_cu_last_error() holds the message of the last failing call.
 *
 * Every entry point names the reference interface it replaces (file:line in
 * proj/).  INTEGRATION.md shows the C++ shim that binds them behind the
 * unchanged reference headers.
 */
#ifndef SAMELDA_CU_H
#define SAMELDA_CU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAMELDA_CU_OK 0
#define SAMELDA_CU_CONFIG 1
#define SAMELDA_CU_IO 2
#define SAMELDA_CU_NUMERICAL 3
#define SAMELDA_CU_CUDA 4

/* sampling modes */
#define SAMELDA_CU_MODE_PARITY 0   /* reference-identical Poisson replicas, f64 */
#define SAMELDA_CU_MODE_EXPECTED 1 /* deterministic factored expected counts, f64 */
#define SAMELDA_CU_MODE_THROUGHPUT 2 /* the same Poisson replicas on this library's own
                                        random streams in f32: statistically, not
                                        bit-for-bit, the reference's sampler */
#define SAMELDA_CU_MODE_MULTINOMIAL 3 /* north_star's multinomial(c m) replicas: per
                                         nonzero floor(c m_t) (+1 with the fractional
                                         part's probability) categorical trials, so
                                         E z = c m_t r as the Poisson replicas and
                                         sum_k z_k = the trial count; own f32 streams,
                                         K <= 1024; no reference implementation */

/* AnnealSchedule (sampler.hpp:17) */
#define SAMELDA_CU_SCHEDULE_CONSTANT 0
#define SAMELDA_CU_SCHEDULE_LINEAR 1
#define SAMELDA_CU_SCHEDULE_LOG 2
#define SAMELDA_CU_SCHEDULE_INVLINEAR 3

typedef struct samelda_cu_ctx samelda_cu_ctx;

/* Corpus view (corpus.hpp:15-32): CSR over documents, word ids strictly
 * increasing per row, counts >= 1, doc_offsets[n_docs] == nnz. */
typedef struct {
  const int64_t* doc_offsets; /* n_docs + 1 */
  const int32_t* word_ids;    /* nnz */
  const int32_t* counts;      /* nnz */
  int64_t n_docs;
  int64_t n_words; /* vocabulary size W */
} samelda_cu_corpus;

/* SamplerConfig (sampler.hpp:23-42); n_threads has no meaning here. */
typedef struct {
  int64_t n_topics;
  double m;
  int32_t schedule;
  double tau0;
  double gamma;
  double batch_fraction;
  int64_t t_max;
  int64_t inner_sweeps;
  uint64_t seed;
  double alpha;
  double beta;
  double init_noise;
  int32_t mode; /* SAMELDA_CU_MODE_* */
} samelda_cu_config;

/* TraceRow (eval.hpp:16-23) */
typedef struct {
  int64_t t;
  double passes;
  double samples_per_word;
  double ll;
  double wall_seconds;
  double m_t;
} samelda_cu_trace_row;

/* ------------------------------------------------------------ context */
int samelda_cu_version(void);
/* number of visible CUDA devices (0 without a usable driver) */
int samelda_cu_device_count(void);
int samelda_cu_create(int device, samelda_cu_ctx** out);
void samelda_cu_destroy(samelda_cu_ctx* ctx);
const char* samelda_cu_last_error(const samelda_cu_ctx* ctx);
/* Run every kernel of this context on `cuda_stream` (a cudaStream_t), e.g.
 * the caller's framework stream; NULL is the legacy default stream.  A new
 * context runs on its own non-blocking stream; samelda_cu_use_own_stream
 * returns to it. */
int samelda_cu_set_stream(samelda_cu_ctx* ctx, void* cuda_stream);
int samelda_cu_use_own_stream(samelda_cu_ctx* ctx);
int samelda_cu_synchronize(samelda_cu_ctx* ctx);
/* number of kernel launches this context issued since creation */
int64_t samelda_cu_launch_count(const samelda_cu_ctx* ctx);

/* ------------------------------------------ per-call mirrors (host buffers) */

/* replaces samelda::sddmm, sampler.hpp:74-81 / sampler.cpp:88-123.
 * theta_batch B x K_theta row-major, phi K x W row-major; mu_out receives
 * sum_b nnz(doc_ids[b]) values in concatenated batch order (*mu_len). */
int samelda_cu_sddmm(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                     const double* theta_batch, int64_t B, int64_t K_theta, const double* phi,
                     int64_t K, int64_t W, const int32_t* doc_ids, double* mu_out,
                     int64_t mu_cap, int64_t* mu_len);

/* replaces samelda::sample_counts, sampler.hpp:83-91 / sampler.cpp:125-195.
 * Outputs SampledCounts' arrays: theta_counts B x K, phi_counts W x K. */
int samelda_cu_sample_counts(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                             const double* theta_batch, int64_t B, int64_t K_theta,
                             const double* phi, int64_t K, int64_t W, const double* mu,
                             int64_t mu_len, const int32_t* doc_ids, double m_t, uint64_t seed,
                             int64_t t, int32_t sweep, int64_t* theta_counts,
                             int64_t* phi_counts);

/* Throughput mode (SURVEY 8(b) "mode 2 fast"): sample_counts on this
 * library's own f32 random streams -- the same Poisson replicas, so the same
 * law, but not the reference's draws.  mu is validated for alignment and not
 * read (the kernel forms its own f32 mu).  Counts are deterministic for given
 * inputs (integer scatter; streams keyed by coordinates, not by schedule). */
int samelda_cu_sample_counts_fast(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                                  const double* theta_batch, int64_t B, int64_t K_theta,
                                  const double* phi, int64_t K, int64_t W, const double* mu,
                                  int64_t mu_len, const int32_t* doc_ids, double m_t,
                                  uint64_t seed, int64_t t, int32_t sweep, int64_t* theta_counts,
                                  int64_t* phi_counts);

/* Throughput mode, non-final inner sweep (sampler.cpp:318-319: only the
 * theta counts of a sweep before the last are used): theta_counts[b,k] drawn
 * ONCE per (document, topic) as Poisson(theta_bk sum_w (m_t c_w / mu_w)
 * phi_wk) -- the law of the per-(nonzero, topic) draws' sum (a sum of
 * independent Poissons), with mu the f32 dot the kernel forms.  This is what
 * the device-resident period runs for its inner sweeps in
 * SAMELDA_CU_MODE_THROUGHPUT; deterministic for given inputs. */
int samelda_cu_sample_theta_counts_fast(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                                        const double* theta_batch, int64_t B, int64_t K_theta,
                                        const double* phi, int64_t K, int64_t W, const int32_t* doc_ids,
                                        double m_t, uint64_t seed, int64_t t, int32_t sweep,
                                        int64_t* theta_counts);

/* Multinomial mode (SAMELDA_CU_MODE_MULTINOMIAL): sample_counts with the
 * c m_t replicas of each nonzero drawn jointly as Multinomial(n, theta phi /
 * mu), n = floor(c m_t) (+1 with probability frac(c m_t)); this library's own
 * streams, deterministic for given inputs.  mu is validated for alignment and
 * not read.  K <= 1024. */
int samelda_cu_sample_counts_multinomial(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                                         const double* theta_batch, int64_t B, int64_t K_theta,
                                         const double* phi, int64_t K, int64_t W, const double* mu,
                                         int64_t mu_len, const int32_t* doc_ids, double m_t,
                                         uint64_t seed, int64_t t, int32_t sweep,
                                         int64_t* theta_counts, int64_t* phi_counts);

/* Deterministic factored path: sample_counts with z := E[z] = rate, f64. */
int samelda_cu_expected_counts(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                               const double* theta_batch, int64_t B, int64_t K_theta,
                               const double* phi, int64_t K, int64_t W, const double* mu,
                               int64_t mu_len, const int32_t* doc_ids, double m_t,
                               double* theta_expected, double* phi_expected);

/* replaces samelda::update_model, sampler.hpp:93-97 / sampler.cpp:197-229.
 * theta D x K and phi K x W are updated in place. */
int samelda_cu_update_model(samelda_cu_ctx* ctx, double* theta, int64_t D, double* phi,
                            int64_t K, int64_t W, double alpha, double beta,
                            const int32_t* doc_ids, int64_t B, const int64_t* theta_counts,
                            const int64_t* phi_counts, double m_t, double rho_t);
int samelda_cu_update_model_expected(samelda_cu_ctx* ctx, double* theta, int64_t D,
                                     double* phi, int64_t K, int64_t W, double alpha,
                                     double beta, const int32_t* doc_ids, int64_t B,
                                     const double* theta_expected, const double* phi_expected,
                                     double m_t, double rho_t);

/* replaces samelda::rho_schedule / anneal_m, sampler.cpp:231-267 (host math) */
int samelda_cu_rho_schedule(int64_t t, double tau0, double gamma, double* out);
int samelda_cu_anneal_m(int32_t schedule, int64_t t, int64_t t_max, double m, double* out);

/* replaces samelda::fold_in_theta, eval.hpp:32-36 / eval.cpp:68-73 */
int samelda_cu_fold_in_theta(samelda_cu_ctx* ctx, const double* phi, int64_t K, int64_t W,
                             const int32_t* words, const int32_t* counts, int64_t n,
                             double alpha, int32_t sweeps, double* theta_out);

/* Held-out evaluation arithmetic (fold_in_theta, perword_loglik, evaluate).
 * exact = 0 (default): per-document fold-in with tree-ordered f64 sums and
 *   FMA -- ll within SURVEY 8(d)'s 1e-12 relative of the reference, theta
 *   within 1e-12 relative (k_eval_fold);
 * exact = 1: the reference's summation order (eval.cpp:30-62), ll and theta
 *   bit-identical, ~10x slower.  SAMELDA_EVAL=x sets it at create. */
int samelda_cu_set_eval_exact(samelda_cu_ctx* ctx, int exact);

/* replaces samelda::perword_loglik, eval.hpp:38-43 / eval.cpp:75-159 */
int samelda_cu_perword_loglik(samelda_cu_ctx* ctx, const double* phi, int64_t K, int64_t W,
                              const samelda_cu_corpus* test, double alpha, uint64_t seed,
                              double* ll_out);

/* --------------------------------------- device-resident trainer (train()) */

/* Minibatch stream (corpus.hpp:62-84, corpus.cpp:252-285), host-side. */
typedef struct samelda_cu_batches samelda_cu_batches;
int samelda_cu_batches_create(int64_t n_docs, double batch_fraction, uint64_t seed,
                              samelda_cu_batches** out);
int64_t samelda_cu_batches_size(const samelda_cu_batches* s);
int64_t samelda_cu_batches_per_pass(const samelda_cu_batches* s);
/* writes the next batch's doc ids into out (capacity >= batch size) */
int64_t samelda_cu_batches_next(samelda_cu_batches* s, int32_t* out);
void samelda_cu_batches_destroy(samelda_cu_batches* s);

/* sampler.cpp:269-300: validate, upload the corpus, init_model + init noise
 * on the device.  The model stays resident until the next train_begin. */
int samelda_cu_train_begin(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                           const samelda_cu_config* config);
/* held-out corpus + split seed for samelda_cu_evaluate; the 50/50 token split
 * (eval.cpp:99-121) depends only on (corpus, seed) and is computed once. */
int samelda_cu_heldout(samelda_cu_ctx* ctx, const samelda_cu_corpus* test, uint64_t seed);

/* One period (sampler.cpp:307-333) on the resident model: gather theta rows,
 * inner_sweeps x (sddmm, sample), persist theta, M-step on phi.
 * Asynchronous: the host does not wait for the device; a NumericalError raised
 * on the device (non-finite rate, bad phi row mass) is reported by the next
 * period call or by the next synchronising call (samelda_cu_synchronize,
 * _evaluate, _model_download, _batch_theta, _count_totals). */
int samelda_cu_period(samelda_cu_ctx* ctx, const int32_t* doc_ids, int64_t B, int64_t t,
                      double m_t, double rho_t);
/* The same period split at the topic-word count exchange, for doc-sharded
 * multi-GPU runs: sample -> caller all-reduces the phi counts buffer
 * (samelda_cu_phi_counts_device) -> update. */
int samelda_cu_period_sample(samelda_cu_ctx* ctx, const int32_t* doc_ids, int64_t B,
                             int64_t t, double m_t);
int samelda_cu_period_update(samelda_cu_ctx* ctx, double rho_t);
/* device address of the W x K phi count buffer of the last sampled sweep;
 * elem_bytes is 8 (u64 parity counts or f64 expected counts); is_float 1 for f64. */
int samelda_cu_phi_counts_device(samelda_cu_ctx* ctx, void** ptr, int64_t* n_elems,
                                 int32_t* elem_bytes, int32_t* is_float);
/* The count exchange in 32-bit words (half the bytes of the u64
 * all-reduce), integer-count modes: pack32 writes lo[i] = count[i] as int32
 * into the caller's device buffer and the number of cells >= (2^31 - 1) /
 * world_size into the caller's device u64 *n_over (zeroed first), on the
 * context's stream.  When the all-reduced n_over is 0, the int32 all-reduce
 * of lo is exact (its sums stay below 2^31) and unpack32 writes the summed
 * counts back into the W x K buffer; otherwise the caller all-reduces the
 * untouched u64 buffer instead. */
int samelda_cu_phi_counts_pack32(samelda_cu_ctx* ctx, void* lo, int64_t n_elems, int32_t world_size,
                                 void* n_over);
int samelda_cu_phi_counts_unpack32(samelda_cu_ctx* ctx, const void* lo, int64_t n_elems);
/* Doc-sharded runs: this context holds documents [doc_base, doc_base + D)
 * of the global corpus under local ids 0..D-1; Philox stream keys use the
 * global id, so every shard draws exactly what a single GPU would. */
int samelda_cu_set_doc_base(samelda_cu_ctx* ctx, int64_t doc_base);
/* CUDA-event timing of the period kernels (0 sampling of a non-final inner
 * sweep, 1 sddmm, 2 M-step, 3 sampling of the final inner sweep -- the one
 * that scatters phi counts). */
int samelda_cu_profile(samelda_cu_ctx* ctx, int32_t enable);
/* ms_out[4] summed event time, launches_out[4] launches timed; batch nonzeros
 * and docs seen by the timed sample launches, and the deferred exact-draw
 * records they produced (profiling synchronises after every sample launch to
 * read that count).  Resets the accumulators. */
int samelda_cu_profile_read(samelda_cu_ctx* ctx, double* ms_out, int64_t* launches_out,
                            int64_t* nnz_sampled, int64_t* docs_sampled, int64_t* deferred);
/* copy the batch theta rows (B x K, f64, batch order) of the last period */
int samelda_cu_batch_theta(samelda_cu_ctx* ctx, double* out, int64_t cap);
/* the same copy without a host wait: the rows are gathered on the context
 * stream and copied on a context-owned copy stream, so the transfer overlaps
 * the next periods' kernels (two row buffers rotate); `out` (page-locked)
 * holds the rows after samelda_cu_synchronize or a device-wide synchronize. */
int samelda_cu_batch_theta_async(samelda_cu_ctx* ctx, double* out, int64_t cap);
/* sums of the last sweep's integer theta and phi counts (mass balance) */
int samelda_cu_count_totals(samelda_cu_ctx* ctx, int64_t* theta_total, int64_t* phi_total);

/* perword_loglik(phi_resident, heldout, alpha, seed) (sampler.cpp:341-345) */
int samelda_cu_evaluate(samelda_cu_ctx* ctx, double* ll_out);

/* phi K x W (reference layout) and theta D x K; either may be NULL */
int samelda_cu_model_download(samelda_cu_ctx* ctx, double* phi, double* theta);
int samelda_cu_model_upload(samelda_cu_ctx* ctx, const double* phi, const double* theta);

/* replaces samelda::train, sampler.hpp:105-110 / sampler.cpp:269-353, end to
 * end: returns phi (K x W), theta (D x K) and the metrics trace. */
int samelda_cu_train(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus,
                     const samelda_cu_config* config, const samelda_cu_corpus* heldout,
                     int64_t eval_every, double* phi_out, double* theta_out,
                     samelda_cu_trace_row* trace, int64_t trace_cap, int64_t* n_trace);

/* ------------------------------------ collapsed Gibbs sampler (the baseline)
 *
 * The paper's comparison method: cgs.hpp:17-49 /
 * cgs.cpp:11-157 with the reference's draws (state in the context; the
 * corpus is the context's training corpus).  The sweep is sequential by
 * definition (one token at a time); on the device it is one warp. */
/* replaces samelda::cgs_init, cgs.hpp:29-31 / cgs.cpp:11-55 (n_topics <= 1024) */
int samelda_cu_cgs_init(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus, int64_t n_topics,
                        double alpha, double beta, uint64_t seed);
/* replaces samelda::cgs_sweep, cgs.hpp:33-38 / cgs.cpp:57-98 (asynchronous) */
int samelda_cu_cgs_sweep(samelda_cu_ctx* ctx, uint64_t seed, int64_t sweep_index);
/* CgsState's arrays (cgs.hpp:17-27): z (n_tokens), doc_topic D x K, word_topic
 * W x K, topic_total K; any may be NULL */
int samelda_cu_cgs_state(samelda_cu_ctx* ctx, int32_t* z, int32_t* doc_topic, int32_t* word_topic,
                         int64_t* topic_total);
int samelda_cu_cgs_set_state(samelda_cu_ctx* ctx, const int32_t* z, const int32_t* doc_topic,
                             const int32_t* word_topic, const int64_t* topic_total);
/* replaces samelda::cgs_model, cgs.hpp:40-41 / cgs.cpp:100-129: phi K x W, theta D x K */
int samelda_cu_cgs_model(samelda_cu_ctx* ctx, double* phi, double* theta);
/* replaces samelda::cgs_train, cgs.hpp:43-49 / cgs.cpp:131-157 */
int samelda_cu_cgs_train(samelda_cu_ctx* ctx, const samelda_cu_corpus* corpus, int64_t n_topics,
                         double alpha, double beta, int64_t n_sweeps, uint64_t seed,
                         int64_t eval_every, const samelda_cu_corpus* heldout, double* phi_out,
                         double* theta_out, samelda_cu_trace_row* trace, int64_t trace_cap,
                         int64_t* n_trace);

/* ------------------------------------- multi-GPU group (one process, N GPUs)
 *
 * SURVEY.md 8(e) behind the ABI: documents are split into contiguous ranges
 * balanced by nonzeros, one context per device; every period each device
 * samples the batch documents it owns (Philox keys use global document ids),
 * the W x K topic-word counts are summed in place over the devices with
 * ncclAllReduce (communicator from ncclCommInitAll over `devices`; NCCL is
 * loaded at run time), and the M-step runs replicated.  In the integer-count
 * modes the model is bit-identical to one GPU's for any device count.
 * A list that repeats one device (tests on a one-GPU box) exchanges with a
 * device-side sum instead of NCCL. */
typedef struct samelda_cu_group samelda_cu_group;
int samelda_cu_group_create(const int* devices, int n, samelda_cu_group** out);
void samelda_cu_group_destroy(samelda_cu_group* g);
const char* samelda_cu_group_last_error(const samelda_cu_group* g);
int samelda_cu_group_size(const samelda_cu_group* g);
/* 1 when the exchange runs over an NCCL communicator */
int samelda_cu_group_uses_nccl(const samelda_cu_group* g);
/* the sharded counterparts of samelda_cu_train_begin / _heldout / _period /
 * _synchronize / _evaluate / _model_download (doc ids are GLOBAL ids) */
int samelda_cu_group_train_begin(samelda_cu_group* g, const samelda_cu_corpus* corpus,
                                 const samelda_cu_config* config);
int samelda_cu_group_heldout(samelda_cu_group* g, const samelda_cu_corpus* test, uint64_t seed);
int samelda_cu_group_period(samelda_cu_group* g, const int32_t* doc_ids, int64_t B, int64_t t,
                            double m_t, double rho_t);
int samelda_cu_group_synchronize(samelda_cu_group* g);
int samelda_cu_group_evaluate(samelda_cu_group* g, double* ll_out);
int samelda_cu_group_model_download(samelda_cu_group* g, double* phi, double* theta);
/* replaces samelda::train (sampler.hpp:105-110 / sampler.cpp:269-353) on N GPUs */
int samelda_cu_group_train(samelda_cu_group* g, const samelda_cu_corpus* corpus,
                           const samelda_cu_config* config, const samelda_cu_corpus* heldout,
                           int64_t eval_every, double* phi_out, double* theta_out,
                           samelda_cu_trace_row* trace, int64_t trace_cap, int64_t* n_trace);

#ifdef __cplusplus
}
#endif
#endif
