/*
 * samelda_synth.h -- synthetic LDA corpora at NYTimes / PubMed shape
 * (BASELINE.json configs 1-4).  Host-side data generation for the bench and
 * tests; not part of the hot path.  Replaces, for scale, the reference's
 * tests/support/synthetic.cpp:61-106 make_corpus (O(tokens x W)).
 */
#ifndef SAMELDA_SYNTH_H
#define SAMELDA_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t n_docs;
  int64_t n_words;
  int64_t n_topics_gen;  /* generating topics */
  double mean_len;       /* mean tokens per document */
  double len_shape;      /* gamma shape of the length distribution */
  double zipf_s;         /* Zipf exponent of topic-word distributions */
  double background;     /* weight of the shared background distribution */
  double topics_per_doc; /* mean extra topics per document (geometric) */
  uint64_t seed;
  int64_t first_doc; /* global id of the first generated doc (sharded generation) */
} samelda_synth_params;

/* Generates into an opaque handle; returns 0 or 1 (bad parameters). */
int samelda_synth_generate(const samelda_synth_params* params, int n_threads, void** handle,
                           int64_t* nnz, int64_t* n_tokens);
/* The reference's own generator, synthetic::make_corpus
 * (tests/support/synthetic.cpp:61-106; defaults theta_conc 0.2, phi_conc 0.08),
 * value for value on the reference's Philox streams, documents in parallel.
 * BASELINE.json configs[0] = (10000, 5000, 32, 100.0, seed 1). */
int samelda_synth_make_corpus_ref(int64_t n_docs, int64_t n_words, int64_t n_topics,
                                  double len_mean, uint64_t seed, double theta_conc,
                                  double phi_conc, int n_threads, void** handle, int64_t* nnz,
                                  int64_t* n_tokens);
/* split_holdout's document ids (corpus.cpp:231-250): test_ids (capacity
 * n_docs) and train_ids (capacity n_docs), both sorted; *n_test written. */
int samelda_synth_split_holdout(int64_t n_docs, double test_fraction, uint64_t seed,
                                int32_t* test_ids, int64_t* n_test, int32_t* train_ids);
/* offsets n_docs + 1, words / counts nnz */
void samelda_synth_copy(void* handle, int64_t* offsets, int32_t* words, int32_t* counts);
void samelda_synth_free(void* handle);

#ifdef __cplusplus
}
#endif
#endif
