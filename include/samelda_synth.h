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
/* offsets n_docs + 1, words / counts nnz */
void samelda_synth_copy(void* handle, int64_t* offsets, int32_t* words, int32_t* counts);
void samelda_synth_free(void* handle);

#ifdef __cplusplus
}
#endif
#endif
