/*
 * samelda_io.h -- host-side data formats either side of the sampler hot path
 * (SURVEY.md 8(f) rows 1 and 3), exported by libsamelda_cuda.so.
 *
 *   corpus ingest   load_uci_bow (corpus.cpp:62-183) as a parallel mmap
 *                   parser with the reference's validation order and error
 *                   messages; save_uci_bow (corpus.cpp:186-213);
 *                   a binary CSR cache (no reference equivalent: loading a
 *                   NYTimes/PubMed docword text file dominates wall time at
 *                   GPU speeds);
 *   model output    save_checkpoint / load_checkpoint (model.cpp:54-111),
 *                   byte-identical files;
 *   metrics output  write_metrics_csv / read_metrics_csv (eval.cpp:161-210),
 *                   byte-identical files.
 *
 * Return codes as samelda_cu.h (1 ConfigError, 2 IoError); the message of
 * the last failing call on this thread is samelda_io_last_error().
 * Vocabularies cross the boundary as one buffer of n_words lines, each
 * terminated by '\n' (vocab_bytes counts the terminators).
 */
#ifndef SAMELDA_IO_H
#define SAMELDA_IO_H

#include <stdint.h>

#include "samelda_cu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct samelda_io_corpus samelda_io_corpus; /* owned host CSR + vocab */

const char* samelda_io_last_error(void);

/* replaces load_uci_bow (corpus.cpp:62-183): same result (rows sorted by word
 * id, duplicates merged, empty documents dropped with the same stderr note),
 * same IoError conditions checked in the same order.  n_threads <= 0: all
 * hardware threads. */
int samelda_io_load_uci(const char* docword_path, const char* vocab_path, int n_threads,
                        samelda_io_corpus** out);

/* binary CSR cache: header + doc_offsets + word_ids + counts + vocab */
int samelda_io_save_csr(const char* path, const samelda_cu_corpus* corpus, const char* vocab,
                        int64_t vocab_bytes);
int samelda_io_load_csr(const char* path, int n_threads, samelda_io_corpus** out);

/* dimensions and a zero-copy view (valid until samelda_io_corpus_free) */
void samelda_io_corpus_dims(const samelda_io_corpus* c, int64_t* n_docs, int64_t* n_words,
                            int64_t* nnz, int64_t* n_tokens, int64_t* vocab_bytes,
                            int64_t* dropped_docs);
void samelda_io_corpus_view(const samelda_io_corpus* c, samelda_cu_corpus* view,
                            const char** vocab);
void samelda_io_corpus_free(samelda_io_corpus* c);

/* replaces save_uci_bow (corpus.cpp:186-213) */
int samelda_io_save_uci(const samelda_cu_corpus* corpus, const char* vocab, int64_t vocab_bytes,
                        const char* docword_path, const char* vocab_path);

/* replaces save_checkpoint / load_checkpoint (model.cpp:54-111); phi is
 * K x W row-major (Model::phi) */
int samelda_io_save_checkpoint(const char* path, int64_t n_topics, int64_t n_words, double alpha,
                               double beta, const double* phi_kw);
int samelda_io_checkpoint_header(const char* path, int64_t* n_topics, int64_t* n_words,
                                 double* alpha, double* beta);
int samelda_io_load_checkpoint(const char* path, double* phi_kw, int64_t cap_elems);

/* replaces write_metrics_csv / read_metrics_csv (eval.cpp:161-210) */
int samelda_io_write_metrics_csv(const char* path, const samelda_cu_trace_row* rows, int64_t n);
int samelda_io_read_metrics_csv(const char* path, samelda_cu_trace_row* rows, int64_t cap,
                                int64_t* n);

#ifdef __cplusplus
}
#endif
#endif
