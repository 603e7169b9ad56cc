// kernels_eval.cu -- sm_100a held-out evaluation (perword_loglik /
// fold_in_theta, eval.cpp:19-159): token split, fold-in + scoring kernels,
// document-order reduction.
#include "kernels_common.cuh"

#include <cstdio>

namespace scu {

namespace {

// --------------------------------------------------------------------- eval
// eval.cpp:99-121, one thread per test document.
// Besides the per-cell halves it writes each document's compacted fold and
// score cell lists (word, count of the cells with a nonzero half, in cell
// order) at the document's CSR offset, with their lengths per document: the
// inputs of k_eval_fold.  The split depends only on (test corpus, seed), so it
// runs once per corpus and seed.
__global__ void k_eval_split(const int64_t* __restrict__ doc_offsets,
                             const int32_t* __restrict__ word_ids,
                             const int32_t* __restrict__ counts,
                             const int64_t* __restrict__ token_offsets, int64_t n_docs,
                             uint64_t seed, int32_t* __restrict__ slots,
                             int32_t* __restrict__ fold_counts,
                             int32_t* __restrict__ score_counts, EvalLists lists) {
  const int64_t d = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (d >= n_docs) return;
  const int64_t begin = doc_offsets[d], end = doc_offsets[d + 1];
  int32_t* sl = slots + token_offsets[d];
  int64_t pos = 0;
  for (int64_t i = begin; i < end; ++i) {
    fold_counts[i] = 0;
    score_counts[i] = 0;
    for (int32_t r = 0; r < counts[i]; ++r) sl[pos++] = static_cast<int32_t>(i - begin);
  }
  const int64_t n_tokens = pos;
  Stream s;
  s.init(seed, 0u, static_cast<uint32_t>(d), 0u, make_tag(kEvalSplit, 0, 0));
  for (int64_t i = n_tokens - 1; i > 0; --i) {
    const int64_t j = static_cast<int64_t>(s.uniform_below(static_cast<uint64_t>(i) + 1));
    const int32_t tmp = sl[i];
    sl[i] = sl[j];
    sl[j] = tmp;
  }
  const int64_t n_fold = (n_tokens + 1) / 2;
  for (int64_t i = 0; i < n_tokens; ++i) {
    if (i < n_fold) ++fold_counts[begin + sl[i]]; else ++score_counts[begin + sl[i]];
  }
  if (lists.fold == nullptr) return;
  int32_t nf = 0, ns = 0;
  for (int64_t i = begin; i < end; ++i) {
    const int32_t w = word_ids[i], f = fold_counts[i], s = score_counts[i];
    if (f != 0) lists.fold[begin + nf++] = make_int2(w, f);
    if (s != 0) lists.score[begin + ns++] = make_int2(w, s);
  }
  lists.n_fold[d] = nf;
  lists.n_score[d] = ns;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One warp per test document: fold-in (eval.cpp:19-64) then scoring
// (eval.cpp:125-145).  Dot products mu / p run lane-per-cell in sequential k
// order; the responsibility update runs lane-per-topic in cell order, so all
// f64 sums accumulate in the reference's order.
constexpr int kEvalWarps = 4;

// sum_k th[k] * row[k] in sequential k order (product then add, no FMA),
// 16-byte loads when the row is 16-byte aligned (K even)
__device__ __forceinline__ double seq_dot(const double* __restrict__ th,
                                          const double* __restrict__ row, int K) {
  double dot = 0.0;
  if ((K & 1) == 0) {
    const double2* r2 = reinterpret_cast<const double2*>(row);
    // unrolled so several row loads are in flight ahead of the (sequential) adds
#pragma unroll 8
    for (int k2 = 0; k2 < (K >> 1); ++k2) {
      const double2 v = __ldg(r2 + k2);
      dot = __dadd_rn(dot, __dmul_rn(th[2 * k2], v.x));
      dot = __dadd_rn(dot, __dmul_rn(th[2 * k2 + 1], v.y));
    }
  } else {
    for (int k = 0; k < K; ++k) dot = __dadd_rn(dot, __dmul_rn(th[k], __ldg(row + k)));
  }
  return dot;
}

// seq_dot over a row in global memory with deeper memory-level parallelism:
// 16-double blocks (8 x 16-byte loads) double-buffered in registers, so the
// next block's loads are in flight while the current block's sequential
// adds run (same order, same rounding as seq_dot).  K % 16 == 0.
__device__ __forceinline__ double seq_dot_pipe(const double* __restrict__ th,
                                               const double* __restrict__ row, int K) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
  double2 cur[8], nxt[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) cur[j] = __ldg(r2 + j);
  double dot = 0.0;
  for (int b = 0; b < K; b += 16) {
    if (b + 16 < K) {
#pragma unroll
      for (int j = 0; j < 8; ++j) nxt[j] = __ldg(r2 + (b + 16) / 2 + j);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      dot = __dadd_rn(dot, __dmul_rn(th[b + 2 * j], cur[j].x));
      dot = __dadd_rn(dot, __dmul_rn(th[b + 2 * j + 1], cur[j].y));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) cur[j] = nxt[j];
  }
  return dot;
}

__device__ __forceinline__ double seq_dot_g(const double* __restrict__ th,
                                            const double* __restrict__ row, int K) {
  return (K & 15) == 0 ? seq_dot_pipe(th, row, K) : seq_dot(th, row, K);
}

__global__ void __launch_bounds__(kEvalWarps * 32) k_eval_docs(
    const int64_t* __restrict__ doc_offsets, const int32_t* __restrict__ word_ids,
    const int32_t* __restrict__ fold_counts, const int32_t* __restrict__ score_counts,
    int64_t n_docs, const double* __restrict__ phi_wk, int K, double alpha, int sweeps,
    double* __restrict__ doc_logp, int64_t* __restrict__ doc_scored,
    double* __restrict__ theta_out, double* __restrict__ scratch, int* __restrict__ err) {
  extern __shared__ double smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t slot = blockIdx.x * static_cast<int64_t>(kEvalWarps) + wib;
  const int64_t per = 2 * static_cast<int64_t>(K);
  double* th = scratch ? scratch + slot * per : smem + wib * per;
  double* nx = th + K;
  const double inv_k = 1.0 / static_cast<double>(K);
  for (int64_t doc = slot; doc < n_docs; doc += static_cast<int64_t>(gridDim.x) * kEvalWarps) {
    const int64_t base = doc_offsets[doc];
    const int64_t n = doc_offsets[doc + 1] - base;
    for (int k = lane; k < K; k += 32) th[k] = inv_k;
    __syncwarp();
    for (int sweep = 0; sweep < sweeps && n > 0; ++sweep) {
      for (int k = lane; k < K; k += 32) nx[k] = alpha;
      for (int64_t i0 = 0; i0 < n; i0 += 32) {
        const int64_t i = i0 + lane;
        int32_t w = 0;
        double scale = 0.0;
        bool use = false;
        if (i < n) {
          const int32_t fc = fold_counts[base + i];
          w = word_ids[base + i];
          if (fc != 0) {  // a zero-count cell adds exactly +0 (eval.cpp:43-47)
            const double mu = seq_dot(th, phi_wk + static_cast<int64_t>(w) * K, K);
            if (mu > 0.0) {
              scale = __ddiv_rn(static_cast<double>(fc), mu);
              use = true;
            }
          }
        }
        unsigned mask = __ballot_sync(0xffffffffu, use);
        __syncwarp();
        while (mask) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1;
          const double s = __shfl_sync(0xffffffffu, scale, src);
          const int32_t ww = __shfl_sync(0xffffffffu, w, src);
          const double* ph = phi_wk + static_cast<int64_t>(ww) * K;
          for (int k = lane; k < K; k += 32)
            nx[k] = __dadd_rn(nx[k], __dmul_rn(__dmul_rn(s, th[k]), __ldg(ph + k)));
        }
      }
      __syncwarp();
      double total = 0.0;
      if (lane == 0)
        for (int k = 0; k < K; ++k) total = __dadd_rn(total, nx[k]);
      total = __shfl_sync(0xffffffffu, total, 0);
      double delta = 0.0;
      for (int k = lane; k < K; k += 32) {
        const double v = __ddiv_rn(nx[k], total);
        delta = fmax(delta, fabs(__dadd_rn(v, -th[k])));
        th[k] = v;
      }
      delta = warp_max(delta);
      __syncwarp();
      if (delta < 1e-12) break;
    }
    // score the held-back half in cell order
    double logp = 0.0;
    int64_t scored = 0;
    for (int64_t i0 = 0; i0 < n; i0 += 32) {
      const int64_t i = i0 + lane;
      int32_t sc = 0;
      double term = 0.0;
      if (i < n) {
        sc = score_counts[base + i];
        if (sc != 0) {
          const double p = seq_dot(th, phi_wk + static_cast<int64_t>(word_ids[base + i]) * K, K);
          if (!(p > 0.0)) atomicOr(err, kErrNumerical);
          term = __dmul_rn(static_cast<double>(sc), log(p));
        }
      }
      const int n_here = static_cast<int>(min(static_cast<int64_t>(32), n - i0));
      for (int j = 0; j < n_here; ++j) {
        const int32_t scj = __shfl_sync(0xffffffffu, sc, j);
        const double tj = __shfl_sync(0xffffffffu, term, j);
        if (scj != 0) {
          logp = __dadd_rn(logp, tj);
          scored += scj;
        }
      }
    }
    if (lane == 0) {
      doc_logp[doc] = logp;
      doc_scored[doc] = scored;
    }
    if (theta_out)
      for (int k = lane; k < K; k += 32) theta_out[doc * K + k] = th[k];
    __syncwarp();
  }
}

// CTA per test document (K <= kEvalCtaMaxK): the same arithmetic in the same
// order as k_eval_docs / eval.cpp:19-64, laid out so a document's phi rows
// stay L2-resident across its fold-in sweeps (~600 documents in flight, their
// fold rows ~90 MB) and every step has block-wide parallelism:
//   phase 1, thread = cell: mu_i = sequential-k dot (eval.cpp:38-41), scale
//     c_i / mu_i for the cells that inform theta;
//   phase 2, thread = topic: next[k] += (scale_i theta[k]) phi[w_i][k] over
//     the chunk's cells in cell order (eval.cpp:45-49) -- coalesced rows;
//   phase 3: total in sequential k order (one thread), theta = next / total,
//     block max of |delta| (eval.cpp:51-60).
// Scoring: thread = cell dot, doc log p summed in cell order by one thread.
constexpr int kEvalCtaThreads = 256;
constexpr int kEvalCtaMaxK = 4096;

__global__ void __launch_bounds__(kEvalCtaThreads) k_eval_cta(
    const int64_t* __restrict__ doc_offsets, const int32_t* __restrict__ word_ids,
    const int32_t* __restrict__ fold_counts, const int32_t* __restrict__ score_counts,
    int64_t n_docs, const double* __restrict__ phi_wk, int K, double alpha, int sweeps,
    double* __restrict__ doc_logp, int64_t* __restrict__ doc_scored,
    double* __restrict__ theta_out, int* __restrict__ err) {
  extern __shared__ double smem[];
  const int KE = (K + 1) & ~1;       // even padding, as k_eval_stage
  double* th = smem;                 // K (+ pad)
  double* nx = th + KE;              // K (+ pad)
  double* cs = nx + KE;              // [256] cell scale (0 = skip) / score term
  int32_t* cw = reinterpret_cast<int32_t*>(cs + kEvalCtaThreads);  // [256] cell word
  __shared__ double s_red[kEvalCtaThreads / 32];
  __shared__ int64_t s_cnt[kEvalCtaThreads];
  __shared__ double s_total;
  __shared__ int s_done;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double inv_k = 1.0 / static_cast<double>(K);
  for (int64_t doc = blockIdx.x; doc < n_docs; doc += gridDim.x) {
    const int64_t base = doc_offsets[doc];
    const int64_t n = doc_offsets[doc + 1] - base;
    for (int k = tid; k < K; k += kEvalCtaThreads) th[k] = inv_k;
    __syncthreads();
    for (int sweep = 0; sweep < sweeps && n > 0; ++sweep) {
      for (int k = tid; k < K; k += kEvalCtaThreads) nx[k] = alpha;
      for (int64_t i0 = 0; i0 < n; i0 += kEvalCtaThreads) {
        const int n_here = static_cast<int>(min(static_cast<int64_t>(kEvalCtaThreads), n - i0));
        if (tid < n_here) {
          const int64_t i = base + i0 + tid;
          const int32_t fc = __ldg(fold_counts + i);
          const int32_t w = __ldg(word_ids + i);
          double scale = 0.0;
          if (fc != 0) {  // a zero-count cell adds exactly +0 (eval.cpp:43-47)
            const double mu = seq_dot(th, phi_wk + static_cast<int64_t>(w) * K, K);
            if (mu > 0.0) scale = __ddiv_rn(static_cast<double>(fc), mu);
          }
          cs[tid] = scale;
          cw[tid] = w;
        }
        __syncthreads();
        for (int k = tid; k < K; k += kEvalCtaThreads) {
          double acc = nx[k];
          const double tk = th[k];
#pragma unroll 4
          for (int c = 0; c < n_here; ++c) {
            const double sc = cs[c];
            if (sc != 0.0)
              acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(sc, tk),
                                             __ldg(phi_wk + static_cast<int64_t>(cw[c]) * K + k)));
          }
          nx[k] = acc;
        }
        __syncthreads();
      }
      if (tid == 0) {
        double total = 0.0;
        for (int k = 0; k < K; ++k) total = __dadd_rn(total, nx[k]);
        s_total = total;
      }
      __syncthreads();
      const double total = s_total;
      double delta = 0.0;
      for (int k = tid; k < K; k += kEvalCtaThreads) {
        const double v = __ddiv_rn(nx[k], total);
        delta = fmax(delta, fabs(__dadd_rn(v, -th[k])));
        th[k] = v;
      }
      delta = warp_max(delta);
      if (lane == 0) s_red[wid] = delta;
      __syncthreads();
      if (tid == 0) {
        double d = s_red[0];
        for (int w = 1; w < kEvalCtaThreads / 32; ++w) d = fmax(d, s_red[w]);
        s_done = d < 1e-12;
      }
      __syncthreads();
      if (s_done) break;
    }
    // score the held-back half (eval.cpp:125-145), log p summed in cell order
    double logp = 0.0;
    int64_t scored = 0;
    for (int64_t i0 = 0; i0 < n; i0 += kEvalCtaThreads) {
      const int n_here = static_cast<int>(min(static_cast<int64_t>(kEvalCtaThreads), n - i0));
      if (tid < n_here) {
        const int64_t i = base + i0 + tid;
        const int32_t sc = __ldg(score_counts + i);
        double term = 0.0;
        if (sc != 0) {
          const double pr = seq_dot(th, phi_wk + static_cast<int64_t>(__ldg(word_ids + i)) * K, K);
          if (!(pr > 0.0)) atomicOr(err, kErrNumerical);
          term = __dmul_rn(static_cast<double>(sc), log(pr));
        }
        cs[tid] = term;
        s_cnt[tid] = sc;
      }
      __syncthreads();
      if (tid == 0)
        for (int c = 0; c < n_here; ++c)
          if (s_cnt[c] != 0) {
            logp = __dadd_rn(logp, cs[c]);
            scored += s_cnt[c];
          }
      __syncthreads();
    }
    if (tid == 0) {
      doc_logp[doc] = logp;
      doc_scored[doc] = scored;
    }
    if (theta_out)
      for (int k = tid; k < K; k += kEvalCtaThreads) theta_out[doc * K + k] = th[k];
    __syncthreads();
  }
}

// k_eval_stage: k_eval_cta with a document's first R fold rows staged in
// shared memory once per document, so the 2 x sweeps row reads of those cells
// come from shared memory instead of L2 (the fold-in is L2-bound: 845 GB at
// NYTimes shape).  Fold cells (fold count > 0; a zero-count cell adds exactly
// +0, eval.cpp:43-47) are compacted per window of <= kEvalFoldMax in cell
// order; arithmetic and order are k_eval_cta's (eval.cpp:19-64):
//   phase 1, thread = fold cell: sequential-k mu, scale = c / mu (or skip);
//   phase 2, thread = topic: next[k] += (scale theta[k]) phi[w][k] in fold order;
//   phase 3: sequential total (one thread), theta = next / total, max |delta|.
// Staged rows use an odd stride (K | 1 doubles): the thread-per-cell dots hit
// distinct banks.
constexpr int kEvalFoldMax = 1024;

__device__ __forceinline__ double seq_dot_stride1(const double* __restrict__ th,
                                                  const double* row, int K) {
  double dot = 0.0;
#pragma unroll 8
  for (int k = 0; k < K; ++k) dot = __dadd_rn(dot, __dmul_rn(th[k], row[k]));
  return dot;
}

__global__ void __launch_bounds__(kEvalCtaThreads) k_eval_stage(
    const int64_t* __restrict__ doc_offsets, const int32_t* __restrict__ word_ids,
    const int32_t* __restrict__ fold_counts, const int32_t* __restrict__ score_counts,
    int64_t n_docs, const double* __restrict__ phi_wk, int K, double alpha, int sweeps,
    int R, double* __restrict__ doc_logp, int64_t* __restrict__ doc_scored,
    double* __restrict__ theta_out, int* __restrict__ err) {
  extern __shared__ double smem[];
  const int KP = K | 1;
  // th / nx padded to an even length: the uniform th[k] loads are paired
  // into 16-byte LDS, which for odd K would touch nx[0] (harmless, but a
  // racecheck hazard against nx's writes)
  const int KE = (K + 1) & ~1;
  double* th = smem;                     // K (+ pad)
  double* nx = th + KE;                  // K (+ pad)
  double* fs = nx + KE;                  // [kEvalFoldMax] scale per fold cell
  int32_t* fw = reinterpret_cast<int32_t*>(fs + kEvalFoldMax);  // word per fold cell
  int32_t* fc = fw + kEvalFoldMax;                              // fold count per fold cell
  double* rows = reinterpret_cast<double*>(fc + kEvalFoldMax);   // R x KP staged rows
  __shared__ double s_red[kEvalCtaThreads / 32];
  __shared__ int s_wc[kEvalCtaThreads / 32];
  __shared__ int64_t s_cnt[kEvalCtaThreads];
  __shared__ double s_total;
  __shared__ int s_done;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double inv_k = 1.0 / static_cast<double>(K);

  // documents are handed out dynamically (their fold-in lengths differ:
  // 1 to 50 sweeps, tens to thousands of cells): counter at doc_scored[n_docs]
  __shared__ int64_t s_doc;
  unsigned long long* next_doc = reinterpret_cast<unsigned long long*>(doc_scored + n_docs);
  for (;;) {
    if (threadIdx.x == 0) s_doc = static_cast<int64_t>(atomicAdd(next_doc, 1ull));
    __syncthreads();
    const int64_t doc = s_doc;
    __syncthreads();
    if (doc >= n_docs) break;
    const int64_t base = doc_offsets[doc];
    const int64_t n = doc_offsets[doc + 1] - base;
    // compact the fold cells of cells [c_begin, ...) into fw/fc, whole chunks
    // of 256 cells while they fit; returns the first cell not taken
    auto build = [&](int64_t c_begin, int& nf) -> int64_t {
      nf = 0;
      int64_t c0 = c_begin;
      while (c0 < n && nf + kEvalCtaThreads <= kEvalFoldMax) {
        const int64_t c = c0 + tid;
        const int32_t f = c < n ? __ldg(fold_counts + base + c) : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f > 0);
        if (lane == 0) s_wc[wid] = __popc(bal);
        __syncthreads();
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kEvalCtaThreads / 32; ++w) {
          before += w < wid ? s_wc[w] : 0;
          total += s_wc[w];
        }
        if (f > 0) {
          const int pos = nf + before + __popc(bal & ((1u << lane) - 1u));
          fw[pos] = __ldg(word_ids + base + c);
          fc[pos] = f;
        }
        nf += total;
        c0 += kEvalCtaThreads;
        __syncthreads();
      }
      return c0;
    };
    int nf0 = 0;
    const int64_t end0 = build(0, nf0);
    const bool multi = end0 < n;
    const int Reff = min(nf0, R);
    for (int i = tid; i < Reff * K; i += kEvalCtaThreads) {
      const int f = i / K, k = i - f * K;
      rows[f * KP + k] = __ldg(phi_wk + static_cast<int64_t>(fw[f]) * K + k);
    }
    for (int k = tid; k < K; k += kEvalCtaThreads) th[k] = inv_k;
    __syncthreads();
    for (int sweep = 0; sweep < sweeps && n > 0; ++sweep) {
      for (int k = tid; k < K; k += kEvalCtaThreads) nx[k] = alpha;
      int64_t cw0 = 0;
      bool first = true;
      while (cw0 < n) {
        int nf = nf0;
        int64_t cnext = end0;
        if (multi) cnext = build(cw0, nf);  // lists of later windows overwrite window 0's
        const int rs = first ? Reff : 0;     // staged rows belong to window 0
        for (int f0 = 0; f0 < nf; f0 += kEvalCtaThreads) {
          const int f = f0 + tid;
          if (f < nf) {
            const double mu = f < rs ? seq_dot_stride1(th, rows + f * KP, K)
                                     : seq_dot_g(th, phi_wk + static_cast<int64_t>(fw[f]) * K, K);
            fs[f] = mu > 0.0 ? __ddiv_rn(static_cast<double>(fc[f]), mu) : 0.0;
          }
        }
        __syncthreads();
        for (int k = tid; k < K; k += kEvalCtaThreads) {
          double acc = nx[k];
          const double tk = th[k];
          // branch-free (scale 0 adds +0 exactly), loads batch across iterations
#pragma unroll 8
          for (int f = 0; f < rs; ++f)
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(fs[f], tk), rows[f * KP + k]));
#pragma unroll 16
          for (int f = rs; f < nf; ++f)
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(fs[f], tk),
                                           __ldg(phi_wk + static_cast<int64_t>(fw[f]) * K + k)));
          nx[k] = acc;
        }
        __syncthreads();
        cw0 = cnext;
        first = false;
      }
      if (tid == 0) {
        double total = 0.0;
        for (int k = 0; k < K; ++k) total = __dadd_rn(total, nx[k]);
        s_total = total;
      }
      __syncthreads();
      const double total = s_total;
      double delta = 0.0;
      for (int k = tid; k < K; k += kEvalCtaThreads) {
        const double v = __ddiv_rn(nx[k], total);
        delta = fmax(delta, fabs(__dadd_rn(v, -th[k])));
        th[k] = v;
      }
      delta = warp_max(delta);
      if (lane == 0) s_red[wid] = delta;
      __syncthreads();
      if (tid == 0) {
        double d = s_red[0];
        for (int w = 1; w < kEvalCtaThreads / 32; ++w) d = fmax(d, s_red[w]);
        s_done = d < 1e-12;
      }
      __syncthreads();
      if (s_done) break;
    }
    // score the held-back half (eval.cpp:125-145), log p summed in cell order
    double logp = 0.0;
    int64_t scored = 0;
    for (int64_t i0 = 0; i0 < n; i0 += kEvalCtaThreads) {
      const int n_here = static_cast<int>(min(static_cast<int64_t>(kEvalCtaThreads), n - i0));
      if (tid < n_here) {
        const int64_t i = base + i0 + tid;
        const int32_t sc = __ldg(score_counts + i);
        double term = 0.0;
        if (sc != 0) {
          const double pr = seq_dot_g(th, phi_wk + static_cast<int64_t>(__ldg(word_ids + i)) * K, K);
          if (!(pr > 0.0)) atomicOr(err, kErrNumerical);
          term = __dmul_rn(static_cast<double>(sc), log(pr));
        }
        fs[tid] = term;
        s_cnt[tid] = sc;
      }
      __syncthreads();
      if (tid == 0)
        for (int c = 0; c < n_here; ++c)
          if (s_cnt[c] != 0) {
            logp = __dadd_rn(logp, fs[c]);
            scored += s_cnt[c];
          }
      __syncthreads();
    }
    if (tid == 0) {
      doc_logp[doc] = logp;
      doc_scored[doc] = scored;
    }
    if (theta_out)
      for (int k = tid; k < K; k += kEvalCtaThreads) theta_out[doc * K + k] = th[k];
    __syncthreads();
  }
}

// eval.cpp:148-158: the document-order reduction.  The block stages 1024
// documents at a time in shared memory (coalesced); one thread then adds
// them in document order at the f64 add latency instead of a global-load
// latency per document.
constexpr int kOrderedBlock = 1024;

__global__ void __launch_bounds__(kOrderedBlock) k_ordered_ll(
    const double* __restrict__ doc_logp, const int64_t* __restrict__ doc_scored, int64_t n_docs,
    double* __restrict__ ll_out, int* __restrict__ err) {
  __shared__ double s_lp[kOrderedBlock];
  __shared__ int64_t s_sc[kOrderedBlock];
  double total = 0.0;
  int64_t scored = 0;
  for (int64_t d0 = 0; d0 < n_docs; d0 += kOrderedBlock) {
    const int n = static_cast<int>(min(static_cast<int64_t>(kOrderedBlock), n_docs - d0));
    if (threadIdx.x < n) {
      s_lp[threadIdx.x] = doc_logp[d0 + threadIdx.x];
      s_sc[threadIdx.x] = doc_scored[d0 + threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll 8
      for (int i = 0; i < n; ++i) {
        total = __dadd_rn(total, s_lp[i]);
        scored += s_sc[i];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  if (scored == 0) {
    atomicOr(err, kErrNumerical);
    *ll_out = 0.0;
    return;
  }
  *ll_out = __ddiv_rn(total, static_cast<double>(scored));
}

// ------------------------------------------------------ fast fold-in (k_eval_fold)
// perword_loglik / fold_in_theta (eval.cpp:19-159) at SURVEY 8(d)'s tolerance
// (1e-12 relative on ll) instead of the reference's summation order: the
// exact kernels above are latency-bound on sequential f64 chains (a K-term
// chain per fold cell and sweep) and re-read every fold row from L2 twice per
// sweep.  Here one CTA owns a document at a time (K <= 256: two CTAs of 4
// warps per SM, so one document's barriers and staging overlap the other's
// cells):
//   * lane l owns topics k = 64 j + 2 l + {0, 1} (j < NJ), theta in registers;
//   * a warp takes groups of G consecutive fold cells (G x 2 NJ = 32 row
//     values per lane); per group: the lane's partial dots (FMA), one
//     transposed butterfly that leaves cell c's mu on lanes c << SH ..
//     (1.5 f64 shuffles per cell at G = 4, not 5), s = count / mu once per
//     cell (MUFU reciprocal + Newton), then g_k += s_c phi[w_c][k] (FMA) from
//     the same registers -- one read of each row per sweep;
//   * rows stay on chip across the <= 50 sweeps: the first group of every
//     warp in registers (RES), the next R rows in shared memory (staged once
//     per document), the rest re-read from L2;
//   * next_k = alpha + theta_k g_k (FMA).  The total sum_k next_k =
//     K alpha + sum_k theta_k g_k comes from per-warp partials written with
//     the warps' g, so after ONE barrier the topic owners form
//     theta = next / total and the stopping test (eval.cpp:51-61: same 1e-12
//     rule, same 1 / K start, no sweeps for a document without cells), and a
//     second barrier (__syncthreads_or) ORs the test.
// Scoring (eval.cpp:125-145) runs the same group dots over the score cells;
// the document's log p terms are added in cell order with the reference's
// rounding (c * log p, then add), the doc-order reduction is k_ordered_ll.
// Zero-count cells are absent from the lists: the reference adds exactly +0
// for them.  Measured at NYTimes shape (30K test docs, 127 fold cells on
// average, all 50 sweeps): 45 ms against 117 ms for the exact kernel; per
// cell the loop costs ~32-46 SM cycles (16 of them the 2 KB shared-memory
// row read, the rest shuffles / reciprocal latency), see profiles/r2_eval.md.
// v[0..2H) -> after log2(2H) halving stages and the remaining full stages,
// v[0] on every lane = sum over the lane's group of the partials of cell
// (lane >> SH); offsets O, O/2, ..., 1
template <int H, int O>
__device__ __forceinline__ void fold_tree(double* v, int lane) {
  if constexpr (H >= 1) {
    const bool up = (lane & O) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double send = up ? v[i] : v[i + H];
      const double keep = up ? v[i + H] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
    if constexpr (O > 1) fold_tree<H / 2, O / 2>(v, lane);
  } else {
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], O);
    if constexpr (O > 1) fold_tree<0, O / 2>(v, lane);
  }
}

__device__ __forceinline__ double2 load_pair_g(const double* __restrict__ row, int k, int K,
                                               bool keven) {
  if (keven && k + 1 < K) return __ldg(reinterpret_cast<const double2*>(row + k));
  double2 v;
  v.x = k < K ? __ldg(row + k) : 0.0;
  v.y = k + 1 < K ? __ldg(row + k + 1) : 0.0;
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 1 / x for x > 0: MUFU reciprocal + two Newton steps (relative error ~1 ulp;
// IEEE division below the f64 normal range, where the approximation flushes)
__device__ __forceinline__ double fold_rcp(double x) {
  if (x < 1e-300) return __ddiv_rn(1.0, x);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}

// Kernel shape: NJ topic pairs per lane (K <= 64 NJ), NW warps; NRES
// register-resident groups of G fold cells per warp (their rows stay in
// registers across sweeps); the other cells in streaming groups of GS (rows
// from shared memory or L2), one transposed butterfly per group.
template <int NJ_, int G_, int NW_, int NRES_, int GS_, int CPS_ = 1>
struct FoldCfg {
  static constexpr int NJ = NJ_, G = G_, NW = NW_, NRES = NRES_, GS = GS_;
  static constexpr int CPS = CPS_;  // CTAs (documents) per SM
  static constexpr int NT = 32 * NW;
  static constexpr int KP = 64 * NJ;         // padded topics (row stride in shared memory)
  static constexpr int S0 = NRES * G * NW;   // first cell past the register-resident ones
  static constexpr int GW = GS * NW;         // streaming cells per round of groups
  static constexpr int TPT = (KP + NT - 1) / NT;  // topics per thread in the epilogue
};

template <int G>
struct GroupShape {
  static constexpr int LG = G == 1 ? 0 : G == 2 ? 1 : G == 4 ? 2 : G == 8 ? 3 : 4;
  static constexpr int SH = 5 - LG;  // lane >> SH = the lane's cell in a group
};

// fold-list entries staged per document (longer lists are read from global)
constexpr int kFoldList = 768;

template <int NJ, int G>
__device__ __forceinline__ void fold_dots(const double2 (&th)[NJ], const double2 (&r)[G][NJ],
                                          double (&v)[G]) {
#pragma unroll
  for (int c = 0; c < G; ++c) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      a = __fma_rn(th[j].x, r[c][j].x, a);
      b = __fma_rn(th[j].y, r[c][j].y, b);
    }
    v[c] = a + b;
  }
}

// one group of G cells (rows r; cnt = count of the lane's cell, 0 past the
// list) into the warp's g sums: partial dots, one transposed butterfly (the
// lanes of cell c end with its mu), s = c / mu (eval.cpp:38-44; mu <= 0 or
// NaN: 0), g_k += s_c phi[w_c][k] (eval.cpp:45-49)
template <int NJ, int G>
__device__ __forceinline__ void fold_group(const double2 (&th)[NJ], const double2 (&r)[G][NJ],
                                           double2 (&acc)[NJ], int cnt, int lane) {
  double v[G];
  fold_dots<NJ, G>(th, r, v);
  fold_tree<G / 2, 16>(v, lane);
  const double s = v[0] > 0.0 ? static_cast<double>(cnt) * fold_rcp(v[0]) : 0.0;
#pragma unroll
  for (int c = 0; c < G; ++c) {
    const double sc = __shfl_sync(0xffffffffu, s, c << GroupShape<G>::SH);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      acc[j].x = __fma_rn(sc, r[c][j].x, acc[j].x);
      acc[j].y = __fma_rn(sc, r[c][j].y, acc[j].y);
    }
  }
}

template <int NJ>
__device__ __forceinline__ void fold_row_g(double2 (&r)[NJ], const double* __restrict__ phi_wk,
                                           int w, int K, bool keven, int lane) {
  const double* row = phi_wk + static_cast<int64_t>(w) * K;
#pragma unroll
  for (int j = 0; j < NJ; ++j) r[j] = load_pair_g(row, 64 * j + 2 * lane, K, keven);
}

template <int NJ>
__device__ __forceinline__ void fold_row_zero(double2 (&r)[NJ]) {
#pragma unroll
  for (int j = 0; j < NJ; ++j) r[j] = make_double2(0.0, 0.0);
}

#ifdef SAMELDA_FOLD_PROF
__device__ unsigned long long g_fold_prof[8];  // cycles of thread 0: stage, cells, bar1, epi, bar2, -, score
#define FOLD_T(i) if (tid == 0) { const long long _n = clock64(); atomicAdd(&g_fold_prof[i], _n - _t); _t = _n; }
#else
#define FOLD_T(i)
#endif

template <class C>
__global__ void __launch_bounds__(C::NT, C::CPS) k_eval_fold(
    const int64_t* __restrict__ doc_offsets, EvalLists L, int64_t n_docs,
    const double* __restrict__ phi_wk, int K, double alpha, int sweeps, int R,
    double* __restrict__ doc_logp, int64_t* __restrict__ doc_scored,
    double* __restrict__ theta_out, int* __restrict__ err) {
  constexpr int NJ = C::NJ, G = C::G, GS = C::GS, NW = C::NW, NT = C::NT, KP = C::KP;
  constexpr int GW = C::GW, S0 = C::S0, TPT = C::TPT, NRES = C::NRES;
  constexpr int SH = GroupShape<G>::SH, SHS = GroupShape<GS>::SH;
  extern __shared__ __align__(16) double smem[];
  double* red = smem;                                // [NW][KP] per-warp g
  double* ths = red + NW * KP;                       // [KP] theta (zero past K)
  int2* lst_s = reinterpret_cast<int2*>(ths + KP);   // [kFoldList] (word, count)
  double* rows = ths + KP + kFoldList;               // [R][KP] staged fold rows
  __shared__ double s_part[NW], s_term[G * NW];
  __shared__ long long s_cnt[NW];
  __shared__ int64_t s_doc;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool keven = (K & 1) == 0;
  const double inv_k = 1.0 / static_cast<double>(K);
  const double k_alpha = static_cast<double>(K) * alpha;
  unsigned long long* next_doc = reinterpret_cast<unsigned long long*>(doc_scored + n_docs);

  for (;;) {
    __syncthreads();  // the previous document's shared-memory readers are done
    if (tid == 0) s_doc = static_cast<int64_t>(atomicAdd(next_doc, 1ull));
    __syncthreads();
    const int64_t doc = s_doc;
    if (doc >= n_docs) break;
#ifdef SAMELDA_FOLD_PROF
    long long _t = clock64();
#endif
    const int64_t base = doc_offsets[doc];
    const int64_t ncell = doc_offsets[doc + 1] - base;
    const int F = L.n_fold[doc];
    const int2* __restrict__ gl = L.fold + base;
    const int2* lst = F <= kFoldList ? lst_s : gl;  // generic: shared or global

    // stage: list, shared-memory rows [S0, s_end), register-resident group, theta
    if (F <= kFoldList)
      for (int i = tid; i < F; i += NT) lst_s[i] = __ldg(gl + i);
    const int Rn = max(0, min(R, F - S0));
    const int s_end = S0 + Rn;
    for (int i = tid; i < Rn * (KP / 2); i += NT) {
      const int f = i / (KP / 2), k = 2 * (i - f * (KP / 2));
      *reinterpret_cast<double2*>(rows + f * KP + k) =
          load_pair_g(phi_wk + static_cast<int64_t>(__ldg(&gl[S0 + f].x)) * K, k, K, keven);
    }
    double2 res[NRES > 0 ? NRES : 1][G][NJ];
    int res_cnt[NRES > 0 ? NRES : 1];
#pragma unroll
    for (int q = 0; q < NRES; ++q) {  // group q of warp w: cells q G NW + G w + [0, G)
#pragma unroll
      for (int c = 0; c < G; ++c) {
        const int f = q * G * NW + G * wid + c;
        if (f < F) fold_row_g<NJ>(res[q][c], phi_wk, __ldg(&gl[f].x), K, keven, lane);
        else fold_row_zero<NJ>(res[q][c]);
      }
      const int my = q * G * NW + G * wid + (lane >> SH);
      res_cnt[q] = my < F ? __ldg(&gl[my].y) : 0;
    }
    double2 th[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = 64 * j + 2 * lane;
      th[j].x = k < K ? inv_k : 0.0;
      th[j].y = k + 1 < K ? inv_k : 0.0;
    }
    for (int t = tid; t < KP; t += NT) ths[t] = t < K ? inv_k : 0.0;
    __syncthreads();
    FOLD_T(0)

    const int nsw = ncell > 0 ? sweeps : 0;
    for (int sweep = 0; sweep < nsw; ++sweep) {
      double2 acc[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[j] = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < NRES; ++q)
        if (q * G * NW + G * wid < F) fold_group<NJ, G>(th, res[q], acc, res_cnt[q], lane);
      for (int f0 = S0 + GS * wid; f0 < F; f0 += GW) {
        const int my = f0 + (lane >> SHS);
        const int cnt = my < F ? lst[my].y : 0;
        double2 r[GS][NJ];
        if (f0 + GS <= s_end) {  // whole group staged
#pragma unroll
          for (int c = 0; c < GS; ++c)
#pragma unroll
            for (int j = 0; j < NJ; ++j)
              r[c][j] = *reinterpret_cast<const double2*>(rows + (f0 - S0 + c) * KP + 64 * j + 2 * lane);
        } else if (f0 >= s_end && f0 + GS <= F && K == KP) {
          // whole group from L2, full-width rows: unconditional 16-byte loads
          // (the generic path below costs ~160 extra instructions per group)
#pragma unroll
          for (int c = 0; c < GS; ++c) {
            const double2* row = reinterpret_cast<const double2*>(phi_wk + static_cast<int64_t>(lst[f0 + c].x) * KP);
#pragma unroll
            for (int j = 0; j < NJ; ++j) r[c][j] = __ldg(row + 32 * j + lane);
          }
        } else {  // the staged / L2 boundary and the past-the-end edge
#pragma unroll
          for (int c = 0; c < GS; ++c) {
            const int f = f0 + c;
            if (f < s_end) {
#pragma unroll
              for (int j = 0; j < NJ; ++j)
                r[c][j] = *reinterpret_cast<const double2*>(rows + (f - S0) * KP + 64 * j + 2 * lane);
            } else if (K == KP) {
              // past the end: the last cell's row with count 0 (adds exactly 0)
              const double2* row = reinterpret_cast<const double2*>(
                  phi_wk + static_cast<int64_t>(lst[min(f, F - 1)].x) * KP);
#pragma unroll
              for (int j = 0; j < NJ; ++j) r[c][j] = __ldg(row + 32 * j + lane);
            } else if (f < F) {
              fold_row_g<NJ>(r[c], phi_wk, lst[f].x, K, keven, lane);
            } else {
              fold_row_zero<NJ>(r[c]);
            }
          }
        }
        fold_group<NJ, GS>(th, r, acc, cnt, lane);
      }
      // ---- epilogue (eval.cpp:51-61).  total = K alpha + sum_k theta_k g_k
      // from per-warp partials, so theta = next / total and the stopping test
      // are formed by the topic owners right after the first barrier; the
      // second barrier ORs the test
      double part = 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        part = __fma_rn(th[j].x, acc[j].x, part);
        part = __fma_rn(th[j].y, acc[j].y, part);
        *reinterpret_cast<double2*>(red + wid * KP + 64 * j + 2 * lane) = acc[j];
      }
      part = warp_sum_d(part);
      if (lane == 0) s_part[wid] = part;
      FOLD_T(1)
      __syncthreads();
      FOLD_T(2)
      const double rt = fold_rcp(k_alpha + warp_sum_d(lane < NW ? s_part[lane] : 0.0));
      bool big = false;
#pragma unroll
      for (int q = 0; q < TPT; ++q) {
        const int t = tid + q * NT;
        if (t < K) {
          double g = red[t];
#pragma unroll
          for (int w = 1; w < NW; ++w) g += red[w * KP + t];
          const double old = ths[t];
          const double val = __fma_rn(old, g, alpha) * rt;
          // stop when max_k |delta_k| < 1e-12 (a NaN delta never raises the
          // reference's std::max)
          big |= fabs(val - old) >= 1e-12;
          ths[t] = val;
        }
      }
      FOLD_T(3)
      const bool more = __syncthreads_or(big);
      FOLD_T(4)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        th[j] = *reinterpret_cast<const double2*>(ths + 64 * j + 2 * lane);
      if (!more) break;
    }

    // scoring (eval.cpp:125-145): the document's log p is summed in cell
    // order with the reference's rounding (term = c * log p, then add), one
    // round of G NW cells at a time
    const int Sn = L.n_score[doc];
    const int2* sl = L.score + base;
    constexpr int GWS = G * NW;
    double lp = 0.0;
    long long scored = 0;
    for (int r0 = 0; r0 < Sn; r0 += GWS) {
      const int f0 = r0 + G * wid;
      double2 r[G][NJ];
#pragma unroll
      for (int c = 0; c < G; ++c) {
        if (f0 + c < Sn) fold_row_g<NJ>(r[c], phi_wk, __ldg(&sl[f0 + c].x), K, keven, lane);
        else fold_row_zero<NJ>(r[c]);
      }
      double v[G];
      fold_dots<NJ, G>(th, r, v);
      fold_tree<G / 2, 16>(v, lane);
      const int my = f0 + (lane >> SH);
      if ((lane & ((1 << SH) - 1)) == 0) {
        double term = 0.0;
        if (my < Sn) {
          const int32_t c = __ldg(&sl[my].y);
          if (!(v[0] > 0.0)) atomicOr(err, kErrNumerical);
          term = __dmul_rn(static_cast<double>(c), log(v[0]));
          scored += c;
        }
        s_term[G * wid + (lane >> SH)] = term;
      }
      __syncthreads();
      if (tid == 0) {
        const int n = min(GWS, Sn - r0);
        for (int i = 0; i < n; ++i) lp = __dadd_rn(lp, s_term[i]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) scored += __shfl_xor_sync(0xffffffffu, scored, o);
    if (lane == 0) s_cnt[wid] = scored;
    __syncthreads();
    FOLD_T(6)
    if (tid == 0) {
      long long n = s_cnt[0];
      for (int w = 1; w < NW; ++w) n += s_cnt[w];
      doc_logp[doc] = lp;
      doc_scored[doc] = n;
    }
    if (theta_out)
      for (int t = tid; t < K; t += NT) theta_out[doc * K + t] = ths[t];
  }
}

template <class C>
int launch_fold(const int64_t* doc_offsets, const EvalLists& L, int64_t n_docs,
                const double* phi_wk, int K, double alpha, int sweeps, double* doc_logp,
                int64_t* doc_scored, double* theta_out, int* err, cudaStream_t st) {
  int dev = 0, sms = 148, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int per_sm = 0;
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, k_eval_fold<C>);
  const size_t fixed = (static_cast<size_t>(C::NW + 1) * C::KP + kFoldList) * sizeof(double);
  // per CTA: the SM's shared memory split CPS ways, less each CTA's static
  // part and the 1 KB the runtime reserves per block
  const size_t cap = C::CPS == 1 ? static_cast<size_t>(optin)
                                 : static_cast<size_t>(per_sm) / C::CPS - 1024;
  const size_t budget = std::min(static_cast<size_t>(optin), cap) - fa.sharedSizeBytes;
  const size_t row = static_cast<size_t>(C::KP) * sizeof(double);
  const int R = budget > fixed ? static_cast<int>((budget - fixed) / row) : 0;
  const size_t bytes = fixed + static_cast<size_t>(R) * row;
  static std::atomic<unsigned long long> configured{0};
  smem_opt_in(k_eval_fold<C>, static_cast<int>(bytes), configured);
  const int64_t blocks = min(n_docs, static_cast<int64_t>(sms) * C::CPS);
#ifdef SAMELDA_FOLD_PROF
  unsigned long long z[8] = {};
  cudaMemcpyToSymbolAsync(g_fold_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
#endif
  // the dynamic document counter lives one past the per-document results
  cudaMemsetAsync(doc_scored + n_docs, 0, sizeof(int64_t), st);
  k_eval_fold<C><<<static_cast<unsigned>(blocks), C::NT, bytes, st>>>(
      doc_offsets, L, n_docs, phi_wk, K, alpha, sweeps, R, doc_logp, doc_scored, theta_out, err);
#ifdef SAMELDA_FOLD_PROF
  cudaMemcpyFromSymbolAsync(z, g_fold_prof, sizeof(z), 0, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  fprintf(stderr, "fold prof (cycles summed over CTAs, thread 0): stage %.3g cells %.3g bar1 %.3g epi %.3g bar2 %.3g score %.3g  R=%d\n",
          (double)z[0], (double)z[1], (double)z[2], (double)z[3], (double)z[4], (double)z[6], R);
#endif
  return 1;
}

constexpr size_t kEvalSmemMax = 200 * 1024;

}  // namespace

// ------------------------------------------------------------- launchers

int launch_eval_split(const int64_t* doc_offsets, const int32_t* word_ids, const int32_t* counts,
                      const int64_t* token_offsets, int64_t n_docs, uint64_t seed,
                      int32_t* slots, int32_t* fold_counts, int32_t* score_counts,
                      const EvalLists& lists, cudaStream_t st) {
  if (n_docs == 0) return 0;
  k_eval_split<<<grid_for(n_docs, 128), 128, 0, st>>>(doc_offsets, word_ids, counts,
                                                      token_offsets, n_docs, seed, slots,
                                                      fold_counts, score_counts, lists);
  return 1;
}

int64_t eval_scratch_doubles(int K) {
  // theta / next (2K doubles per warp) live in shared memory up to
  // kEvalSmemMax per block; beyond that, a global scratch for a capped grid
  const size_t smem = static_cast<size_t>(kEvalWarps) * 2 * K * sizeof(double);
  if (smem <= kEvalSmemMax) return 0;
  return static_cast<int64_t>(148) * 4 * kEvalWarps * 2 * K;
}

int launch_eval_docs(const int64_t* doc_offsets, const int32_t* word_ids,
                     const int32_t* fold_counts, const int32_t* score_counts, int64_t n_docs,
                     const double* phi_wk, int K, double alpha, int sweeps, double* doc_logp,
                     int64_t* doc_scored, double* theta_out, double* scratch,
                     int64_t scratch_doubles, int* err, cudaStream_t st) {
  if (n_docs == 0) return 0;
  const char ev = tuning().eval_variant;  // A/B: 'c' cta, 'w' warp; default staged
  if (K <= 1024 && ev != 'c' && ev != 'w') {
    // staged rows: 2 CTAs per SM share (almost) all of shared memory; the
    // global-row dots (seq_dot_pipe, 128 registers) allow 2 resident CTAs
    // (measured at NYTimes shape: 1 / 2 / 3 CTAs 134 / 117 / 126 ms;
    // SAMELDA_EVAL_CTAS_PER_SM overrides)
    const int cps = tuning().eval_ctas_per_sm > 0 ? tuning().eval_ctas_per_sm : 2;
    const int KP = K | 1;
    const size_t fixed = (2 * static_cast<size_t>((K + 1) & ~1) + kEvalFoldMax) * sizeof(double) +
                         2 * kEvalFoldMax * sizeof(int32_t);
    const size_t budget = (220u * 1024u) / static_cast<size_t>(cps);
    if (budget > fixed + static_cast<size_t>(KP) * sizeof(double)) {
      const int R = static_cast<int>(std::min<size_t>((budget - fixed) / (KP * sizeof(double)), static_cast<size_t>(kEvalFoldMax)));
      const size_t smem_s = fixed + static_cast<size_t>(R) * KP * sizeof(double);
      static std::atomic<unsigned long long> configured_s{0};
      smem_opt_in(k_eval_stage, static_cast<int>(220 * 1024), configured_s);
      const int64_t blocks = min(n_docs, static_cast<int64_t>(148 * cps));
      // the dynamic document counter lives one past the per-document results
      cudaMemsetAsync(doc_scored + n_docs, 0, sizeof(int64_t), st);
      k_eval_stage<<<static_cast<unsigned>(blocks), kEvalCtaThreads, smem_s, st>>>(
          doc_offsets, word_ids, fold_counts, score_counts, n_docs, phi_wk, K, alpha, sweeps, R,
          doc_logp, doc_scored, theta_out, err);
      return 1;
    }
  }
  if (K <= kEvalCtaMaxK && ev != 'w') {
    const size_t smem_c = (2 * static_cast<size_t>((K + 1) & ~1) + kEvalCtaThreads) * sizeof(double) +
                          kEvalCtaThreads * sizeof(int32_t);
    static std::atomic<unsigned long long> configured_c{0};
    // largest smem_c over K <= kEvalCtaMaxK
    smem_opt_in(k_eval_cta,
                static_cast<int>((2 * static_cast<size_t>(kEvalCtaMaxK) + kEvalCtaThreads) * sizeof(double) +
                                 kEvalCtaThreads * sizeof(int32_t)),
                configured_c);
    // ~600 documents in flight: their fold rows stay L2-resident across sweeps
    const int64_t blocks = min(n_docs, static_cast<int64_t>(148 * 4));
    k_eval_cta<<<static_cast<unsigned>(blocks), kEvalCtaThreads, smem_c, st>>>(
        doc_offsets, word_ids, fold_counts, score_counts, n_docs, phi_wk, K, alpha, sweeps,
        doc_logp, doc_scored, theta_out, err);
    return 1;
  }
  const size_t smem = static_cast<size_t>(kEvalWarps) * 2 * K * sizeof(double);
  int64_t blocks = (n_docs + kEvalWarps - 1) / kEvalWarps;
  if (smem <= kEvalSmemMax) {
    static std::atomic<unsigned long long> configured{0};
    smem_opt_in(k_eval_docs, static_cast<int>(kEvalSmemMax), configured);
    k_eval_docs<<<static_cast<unsigned>(blocks), kEvalWarps * 32, smem, st>>>(
        doc_offsets, word_ids, fold_counts, score_counts, n_docs, phi_wk, K, alpha, sweeps,
        doc_logp, doc_scored, theta_out, nullptr, err);
  } else {
    const int64_t per_block = static_cast<int64_t>(kEvalWarps) * 2 * K;
    int64_t cap = scratch_doubles / per_block;
    if (cap < 1) cap = 1;
    if (blocks > cap) blocks = cap;
    k_eval_docs<<<static_cast<unsigned>(blocks), kEvalWarps * 32, 0, st>>>(
        doc_offsets, word_ids, fold_counts, score_counts, n_docs, phi_wk, K, alpha, sweeps,
        doc_logp, doc_scored, theta_out, scratch, err);
  }
  return 1;
}

int launch_eval_fold(const int64_t* doc_offsets, const EvalLists& lists, int64_t n_docs,
                     const double* phi_wk, int K, double alpha, int sweeps, double* doc_logp,
                     int64_t* doc_scored, double* theta_out, int* err, cudaStream_t st) {
  if (n_docs == 0) return 0;
#define SCU_FOLD(...)                                                                        \
  launch_fold<FoldCfg<__VA_ARGS__>>(doc_offsets, lists, n_docs, phi_wk, K, alpha, sweeps,      \
                                    doc_logp, doc_scored, theta_out, err, st)
  // K <= 256 measured at NYTimes shape (30K test docs, 127 fold cells on
  // average), after the lean L2 path (unconditional 16-byte row loads): four
  // documents per SM, CTAs of 4 warps, no register-resident group, streaming
  // groups of 4 -- 29.5 ms; two documents per SM with two resident groups per
  // warp 34.6 (40.6 before the lean path); 3 CTAs / one resident group 31.1;
  // 8-warp CTAs x 2 30.4; 5-6 CTAs per SM spill (34-57)
  if (K <= 64) return SCU_FOLD(1, 16, 8, 1, 16);
  if (K <= 128) return SCU_FOLD(2, 8, 8, 1, 8);
  if (K <= 256) return SCU_FOLD(4, 4, 4, 0, 4, 4);
  if (K <= 512) return SCU_FOLD(8, 2, 8, 0, 2);
  if (K <= 1024) return SCU_FOLD(16, 1, 8, 0, 1);
#undef SCU_FOLD
  return -1;  // K > 1024: the exact kernels
}

int launch_ordered_ll(const double* doc_logp, const int64_t* doc_scored, int64_t n_docs,
                      double* ll_out, int* err, cudaStream_t st) {
  k_ordered_ll<<<1, kOrderedBlock, 0, st>>>(doc_logp, doc_scored, n_docs, ll_out, err);
  return 1;
}

}  // namespace scu
