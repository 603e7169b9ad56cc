// kernels_eval.cu -- sm_100a held-out evaluation (perword_loglik /
// fold_in_theta, eval.cpp:19-159): token split, fold-in + scoring kernels,
// document-order reduction.
#include "kernels_common.cuh"

namespace scu {

namespace {

// --------------------------------------------------------------------- eval
// eval.cpp:99-121, one thread per test document.
__global__ void k_eval_split(const int64_t* __restrict__ doc_offsets,
                             const int32_t* __restrict__ counts,
                             const int64_t* __restrict__ token_offsets, int64_t n_docs,
                             uint64_t seed, int32_t* __restrict__ slots,
                             int32_t* __restrict__ fold_counts,
                             int32_t* __restrict__ score_counts) {
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

constexpr size_t kEvalSmemMax = 200 * 1024;

}  // namespace

// ------------------------------------------------------------- launchers

int launch_eval_split(const int64_t* doc_offsets, const int32_t* counts,
                      const int64_t* token_offsets, int64_t n_docs, uint64_t seed,
                      int32_t* slots, int32_t* fold_counts, int32_t* score_counts,
                      cudaStream_t st) {
  if (n_docs == 0) return 0;
  k_eval_split<<<grid_for(n_docs, 128), 128, 0, st>>>(doc_offsets, counts, token_offsets,
                                                      n_docs, seed, slots, fold_counts,
                                                      score_counts);
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

int launch_ordered_ll(const double* doc_logp, const int64_t* doc_scored, int64_t n_docs,
                      double* ll_out, int* err, cudaStream_t st) {
  k_ordered_ll<<<1, kOrderedBlock, 0, st>>>(doc_logp, doc_scored, n_docs, ll_out, err);
  return 1;
}

}  // namespace scu
