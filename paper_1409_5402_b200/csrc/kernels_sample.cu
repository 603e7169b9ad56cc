// kernels_sample.cu -- sm_100a sampling kernels: theta gather, SDDMM, the
// exact f64 sampler, the fast-exact period sampler (k_sample_v2) with its
// deferred exact passes, the K > 256 mu pre-pass and the expected-count
// kernel.  Each kernel cites the reference loop it replaces.
#include <cmath>

#include "kernels_common.cuh"
#include "poisson.cuh"

namespace scu {

namespace {

// ------------------------------------------------------------------- gather

__global__ void k_gather_theta(const double* __restrict__ theta,
                               const int32_t* __restrict__ batch_docs, int64_t B, int K,
                               double* __restrict__ out, float* __restrict__ out32) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= B * K) return;
  const int64_t b = i / K;
  const int k = static_cast<int>(i - b * K);
  const double v = theta[static_cast<int64_t>(batch_docs[b]) * K + k];
  out[i] = v;
  if (out32) out32[i] = __double2float_rn(v);
}

// -------------------------------------------------------------------- sddmm
// One thread per batch nonzero; the dot product runs in the reference's
// sequential k order (sampler.cpp:111-119), product then add, no FMA.
__global__ void __launch_bounds__(256) k_sddmm(BatchView bv,
                                               const double* __restrict__ theta_batch,
                                               const double* __restrict__ phi_wk, int K,
                                               double* __restrict__ mu) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= bv.nnz) return;
  const int64_t b = find_row(bv.batch_prefix, bv.B, p);
  const int32_t d = bv.batch_docs[b];
  const int64_t g = bv.doc_offsets[d] + (p - bv.batch_prefix[b]);
  const int32_t w = bv.word_ids[g];
  const double* th = theta_batch + b * K;
  const double* ph = phi_wk + static_cast<int64_t>(w) * K;
  double dot = 0.0;
  if ((K & 1) == 0) {
    const double2* th2 = reinterpret_cast<const double2*>(th);
    const double2* ph2 = reinterpret_cast<const double2*>(ph);
    for (int k = 0; k < (K >> 1); ++k) {
      const double2 a = __ldg(th2 + k);
      const double2 c = __ldg(ph2 + k);
      dot = __dadd_rn(dot, __dmul_rn(a.x, c.x));
      dot = __dadd_rn(dot, __dmul_rn(a.y, c.y));
    }
  } else {
    for (int k = 0; k < K; ++k) dot = __dadd_rn(dot, __dmul_rn(__ldg(th + k), __ldg(ph + k)));
  }
  mu[p] = dot;
}

// The same exact mu with the phi rows staged through shared memory (K a
// multiple of 16): lane = nonzero for the sequential sum, but the rows arrive
// with coalesced 16-byte cp.async copies (four rows' 16 topics per
// instruction) into a per-warp tile, double-buffered over 16-topic chunks,
// instead of 32 lane-divergent row streams per load instruction (0.75 against
// 1.63 ms per NYTimes-shape sweep; 8-byte copies 1.16 ms).  theta rows are read directly (a warp's
// nonzeros mostly share one document).  Used by the converged-model regime,
// where the deferred draws need the exact mu of nearly every nonzero.
constexpr int kSdWarps = 4;
constexpr int kSdChunk = 16;            // topics per staged chunk (two rows per copy instruction)
constexpr int kSdStride = kSdChunk + 2; // doubles per staged row (16-byte aligned rows)

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

__global__ void __launch_bounds__(kSdWarps * 32) k_sddmm_staged(BatchView bv,
                                                                const double* __restrict__ theta_batch,
                                                                const double* __restrict__ phi_wk, int K,
                                                                double* __restrict__ mu) {
  __shared__ __align__(16) double tile[kSdWarps][2][32 * kSdStride];  // 2 buffers x 32 rows x 16 topics
  __shared__ int32_t s_w[kSdWarps][32];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int64_t p0 = (static_cast<int64_t>(blockIdx.x) * kSdWarps + wq) * 32;
  if (p0 >= bv.nnz) return;
  const int64_t p = p0 + lane;
  const bool live = p < bv.nnz;
  const int n_live = static_cast<int>(min(static_cast<int64_t>(32), bv.nnz - p0));
  int64_t b = 0;
  int32_t w = 0;
  if (live) {
    b = find_row(bv.batch_prefix, bv.B, p);
    const int32_t d = bv.batch_docs[b];
    w = bv.word_ids[bv.doc_offsets[d] + (p - bv.batch_prefix[b])];
  }
  s_w[wq][lane] = w;
  __syncwarp();
  // 16-byte copies: lanes 8q .. 8q + 7 copy row i + q's 16 topics
  const int quarter = lane >> 3, col = 2 * (lane & 7);
  auto stage = [&](int kc, int buf) {
    double* t = tile[wq][buf];
    for (int i = quarter; i < n_live; i += 4)
      cp_async16(t + i * kSdStride + col, phi_wk + static_cast<int64_t>(s_w[wq][i]) * K + kc + col);
    cp_async_commit();
  };
  const double* th = theta_batch + b * K;
  double dot = 0.0;
  stage(0, 0);
  for (int kc = 0, buf = 0; kc < K; kc += kSdChunk, buf ^= 1) {
    if (kc + kSdChunk < K) {
      stage(kc + kSdChunk, buf ^ 1);
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    __syncwarp();
    if (live) {
      const double* row = tile[wq][buf] + lane * kSdStride;
#pragma unroll
      for (int k = 0; k < kSdChunk; ++k) dot = __dadd_rn(dot, __dmul_rn(__ldg(th + kc + k), row[k]));
    }
    __syncwarp();  // the buffer is refilled two chunks later
  }
  if (live) mu[p] = dot;
}

// ------------------------------------------------------------------- sample
// Work item = (chunk of `chunk` consecutive batch nonzeros, slice of 32*KPL
// topics); one warp per item, lane owns topics kbase + lane + 32 j.  The warp
// walks its nonzeros in order; every lane draws its topics' Poisson replicas
// from the stream keyed (t, doc, word, tag(poisson_counts, sweep, k))
// (sampler.cpp:152-190).  theta counts accumulate in registers and are
// flushed with one integer atomic per (doc, topic) when the warp leaves a
// doc; phi counts go straight to word-major rows with red.global.add (the 32
// lanes of a warp hit 32 consecutive topics of one word, so each scatter is
// one coalesced 256 B transaction).  Integer adds commute, so the result is
// independent of the work split.
constexpr int kSampleBlock = 256;
constexpr int kSampleWarps = kSampleBlock / 32;

template <int KPL, int MODE>
__global__ void __launch_bounds__(kSampleBlock) k_sample(
    BatchView bv, const double* __restrict__ theta_batch, const double* __restrict__ phi_wk,
    const double* __restrict__ mu, int K, double m_t, uint64_t seed, uint32_t t,
    uint32_t sweep, int64_t chunk, int n_slices, unsigned long long* __restrict__ theta_counts,
    unsigned long long* __restrict__ phi_counts, double* __restrict__ theta_exp,
    double* __restrict__ phi_exp, int* __restrict__ err) {
  // per-warp topic state in shared memory, lane-interleaved (conflict-free):
  // theta_batch row slice and the running theta counts of the current doc
  __shared__ double s_th[kSampleWarps][KPL * kWarp];
  __shared__ unsigned long long s_acc[kSampleWarps][KPL * kWarp];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t item = gw / n_slices;
  const int slice = static_cast<int>(gw - item * n_slices);
  const int64_t p0 = item * chunk;
  if (p0 >= bv.nnz) return;
  const int64_t p1 = min(p0 + chunk, bv.nnz);
  const int kbase = slice * kWarp * KPL;
  const double uniform_weight = 1.0 / static_cast<double>(K);
  double* th = s_th[wib];
  unsigned long long* acc = s_acc[wib];
  double* accf = reinterpret_cast<double*>(s_acc[wib]);

  int64_t cur_b = -1;
  auto flush = [&](int64_t b) {
    if (b < 0) return;
    for (int j = 0; j < KPL; ++j) {
      const int k = kbase + lane + kWarp * j;
      if (k < K) {
        if (MODE == kModeExpected) {
          if (accf[j * kWarp + lane] != 0.0) atomicAdd(theta_exp + b * K + k, accf[j * kWarp + lane]);
        } else {
          if (acc[j * kWarp + lane] != 0ull) atomicAdd(theta_counts + b * K + k, acc[j * kWarp + lane]);
        }
      }
    }
  };

  for (int64_t g0 = p0; g0 < p1; g0 += kWarp) {
    const int64_t p = g0 + lane;
    int64_t b = 0;
    int32_t d = 0, w = 0, c = 0;
    double mu_v = 0.0;
    if (p < p1) {
      b = find_row(bv.batch_prefix, bv.B, p);
      d = __ldg(bv.batch_docs + b);
      const int64_t gi = __ldg(bv.doc_offsets + d) + (p - __ldg(bv.batch_prefix + b));
      w = __ldg(bv.word_ids + gi);
      c = __ldg(bv.counts + gi);
      mu_v = __ldg(mu + p);
    }
    const int n_here = static_cast<int>(min(static_cast<int64_t>(kWarp), p1 - g0));
    for (int i = 0; i < n_here; ++i) {
      const int64_t bi = __shfl_sync(0xffffffffu, b, i);
      const uint32_t di = static_cast<uint32_t>(__shfl_sync(0xffffffffu, d, i) + bv.doc_base);
      const int32_t wi = __shfl_sync(0xffffffffu, w, i);
      const int32_t ci = __shfl_sync(0xffffffffu, c, i);
      const double mui = __shfl_sync(0xffffffffu, mu_v, i);
      if (bi != cur_b) {
        flush(cur_b);
        cur_b = bi;
        for (int j = 0; j < KPL; ++j) {
          const int k = kbase + lane + kWarp * j;
          th[j * kWarp + lane] = k < K ? __ldg(theta_batch + bi * K + k) : 0.0;
          acc[j * kWarp + lane] = 0ull;
        }
      }
      const double cell_scale = __dmul_rn(m_t, static_cast<double>(ci));
      const bool degenerate = mui < 1e-30;  // sampler.cpp:164, 0/0 guard
      const double* prow = phi_wk + static_cast<int64_t>(wi) * K;
#pragma unroll 1
      for (int j = 0; j < KPL; ++j) {
        const int k = kbase + lane + kWarp * j;
        if (k >= K) break;
        const double ph = __ldg(prow + k);
        const double weight =
            degenerate ? uniform_weight : __ddiv_rn(__dmul_rn(th[j * kWarp + lane], ph), mui);
        const double rate = __dmul_rn(weight, cell_scale);
        if (!(rate >= 0.0) || isinf(rate)) {  // sampler.cpp:173-175 and rng.cpp:140-142
          atomicOr(err, kErrNumerical);
          continue;
        }
        if (MODE == kModeExpected) {
          accf[j * kWarp + lane] = __dadd_rn(accf[j * kWarp + lane], rate);
          atomicAdd(phi_exp + static_cast<int64_t>(wi) * K + k, rate);
        } else {
          if (rate == 0.0) continue;
          const uint32_t tag = make_tag(kPoissonCounts, sweep, static_cast<uint32_t>(k));
          uint32_t k0, k1;
          stream_key(seed, tag, k0, k1);
          const U4 blk = philox10(U4{0u, static_cast<uint32_t>(wi), di, t}, k0, k1);
          int64_t z;
          if (rate < 10.0) {
            z = poisson_inversion(rate, u64_to_uniform(join64(blk.x, blk.y)));
          } else {
            Stream s;
            s.init_with_block0(seed, t, di, static_cast<uint32_t>(wi), tag, blk, 0);
            z = poisson_ptrs(rate, s);
          }
          if (z != 0) {
            acc[j * kWarp + lane] += static_cast<unsigned long long>(z);
            atomicAdd(phi_counts + static_cast<int64_t>(wi) * K + k,
                      static_cast<unsigned long long>(z));
          }
        }
      }
    }
  }
  flush(cur_b);
}

// ------------------------------------------------------ sample (fast-exact)
// Same draws as k_sample, bit for bit, at a fraction of the cost.  A draw's
// outcome z is the first k with u <= cdf_k, where u is the stream's first
// uniform and cdf_k the reference's f64 inversion recurrence (rng.cpp:39-52).
// The fast path evaluates rate, exp and the recurrence in f32 and decides a
// comparison only when u lies outside [cdf_k - m_k, cdf_k + m_k], m_k a
// rigorous bound on |cdf_f32 - cdf_ref| (below); otherwise (~3e-5 per draw),
// for lambda near or above 10 (PTRS), non-finite / tiny inputs, or k > 40,
// the draw is deferred to the exact path (k_deferred_*): sequential f64 mu,
// __ddiv_rn rate, full Philox block, exact inversion or PTRS.
// Error bound (u = 2^-24):
//   lambda_f: theta, phi rounded to f32 (2u), product (u), mu by tree sum of
//     positive terms (<= 12u), m*c (u), __fdividef (4u), lambda (u)
//     -> |lambda_f - lambda| <= dl = 24u lambda = 1.43e-6 lambda
//   |cdf_f32(k; lambda_f) - cdf_ref(k; lambda)| <=
//       |cdf_f32(k; lambda_f) - F_k(lambda_f)|       f32 evaluation
//     + |F_k(lambda_f) - F_k(lambda)|                 <= dl pmf_k (dF_k/dl = -pmf_k)
//     + |F_k(lambda) - cdf_ref(k; lambda)|            f64, < 1e-14
//   f32 evaluation: e0 = ex2.approx(-lambda log2 e): 2^-22 + 1.5u lambda
//     = eps0 <= 2.4e-7 + 1.2e-7 lambda; pmf_i carries eps0 + 4u i (rcp.approx
//     1 ulp + 2 roundings per step); each cdf add one rounding
//     -> <= cdf_k (eps0 + 5u k) = cdf_k (2.4e-7 + 1.2e-7 lambda + 3e-7 k)
//   m_k = 2 x the sum = cdf_k (4.8e-7 + 2.4e-7 lambda + 6e-7 k)
//         + 3e-6 lambda pmf_k + 2.5e-7
//   (k <= 2 share the upper bound M = 2e-6 + 3.3e-6 lambda >= m_0, m_1, m_2:
//   one FFMA instead of ten instructions, at ~1.3x the deferral rate)
//   (2.5e-7 >= 2x the u quantisation: u is taken from the top 23 bits of the
//   high word, true u in [u_f, u_f + 2^-23)).
// The mu used is the caller's mu array when given (per-call sample_counts),
// else the warp computes it (f32 tree).

constexpr int kFastBlock = 256;
// the decision variant of the production kernel (fast_poisson3 DEC 1: z in
// {0, 1, 2} branch-free, the sequential search beyond; a fourth branch-free
// threshold was measured equal -- its extra instructions cost what the rarer
// search saves -- with 9% more deferrals from the wider band)
constexpr int kDecDefault = 1;
#ifndef SAMELDA_V2_MINB
#define SAMELDA_V2_MINB 4
#endif
constexpr int kV2Minb = SAMELDA_V2_MINB;  // blocks per SM of the period kernel

// Nonzeros per warp work item: 128 (the packed u16 theta-count pairs hold
// <= 128 nonzeros x z <= 40), fewer on small batches so the grid keeps ~4
// waves of resident warps (148 SMs x 32 warps) -- a C1 sweep (0.87M nonzeros,
// K = 32, one topic slice) has only 1.4 waves at 128
inline int64_t work_chunk(int64_t nnz, int n_slices) {
  const int64_t target_warps = int64_t{148} * 32 * 4;
  int64_t c = nnz * n_slices / target_warps;
  c = std::max<int64_t>(32, std::min<int64_t>(128, (c + 31) / 32 * 32));
  return c;
}
// inversion below 10 (rng.cpp:139-150): decided only when lambda_f's whole
// error interval (1.5e-6 relative, 2x) lies below 10; PTRS draws defer
constexpr float kInvMax = 9.99997f;

// MUFU-only exp2 (no denormal range fix-up: arguments here are in
// [-14.5, 0]); its error is inside the fast-path budget.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Fast-path Poisson decision (fast_poisson3 + fast_poisson_tail_z below; the
// error bound above).  z is the first k with u <= cdf_k; a draw is left
// undecided when u falls inside a threshold's band, or the search passes
// z = 40.  The first three thresholds (z in {0, 1, 2}, ~99% of draws at
// lambda ~ 0.4) are evaluated branch-free with one band: with cdf_k, pmf_k <= 1
// (+ rounding slack), m_k <= (r0 + 1.2e-6) + pl + 2.5e-7 = 1.93e-6 + 3.24e-6
// lambda <= M = 2e-6 + 3.3e-6 lambda (r0 = 4.8e-7 + 2.4e-7 lambda,
// pl = 3e-6 lambda); only u beyond cdf_2 + M enters the sequential search,
// with m_k = cdf_k (r0 + 1.2e-6 + 6e-7 (k - 2)) + pl pmf_k + 2.5e-7.  Terms:
// t1 = e0 lambda, pmf_2 = t1 lambda / 2 (the reference recurrence
// pmf *= lambda / k with an exact 1/2).

#ifdef SAMELDA_DEFER_STATS
// Diagnostics build only (tools/defer_stats.sh): why draws defer.
//   [0] nz_exact  [1] tiny product  [2] lambda >= kInvMax  [3] band / search
//   [8 + b]  deferred draws by lambda bin b = floor(log2 lambda) + 20
//   [48 + b] all draws with lambda >= 2^-4, by the same bins
__device__ unsigned long long g_defer_stats[96];
__device__ __forceinline__ void defer_stats(bool nz_exact, float prod, float lam, bool undecided) {
  const int bin = lam > 0.0f ? max(0, min(39, static_cast<int>(floorf(log2f(lam))) + 20)) : 0;
  if (lam >= 0.0625f) atomicAdd(&g_defer_stats[48 + bin], 1ull);
  if (!undecided) return;
  const int cat = nz_exact ? 0 : !(prod >= 1e-30f) ? 1 : !(lam < kInvMax) ? 2 : 3;
  atomicAdd(&g_defer_stats[cat], 1ull);
  atomicAdd(&g_defer_stats[8 + bin], 1ull);
}
#endif

struct Philox1 {
  // round-1 specialisation for counter {0, w, d, t}: M0 * 0 = 0, so the
  // only per-draw work in round 1 is one xor; M1 * d is per nonzero
  uint32_t hw;  // hi(M1 * d) ^ w
  uint32_t lo;  // lo(M1 * d)
};

// Deferred exact draws: one record per (nonzero, topic slice) that has at
// least one draw the fast path could not decide (a PTRS decision inside its band,
// an ambiguous comparison, z > 40, or non-finite / tiny inputs).
struct Deferred {
  int64_t p;          // batch nonzero index
  int32_t b, w, c;    // batch row, word id, token count
  int32_t kbase;      // first topic of the slice
  uint32_t mask[8];   // bit lane of mask[j]: topic kbase + lane + 32 j
  float scale;        // the fast path's m c / mu_f (its lambda_f = (theta32 phi32) scale)
  uint32_t spare;     // written (0): the 64-byte record has no uninitialised bytes
};

// Round keys a draw of topic k needs (philox_y_sched), precomputed once per topic:
// ks[0] = k0, ks[1] = p2lo, ks[2] = p2hi (M1 * (t ^ k1)), then for r = 1..8
// ks[1 + 2r] = k0 + r W0, ks[2 + 2r] = k1 + r W1 (ks[17] = k0 + 8 W0 unused).
constexpr int kKeyWords = 20;

__device__ __forceinline__ void topic_schedule(uint64_t seed, uint32_t t, uint32_t sweep,
                                               uint32_t k, uint32_t* ks) {
  uint32_t k0, k1;
  stream_key(seed, make_tag(kPoissonCounts, sweep, k), k0, k1);
  uint32_t p2lo, p2hi;
  mulhilo(kPhiloxM1, t ^ k1, p2lo, p2hi);
  ks[0] = k0;
  ks[1] = p2lo;
  ks[2] = p2hi;
#pragma unroll
  for (int r = 1; r <= 8; ++r) {
    ks[1 + 2 * r] = k0 + static_cast<uint32_t>(r) * kPhiloxW0;
    ks[2 + 2 * r] = k1 + static_cast<uint32_t>(r) * kPhiloxW1;
  }
  ks[19] = 0;
}

__device__ __forceinline__ uint32_t philox_y_sched(const Philox1 r1, const uint32_t* ks) {
  uint32_t lo0, hi0;
  mulhilo(kPhiloxM0, r1.hw ^ ks[0], lo0, hi0);
  uint32_t x0 = ks[2] ^ r1.lo ^ ks[3], x1 = ks[1], x2 = hi0 ^ ks[4], x3 = lo0;
#pragma unroll
  for (int r = 2; r < 9; ++r) {
    uint32_t a0, b0, a1, b1;
    mulhilo(kPhiloxM0, x0, a0, b0);
    mulhilo(kPhiloxM1, x2, a1, b1);
    const uint32_t n0 = b1 ^ x1 ^ ks[1 + 2 * r], n2 = b0 ^ x3 ^ ks[2 + 2 * r];
    x0 = n0;
    x1 = a1;
    x2 = n2;
    x3 = a0;
  }
  return kPhiloxM1 * x2;
}

// f32 mu of every batch nonzero over all K topics (fast path only; the exact
// f64 mu of deferred draws is computed separately).  Warp per 32 nonzeros:
// lanes over topics, shuffle tree per nonzero, lane i keeps nonzero i's.
__global__ void __launch_bounds__(256) k_mu_f32(BatchView bv, const float* __restrict__ theta_b32,
                                                const float* __restrict__ phi32, int K,
                                                float* __restrict__ mu_f) {
  const int lane = threadIdx.x & 31;
  const int64_t g0 = ((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5) * 32;
  if (g0 >= bv.nnz) return;
  const int n_here = static_cast<int>(min(static_cast<int64_t>(32), bv.nnz - g0));
  int64_t b = 0;
  int32_t w = 0;
  if (lane < n_here) {
    const int64_t p = g0 + lane;
    b = find_row(bv.batch_prefix, bv.B, p);
    const int32_t d = __ldg(bv.batch_docs + b);
    w = __ldg(bv.word_ids + __ldg(bv.doc_offsets + d) + (p - __ldg(bv.batch_prefix + b)));
  }
  float mine = 0.0f;
  for (int i = 0; i < n_here; ++i) {
    const int64_t bi = __shfl_sync(0xffffffffu, b, i);
    const int32_t wi = __shfl_sync(0xffffffffu, w, i);
    const float* tr = theta_b32 + bi * K;
    const float* pr = phi32 + static_cast<int64_t>(wi) * K;
    // f64 accumulation of the exact f32 x f32 products: mu_f is then within
    // ~1 ulp of the f32-input dot for any K (the fast-path budget assumes 16u)
    double part = 0.0;
    if ((K & 3) == 0) {
      // 16-byte loads: lane takes topics 4 lane .. 4 lane + 3 of each 128
      const float4* t4 = reinterpret_cast<const float4*>(tr);
      const float4* p4 = reinterpret_cast<const float4*>(pr);
#pragma unroll 4
      for (int q = lane; q < (K >> 2); q += 32) {
        const float4 a = __ldg(t4 + q), b = __ldg(p4 + q);
        part = __dadd_rn(part, static_cast<double>(a.x) * static_cast<double>(b.x));
        part = __dadd_rn(part, static_cast<double>(a.y) * static_cast<double>(b.y));
        part = __dadd_rn(part, static_cast<double>(a.z) * static_cast<double>(b.z));
        part = __dadd_rn(part, static_cast<double>(a.w) * static_cast<double>(b.w));
      }
    } else {
      for (int k = lane; k < K; k += 32)
        part = __dadd_rn(part, static_cast<double>(__ldg(tr + k)) * static_cast<double>(__ldg(pr + k)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
    if (lane == i) mine = __double2float_rn(part);
  }
  if (lane < n_here) mu_f[g0 + lane] = mine;
}

// ---------------------------------------------- sample (fast-exact, v2)
// k_sample_v2: the same draws as round 1's first fast-exact kernel
// (k_sample_fast, since removed), bit for bit, with about a tenth fewer
// instructions per draw (the kernel is issue-bound; ncu on the
// fast kernel: 110 warp instructions per draw of which ~38 are the Philox
// rounds and their round keys).  Differences:
//   * the mu source is a template parameter (the period path's fused tree
//     carries no mu shuffles or branches);
//   * Philox chains run in groups of KG topics (register pressure: no spills
//     at 64 registers), decisions follow each group;
//   * decision: c2 by one FFMA (one rounding instead of two: inside the same
//     bound), the count z = #(d_k > M) from three set.gt (0 / -1) and one
//     IADD3 instead of predicate selects;
//   * the phi-count scatter address is formed once per nonzero and every
//     draw issues one unpredicated RED with an immediate offset (a warp-wide
//     RED is issued for virtually every draw anyway; lanes with z = 0 add 0);
//   * theta counts accumulate as packed u16 pairs (per lane and topic a
//     chunk holds <= 128 nonzeros x z <= 40 < 2^16), flushed per doc.

__device__ __forceinline__ void red_add_u64(unsigned long long* addr, uint32_t z) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(addr),
               "l"(static_cast<unsigned long long>(z)));
}

// z in {0, 1, 2} decided branch-free, 3 = continue the search from k = 3
// (bound above; c2 = fma(t1, lambda/2, c1) rounds once).
// DEC selects how z and the band flag are formed (same decisions):
//   0: predicates + nested selects (ALU pipe)
//   1: z = sum of sat(2^100 (d_k - M)) on the FMA pipe, band by predicates
//   2: band too: und iff sum_k sat(2^100 (d_k - M)) + sat(2^100 (-d_k - M)) != 3
//      (counts d_k > M and d_k < -M; equality on either side is in the band)
// Mb = M 2^100 exactly (power-of-two scaling).
template <int DEC>
__device__ __forceinline__ uint32_t fast_poisson3(float lam, float M, float Mb, float u, bool& und,
                                                  float& t1_out, float& c2_out) {
  const float e0 = ex2_approx(__fmul_rn(lam, -1.4426950408889634f));
  const float t1 = __fmul_rn(e0, lam);
  const float c1 = __fadd_rn(e0, t1);
  const float c2 = __fmaf_rn(t1, __fmul_rn(lam, 0.5f), c1);
  const float d0 = __fsub_rn(u, e0), d1 = __fsub_rn(u, c1), d2 = __fsub_rn(u, c2);
  t1_out = t1;
  c2_out = c2;
  if (DEC == 0) {
    und = und || (fabsf(d0) <= M) || (fabsf(d1) <= M) || (fabsf(d2) <= M);
    // d0 >= d1 >= d2 (the cdf terms are non-decreasing): nested selects
    return d2 > M ? 3u : (d1 > M ? 2u : (d0 > M ? 1u : 0u));
  }
  // sign of 2^100 d_k - Mb is the sign of d_k - M (one rounding, no overflow:
  // |d_k| <= 1); any nonzero difference is >= 2^-149 * 2^100 -> saturates to 1
  const float s0 = __saturatef(__fmaf_rn(d0, 0x1p100f, -Mb));
  const float s1 = __saturatef(__fmaf_rn(d1, 0x1p100f, -Mb));
  const float s2 = __saturatef(__fmaf_rn(d2, 0x1p100f, -Mb));
  const float zf = __fadd_rn(__fadd_rn(s0, s1), s2);
  if (DEC == 1) {
    und = und || (fabsf(d0) <= M) || (fabsf(d1) <= M) || (fabsf(d2) <= M);
  } else {
    const float l0 = __saturatef(__fmaf_rn(d0, -0x1p100f, -Mb));
    const float l1 = __saturatef(__fmaf_rn(d1, -0x1p100f, -Mb));
    const float l2 = __saturatef(__fmaf_rn(d2, -0x1p100f, -Mb));
    und = und || (__fadd_rn(zf, __fadd_rn(__fadd_rn(l0, l1), l2)) != 3.0f);
  }
  return __float_as_uint(__fadd_rn(zf, 8388608.0f)) - 0x4B000000u;
}

// sequential search from k = 3 (u beyond cdf_2 + M) with the bound above,
// 1/k and the bound's k-term r_k - r_0 = 1.2e-6 + 6e-7 (k - 2)
// read from constant tables (the step index is the same for every lane still
// searching: one broadcast load) instead of rcp.approx and running sums; the
// correctly rounded 1/k is within the 1-ulp rcp.approx the budget assumed.
// Returns z, or kUndZ when undecided (also past z = 40): the outcome as a
// value, so no flag state lives across the loop.
__constant__ float c_tail_inv[41] = {
    0.0f,        1.0f,         0.5f,         1.0f / 3,  0.25f,     0.2f,      1.0f / 6,
    1.0f / 7,    0.125f,       1.0f / 9,     0.1f,      1.0f / 11, 1.0f / 12, 1.0f / 13,
    1.0f / 14,   1.0f / 15,    0.0625f,      1.0f / 17, 1.0f / 18, 1.0f / 19, 0.05f,
    1.0f / 21,   1.0f / 22,    1.0f / 23,    1.0f / 24, 0.04f,     1.0f / 26, 1.0f / 27,
    1.0f / 28,   1.0f / 29,    1.0f / 30,    1.0f / 31, 0.03125f,  1.0f / 33, 1.0f / 34,
    1.0f / 35,   1.0f / 36,    1.0f / 37,    1.0f / 38, 1.0f / 39, 0.025f};
__constant__ float c_tail_rk[41] = {
    0.0f,     0.0f,     1.2e-6f,  1.8e-6f,  2.4e-6f,  3.0e-6f,  3.6e-6f,  4.2e-6f,  4.8e-6f,
    5.4e-6f,  6.0e-6f,  6.6e-6f,  7.2e-6f,  7.8e-6f,  8.4e-6f,  9.0e-6f,  9.6e-6f,  1.02e-5f,
    1.08e-5f, 1.14e-5f, 1.2e-5f,  1.26e-5f, 1.32e-5f, 1.38e-5f, 1.44e-5f, 1.5e-5f,  1.56e-5f,
    1.62e-5f, 1.68e-5f, 1.74e-5f, 1.8e-5f,  1.86e-5f, 1.92e-5f, 1.98e-5f, 2.04e-5f, 2.1e-5f,
    2.16e-5f, 2.22e-5f, 2.28e-5f, 2.34e-5f, 2.4e-5f};

constexpr uint32_t kUndZ = 64;
__device__ __forceinline__ uint32_t fast_poisson_tail_z(float lam, float u, float t1, float c2) {
  const float r0 = __fmaf_rn(2.4e-7f, lam, 4.8e-7f);
  const float pl = __fmul_rn(3e-6f, lam);
  float pmf = __fmul_rn(t1, __fmul_rn(lam, 0.5f)), cdf = c2;
#pragma unroll 1
  for (uint32_t k = 3; k <= 40; ++k) {
    pmf = __fmul_rn(pmf, __fmul_rn(lam, c_tail_inv[k]));
    cdf = __fadd_rn(cdf, pmf);
    const float mk = __fmaf_rn(cdf, __fadd_rn(r0, c_tail_rk[k]), __fmaf_rn(pmf, pl, 2.5e-7f));
    const float dk = __fsub_rn(u, cdf);
    if (dk < -mk) return k;
    if (!(dk > mk)) return kUndZ;
  }
  return kUndZ;
}

// PHI = false: a non-final inner sweep -- only the last sweep's phi counts feed
// update_model (sampler.cpp:320-332), so the phi-count scatter is skipped.
template <int KPL, bool FULL, int MUSRC, int MINB, int DEC = 1, int TAIL = 0, bool PHI = true>
__global__ void __launch_bounds__(kFastBlock, MINB) k_sample_v2(
    BatchView bv, const float* __restrict__ theta_b32, const float* __restrict__ phi32,
    const double* __restrict__ mu_in, const float* __restrict__ mu_f_in, int K, double m_t,
    uint64_t seed, uint32_t t, uint32_t sweep, int64_t chunk,
    unsigned long long* __restrict__ theta_counts, unsigned long long* __restrict__ phi_counts,
    Deferred* __restrict__ deferred, uint32_t* __restrict__ rec_count,
    unsigned long long* __restrict__ n_deferred) {
  constexpr int KG = KPL < 4 ? KPL : 4;  // Philox chains in flight per group
  const int lane = threadIdx.x & 31;
  const int kbase = static_cast<int>(blockIdx.y) * kWarp * KPL;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * (kFastBlock / kWarp) + (threadIdx.x >> 5);

  __shared__ uint4 s_keys[KPL][kKeyWords / 4][kWarp];
  // TAIL 1: draws that need the sequential search (u beyond cdf_2 + M) are
  // provisionally counted as z = 3 (certain lower bound) and parked here;
  // one combined pass per nonzero finishes them (lanes run their own parked
  // topics back to back instead of entering a divergent loop per topic)
  __shared__ float2 s_park[TAIL ? kFastBlock / kWarp : 1][TAIL ? KPL : 1][kWarp];
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < KPL * kWarp; e += blockDim.x) {
    const int jj = e / kWarp, ll = e % kWarp;
    uint32_t ks[kKeyWords];
    topic_schedule(seed, t, sweep, static_cast<uint32_t>(kbase + ll + kWarp * jj), ks);
#pragma unroll
    for (int q = 0; q < kKeyWords / 4; ++q)
      s_keys[jj][q][ll] = make_uint4(ks[4 * q], ks[4 * q + 1], ks[4 * q + 2], ks[4 * q + 3]);
  }
  __syncthreads();
  const int64_t p0 = item * chunk;
  const int64_t p1 = min(p0 + chunk, bv.nnz);
  // this work item's deferred records live at fixed slots [item_g chunk,
  // item_g chunk + rec_count[item_g]): no global counter per record (late in
  // training nearly every nonzero carries a PTRS draw, and one contended
  // atomic per record serialised the kernel); k_deferred_expand walks them item by item
  const int64_t item_g = static_cast<int64_t>(blockIdx.y) * gridDim.x * (kFastBlock / kWarp) + item;
  if (p0 >= p1) {
    if (lane == 0) rec_count[item_g] = 0;
    return;
  }
  Deferred* const rec_out = deferred + item_g * chunk;
  uint32_t n_rec = 0;

  int cur_b = -1;
  // the document's theta slice lives in shared memory (lane-private 16-byte
  // slots, two LDS.128 per nonzero), not in eight registers: the freed
  // registers end the per-draw rematerialisation of addresses (last sweep
  // 3.30 -> 3.22 ms at K = 256)
  constexpr bool kThS = KPL % 4 == 0;
  __shared__ float4 s_th[kThS ? kFastBlock / kWarp : 1][kThS ? KPL / 4 : 1][kWarp];
  (void)s_th;
  float th[kThS ? 1 : KPL];
  uint32_t acc[(KPL + 1) / 2];
#pragma unroll
  for (int j = 0; j < (kThS ? 1 : KPL); ++j) th[j] = 0.0f;
#pragma unroll
  for (int j = 0; j < (KPL + 1) / 2; ++j) acc[j] = 0u;

  auto flush = [&](int b) {
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int k = kbase + lane + kWarp * j;
      const uint32_t v = (j & 1) ? (acc[j >> 1] >> 16) : (acc[j >> 1] & 0xffffu);
      if ((FULL || k < K) && v)
        atomicAdd(theta_counts + static_cast<int64_t>(b) * K + k, static_cast<unsigned long long>(v));
    }
  };

  for (int64_t g0 = p0; g0 < p1; g0 += kWarp) {
    const int64_t p = g0 + lane;
    int32_t b = 0, d = 0, w = 0, c = 0;
    double mu_v = 0.0;
    float muf_v = 0.0f;
    if (p < p1) {
      b = static_cast<int32_t>(find_row(bv.batch_prefix, bv.B, p));
      d = __ldg(bv.batch_docs + b);
      const int64_t gi = __ldg(bv.doc_offsets + d) + (p - __ldg(bv.batch_prefix + b));
      w = __ldg(bv.word_ids + gi);
      c = __ldg(bv.counts + gi);
      if (MUSRC == 1) mu_v = __ldg(mu_in + p);
      if (MUSRC == 2) muf_v = __ldg(mu_f_in + p);
    }
    const int n_here = static_cast<int>(min(static_cast<int64_t>(kWarp), p1 - g0));
    for (int i = 0; i < n_here; ++i) {
      const int32_t bi = __shfl_sync(0xffffffffu, b, i);
      const uint32_t di = static_cast<uint32_t>(__shfl_sync(0xffffffffu, d, i) + static_cast<int32_t>(bv.doc_base));
      const int32_t wi = __shfl_sync(0xffffffffu, w, i);
      const int32_t ci = __shfl_sync(0xffffffffu, c, i);
      float ph[KPL];
      {
        const float* prow = phi32 + static_cast<int64_t>(wi) * K + kbase + lane;
#pragma unroll
        for (int j = 0; j < KPL; ++j) ph[j] = (FULL || kbase + lane + kWarp * j < K) ? __ldg(prow + kWarp * j) : 0.0f;
      }
      if (bi != cur_b) {
        if (cur_b >= 0) flush(cur_b);
        cur_b = bi;
        const float* trow = theta_b32 + static_cast<int64_t>(bi) * K + kbase + lane;
        if constexpr (kThS) {
          float tv[KPL];
#pragma unroll
          for (int j = 0; j < KPL; ++j) tv[j] = (FULL || kbase + lane + kWarp * j < K) ? __ldg(trow + kWarp * j) : 0.0f;
#pragma unroll
          for (int q = 0; q < KPL / 4; ++q)
            s_th[warp][q][lane] = make_float4(tv[4 * q], tv[4 * q + 1], tv[4 * q + 2], tv[4 * q + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < KPL; ++j) th[j] = (FULL || kbase + lane + kWarp * j < K) ? __ldg(trow + kWarp * j) : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < (KPL + 1) / 2; ++j) acc[j] = 0u;
      }
      float prod[KPL];
      if constexpr (kThS) {
#pragma unroll
        for (int q = 0; q < KPL / 4; ++q) {
          const float4 tv = s_th[warp][q][lane];
          prod[4 * q] = __fmul_rn(tv.x, ph[4 * q]);
          prod[4 * q + 1] = __fmul_rn(tv.y, ph[4 * q + 1]);
          prod[4 * q + 2] = __fmul_rn(tv.z, ph[4 * q + 2]);
          prod[4 * q + 3] = __fmul_rn(tv.w, ph[4 * q + 3]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < KPL; ++j) prod[j] = __fmul_rn(th[j], ph[j]);
      }
      float mu_f;
      if (MUSRC == 1) {
        mu_f = __double2float_rn(__shfl_sync(0xffffffffu, mu_v, i));
      } else if (MUSRC == 2) {
        mu_f = __shfl_sync(0xffffffffu, muf_v, i);
      } else {
        mu_f = 0.0f;
#pragma unroll
        for (int j = 0; j < KPL; ++j) mu_f = __fadd_rn(mu_f, prod[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mu_f = __fadd_rn(mu_f, __shfl_xor_sync(0xffffffffu, mu_f, o));
      }
      const bool nz_exact = !(mu_f >= 1e-20f) || isinf(mu_f);
      // an unusable mu defers the whole nonzero: scale = NaN makes every
      // lambda fail the lambda < kInvMax eligibility test (no per-draw flag)
      const float scale = nz_exact ? __int_as_float(0x7fffffff)
                                   : __fdividef(__double2float_rn(__dmul_rn(m_t, static_cast<double>(ci))), mu_f);
      // band slope per nonzero: M = prod (3.3e-6 scale) + 2e-6 is within 2.4e-7
      // relative of 3.3e-6 lambda + 2e-6 >= 3.24e-6 lambda + 1.93e-6 >= m_0..2
      const float mslope = __fmul_rn(scale, 3.3e-6f);
      uint32_t m1lo, m1hi;
      mulhilo(kPhiloxM1, di, m1lo, m1hi);
      const Philox1 r1{m1hi ^ static_cast<uint32_t>(wi), m1lo};
      unsigned long long* pc = phi_counts + static_cast<int64_t>(wi) * K + kbase + lane;
      uint32_t defer_bits = 0, parked = 0;
#pragma unroll
      for (int g = 0; g < KPL; g += KG) {
        uint32_t y[KG];
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) {
          uint32_t ks[kKeyWords];
#pragma unroll
          for (int q = 0; q < kKeyWords / 4; ++q) {
            const uint4 v = s_keys[g + jj][q][lane];
            ks[4 * q] = v.x;
            ks[4 * q + 1] = v.y;
            ks[4 * q + 2] = v.z;
            ks[4 * q + 3] = v.w;
          }
          y[jj] = philox_y_sched(r1, ks);
        }
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) asm volatile("" : "+r"(y[jj]));
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) {
          const int j = g + jj;
          const float lam = __fmul_rn(prod[j], scale);
          bool und = !(prod[j] >= 1e-30f) || !(lam < kInvMax);
          const float u = __fsub_rn(__int_as_float(0x3f800000 | (y[jj] >> 9)), 1.0f);
          float t1, c2;
          const float M = __fmaf_rn(prod[j], mslope, 2e-6f);
          uint32_t z = fast_poisson3<DEC>(lam, M, __fmul_rn(M, 0x1p100f), u, und, t1, c2);
          if constexpr (TAIL == 0) {
            // z carries the band flag (kUndZ: undecided): no flag state lives
            // across the search (first sweep 3.18 -> 3.14 ms)
            z = und ? kUndZ : z;
            if (z == 3) z = fast_poisson_tail_z(lam, u, t1, c2);
            if (!FULL && kbase + lane + kWarp * j >= K) z = 0;
#ifdef SAMELDA_DEFER_STATS
            if (FULL || kbase + lane + kWarp * j < K) defer_stats(nz_exact, prod[j], lam, z == kUndZ);
#endif
            defer_bits += (z & kUndZ) << j;  // bit 6 + j
            z &= kUndZ - 1;
            acc[j >> 1] += (j & 1) ? (z << 16) : z;
            if (PHI && (FULL || kbase + lane + kWarp * j < K)) red_add_u64(pc + kWarp * j, z);
            continue;
          }
          bool park = z == 3 && !und;  // TAIL 1
          if (!FULL && kbase + lane + kWarp * j >= K) {
            und = false;
            z = 0;
            park = false;
          }
          if (park) {
            s_park[warp][j][lane] = make_float2(lam, u);
            parked |= 1u << j;
          }
          if (und) {
            defer_bits |= 1u << j;
            z = 0;
          }
          acc[j >> 1] += (j & 1) ? (z << 16) : z;
          if (PHI && (FULL || kbase + lane + kWarp * j < K)) red_add_u64(pc + kWarp * j, z);
        }
      }
      if (TAIL == 0) defer_bits >>= 6;
      if (TAIL && __any_sync(0xffffffffu, parked != 0)) {
        // finish parked draws: z = 3 was counted; add z - 3, or undo the 3
        // (u64 wrap-around) and defer the draw when the search is undecided
        unsigned long long* tcrow = theta_counts + static_cast<int64_t>(bi) * K + kbase + lane;
        do {
          if (parked) {
            const int j = __ffs(parked) - 1;
            parked &= parked - 1;
            const float2 st = s_park[warp][j][lane];
            // t1, c2 recomputed exactly as fast_poisson3 formed them
            const float e0 = ex2_approx(__fmul_rn(st.x, -1.4426950408889634f));
            const float t1 = __fmul_rn(e0, st.x);
            const float c2 = __fmaf_rn(t1, __fmul_rn(st.x, 0.5f), __fadd_rn(e0, t1));
            const uint32_t z = fast_poisson_tail_z(st.x, st.y, t1, c2);
            const bool und = z == kUndZ;
            const unsigned long long delta =
                und ? ~2ull : static_cast<unsigned long long>(z - 3u);
            if (und) defer_bits |= 1u << j;
            if (delta) {
              if (PHI) atomicAdd(pc + kWarp * j, delta);
              atomicAdd(tcrow + kWarp * j, delta);
            }
          }
        } while (__any_sync(0xffffffffu, parked != 0));
      }
      if (__any_sync(0xffffffffu, defer_bits != 0)) {
        uint32_t masks[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) masks[j] = j < KPL ? __ballot_sync(0xffffffffu, (defer_bits >> j) & 1u) : 0u;
        if (lane == 0) {
          const uint32_t slot = n_rec;
          Deferred rec;
          rec.p = g0 + i;
          rec.b = bi;
          rec.w = wi;
          rec.c = ci;
          rec.kbase = kbase;
          rec.scale = scale;
          rec.spare = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) rec.mask[j] = masks[j];
          rec_out[slot] = rec;
        }
        ++n_rec;
      }
    }
  }
  if (cur_b >= 0) flush(cur_b);
  if (lane == 0) {
    rec_count[item_g] = n_rec;
    if (n_rec) atomicAdd(n_deferred, static_cast<unsigned long long>(n_rec));
  }
}

// Deferred exact draws in two passes.
// Phase A (k_deferred_expand), lane = record: the record's exact mu -- the
// reference's sequential-k f64 dot (sampler.cpp:111-119), unless the caller
// supplied mu -- and one flat-list entry per flagged topic (slots reserved
// with one atomic per record; integer count scatter makes order irrelevant).
// Phase B (k_deferred_draw), thread = draw: rate with __ddiv_rn, full Philox
// block, f64 inversion or PTRS (rng.cpp:39-86), exactly as k_sample.
struct DeferredDraw {
  uint32_t rec;
  uint32_t k;
};

__device__ __forceinline__ void deferred_one(const BatchView& bv, const Deferred& rec, double mu,
                                             int k, const double* __restrict__ theta_b64,
                                             const double* __restrict__ phi64, int K, double m_t,
                                             uint64_t seed, uint32_t t, uint32_t sweep,
                                             unsigned long long* __restrict__ theta_counts,
                                             unsigned long long* __restrict__ phi_counts,
                                             int* __restrict__ err) {
  const uint32_t d = static_cast<uint32_t>(__ldg(bv.batch_docs + rec.b) + bv.doc_base);
  const double cs = __dmul_rn(m_t, static_cast<double>(rec.c));
  const double weight =
      mu < 1e-30 ? 1.0 / static_cast<double>(K)
                 : __ddiv_rn(__dmul_rn(__ldg(theta_b64 + static_cast<int64_t>(rec.b) * K + k),
                                       __ldg(phi64 + static_cast<int64_t>(rec.w) * K + k)),
                             mu);
  const double rate = __dmul_rn(weight, cs);
  if (!(rate >= 0.0) || isinf(rate)) {
    atomicOr(err, kErrNumerical);
    return;
  }
  if (rate == 0.0) return;
  const uint32_t tag = make_tag(kPoissonCounts, sweep, static_cast<uint32_t>(k));
  uint32_t k0, k1;
  stream_key(seed, tag, k0, k1);
  const U4 blk = philox10(U4{0u, static_cast<uint32_t>(rec.w), d, t}, k0, k1);
  long long z;
  if (rate < 10.0) {
    z = poisson_inversion(rate, u64_to_uniform(join64(blk.x, blk.y)));
  } else {
    Stream st;
    st.init_with_block0(seed, t, d, static_cast<uint32_t>(rec.w), tag, blk, 0);
    z = poisson_ptrs(rate, st);
  }
  if (z != 0) {
    atomicAdd(theta_counts + static_cast<int64_t>(rec.b) * K + k, static_cast<unsigned long long>(z));
    if (phi_counts)  // null for a non-final inner sweep (only theta counts are used)
      atomicAdd(phi_counts + static_cast<int64_t>(rec.w) * K + k, static_cast<unsigned long long>(z));
  }
}

// The reference's sequential-k exact mu of a record (sampler.cpp:111-119).
__device__ __forceinline__ double record_mu(const Deferred& rec, const double* __restrict__ theta_b64,
                                            const double* __restrict__ phi64, int K) {
  const double* th = theta_b64 + static_cast<int64_t>(rec.b) * K;
  const double* ph = phi64 + static_cast<int64_t>(rec.w) * K;
  double mu = 0.0;
  if ((K & 1) == 0) {
    const double2* th2 = reinterpret_cast<const double2*>(th);
    const double2* ph2 = reinterpret_cast<const double2*>(ph);
#pragma unroll 8
    for (int k2 = 0; k2 < (K >> 1); ++k2) {
      const double2 a = __ldg(th2 + k2), b = __ldg(ph2 + k2);
      mu = __dadd_rn(mu, __dmul_rn(a.x, b.x));
      mu = __dadd_rn(mu, __dmul_rn(a.y, b.y));
    }
  } else {
    for (int k = 0; k < K; ++k) mu = __dadd_rn(mu, __dmul_rn(__ldg(th + k), __ldg(ph + k)));
  }
  return mu;
}

// PTRS (rng.cpp:57-86) for a rate known only to lie in [L (1 - e), L (1 + e)],
// e = kLamRel (the fast path's f32 lambda: 1.5e-6 relative, 2x): every
// decision the reference takes is evaluated at L and accepted only when no
// rate in the interval could change it, with bounds on its derivative in
// lambda >= 10 (b' = 1.265 / sqrt(lambda) <= 0.4, a' = 0.02483 b'):
//   v_r:  |dv_r/dlambda| lambda <= 1.46 / sqrt(lambda) <= 0.46      -> band e
//   g:    |dg/dlambda| <= 1 + |u| (2 a' / us + b') <= 1.2 + 0.00993 / us
//   lhs:  lambda |dlhs/dlambda| <= 0.111 (inv_alpha) + 0.61 (a / us^2 + b)
//   rhs:  |drhs/dlambda| = |k / lambda - 1|
// plus slack for the reference's f64 rounding and the libdevice / glibc ulp
// differences of log, sqrt and lgamma.  The uniforms, us and the rejection
// tests that do not involve lambda are the reference's exactly.  Returns
// false when any decision is inside its band (the caller then forms the
// exact rate), true with the draw in *z otherwise.
constexpr double kLamRel = 3e-6;
constexpr float kPtrsMinF = 10.0001f;  // lambda_f (1 - kLamRel) >= 10: PTRS for every rate
__device__ __noinline__ bool ptrs_banded(double L, U4 blk, uint32_t k0, uint32_t k1, uint32_t w,
                                            uint32_t d, uint32_t t, long long* z) {
  constexpr double e = kLamRel;
  const double log_lambda = log(L);
  const double b = __dadd_rn(0.931, __dmul_rn(2.53, sqrt(L)));
  const double a = __dadd_rn(-0.059, __dmul_rn(0.02483, b));
  const double v_r = __dadd_rn(0.9277, -__ddiv_rn(3.6224, __dadd_rn(b, -2.0)));
  const double e_vr = e + 1e-12;
  const double a2 = __dmul_rn(2.0, a);
  // each iteration consumes one Philox block (two uniforms, rng.cpp:70-71)
  for (uint32_t it = 0; it < 16; ++it) {
    if (it) blk = philox10(U4{it, w, d, t}, k0, k1);
    const double u = __dadd_rn(u64_to_uniform_oo(join64(blk.x, blk.y)), -0.5);
    const double v = u64_to_uniform_oo(join64(blk.z, blk.w));
    const double us = __dadd_rn(0.5, -fabs(u));
    const double g = __dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(__ddiv_rn(a2, us), b), u), L), 0.43);
    const double slack = 1e-12 * (fabs(g) + 2.0 * L + 1.0);
    if (us >= 0.07) {
      if (v <= v_r - e_vr) {  // quick acceptance for every rate in the interval
        const double e_g = 1.35 * e * L * 1.01 + slack;  // 1.2 + 0.00993 / 0.07 < 1.35
        const double lo = g - e_g, hi = g + e_g;
        if (!(lo >= 0.0) || !(hi < 9.0e18) || floor(lo) != floor(hi)) return false;
        *z = static_cast<long long>(g);
        return true;
      }
      if (!(v > v_r + e_vr)) return false;
    }
    const double e_g = (1.2 + 0.01 / us) * e * L * 1.01 + slack;
    if (g + e_g < 0.0 || (us < 0.013 && v > us)) continue;  // rejected for every rate
    if (!(g - e_g >= 0.0) || !(g + e_g <= 9.0e18) || floor(g - e_g) != floor(g + e_g)) return false;
    const long long k = static_cast<long long>(g);
    const double inv_alpha = __dadd_rn(1.1239, __ddiv_rn(1.1328, __dadd_rn(b, -3.4)));
    const double lhs =
        log(__ddiv_rn(__dmul_rn(v, inv_alpha), __dadd_rn(__ddiv_rn(a, __dmul_rn(us, us)), b)));
    const double lg = k < kLgammaTab && g_lgamma_ready ? g_lgamma_int[k]
                                                       : lgamma(__dadd_rn(static_cast<double>(k), 1.0));
    const double kl = __dmul_rn(static_cast<double>(k), log_lambda);
    const double rhs = __dadd_rn(__dadd_rn(-L, kl), -lg);
    const double mag = fabs(lhs) + L + fabs(kl) + fabs(lg);
    const double e_log = 0.74 * e + (fabs(static_cast<double>(k) - L) + e * L) * e * 1.01 + 1e-13 * mag;
    if (lhs <= rhs - e_log) {
      *z = k;
      return true;
    }
    if (!(lhs > rhs + e_log)) return false;
  }
  return false;
}

// The fast path's lambda_f of a deferred draw, exactly as k_sample_v2 formed it
__device__ __forceinline__ float draw_lambda_f(const Deferred& rec, int k,
                                               const float* __restrict__ theta_b32,
                                               const float* __restrict__ phi32, int K) {
  const float prod = __fmul_rn(__ldg(theta_b32 + static_cast<int64_t>(rec.b) * K + k),
                               __ldg(phi32 + static_cast<int64_t>(rec.w) * K + k));
  return prod >= 1e-30f ? __fmul_rn(prod, rec.scale) : 0.0f;
}

// A deferred draw without a precomputed mu: a PTRS draw is decided from the
// fast path's lambda_f when its interval allows (ptrs_banded).  Returns false
// when the draw needs the exact rate (the record's mu, deferred_one).
__device__ __forceinline__ bool deferred_try_fast(const BatchView& bv, const Deferred& rec, int k,
                                                  const float* __restrict__ theta_b32,
                                                  const float* __restrict__ phi32, int K,
                                                  uint64_t seed, uint32_t t, uint32_t sweep,
                                                  unsigned long long* __restrict__ theta_counts,
                                                  unsigned long long* __restrict__ phi_counts) {
  const float lam = draw_lambda_f(rec, k, theta_b32, phi32, K);
  if (!(lam >= kPtrsMinF && lam <= 1e30f)) return false;
  const uint32_t d = static_cast<uint32_t>(__ldg(bv.batch_docs + rec.b) + bv.doc_base);
  const uint32_t tag = make_tag(kPoissonCounts, sweep, static_cast<uint32_t>(k));
  uint32_t k0, k1;
  stream_key(seed, tag, k0, k1);
  const U4 blk = philox10(U4{0u, static_cast<uint32_t>(rec.w), d, t}, k0, k1);
  long long z = 0;
  if (!ptrs_banded(static_cast<double>(lam), blk, k0, k1, static_cast<uint32_t>(rec.w), d, t, &z))
    return false;
  if (z != 0) {
    atomicAdd(theta_counts + static_cast<int64_t>(rec.b) * K + k, static_cast<unsigned long long>(z));
    if (phi_counts)
      atomicAdd(phi_counts + static_cast<int64_t>(rec.w) * K + k, static_cast<unsigned long long>(z));
  }
  return true;
}


// Phase A, thread = record: the record's exact mu -- the reference's
// sequential-k f64 dot (sampler.cpp:111-119: product then add, no FMA) over
// the batch row's theta and the word's phi, both read as 16-byte pairs --
// unless the caller supplied mu, then the record's flagged draws into the flat
// list (one atomic per warp reserves the warp's slots).  No shared-memory
// tiles and no block barriers: late in training nearly every nonzero carries a
// PTRS draw and this pass is the exact SDDMM of the whole batch (staging the
// phi rows through shared memory for coalesced loads measured slower: 7.7 and
// 9.0 ms per sweep against 5.7).
__global__ void __launch_bounds__(256) k_deferred_expand(
    BatchView bv, const double* __restrict__ theta_b64, const double* __restrict__ phi64,
    const float* __restrict__ theta_b32, const float* __restrict__ phi32, bool fast,
    const double* __restrict__ mu_in, int K, double m_t, uint64_t seed, uint32_t t,
    uint32_t sweep, const Deferred* __restrict__ deferred, const uint32_t* __restrict__ rec_count,
    int64_t n_items, int chunk, double* __restrict__ rec_mu,
    DeferredDraw* __restrict__ draws, unsigned long long* __restrict__ n_draws,
    unsigned long long draw_cap, unsigned long long* __restrict__ theta_counts,
    unsigned long long* __restrict__ phi_counts, int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_g = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  // a warp takes a window of kExpItems work items of k_sample_v2 (item i's
  // records at slots i chunk + [0, rec_count[i])) and numbers their records
  // densely (warp scan of the counts), lane = record, 32 at a time: early in
  // training an item holds ~2 records, late ~chunk
  constexpr int kExpItems = 8;
  for (int64_t i0 = warp_g * kExpItems; i0 < n_items; i0 += n_warps * kExpItems) {
   const uint32_t cnt_i = lane < kExpItems && i0 + lane < n_items ? __ldg(rec_count + i0 + lane) : 0u;
   uint32_t inc_i = cnt_i;
#pragma unroll
   for (int o = 1; o < kExpItems; o <<= 1) {
     const uint32_t v = __shfl_up_sync(0xffffffffu, inc_i, o);
     if (lane >= o) inc_i += v;
   }
   const uint32_t excl_i = inc_i - cnt_i;
   const uint32_t total = __shfl_sync(0xffffffffu, inc_i, kExpItems - 1);
   for (uint32_t q0 = 0; q0 < total; q0 += 32) {
    const uint32_t q = q0 + lane;
    const bool live = q < total;
    int j = 0;  // last window item with excl <= q
#pragma unroll
    for (int step = kExpItems / 2; step > 0; step >>= 1)
      if (__shfl_sync(0xffffffffu, excl_i, j + step) <= q) j += step;
    const uint32_t slot =
        static_cast<uint32_t>((i0 + j) * chunk + (q - __shfl_sync(0xffffffffu, excl_i, j)));
    Deferred me{};
    double mu = 0.0;
    bool mu_ok = false;
    uint32_t cnt = 0;
    if (live) {
      me = deferred[slot];
      // fast mode (late in training: nearly every record is one PTRS draw):
      // no mu here (NaN); the draw pass decides PTRS draws from lambda_f and
      // forms the record's mu itself for the others
      const bool need_mu = !fast;
      if (mu_in) mu = __ldg(mu_in + me.p);
      else if (need_mu) mu = record_mu(me, theta_b64, phi64, K);
      else mu = __longlong_as_double(0x7ff8000000000000ll);
      rec_mu[slot] = mu;
      mu_ok = mu_in != nullptr || need_mu;
#pragma unroll
      for (int j = 0; j < 8; ++j) cnt += __popc(me.mask[j]);
    }
    // the warp's draw-list slots: inclusive scan + one atomic
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    unsigned long long b0 = 0;
    if (lane == 31 && inc) b0 = atomicAdd(n_draws, static_cast<unsigned long long>(inc));
    b0 = __shfl_sync(0xffffffffu, b0, 31);
    unsigned long long base = b0 + inc - cnt;
    if (!live) continue;
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
      uint32_t m = me.mask[j];
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        const int k = me.kbase + bit + 32 * j;
        // every reserved slot below draw_cap is written (phase B reads exactly
        // [0, min(n_draws, draw_cap))), the rest is drawn here
        if (base < draw_cap) {
          draws[base] = DeferredDraw{slot, static_cast<uint32_t>(k)};
        } else {
          if (!mu_ok) {
            mu = record_mu(me, theta_b64, phi64, K);
            mu_ok = true;
          }
          deferred_one(bv, me, mu, k, theta_b64, phi64, K, m_t, seed, t, sweep, theta_counts,
                       phi_counts, err);
        }
        ++base;
      }
    }
   }
  }
}

// 4 blocks per SM (64 registers, some spills): the pass is latency-bound on
// its record / row loads; 108 registers at 2 blocks cost 0.17 ms per
// converged sweep and 0.05 early
__global__ void __launch_bounds__(256, 4) k_deferred_draw(
    BatchView bv, const double* __restrict__ theta_b64, const double* __restrict__ phi64,
    const float* __restrict__ theta_b32, const float* __restrict__ phi32, bool fast, int K,
    double m_t, uint64_t seed, uint32_t t, uint32_t sweep, const Deferred* __restrict__ deferred,
    const double* __restrict__ rec_mu, const DeferredDraw* __restrict__ draws,
    const unsigned long long* __restrict__ n_draws, unsigned long long draw_cap,
    unsigned long long* __restrict__ theta_counts, unsigned long long* __restrict__ phi_counts,
    int* __restrict__ err) {
  const int64_t n = static_cast<int64_t>(min(*n_draws, draw_cap));
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const DeferredDraw dd = draws[i];
    // fast mode: PTRS from lambda_f where its interval decides, else the
    // record's exact mu (from the expand pass, or formed here: NaN) and the
    // reference's draw
    if (fast && deferred_try_fast(bv, deferred[dd.rec], static_cast<int>(dd.k), theta_b32, phi32, K,
                                  seed, t, sweep, theta_counts, phi_counts))
      continue;
    const Deferred rec = deferred[dd.rec];
    double mu = rec_mu[dd.rec];
    if (isnan(mu)) mu = record_mu(rec, theta_b64, phi64, K);
    deferred_one(bv, rec, mu, static_cast<int>(dd.k), theta_b64, phi64, K, m_t, seed, t, sweep,
                 theta_counts, phi_counts, err);
  }
}

// Both passes.  aux = [rec_mu: max_records f64][n_draws: u64][pad][draws: draw_cap]
// fast (the caller's choice: late in training, when most nonzeros defer a
// PTRS draw), tb32 / phi32 given and no caller mu: the expand pass forms no
// mu; the draw pass decides PTRS draws from the fast path's lambda_f
// (deferred_try_fast, thread per draw) and forms the record's exact mu only
// for the rest.
void launch_deferred(const BatchView& bv, const double* tb64, const double* phi64, const float* tb32,
                     const float* phi32, bool fast, const double* mu, int K, double m_t, uint64_t seed,
                     uint32_t t, uint32_t sweep, Deferred* rec, uint32_t* rec_count, int64_t n_items,
                     int chunk, unsigned long long* n_deferred, void* aux, int64_t max_records,
                     int64_t draw_cap, unsigned long long* tc, unsigned long long* pc, int* err,
                     cudaStream_t st) {
  fast = fast && mu == nullptr && tb32 != nullptr && phi32 != nullptr;
  double* rec_mu = static_cast<double*>(aux);
  auto* n_draws = reinterpret_cast<unsigned long long*>(rec_mu + max_records);
  auto* draws = reinterpret_cast<DeferredDraw*>(n_draws + 2);
  cudaMemsetAsync(n_draws, 0, sizeof(unsigned long long), st);
  k_deferred_expand<<<148 * 8, 256, 0, st>>>(bv, tb64, phi64, tb32, phi32, fast, mu, K, m_t, seed, t, sweep, rec,
                                             rec_count, n_items, chunk, rec_mu, draws, n_draws,
                                             static_cast<unsigned long long>(draw_cap), tc, pc, err);
  k_deferred_draw<<<148 * 16, 256, 0, st>>>(bv, tb64, phi64, tb32, phi32, fast, K, m_t, seed, t, sweep, rec, rec_mu,
                                            draws, n_draws, static_cast<unsigned long long>(draw_cap),
                                            tc, pc, err);
}

// ----------------------------------------------- sample (throughput mode)
// k_sample_thru: SURVEY 7 step 9's throughput mode -- the same SAME sampler
// (Poisson replicas of rate (theta phi / mu) m c, counts scattered as in
// parity mode) on this library's own random streams in f32, so statistically,
// not bit-for-bit, the reference's sampler.
//
//   * one Philox-4x32-10 block per four draws; the stream key is per topic
//     slice (warp-uniform: the ten round keys live in uniform registers) and
//     the lane is in the counter {lane << 8 | block, word, doc, period};
//   * inversion against u = the raw 32-bit word as a float, with the
//     thresholds scaled by 2^32 (e^-lambda 2^32 = ex2(32 - lambda log2 e)):
//     z in {0, 1, 2} branch-free;
//   * draws with z >= 3 or lambda >= 10 are rare but would serialise the warp
//     (one lane's search costs all 32): they are queued per warp in shared
//     memory and drained 32 at a time, one per lane -- the sequential search
//     resumes from z = 3 on the same thresholds; lambda >= 10 takes PTRS
//     (Hormann 1993, the reference's rng.cpp:57-86 algorithm) in f32 on
//     blocks {lane << 8 | 2 + 16 j + i} of the same stream.
constexpr int kThruQueue = 288;  // 31 left over + 8 draws x 32 lanes, + 1 spare

// PTRS conditioned on z >= 3 (rejecting accepted draws below 3 -- exact for
// the conditional law; P(z < 3) < 3e-3 at lambda >= 10)
__device__ __forceinline__ uint32_t ptrs_f32_ge3(float lam, uint32_t k0, uint32_t k1, uint32_t blk0,
                                                 uint32_t w, uint32_t d, uint32_t t) {
  const float slam = sqrtf(lam);
  const float b = 0.931f + 2.53f * slam;
  const float a = -0.059f + 0.02483f * b;
  const float inv_alpha = 1.1239f + 1.1328f / (b - 3.4f);
  const float v_r = 0.9277f - 3.6224f / (b - 2.0f);
  for (uint32_t blk = blk0;; ++blk) {
    const U4 r = philox10(U4{blk, w, d, t}, k0, k1);
    const uint32_t words[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float u = (static_cast<float>(words[2 * h] >> 8) + 0.5f) * 0x1p-24f - 0.5f;
      const float v = (static_cast<float>(words[2 * h + 1] >> 8) + 0.5f) * 0x1p-24f;
      const float us = 0.5f - fabsf(u);
      const float g = (2.0f * a / us + b) * u + lam + 0.43f;
      if (us >= 0.07f && v <= v_r) {
        if (g >= 3.0f) return static_cast<uint32_t>(g);
        continue;
      }
      if (g < 3.0f || (us < 0.013f && v > us)) continue;
      // the (rare) non-squeeze acceptance test in f64: at rates ~1e4 the
      // right-hand side is a difference of ~1e5-sized terms, where lgammaf's
      // few-ulp error would move the log acceptance ratio by ~0.1
      const double k = floor(static_cast<double>(g));
      const double dl = static_cast<double>(lam);
      if (log(static_cast<double>(v) * inv_alpha / (a / (us * us) + b)) <=
          -dl + k * log(dl) - lgamma(k + 1.0))
        return static_cast<uint32_t>(k);
    }
  }
}

template <int KPL, bool FULL, int MUSRC, bool PHI, int BLK, int MINB>
__global__ void __launch_bounds__(BLK, MINB) k_sample_thru(
    BatchView bv, const float* __restrict__ theta_b32, const float* __restrict__ phi32,
    const float* __restrict__ mu_f_in, int K, float m_t, uint64_t seed, uint32_t t,
    uint32_t sweep, int64_t chunk, unsigned long long* __restrict__ theta_counts,
    unsigned long long* __restrict__ phi_counts) {
  static_assert(KPL % 4 == 0 && KPL <= 8, "four draws per Philox block, u16 pairs");
  constexpr int kWarps = BLK / kWarp;
  // the per-warp queue of deferred draws (SoA rows: conflict-free per lane):
  // rate, u, batch row, word, topic
  __shared__ uint32_t q[kWarps][5][kThruQueue];
  const int lane = threadIdx.x & 31;
  const int wq = threadIdx.x >> 5;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * kWarps + wq;
  const int kbase = static_cast<int>(blockIdx.y) * kWarp * KPL;
  const int64_t p0 = item * chunk;
  if (p0 >= bv.nnz) return;
  const int64_t p1 = min(p0 + chunk, bv.nnz);
  uint32_t k0, k1;  // warp-uniform stream key of this topic slice
  stream_key(seed, make_tag(kThroughput, sweep, blockIdx.y), k0, k1);
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t* const qw = &q[wq][0][0];

  int qn = 0;  // warp-uniform queue length

  // drain n (<= 32) queued draws, one per lane, from the top of the queue; a
  // queued draw has u > c2, which the main path counted as z = 2, so it adds
  // z - 2 with z drawn from the tail law beyond 2
  auto drain = [&](int n) {
    __syncwarp();
    if (lane < n) {
      const int e = qn - n + lane;
      const float lam = __uint_as_float(qw[e]);
      const float u = __uint_as_float(qw[kThruQueue + e]);
      const uint32_t b = qw[2 * kThruQueue + e], w = qw[3 * kThruQueue + e];
      const uint32_t k = qw[4 * kThruQueue + e];
      uint32_t z;
      if (lam < 10.0f) {  // resume the search past z = 2 on the same thresholds
        const float e0 = ex2_approx(__fmaf_rn(lam, -1.4426950408889634f, 32.0f));
        const float t1 = e0 * lam;
        float cdf = __fmaf_rn(t1, 0.5f * lam, e0 + t1);
        float pmf = t1 * 0.5f * lam;
        z = 3;
        for (; z < 40; ++z) {
          pmf *= lam * c_tail_inv[z];
          cdf += pmf;
          if (u <= cdf) break;
        }
      } else {  // the tail beyond 2 of a large rate: PTRS given z >= 3
        const uint32_t kl = k - static_cast<uint32_t>(kbase);
        const uint32_t di = static_cast<uint32_t>(__ldg(bv.batch_docs + b) + static_cast<int32_t>(bv.doc_base));
        z = ptrs_f32_ge3(lam, k0, k1, ((kl & 31u) << 8) | (2u + 16u * (kl >> 5)), w, di, t);
      }
      const unsigned long long dz = z - 2u;  // the main path counted 2
      atomicAdd(theta_counts + static_cast<int64_t>(b) * K + k, dz);
      if (PHI)
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(phi_counts + static_cast<int64_t>(w) * K + k),
                     "l"(dz));
    }
    qn -= n;
    __syncwarp();
  };

  int cur_b = -1;
  uint32_t acc[KPL / 2];  // this lane's theta counts for the current document, u16 pairs
#pragma unroll
  for (int j = 0; j < KPL / 2; ++j) acc[j] = 0u;
  auto flush = [&](int b) {
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int k = kbase + lane + kWarp * j;
      const uint32_t z = (acc[j / 2] >> (16 * (j & 1))) & 0xffffu;
      if ((FULL || k < K) && z)
        atomicAdd(theta_counts + static_cast<int64_t>(b) * K + k, static_cast<unsigned long long>(z));
    }
  };
  for (int64_t g0 = p0; g0 < p1; g0 += kWarp) {
    const int64_t p = g0 + lane;
    int32_t b = 0, d = 0, w = 0, c = 0;
    float muf_v = 0.0f;
    if (p < p1) {
      b = static_cast<int32_t>(find_row(bv.batch_prefix, bv.B, p));
      d = __ldg(bv.batch_docs + b);
      const int64_t gi = __ldg(bv.doc_offsets + d) + (p - __ldg(bv.batch_prefix + b));
      w = __ldg(bv.word_ids + gi);
      c = __ldg(bv.counts + gi);
      if (MUSRC == 2) muf_v = __ldg(mu_f_in + p);
    }
    const int n_here = static_cast<int>(min(static_cast<int64_t>(kWarp), p1 - g0));
    for (int i = 0; i < n_here; ++i) {
      const int32_t bi = __shfl_sync(0xffffffffu, b, i);
      const uint32_t di = static_cast<uint32_t>(__shfl_sync(0xffffffffu, d, i) + static_cast<int32_t>(bv.doc_base));
      const int32_t wi = __shfl_sync(0xffffffffu, w, i);
      const int32_t ci = __shfl_sync(0xffffffffu, c, i);
      if (bi != cur_b) {
        if (cur_b >= 0) flush(cur_b);
        cur_b = bi;
#pragma unroll
        for (int j = 0; j < KPL / 2; ++j) acc[j] = 0u;
      }
      float prod[KPL];
      float mu_f = 0.0f;
      {
        const float* prow = phi32 + static_cast<int64_t>(wi) * K + kbase + lane;
        const float* trow = theta_b32 + static_cast<int64_t>(bi) * K + kbase + lane;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
          prod[j] = FULL || kbase + lane + kWarp * j < K ? __ldg(trow + kWarp * j) * __ldg(prow + kWarp * j) : 0.0f;
          mu_f += prod[j];
        }
      }
      if (MUSRC == 2) {
        mu_f = __shfl_sync(0xffffffffu, muf_v, i);
      } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mu_f += __shfl_xor_sync(0xffffffffu, mu_f, o);
      }
      const float cs = m_t * static_cast<float>(ci);
      float scale = __fdividef(cs, mu_f);
      if (!(mu_f >= 1e-30f)) {  // sampler.cpp:164: mu < 1e-30 -> uniform weights 1/K (warp-uniform)
#pragma unroll
        for (int j = 0; j < KPL; ++j) prod[j] = (FULL || kbase + lane + kWarp * j < K) ? 1.0f : 0.0f;
        scale = __fdividef(cs, static_cast<float>(K));
      }
      unsigned long long* pc = phi_counts + static_cast<int64_t>(wi) * K + kbase + lane;
#pragma unroll
      for (int g = 0; g < KPL; g += 4) {
        const U4 r = philox10(U4{(static_cast<uint32_t>(lane) << 8) | static_cast<uint32_t>(g / 4),
                                 static_cast<uint32_t>(wi), di, t},
                              k0, k1);
        const uint32_t words[4] = {r.x, r.y, r.z, r.w};
        uint32_t tm = 0;  // this lane's draws of the group with u > c2
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = g + jj;
          const float lam = prod[j] * scale;  // 0 for topics past K (prod = 0)
          const float u = __uint2float_rn(words[jj]);  // in [0, 2^32]
          const float e0 = ex2_approx(__fmaf_rn(lam, -1.4426950408889634f, 32.0f));
          const float t1 = e0 * lam;
          const float c1 = e0 + t1;
          const float c2 = __fmaf_rn(t1, 0.5f * lam, c1);
          uint32_t z = u > e0 ? 1u : 0u;
          if (u > c1) ++z;
          acc[j / 2] += z << (16 * (j & 1));
          // unpredicated within the row (z = 0 adds 0); topics past K have no cell
          if (PHI && (FULL || kbase + lane + kWarp * j < K)) red_add_u64(pc + kWarp * j, z);
          // z >= 3 (for any rate: lambda >= 10 takes PTRS given z >= 3); topics
          // past K never queue, whatever ex2.approx returns at lambda = 0
          if ((FULL || kbase + lane + kWarp * j < K) && u > c2) tm |= 1u << jj;
        }
        if (__any_sync(0xffffffffu, tm != 0u)) {  // queue this group's tails (lambda, u recomputed)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const bool tail = (tm >> jj) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, tail);
            if (bal != 0u) {
              if (tail) {
                uint32_t* const qe = qw + qn + __popc(bal & lt_mask);
                qe[0] = __float_as_uint(prod[g + jj] * scale);
                qe[kThruQueue] = __float_as_uint(__uint2float_rn(words[jj]));
                qe[2 * kThruQueue] = static_cast<uint32_t>(bi);
                qe[3 * kThruQueue] = static_cast<uint32_t>(wi);
                qe[4 * kThruQueue] = static_cast<uint32_t>(kbase + lane + kWarp * (g + jj));
              }
              qn += __popc(bal);
            }
          }
        }
      }
      while (qn >= kWarp) drain(kWarp);
    }
  }
  if (qn > 0) drain(qn);
  if (cur_b >= 0) flush(cur_b);
}

// The throughput mode's non-final inner sweep.  Only its theta counts are
// used (update_model reads the last sweep's phi counts, sampler.cpp:320-332),
// and a sum of independent Poisson draws is a Poisson draw of the summed rate:
// theta_counts[b,k] = sum_w Poisson(m c_w theta_bk phi_wk / mu_w) has exactly
// the law Poisson(Lambda_bk), Lambda_bk = theta_bk sum_w (m c_w / mu_w) phi_wk,
// independent over (b, k) (mu_w < 1e-30: weight 1/K, sampler.cpp:164, i.e.
// m c_w / K for every topic).  So no per-(nonzero, topic) draw:
//   k_theta_rates: one warp per batch document, lane = topic (KPL per lane),
//     the phi row gather and the f32 mu of k_sample_thru, rates accumulated
//     in registers and written (not added) to a B x K f32 buffer;
//   k_theta_draws: one thread per (b, k), ONE draw -- f64 inversion / PTRS
//     (poisson_from_block0) on the mode's own streams (purpose
//     kThroughputDoc, counter {0, 2^31 | k, doc, t}) -- written to
//     theta_counts.
// Deterministic (no atomics); K draws per document instead of K per nonzero.
// T = double: the expected-count mode's non-final inner sweep (the expected
// theta counts ARE these rates; f64 rows, f64 mu, K <= 256).
#ifndef SAMELDA_RATES_BLK
#define SAMELDA_RATES_BLK 64  // 128: equal; 256: 5-12% slower (doc-length tail per block)
#endif
constexpr int kRatesBlk = SAMELDA_RATES_BLK;  // documents per block = kRatesBlk / 32
#ifndef SAMELDA_RATES_NU
#define SAMELDA_RATES_NU 4  // nonzeros per step (f32): 4 -> 0.56 ms, 3 -> 0.58, 2 -> 0.60 (NYTimes shape)
#endif
#ifndef SAMELDA_RATES_MINB
#define SAMELDA_RATES_MINB 3  // x 256 threads per SM (85 registers at NU = 4)
#endif
template <typename T, int KPL, bool FULL, int MUSRC, int NU = (sizeof(T) == 4 ? SAMELDA_RATES_NU : 1)>
__global__ void __launch_bounds__(kRatesBlk, (sizeof(T) == 4 ? SAMELDA_RATES_MINB : 3) * 256 / kRatesBlk) k_theta_rates(
    BatchView bv, const T* __restrict__ theta_b32, const T* __restrict__ phi32,
    const float* __restrict__ mu_f_in, int K, T m_t, T* __restrict__ rates) {
  static_assert(MUSRC == 0 || sizeof(T) == 4, "a supplied mu is f32");
  const int lane = threadIdx.x & 31;
  const int64_t b = static_cast<int64_t>(blockIdx.x) * (kRatesBlk / kWarp) + (threadIdx.x >> 5);
  if (b >= bv.B) return;
  const int kbase = static_cast<int>(blockIdx.y) * kWarp * KPL;
  const int64_t p0 = __ldg(bv.batch_prefix + b), p1 = __ldg(bv.batch_prefix + b + 1);
  const int64_t off = __ldg(bv.doc_offsets + __ldg(bv.batch_docs + b)) - p0;
  T th[KPL], acc[KPL];
  {
    const T* trow = theta_b32 + b * K + kbase + lane;
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      th[j] = (FULL || kbase + lane + kWarp * j < K) ? __ldg(trow + kWarp * j) : T(0);
      acc[j] = T(0);
    }
  }
  T acc_u = T(0);  // the uniform-weight nonzeros' m c / K (the same for every topic)
  const T inv_k = T(1) / static_cast<T>(K);
  for (int64_t g0 = p0; g0 < p1; g0 += kWarp) {
    const int64_t p = g0 + lane;
    int32_t w = 0, c = 0;
    float muv = 0.0f;
    if (p < p1) {
      w = __ldg(bv.word_ids + off + p);
      c = __ldg(bv.counts + off + p);
      if (MUSRC == 2) muv = __ldg(mu_f_in + p);
    }
    const int n_here = static_cast<int>(min(static_cast<int64_t>(kWarp), p1 - g0));
    // NU nonzeros per step: their row loads and mu butterflies interleave (the
    // loop is latency-bound); a slot past the group re-reads slot 0's row with
    // a zero count
    for (int i = 0; i < n_here; i += NU) {
      T ph[NU][KPL], mu[NU], cs[NU];
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const bool ok = i + u < n_here;
        const int src = ok ? i + u : i;
        const int32_t wi = __shfl_sync(0xffffffffu, w, src);
        const int32_t ci = __shfl_sync(0xffffffffu, c, src);
        cs[u] = ok ? m_t * static_cast<T>(ci) : T(0);
        if (MUSRC == 2) mu[u] = __shfl_sync(0xffffffffu, muv, src);
        const T* prow = phi32 + static_cast<int64_t>(wi) * K + kbase + lane;
#pragma unroll
        for (int j = 0; j < KPL; ++j) ph[u][j] = (FULL || kbase + lane + kWarp * j < K) ? __ldg(prow + kWarp * j) : T(0);
      }
      if (MUSRC != 2) {
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          mu[u] = T(0);
#pragma unroll
          for (int j = 0; j < KPL; ++j) mu[u] = fma(th[j], ph[u][j], mu[u]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < NU; ++u) mu[u] += __shfl_xor_sync(0xffffffffu, mu[u], o);
      }
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const bool use = mu[u] >= T(1e-30);  // else uniform weights (sampler.cpp:164)
        const T sv = sizeof(T) == 4 ? static_cast<T>(__fdividef(static_cast<float>(cs[u]), static_cast<float>(mu[u])))
                                    : cs[u] / mu[u];
        const T s = use ? sv : T(0);
        acc_u += use ? T(0) : cs[u] * inv_k;
#pragma unroll
        for (int j = 0; j < KPL; ++j) acc[j] = fma(ph[u][j], s, acc[j]);
      }
    }
  }
  T* const out = rates + b * K + kbase + lane;
#pragma unroll
  for (int j = 0; j < KPL; ++j)
    if (FULL || kbase + lane + kWarp * j < K) out[kWarp * j] = fma(th[j], acc[j], acc_u);
}

__global__ void __launch_bounds__(256) k_theta_draws(BatchView bv, const float* __restrict__ rates, int K,
                                                     uint64_t seed, uint32_t t, uint32_t sweep,
                                                     unsigned long long* __restrict__ theta_counts) {
  const int64_t n = bv.B * K;
  const uint32_t tag = make_tag(kThroughputDoc, sweep, 0);
  uint32_t k0, k1;
  stream_key(seed, tag, k0, k1);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / K;
    const uint32_t k = static_cast<uint32_t>(i - b * K);
    const uint32_t dg = static_cast<uint32_t>(__ldg(bv.batch_docs + b) + static_cast<int32_t>(bv.doc_base));
    const uint32_t word = 0x80000000u | k;
    const double lam = static_cast<double>(__ldg(rates + i));
    const U4 b0 = philox10(U4{0u, word, dg, t}, k0, k1);
    theta_counts[i] = static_cast<unsigned long long>(poisson_from_block0(lam, b0, seed, t, dg, word, tag));
  }
}

template <int KPL>
int launch_fast_kpl(const BatchView& bv, const double* tb64, const float* tb32, const double* phi64,
                    const float* phi32, const double* mu, int K, double m_t, uint64_t seed,
                    uint32_t t, uint32_t sweep, unsigned long long* tc, unsigned long long* pc,
                    void* deferred, unsigned long long* n_deferred, void* aux, int64_t draw_cap,
                    float* mu_f, int* err, cudaStream_t st, const double* mu_exact,
                    cudaEvent_t mu_ready, bool fast_ptrs) {
  const int n_slices = (K + kWarp * KPL - 1) / (kWarp * KPL);
  // the deferred passes take the caller's mu, else an exact mu computed
  // concurrently on another stream (mu_exact, ready at mu_ready), else their own
  const double* mu_defer = mu ? mu : mu_exact;
  auto wait_mu = [&] {
    if (!mu && mu_exact && mu_ready) cudaStreamWaitEvent(st, mu_ready, 0);
  };
  const int64_t chunk = work_chunk(bv.nnz, n_slices);
  const int64_t items = (bv.nnz + chunk - 1) / chunk;
  const int warps = kFastBlock / kWarp;
  int launched = 0;
  cudaMemsetAsync(n_deferred, 0, sizeof(unsigned long long), st);
  const float* muf = nullptr;
  if (n_slices > 1 && mu == nullptr) {
    k_mu_f32<<<grid_for((bv.nnz + 31) / 32 * 32, 256), 256, 0, st>>>(bv, tb32, phi32, K, mu_f);
    muf = mu_f;
    ++launched;
  }
  // one chunk per warp (a persistent grid taking chunks from a counter was
  // measured 2% slower)
  const dim3 grid(static_cast<unsigned>((items + warps - 1) / warps), static_cast<unsigned>(n_slices));
  // deferred records: chunk fixed slots per (slice, grid work item), then one
  // record count per work item (deferred_buffer_bytes)
  auto* rec = static_cast<Deferred*>(deferred);
  const int64_t n_items = static_cast<int64_t>(grid.x) * warps * n_slices;
  auto* rec_count = reinterpret_cast<uint32_t*>(rec + n_items * chunk);
  const int64_t max_records = n_items * chunk;
  {
    const int musrc = mu ? 1 : (muf ? 2 : 0);
    const bool full = K % (kWarp * KPL) == 0;
    if (pc == nullptr) {
      // non-final inner sweep (theta counts only): the K = 256 period kernel
      if constexpr (KPL == 8) {
        if (full && musrc == 0 && n_slices == 1) {
          k_sample_v2<8, true, 0, kV2Minb, kDecDefault, 0, false><<<grid, kFastBlock, 0, st>>>(
              bv, tb32, phi32, mu, muf, K, m_t, seed, t, sweep, chunk, tc, pc, rec, rec_count, n_deferred);
          wait_mu();
          launch_deferred(bv, tb64, phi64, tb32, phi32, fast_ptrs, mu_defer, K, m_t, seed, t, sweep, rec, rec_count, n_items,
                          static_cast<int>(chunk), n_deferred, aux, max_records, draw_cap, tc, pc, err, st);
          return launched + 3;
        }
      }
      return -1;  // caller passes phi counts for every other shape
    }
#define SCU_V2_LAUNCH(FULLV, MS, MB, DC, ...)                                                   \
  k_sample_v2<KPL, FULLV, MS, MB, DC __VA_OPT__(,) __VA_ARGS__><<<grid, kFastBlock, 0, st>>>(    \
      bv, tb32, phi32, mu, muf, K, m_t, seed, t, sweep, chunk, tc, pc, rec, rec_count, n_deferred)
    // production: DEC 1, 4 blocks/SM.  A library built with
    // -DSAMELDA_AB_VARIANTS also carries the measured alternatives (all
    // bit-identical, all slower at K = 256): SAMELDA_DEC=0|2, SAMELDA_MINB=3,
    // SAMELDA_TAIL=1
#ifdef SAMELDA_AB_VARIANTS
    const Tuning& tu = tuning();
#define SCU_V2(FULLV, MS)                                                                        \
  do {                                                                                           \
    if constexpr (KPL == 8 && FULLV && MS == 0) {                                                \
      if (tu.minb == 3) { SCU_V2_LAUNCH(FULLV, MS, 3, 1); break; }                               \
      if (tu.dec == 0) { SCU_V2_LAUNCH(FULLV, MS, 4, 0); break; }                                \
      if (tu.dec == 2) { SCU_V2_LAUNCH(FULLV, MS, 4, 2); break; }                                \
      if (tu.tail == 1) { SCU_V2_LAUNCH(FULLV, MS, 4, 1, 1); break; }                            \
    }                                                                                            \
    SCU_V2_LAUNCH(FULLV, MS, kV2Minb, kDecDefault);                                                    \
  } while (0)
#else
#define SCU_V2(FULLV, MS) SCU_V2_LAUNCH(FULLV, MS, kV2Minb, kDecDefault)
#endif
    if (full) {
      if (musrc == 0) SCU_V2(true, 0); else if (musrc == 1) SCU_V2(true, 1); else SCU_V2(true, 2);
    } else {
      if (musrc == 0) SCU_V2(false, 0); else if (musrc == 1) SCU_V2(false, 1); else SCU_V2(false, 2);
    }
#undef SCU_V2
#undef SCU_V2_LAUNCH
  }
  wait_mu();
  launch_deferred(bv, tb64, phi64, tb32, phi32, fast_ptrs, mu_defer, K, m_t, seed, t, sweep, rec, rec_count, n_items,
                  static_cast<int>(chunk), n_deferred, aux, max_records, draw_cap, tc, pc, err, st);
  return launched + 3;
}

// k_expected: the deterministic expected-count path (z := rate,
// sampler.cpp:151-193 with poisson_sample replaced by its mean; tolerance 1e-5
// relative against the oracle) in the period kernel's layout: lane = topic,
// 8 topics per lane, warp = 128 consecutive batch nonzeros.  FUSED: mu is the
// f64 tree sum of the row's products (no separate SDDMM pass); else the
// caller's mu.  The per-nonzero scale m c / mu is formed once; a draw is one
// DMUL, a register add into the document's theta row and one coalesced f64
// RED into the word's phi row.
template <int KPL, bool FULL, bool FUSED>
__global__ void __launch_bounds__(256) k_expected(
    BatchView bv, const double* __restrict__ theta_batch, const double* __restrict__ phi_wk,
    const double* __restrict__ mu_in, int K, double m_t, int64_t chunk,
    double* __restrict__ theta_exp, double* __restrict__ phi_exp, int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int kbase = static_cast<int>(blockIdx.y) * kWarp * KPL;
  const int64_t p0 = item * chunk;
  if (p0 >= bv.nnz) return;
  const int64_t p1 = min(p0 + chunk, bv.nnz);
  const double uniform_weight = 1.0 / static_cast<double>(K);
  int64_t cur_b = -1;
  double th[KPL], acc[KPL];
#pragma unroll
  for (int j = 0; j < KPL; ++j) th[j] = acc[j] = 0.0;
  auto flush = [&](int64_t b) {
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int k = kbase + lane + kWarp * j;
      if ((FULL || k < K) && acc[j] != 0.0) atomicAdd(theta_exp + b * K + k, acc[j]);
    }
  };
  for (int64_t g0 = p0; g0 < p1; g0 += kWarp) {
    const int64_t p = g0 + lane;
    int64_t b = 0;
    int32_t w = 0, c = 0;
    double mu_v = 0.0;
    if (p < p1) {
      b = find_row(bv.batch_prefix, bv.B, p);
      const int32_t d = __ldg(bv.batch_docs + b);
      const int64_t gi = __ldg(bv.doc_offsets + d) + (p - __ldg(bv.batch_prefix + b));
      w = __ldg(bv.word_ids + gi);
      c = __ldg(bv.counts + gi);
      if (!FUSED) mu_v = __ldg(mu_in + p);
    }
    const int n_here = static_cast<int>(min(static_cast<int64_t>(kWarp), p1 - g0));
    for (int i = 0; i < n_here; ++i) {
      const int64_t bi = __shfl_sync(0xffffffffu, b, i);
      const int32_t wi = __shfl_sync(0xffffffffu, w, i);
      const int32_t ci = __shfl_sync(0xffffffffu, c, i);
      double ph[KPL];
      const double* prow = phi_wk + static_cast<int64_t>(wi) * K + kbase + lane;
#pragma unroll
      for (int j = 0; j < KPL; ++j) ph[j] = (FULL || kbase + lane + kWarp * j < K) ? __ldg(prow + kWarp * j) : 0.0;
      if (bi != cur_b) {
        if (cur_b >= 0) flush(cur_b);
        cur_b = bi;
        const double* trow = theta_batch + bi * K + kbase + lane;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
          th[j] = (FULL || kbase + lane + kWarp * j < K) ? __ldg(trow + kWarp * j) : 0.0;
          acc[j] = 0.0;
        }
      }
      double prod[KPL];
#pragma unroll
      for (int j = 0; j < KPL; ++j) prod[j] = __dmul_rn(th[j], ph[j]);
      double mu;
      if (FUSED) {
        mu = 0.0;
#pragma unroll
        for (int j = 0; j < KPL; ++j) mu = __dadd_rn(mu, prod[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mu = __dadd_rn(mu, __shfl_xor_sync(0xffffffffu, mu, o));
      } else {
        mu = __shfl_sync(0xffffffffu, mu_v, i);
      }
      const double cell_scale = __dmul_rn(m_t, static_cast<double>(ci));
      const bool degenerate = mu < 1e-30;  // sampler.cpp:164, 0/0 guard
      const double scale = degenerate ? 0.0 : __ddiv_rn(cell_scale, mu);
      const double uni = __dmul_rn(uniform_weight, cell_scale);
      double* prow_out = phi_exp + static_cast<int64_t>(wi) * K + kbase + lane;
      bool bad = false;
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        if (!FULL && kbase + lane + kWarp * j >= K) continue;
        const double rate = degenerate ? uni : __dmul_rn(prod[j], scale);
        bad = bad || !(rate >= 0.0) || isinf(rate);  // sampler.cpp:173-175
        acc[j] = __dadd_rn(acc[j], rate);
        atomicAdd(prow_out + kWarp * j, rate);
      }
      if (bad) atomicOr(err, kErrNumerical);
    }
  }
  if (cur_b >= 0) flush(cur_b);
}

template <int KPL>
int launch_sample_kpl(const BatchView& bv, const double* theta_batch, const double* phi_wk,
                      const double* mu, int K, double m_t, uint64_t seed, uint32_t t,
                      uint32_t sweep, int mode, unsigned long long* tc, unsigned long long* pc,
                      double* tf, double* pf, int* err, cudaStream_t st) {
  const int n_slices = (K + kWarp * KPL - 1) / (kWarp * KPL);
  const int64_t chunk = work_chunk(bv.nnz, n_slices);
  const int64_t items = (bv.nnz + chunk - 1) / chunk;
  const int64_t threads = items * n_slices * kWarp;
  const int block = kSampleBlock;
  if (mode == kModeExpected) {
    // mu == nullptr (period path): fused f64 tree mu, one topic slice only
    const dim3 grid(static_cast<unsigned>((items + 7) / 8), static_cast<unsigned>(n_slices));
    const bool full = K % (kWarp * KPL) == 0;
    if (mu == nullptr && n_slices == 1) {
      if (full)
        k_expected<KPL, true, true><<<grid, 256, 0, st>>>(bv, theta_batch, phi_wk, mu, K, m_t, chunk, tf, pf, err);
      else
        k_expected<KPL, false, true><<<grid, 256, 0, st>>>(bv, theta_batch, phi_wk, mu, K, m_t, chunk, tf, pf, err);
    } else if (mu != nullptr) {
      if (full)
        k_expected<KPL, true, false><<<grid, 256, 0, st>>>(bv, theta_batch, phi_wk, mu, K, m_t, chunk, tf, pf, err);
      else
        k_expected<KPL, false, false><<<grid, 256, 0, st>>>(bv, theta_batch, phi_wk, mu, K, m_t, chunk, tf, pf, err);
    } else {
      return -1;  // K > 256 needs the caller's mu
    }
  } else {
    k_sample<KPL, kModeParity><<<grid_for(threads, block), block, 0, st>>>(
        bv, theta_batch, phi_wk, mu, K, m_t, seed, t, sweep, chunk, n_slices, tc, pc, tf, pf,
        err);
  }
  return 1;
}

}  // namespace

// ------------------------------------------------------------- launchers


int launch_gather_theta(const double* theta, const int32_t* batch_docs, int64_t B, int K,
                        double* theta_batch, float* theta_batch32, cudaStream_t st) {
  if (B * K == 0) return 0;
  k_gather_theta<<<grid_for(B * K, 256), 256, 0, st>>>(theta, batch_docs, B, K, theta_batch,
                                                      theta_batch32);
  return 1;
}

int launch_sddmm(const BatchView& bv, const double* theta_batch, const double* phi_wk, int K,
                 double* mu, cudaStream_t st) {
  if (bv.nnz == 0) return 0;
  if (K % kSdChunk == 0) {  // K even: 16-byte aligned rows
    k_sddmm_staged<<<grid_for(bv.nnz, kSdWarps * 32), kSdWarps * 32, 0, st>>>(bv, theta_batch, phi_wk, K, mu);
    return 1;
  }
  k_sddmm<<<grid_for(bv.nnz, 256), 256, 0, st>>>(bv, theta_batch, phi_wk, K, mu);
  return 1;
}

int launch_sample(const BatchView& bv, const double* theta_batch, const double* phi_wk,
                  const double* mu, int K, double m_t, uint64_t seed, uint32_t t,
                  uint32_t sweep, int mode, unsigned long long* tc, unsigned long long* pc,
                  double* tf, double* pf, int* err, cudaStream_t st) {
  if (bv.nnz == 0) return 0;
  if (K <= 32)
    return launch_sample_kpl<1>(bv, theta_batch, phi_wk, mu, K, m_t, seed, t, sweep, mode, tc,
                                pc, tf, pf, err, st);
  if (K <= 64)
    return launch_sample_kpl<2>(bv, theta_batch, phi_wk, mu, K, m_t, seed, t, sweep, mode, tc,
                                pc, tf, pf, err, st);
  if (K <= 128)
    return launch_sample_kpl<4>(bv, theta_batch, phi_wk, mu, K, m_t, seed, t, sweep, mode, tc,
                                pc, tf, pf, err, st);
  return launch_sample_kpl<8>(bv, theta_batch, phi_wk, mu, K, m_t, seed, t, sweep, mode, tc, pc,
                              tf, pf, err, st);
}



// per (nonzero, 256-topic block): the record, its mu, and up to 256 flat draws
int64_t deferred_max_records(int64_t nnz, int K) {
  // k_sample_v2's fixed slots: (work items rounded to whole blocks) x chunk
  // per topic slice, chunk <= 128 and a block of 8 warps
  const int n_slices = (K + 255) / 256;
  return (nnz + 8 * 128) * n_slices;
}

int64_t deferred_buffer_bytes(int64_t nnz, int K) {
  // records, then one u32 count per work item (chunk >= 32 nonzeros)
  const int n_slices = (K + 255) / 256;
  const int64_t items = ((nnz + 8 * 128) / 32 + 1) * n_slices;
  return deferred_max_records(nnz, K) * static_cast<int64_t>(sizeof(Deferred)) +
         items * static_cast<int64_t>(sizeof(uint32_t));
}

int64_t deferred_aux_bytes(int64_t max_records, int64_t draw_cap) {
  return max_records * static_cast<int64_t>(sizeof(double)) + 16 +
         draw_cap * static_cast<int64_t>(sizeof(DeferredDraw));
}

template <bool PHI, int BLK, int MINB>
static void launch_thru(const BatchView& bv, const float* theta_b32, const float* phi32, int K,
                        float m_t, uint64_t seed, uint32_t t, uint32_t sweep,
                        unsigned long long* tc, unsigned long long* pc, const float* mu_f,
                        cudaStream_t st) {
  constexpr int KPL = 8;
  const int n_slices = (K + kWarp * KPL - 1) / (kWarp * KPL);
  const int64_t chunk = work_chunk(bv.nnz, n_slices);
  const int64_t items = (bv.nnz + chunk - 1) / chunk;
  const int warps = BLK / kWarp;
  const dim3 grid(static_cast<unsigned>((items + warps - 1) / warps), static_cast<unsigned>(n_slices));
  const bool full = K % (kWarp * KPL) == 0;
  if (mu_f != nullptr) {
    if (full)
      k_sample_thru<KPL, true, 2, PHI, BLK, MINB><<<grid, BLK, 0, st>>>(
          bv, theta_b32, phi32, mu_f, K, m_t, seed, t, sweep, chunk, tc, pc);
    else
      k_sample_thru<KPL, false, 2, PHI, BLK, MINB><<<grid, BLK, 0, st>>>(
          bv, theta_b32, phi32, mu_f, K, m_t, seed, t, sweep, chunk, tc, pc);
  } else if (full) {
    k_sample_thru<KPL, true, 0, PHI, BLK, MINB><<<grid, BLK, 0, st>>>(
        bv, theta_b32, phi32, nullptr, K, m_t, seed, t, sweep, chunk, tc, pc);
  } else {
    k_sample_thru<KPL, false, 0, PHI, BLK, MINB><<<grid, BLK, 0, st>>>(
        bv, theta_b32, phi32, nullptr, K, m_t, seed, t, sweep, chunk, tc, pc);
  }
}

// ----------------------------------------------- sample (multinomial mode)
// k_sample_multi: north_star item 3's multinomial(c m) replicas (SURVEY 7
// step 7, optional; no reference implementation).  Per batch nonzero (doc d,
// word w, count c) the c m_t replicated tokens are drawn jointly:
// n = floor(c m_t) + [u < frac(c m_t)] trials (unbiased rounding), each a
// categorical draw over the K topics with probabilities theta_dk phi_kw / mu,
// so z ~ Multinomial(n, r): E z_k = c m_t r_k as for the Poisson replicas,
// and sum_k z_k = n exactly.  On this library's own streams in f32.
//   * warp = work item of `chunk` consecutive nonzeros; lane l owns topics
//     [l KPL, (l + 1) KPL) for the cdf: f32 products, a lane-local prefix,
//     one warp scan, the cdf into the warp's shared-memory row;
//   * trials 128 at a time (one Philox-4x32-10 block per lane gives 4
//     uniforms, counter {round << 5 | lane, w, d, t}, key (seed,
//     tag(multinomial, sweep))): u * total, binary search for the first k
//     with cdf_k > u, a shared-memory histogram increment;
//   * the histogram is flushed lane = topic mod 32 (k = lane + 32 j): theta
//     counts per document in registers, phi counts with one coalesced u64
//     RED per nonzero topic.
// A row without mass (mu < 1e-30) draws uniformly over the K topics (the
// reference's fallback weight 1 / K, sampler.cpp:160-166).
template <int KPL, bool PHI>
struct MultiShape {
  static constexpr int WPB = KPL >= 16 ? 4 : 8;  // warps per block (shared rows of KP)
};

template <int KPL, bool PHI>
__global__ void __launch_bounds__(MultiShape<KPL, PHI>::WPB * 32) k_sample_multi(
    BatchView bv, const float* __restrict__ theta_b32, const float* __restrict__ phi32, int K,
    double m_t, uint64_t seed, uint32_t t, uint32_t sweep, int64_t chunk,
    unsigned long long* __restrict__ theta_counts, unsigned long long* __restrict__ phi_counts,
    int* __restrict__ err) {
  constexpr int KP = kWarp * KPL, WPB = MultiShape<KPL, PHI>::WPB;
  __shared__ float s_cdf[WPB][KP];
  __shared__ uint32_t s_hist[WPB][KP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * WPB + warp;
  const int64_t p0 = item * chunk;
  const int64_t p1 = min(p0 + chunk, bv.nnz);
  if (p0 >= p1) return;
  float* cdf = s_cdf[warp];
  uint32_t* hist = s_hist[warp];
#pragma unroll
  for (int j = 0; j < KPL; ++j) hist[lane + kWarp * j] = 0u;
  uint32_t k0, k1;
  stream_key(seed, make_tag(kMultinomial, sweep, 0), k0, k1);
  int cur_b = -1;
  uint32_t acc[KPL];
#pragma unroll
  for (int j = 0; j < KPL; ++j) acc[j] = 0u;
  auto flush = [&](int b) {
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int k = lane + kWarp * j;
      if (k < K && acc[j]) atomicAdd(theta_counts + static_cast<int64_t>(b) * K + k,
                                     static_cast<unsigned long long>(acc[j]));
      acc[j] = 0u;
    }
  };
  for (int64_t g0 = p0; g0 < p1; g0 += kWarp) {
    const int64_t p = g0 + lane;
    int32_t b = 0, d = 0, w = 0, c = 0;
    if (p < p1) {
      b = static_cast<int32_t>(find_row(bv.batch_prefix, bv.B, p));
      d = __ldg(bv.batch_docs + b);
      const int64_t gi = __ldg(bv.doc_offsets + d) + (p - __ldg(bv.batch_prefix + b));
      w = __ldg(bv.word_ids + gi);
      c = __ldg(bv.counts + gi);
    }
    const int n_here = static_cast<int>(min(static_cast<int64_t>(kWarp), p1 - g0));
    for (int i = 0; i < n_here; ++i) {
      const int32_t bi = __shfl_sync(0xffffffffu, b, i);
      const uint32_t di = static_cast<uint32_t>(__shfl_sync(0xffffffffu, d, i) + static_cast<int32_t>(bv.doc_base));
      const int32_t wi = __shfl_sync(0xffffffffu, w, i);
      const int32_t ci = __shfl_sync(0xffffffffu, c, i);
      if (bi != cur_b) {
        if (cur_b >= 0) flush(cur_b);
        cur_b = bi;
      }
      // cdf over the lane's contiguous topics, then the warp scan
      const float* trow = theta_b32 + static_cast<int64_t>(bi) * K;
      const float* prow = phi32 + static_cast<int64_t>(wi) * K;
      float pr[KPL];
      float run = 0.0f;
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = lane * KPL + j;
        pr[j] = k < K ? __fmul_rn(__ldg(trow + k), __ldg(prow + k)) : 0.0f;
        run = __fadd_rn(run, pr[j]);
      }
      float incl = run;
#pragma unroll
      for (int o = 1; o < kWarp; o <<= 1) {
        const float v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = __fadd_rn(incl, v);
      }
      float total = __shfl_sync(0xffffffffu, incl, kWarp - 1);
      if (!isfinite(total)) {
        if (lane == 0) atomicOr(err, kErrNumerical);
        continue;
      }
      const bool uniform = !(total >= 1e-30f);
      float base = __fsub_rn(incl, run);
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = lane * KPL + j;
        base = uniform ? static_cast<float>(min(k + 1, K)) : __fadd_rn(base, pr[j]);
        cdf[k] = base;
      }
      if (uniform) total = static_cast<float>(K);
      __syncwarp();
      // n = floor(c m_t) + [u < frac(c m_t)]
      const double cm = m_t * static_cast<double>(ci);
      const double fl = floor(cm);
      const U4 fr = philox10(U4{0x80000000u, static_cast<uint32_t>(wi), di, t}, k0, k1);
      const int64_t n = static_cast<int64_t>(fl) + (u64_to_uniform(join64(fr.x, fr.y)) < cm - fl ? 1 : 0);
      for (int64_t r0 = 0; r0 < n; r0 += 4 * kWarp) {
        const U4 y = philox10(U4{static_cast<uint32_t>(r0 >> 7) << 5 | static_cast<uint32_t>(lane),
                                 static_cast<uint32_t>(wi), di, t}, k0, k1);
        const uint32_t ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (r0 + q * kWarp + lane >= n) continue;
          float u = __fmul_rn(__fmul_rn(static_cast<float>(ys[q] >> 8), 0x1p-24f), total);
          if (!(u < total)) u = 0.0f;  // f32 rounding at the top end
          int lo = 0;  // first k with cdf_k > u (the last cdf entry >= total > u)
#pragma unroll
          for (int step = KP >> 1; step > 0; step >>= 1)
            if (cdf[lo + step - 1] <= u) lo += step;
          atomicAdd(hist + min(lo, K - 1), 1u);
        }
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = lane + kWarp * j;
        const uint32_t z = hist[k];
        hist[k] = 0u;
        acc[j] += z;
        if (PHI && z && k < K)
          red_add_u64(phi_counts + static_cast<int64_t>(wi) * K + k, static_cast<unsigned long long>(z));
      }
      __syncwarp();
    }
  }
  if (cur_b >= 0) flush(cur_b);
}

template <int KPL>
void launch_multi_kpl(const BatchView& bv, const float* tb32, const float* phi32, int K, double m_t,
                      uint64_t seed, uint32_t t, uint32_t sweep, unsigned long long* tc,
                      unsigned long long* pc, int* err, cudaStream_t st) {
  constexpr int WPB = MultiShape<KPL, true>::WPB;
  const int64_t chunk = work_chunk(bv.nnz, 1);
  const int64_t items = (bv.nnz + chunk - 1) / chunk;
  const unsigned grid = static_cast<unsigned>((items + WPB - 1) / WPB);
  if (pc) k_sample_multi<KPL, true><<<grid, WPB * 32, 0, st>>>(bv, tb32, phi32, K, m_t, seed, t, sweep, chunk, tc, pc, err);
  else k_sample_multi<KPL, false><<<grid, WPB * 32, 0, st>>>(bv, tb32, phi32, K, m_t, seed, t, sweep, chunk, tc, pc, err);
}

int launch_sample_multinomial(const BatchView& bv, const float* theta_b32, const float* phi32, int K,
                              double m_t, uint64_t seed, uint32_t t, uint32_t sweep,
                              unsigned long long* tc, unsigned long long* pc, int* err,
                              cudaStream_t st) {
  if (bv.nnz == 0) return 0;
  if (K <= 32) launch_multi_kpl<1>(bv, theta_b32, phi32, K, m_t, seed, t, sweep, tc, pc, err, st);
  else if (K <= 64) launch_multi_kpl<2>(bv, theta_b32, phi32, K, m_t, seed, t, sweep, tc, pc, err, st);
  else if (K <= 128) launch_multi_kpl<4>(bv, theta_b32, phi32, K, m_t, seed, t, sweep, tc, pc, err, st);
  else if (K <= 256) launch_multi_kpl<8>(bv, theta_b32, phi32, K, m_t, seed, t, sweep, tc, pc, err, st);
  else if (K <= 512) launch_multi_kpl<16>(bv, theta_b32, phi32, K, m_t, seed, t, sweep, tc, pc, err, st);
  else if (K <= 1024) launch_multi_kpl<32>(bv, theta_b32, phi32, K, m_t, seed, t, sweep, tc, pc, err, st);
  else return -1;
  return 1;
}

int launch_expected_theta(const BatchView& bv, const double* theta_b, const double* phi_wk, int K,
                          double m_t, double* tf, cudaStream_t st) {
  if (K > kWarp * 8) return -1;
  if (bv.B == 0) return 0;
  const dim3 grid(static_cast<unsigned>((bv.B + kRatesBlk / kWarp - 1) / (kRatesBlk / kWarp)), 1u);
  if (K == kWarp * 8) k_theta_rates<double, 8, true, 0><<<grid, kRatesBlk, 0, st>>>(bv, theta_b, phi_wk, nullptr, K, m_t, tf);
  else k_theta_rates<double, 8, false, 0><<<grid, kRatesBlk, 0, st>>>(bv, theta_b, phi_wk, nullptr, K, m_t, tf);
  return 1;
}

int launch_sample_throughput(const BatchView& bv, const float* theta_b32, const float* phi32, int K,
                             double m_t, uint64_t seed, uint32_t t, uint32_t sweep,
                             unsigned long long* tc, unsigned long long* pc, float* mu_f,
                             float* rate_scratch, cudaStream_t st) {
  if (bv.nnz == 0) return 0;
  int launched = 0;
  const float* mu = nullptr;
  if (K > kWarp * 8) {  // more than one topic slice: mu from its own pass
    k_mu_f32<<<grid_for((bv.nnz + 31) / 32 * 32, 256), 256, 0, st>>>(bv, theta_b32, phi32, K, mu_f);
    mu = mu_f;
    ++launched;
  }
  const float mf = static_cast<float>(m_t);
  // 128-thread blocks at <= 72 registers: 28 resident warps per SM (measured
  // 3% faster than 256 x 80 registers; 64 registers spills)
  if (pc != nullptr) {
    launch_thru<true, 128, 7>(bv, theta_b32, phi32, K, mf, seed, t, sweep, tc, pc, mu, st);
    return launched + 1;
  }
  // a non-final inner sweep: theta counts only, one draw per (document, topic)
  constexpr int KPL = 8;
  const dim3 grid(static_cast<unsigned>((bv.B + kRatesBlk / kWarp - 1) / (kRatesBlk / kWarp)),
                  static_cast<unsigned>((K + kWarp * KPL - 1) / (kWarp * KPL)));
  const bool full = K % (kWarp * KPL) == 0;
  if (mu != nullptr) {
    if (full) k_theta_rates<float, KPL, true, 2><<<grid, kRatesBlk, 0, st>>>(bv, theta_b32, phi32, mu, K, mf, rate_scratch);
    else k_theta_rates<float, KPL, false, 2><<<grid, kRatesBlk, 0, st>>>(bv, theta_b32, phi32, mu, K, mf, rate_scratch);
  } else if (full) {
    k_theta_rates<float, KPL, true, 0><<<grid, kRatesBlk, 0, st>>>(bv, theta_b32, phi32, nullptr, K, mf, rate_scratch);
  } else {
    k_theta_rates<float, KPL, false, 0><<<grid, kRatesBlk, 0, st>>>(bv, theta_b32, phi32, nullptr, K, mf, rate_scratch);
  }
  k_theta_draws<<<grid_for(bv.B * K, 256), 256, 0, st>>>(bv, rate_scratch, K, seed, t, sweep, tc);
  launched += 2;
  return launched + 1;
}

int launch_sample_fast(const BatchView& bv, const double* theta_b64, const float* theta_b32,
                       const double* phi64, const float* phi32, const double* mu, int K,
                       double m_t, uint64_t seed, uint32_t t, uint32_t sweep,
                       unsigned long long* tc, unsigned long long* pc, void* deferred,
                       unsigned long long* n_deferred, void* aux, int64_t draw_cap, float* mu_f,
                       int* err, cudaStream_t st, const double* mu_exact, cudaEvent_t mu_ready,
                       bool fast_ptrs) {
  if (bv.nnz == 0) return 0;
  // lane = topic, 8 topics per lane (k_sample_v2); K > 256 in topic slices of
  // 256 with the full mu from a k_mu_f32 pre-pass.  SAMELDA_SAMPLER=x runs
  // the all-f64 exact kernel instead when the caller supplies mu (per-call
  // sample_counts): a device-side cross-check of the fast-exact path.
  if (tuning().sampler_exact && mu != nullptr && pc != nullptr)
    return launch_sample(bv, theta_b64, phi64, mu, K, m_t, seed, t, sweep, kModeParity, tc, pc,
                         nullptr, nullptr, err, st);
  if (K <= 32)
    return launch_fast_kpl<1>(bv, theta_b64, theta_b32, phi64, phi32, mu, K, m_t, seed, t, sweep, tc, pc,
                              deferred, n_deferred, aux, draw_cap, mu_f, err, st, mu_exact, mu_ready, fast_ptrs);
  if (K <= 64)
    return launch_fast_kpl<2>(bv, theta_b64, theta_b32, phi64, phi32, mu, K, m_t, seed, t, sweep, tc, pc,
                              deferred, n_deferred, aux, draw_cap, mu_f, err, st, mu_exact, mu_ready, fast_ptrs);
  if (K <= 128)
    return launch_fast_kpl<4>(bv, theta_b64, theta_b32, phi64, phi32, mu, K, m_t, seed, t, sweep, tc, pc,
                              deferred, n_deferred, aux, draw_cap, mu_f, err, st, mu_exact, mu_ready, fast_ptrs);
  return launch_fast_kpl<8>(bv, theta_b64, theta_b32, phi64, phi32, mu, K, m_t, seed, t, sweep, tc, pc,
                            deferred, n_deferred, aux, draw_cap, mu_f, err, st, mu_exact, mu_ready, fast_ptrs);
}

// glibc lgamma(k + 1) for the PTRS acceptance test (poisson.cuh), per device
namespace {
struct LgammaTab {
  double v[kLgammaTab];
  LgammaTab() {
    for (int k = 0; k < kLgammaTab; ++k) v[k] = std::lgamma(static_cast<double>(k) + 1.0);
  }
};
}  // namespace

int init_lgamma_table() {
  static const LgammaTab tab;  // filled once, thread-safe (static initialisation)
  const int one = 1;
  if (cudaMemcpyToSymbol(g_lgamma_int, tab.v, sizeof(tab.v)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_lgamma_ready, &one, sizeof(one)) != cudaSuccess)
    return 1;
  return 0;
}

}  // namespace scu

#ifdef SAMELDA_DEFER_STATS
extern "C" int samelda_debug_defer_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, scu::g_defer_stats, sizeof(scu::g_defer_stats)) != cudaSuccess) return 4;
  if (reset) {
    static const unsigned long long zero[96] = {};
    cudaMemcpyToSymbol(scu::g_defer_stats, zero, sizeof(zero));
  }
  return 0;
}
#endif

