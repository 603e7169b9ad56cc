// kernels.cu -- sm_100a kernels for the SAME factored Gibbs sampler (parity and
// expected-count modes).  Compiled with -fmad=false: every f64 expression
// rounds like the reference's x86-64 (no FMA) build.  Each kernel cites the
// reference loop it replaces.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "philox.cuh"
#include "poisson.cuh"

namespace scu {

namespace {

constexpr int kWarp = 32;

__device__ __forceinline__ int64_t find_row(const int64_t* __restrict__ prefix, int64_t B,
                                            int64_t p) {
  // largest b in [0, B) with prefix[b] <= p; prefix[B] > p by construction
  int64_t lo = 0, hi = B;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(prefix + mid) <= p) lo = mid; else hi = mid;
  }
  return lo;
}

inline unsigned grid_for(int64_t threads, int block) {
  return static_cast<unsigned>((threads + block - 1) / block);
}

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
// The fast path evaluates rate, exp and the recurrence in f32 with a
// rigorous relative error bound r(lambda, k) and decides each comparison only
// when u lies outside [cdf - m, cdf + m]; otherwise (probability ~1e-5 per
// draw), or for lambda >= 9.5 (PTRS territory), non-finite / negative /
// denormal inputs, or k > 40, the lane recomputes that draw exactly like
// k_sample: sequential f64 mu, __ddiv_rn rate, full Philox block, exact
// inversion or PTRS.  Error budget (u32 = 2^-24 unit roundoff):
//   lambda_f: theta, phi rounded to f32 (2u), product (u), mu by tree sum of
//     positive terms (<= 16u), cs/mu (3u), lambda (u)  -> |dl| <= 1.5e-6 lambda
//   exp:  __expf max error (2 + 1.2 lambda) ulp       -> <= (1.2e-7 + 7e-8 lambda)
//   step k: pmf *= lambda/k (+ dl + 3u), cdf += pmf (+u)
//   __fdividef steps add <= 2 ulp each
//   r = 4e-6 + 4e-6 lambda + 6e-6 k  (>= 2x the sum above);  u from the top
//   23 bits of the high word: u - u_f in [0, 2^-23) -> m = cdf * r + 2.5e-7.
// The mu used is the caller's mu array when given (per-call sample_counts),
// else the warp computes it (f32 tree for the fast path, exact f64
// sequential sum on fallback, cached per lane and nonzero).

constexpr int kFastBlock = 256;

struct Philox1 {
  // round-1 specialisation for counter {0, w, d, t}: M0 * 0 = 0, so the
  // only per-draw work in round 1 is one xor; M1 * d is per nonzero
  uint32_t hw;  // hi(M1 * d) ^ w
  uint32_t lo;  // lo(M1 * d)
};

__device__ __forceinline__ uint32_t philox_y(const Philox1 r1, uint32_t k0, uint32_t k1,
                                             uint32_t p2lo, uint32_t p2hi) {
  // round 1 -> c = {hw ^ k0, lo, t ^ k1, 0}; round 2 with M1 * (t ^ k1) = p2
  uint32_t c0 = r1.hw ^ k0;
  k0 += kPhiloxW0;
  k1 += kPhiloxW1;
  uint32_t lo0, hi0;
  mulhilo(kPhiloxM0, c0, lo0, hi0);
  uint32_t x0 = p2hi ^ r1.lo ^ k0, x1 = p2lo, x2 = hi0 ^ k1, x3 = lo0;
#pragma unroll
  for (int r = 2; r < 9; ++r) {
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
    uint32_t a0, b0, a1, b1;
    mulhilo(kPhiloxM0, x0, a0, b0);
    mulhilo(kPhiloxM1, x2, a1, b1);
    const uint32_t n0 = b1 ^ x1 ^ k0, n2 = b0 ^ x3 ^ k1;
    x0 = n0;
    x1 = a1;
    x2 = n2;
    x3 = a0;
  }
  // round 10: output word y = lo(M1 * x2)
  return kPhiloxM1 * x2;
}

// Deferred exact draws: one record per (nonzero, topic slice) that has at
// least one draw the fast path could not decide (PTRS range lambda >= 9.5,
// an ambiguous comparison, z > 40, or non-finite / tiny inputs).
struct Deferred {
  int64_t p;          // batch nonzero index
  int32_t b, w, c;    // batch row, word id, token count
  int32_t kbase;      // first topic of the slice
  uint32_t mask[8];   // bit lane of mask[j]: topic kbase + lane + 32 j
};

template <int KPL, bool FULL>
__global__ void __launch_bounds__(kFastBlock, 2) k_sample_fast(
    BatchView bv, const float* __restrict__ theta_b32, const float* __restrict__ phi32,
    const double* __restrict__ mu_in, int K, double m_t, uint64_t seed, uint32_t t,
    uint32_t sweep, int64_t chunk, int n_slices, unsigned long long* __restrict__ theta_counts,
    unsigned long long* __restrict__ phi_counts, Deferred* __restrict__ deferred,
    unsigned long long* __restrict__ n_deferred) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t item = gw / n_slices;
  const int slice = static_cast<int>(gw - item * n_slices);
  const int64_t p0 = item * chunk;
  if (p0 >= bv.nnz) return;
  const int64_t p1 = min(p0 + chunk, bv.nnz);
  const int kbase = slice * kWarp * KPL;
  const int have_mu = mu_in != nullptr;

  // per-topic stream keys, fixed for the whole item
  uint32_t key0[KPL], key1[KPL];
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const uint32_t k = static_cast<uint32_t>(kbase + lane + kWarp * j);
    stream_key(seed, make_tag(kPoissonCounts, sweep, k), key0[j], key1[j]);
  }

  int64_t cur_b = -1;
  float th[KPL];
  uint32_t acc[KPL];
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    th[j] = 0.0f;
    acc[j] = 0u;
  }

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
      if (have_mu) mu_v = __ldg(mu_in + p);
    }
    const int n_here = static_cast<int>(min(static_cast<int64_t>(kWarp), p1 - g0));
    // software pipeline: phi slice of nonzero i+1 is in flight while i draws
    float ph_next[KPL];
    {
      const int32_t w0 = __shfl_sync(0xffffffffu, w, 0);
      const float* prow = phi32 + static_cast<int64_t>(w0) * K;
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = kbase + lane + kWarp * j;
        ph_next[j] = (FULL || k < K) ? __ldg(prow + k) : 0.0f;
      }
    }
    for (int i = 0; i < n_here; ++i) {
      const int64_t bi = __shfl_sync(0xffffffffu, b, i);
      const int32_t dl = __shfl_sync(0xffffffffu, d, i);
      const uint32_t di = static_cast<uint32_t>(dl + bv.doc_base);
      const int32_t wi = __shfl_sync(0xffffffffu, w, i);
      const int32_t ci = __shfl_sync(0xffffffffu, c, i);
      const double mui = __shfl_sync(0xffffffffu, mu_v, i);
      float ph[KPL];
#pragma unroll
      for (int j = 0; j < KPL; ++j) ph[j] = ph_next[j];
      {
        const int32_t wn = __shfl_sync(0xffffffffu, w, (i + 1) & 31);
        if (i + 1 < n_here) {
          const float* prow = phi32 + static_cast<int64_t>(wn) * K;
#pragma unroll
          for (int j = 0; j < KPL; ++j) {
            const int k = kbase + lane + kWarp * j;
            ph_next[j] = (FULL || k < K) ? __ldg(prow + k) : 0.0f;
          }
        }
      }
      if (bi != cur_b) {
        if (cur_b >= 0) {
#pragma unroll
          for (int j = 0; j < KPL; ++j) {
            const int k = kbase + lane + kWarp * j;
            if ((FULL || k < K) && acc[j])
              atomicAdd(theta_counts + cur_b * K + k, static_cast<unsigned long long>(acc[j]));
          }
        }
        cur_b = bi;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
          const int k = kbase + lane + kWarp * j;
          th[j] = (FULL || k < K) ? __ldg(theta_b32 + bi * K + k) : 0.0f;
          acc[j] = 0u;
        }
      }
      float prod[KPL];
      float part = 0.0f;
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        prod[j] = __fmul_rn(th[j], ph[j]);
        part = __fadd_rn(part, prod[j]);
      }
      float mu_f;
      if (have_mu) {
        mu_f = __double2float_rn(mui);
      } else {
        mu_f = part;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mu_f = __fadd_rn(mu_f, __shfl_xor_sync(0xffffffffu, mu_f, o));
        if (n_slices > 1) mu_f = 0.0f;  // partial sums only: defer the nonzero
      }
      const bool nz_exact = !(mu_f >= 1e-20f) || isinf(mu_f);
      const float scale = __fdividef(__double2float_rn(__dmul_rn(m_t, static_cast<double>(ci))), mu_f);
      uint32_t m1lo, m1hi;
      mulhilo(kPhiloxM1, di, m1lo, m1hi);
      const Philox1 r1{m1hi ^ static_cast<uint32_t>(wi), m1lo};
      // phase 1: every topic's uniform (independent Philox chains -> ILP)
      uint32_t y[KPL];
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        uint32_t p2lo, p2hi;
        mulhilo(kPhiloxM1, t ^ key1[j], p2lo, p2hi);
        y[j] = philox_y(r1, key0[j], key1[j], p2lo, p2hi);
      }
      // phase 2: decisions; undecidable draws are deferred
      uint32_t defer_bits = 0;
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = kbase + lane + kWarp * j;
        const float lam = __fmul_rn(prod[j], scale);
        int z = 0;
        bool exact = nz_exact || !(prod[j] >= 1e-30f) || !(lam < 9.5f);
        if (!FULL && k >= K) exact = false;
        else if (!exact) {
          // u in [u_f, u_f + 2^-23): top 23 bits of the high word, no I2F
          const float u = __fsub_rn(__int_as_float(0x3f800000 | (y[j] >> 9)), 1.0f);
          float pmf = __expf(-lam);
          float cdf = pmf;
          float r = __fadd_rn(4e-6f, __fmul_rn(4e-6f, lam));
          for (;;) {
            const float mrg = __fadd_rn(__fmul_rn(cdf, r), 2.5e-7f);
            if (u <= __fsub_rn(cdf, mrg)) break;
            if (!(u > __fadd_rn(cdf, mrg)) || z >= 40) {
              exact = true;
              z = 0;
              break;
            }
            ++z;
            pmf = __fmul_rn(pmf, __fdividef(lam, static_cast<float>(z)));
            cdf = __fadd_rn(cdf, pmf);
            r = __fadd_rn(r, 6e-6f);
          }
          if (z != 0) {
            acc[j] += static_cast<uint32_t>(z);
            atomicAdd(phi_counts + static_cast<int64_t>(wi) * K + k, static_cast<unsigned long long>(z));
          }
        }
        if (exact) defer_bits |= 1u << j;
      }
      if (__any_sync(0xffffffffu, defer_bits != 0)) {
        uint32_t masks[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) masks[j] = j < KPL ? __ballot_sync(0xffffffffu, (defer_bits >> j) & 1u) : 0u;
        if (lane == 0) {
          const unsigned long long slot = atomicAdd(n_deferred, 1ull);
          Deferred rec;
          rec.p = g0 + i;
          rec.b = static_cast<int32_t>(bi);
          rec.w = wi;
          rec.c = ci;
          rec.kbase = kbase;
#pragma unroll
          for (int j = 0; j < 8; ++j) rec.mask[j] = masks[j];
          deferred[slot] = rec;
        }
      }
    }
  }
  if (cur_b >= 0) {
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int k = kbase + lane + kWarp * j;
      if ((FULL || k < K) && acc[j])
        atomicAdd(theta_counts + cur_b * K + k, static_cast<unsigned long long>(acc[j]));
    }
  }
}

// One warp per deferred record: exact mu (sequential k order, coalesced row
// loads, warp-broadcast add chain) unless the caller supplied mu, then each
// flagged draw exactly as k_sample: __ddiv_rn rate, full Philox block, exact
// inversion or PTRS (rng.cpp:39-86).
__global__ void __launch_bounds__(256) k_sample_deferred(
    BatchView bv, const double* __restrict__ theta_b64, const double* __restrict__ phi64,
    const double* __restrict__ mu_in, int K, double m_t, uint64_t seed, uint32_t t,
    uint32_t sweep, const Deferred* __restrict__ deferred,
    const unsigned long long* __restrict__ n_deferred,
    unsigned long long* __restrict__ theta_counts, unsigned long long* __restrict__ phi_counts,
    int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t n = static_cast<int64_t>(*n_deferred);
  const double uniform_weight = 1.0 / static_cast<double>(K);
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < n;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const Deferred rec = deferred[r];
    const double* th = theta_b64 + static_cast<int64_t>(rec.b) * K;
    const double* ph = phi64 + static_cast<int64_t>(rec.w) * K;
    double mu;
    if (mu_in) {
      mu = mu_in[rec.p];
    } else {
      mu = 0.0;
      for (int k0 = 0; k0 < K; k0 += 32) {
        const int k = k0 + lane;
        const double prod = k < K ? __dmul_rn(__ldg(th + k), __ldg(ph + k)) : 0.0;
        const int m = min(32, K - k0);
        for (int l = 0; l < m; ++l) mu = __dadd_rn(mu, __shfl_sync(0xffffffffu, prod, l));
      }
    }
    const uint32_t d = static_cast<uint32_t>(__ldg(bv.batch_docs + rec.b) + bv.doc_base);
    const double cs = __dmul_rn(m_t, static_cast<double>(rec.c));
    const bool degenerate = mu < 1e-30;
    for (int j = 0; j < 8; ++j) {
      if (!((rec.mask[j] >> lane) & 1u)) continue;
      const int k = rec.kbase + lane + 32 * j;
      const double weight = degenerate ? uniform_weight : __ddiv_rn(__dmul_rn(__ldg(th + k), __ldg(ph + k)), mu);
      const double rate = __dmul_rn(weight, cs);
      if (!(rate >= 0.0) || isinf(rate)) {
        atomicOr(err, kErrNumerical);
        continue;
      }
      if (rate == 0.0) continue;
      const uint32_t tag = make_tag(kPoissonCounts, sweep, static_cast<uint32_t>(k));
      uint32_t k0, k1;
      stream_key(seed, tag, k0, k1);
      const U4 blk = philox10(U4{0u, static_cast<uint32_t>(rec.w), d, t}, k0, k1);
      long long z;
      if (rate < 10.0) {
        z = poisson_inversion(rate, u64_to_uniform(join64(blk.x, blk.y)));
      } else {
        Stream s;
        s.init_with_block0(seed, t, d, static_cast<uint32_t>(rec.w), tag, blk, 0);
        z = poisson_ptrs(rate, s);
      }
      if (z != 0) {
        atomicAdd(theta_counts + static_cast<int64_t>(rec.b) * K + k, static_cast<unsigned long long>(z));
        atomicAdd(phi_counts + static_cast<int64_t>(rec.w) * K + k, static_cast<unsigned long long>(z));
      }
    }
  }
}

template <int KPL>
int launch_fast_kpl(const BatchView& bv, const double* tb64, const float* tb32, const double* phi64,
                    const float* phi32, const double* mu, int K, double m_t, uint64_t seed,
                    uint32_t t, uint32_t sweep, unsigned long long* tc, unsigned long long* pc,
                    void* deferred, unsigned long long* n_deferred, int* err, cudaStream_t st) {
  const int n_slices = (K + kWarp * KPL - 1) / (kWarp * KPL);
  const int64_t chunk = 128;
  const int64_t items = (bv.nnz + chunk - 1) / chunk;
  const int64_t threads = items * n_slices * kWarp;
  cudaMemsetAsync(n_deferred, 0, sizeof(unsigned long long), st);
  auto* rec = static_cast<Deferred*>(deferred);
  if (K % (kWarp * KPL) == 0)
    k_sample_fast<KPL, true><<<grid_for(threads, kFastBlock), kFastBlock, 0, st>>>(
        bv, tb32, phi32, mu, K, m_t, seed, t, sweep, chunk, n_slices, tc, pc, rec, n_deferred);
  else
    k_sample_fast<KPL, false><<<grid_for(threads, kFastBlock), kFastBlock, 0, st>>>(
        bv, tb32, phi32, mu, K, m_t, seed, t, sweep, chunk, n_slices, tc, pc, rec, n_deferred);
  k_sample_deferred<<<148 * 8, 256, 0, st>>>(bv, tb64, phi64, mu, K, m_t, seed, t, sweep, rec,
                                             n_deferred, tc, pc, err);
  return 2;
}

// ------------------------------------------------------------------- M-step

__global__ void k_theta_from_counts(const unsigned long long* __restrict__ cu,
                                    const double* __restrict__ cf, int64_t n, double m_t,
                                    double alpha, double* __restrict__ out,
                                    float* __restrict__ out32) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double hat = cu ? __ddiv_rn(static_cast<double>(static_cast<long long>(cu[i])), m_t)
                        : __ddiv_rn(cf[i], m_t);
  const double v = __dadd_rn(hat, alpha);
  out[i] = v;
  if (out32) out32[i] = __double2float_rn(v);
}

__global__ void k_theta_persist(const unsigned long long* __restrict__ cu,
                                const double* __restrict__ cf,
                                const int32_t* __restrict__ batch_docs, int64_t B, int K,
                                double m_t, double alpha, double* __restrict__ theta) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= B * K) return;
  const int64_t b = i / K;
  const int k = static_cast<int>(i - b * K);
  const double hat = cu ? __ddiv_rn(static_cast<double>(static_cast<long long>(cu[i])), m_t)
                        : __ddiv_rn(cf[i], m_t);
  theta[static_cast<int64_t>(batch_docs[b]) * K + k] = __dadd_rn(hat, alpha);
}

// total[k] = sum over w, in order, of x[w,k] (sampler.cpp:214-218): one warp
// per topic.  The 32 lanes fetch and convert 32 consecutive words in
// parallel (x = count/m_t + beta, the reference's `value`), then every lane
// runs the same sequential add chain over the 32 broadcast values, so the
// summation order is exactly the reference's and the total is warp-uniform.
template <int SRC>  // 0: u64 counts, 1: f64 expected counts, 2: plain f64 values
__global__ void __launch_bounds__(256) k_col_totals(const unsigned long long* __restrict__ cu,
                                                    const double* __restrict__ cf, int64_t W,
                                                    int K, double m_t, double beta,
                                                    double* __restrict__ totals,
                                                    int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= K) return;
  double total = 0.0;
  for (int64_t w0 = 0; w0 < W; w0 += 32) {
    const int64_t w = w0 + lane;
    double v = 0.0;
    if (w < W) {
      const int64_t i = w * K + k;
      if (SRC == 0) v = __dadd_rn(__ddiv_rn(static_cast<double>(static_cast<long long>(cu[i])), m_t), beta);
      else if (SRC == 1) v = __dadd_rn(__ddiv_rn(cf[i], m_t), beta);
      else v = cf[i];
    }
    const int n = static_cast<int>(min(static_cast<int64_t>(32), W - w0));
    for (int j = 0; j < n; ++j) total = __dadd_rn(total, __shfl_sync(0xffffffffu, v, j));
  }
  if (lane == 0) {
    totals[k] = total;
    if (err && (!(total > 0.0) || isinf(total))) atomicOr(err, kErrNumerical);
  }
}

// phi = (1 - rho) * phi + rho * cand / total, cand = count/m_t + beta
// (sampler.cpp:209-226); also refreshes the f32 copy the sampler reads.
__global__ void k_phi_blend(const unsigned long long* __restrict__ cu,
                            const double* __restrict__ cf, const double* __restrict__ totals,
                            int64_t n, int K, double m_t, double beta, double one_minus_rho,
                            double rho, double* __restrict__ phi_wk, float* __restrict__ phi32) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int k = static_cast<int>(i % K);
  const double hat = cu ? __ddiv_rn(static_cast<double>(static_cast<long long>(cu[i])), m_t)
                        : __ddiv_rn(cf[i], m_t);
  const double cand = __dadd_rn(hat, beta);
  const double v = __dadd_rn(__dmul_rn(one_minus_rho, phi_wk[i]),
                             __ddiv_rn(__dmul_rn(rho, cand), totals[k]));
  phi_wk[i] = v;
  if (phi32) phi32[i] = __double2float_rn(v);
}

__global__ void k_to_f32(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = __double2float_rn(x[i]);
}

// ---------------------------------------------------------------- init phi
// Entry (k, w) of the reference's row-major K x W walk is uniform number
// i = k*W + w of one stream keyed (0,0,0,phi_init): block i/2, words
// 2(i%2), 2(i%2)+1.  Written into the word-major layout.
__global__ void k_phi_init_values(double* __restrict__ phi_wk, int64_t W, int K,
                                  double init_noise, uint32_t k0, uint32_t k1) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= W * K) return;
  const int64_t w = idx / K;
  const int k = static_cast<int>(idx - w * K);
  const uint64_t i = static_cast<uint64_t>(k) * static_cast<uint64_t>(W) + w;
  const U4 r = philox10(U4{static_cast<uint32_t>(i >> 1), 0u, 0u, 0u}, k0, k1);
  const uint64_t x = (i & 1) ? join64(r.z, r.w) : join64(r.x, r.y);
  phi_wk[idx] = __dadd_rn(1.0, __dmul_rn(init_noise, u64_to_uniform(x)));
}

__global__ void k_div_cols(double* __restrict__ x, int64_t n, int K,
                           const double* __restrict__ totals) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  x[i] = __ddiv_rn(x[i], totals[i % K]);
}

__global__ void k_fill(double* __restrict__ p, int64_t n, double v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_transpose(const double* __restrict__ in, int64_t rows, int64_t cols,
                            double* __restrict__ out) {
  __shared__ double tile[32][33];
  const int64_t c0 = blockIdx.x * 32ll, r0 = blockIdx.y * 32ll;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][dy];
  }
}

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
            const double* ph = phi_wk + static_cast<int64_t>(w) * K;
            double mu = 0.0;
            for (int k = 0; k < K; ++k) mu = __dadd_rn(mu, __dmul_rn(th[k], __ldg(ph + k)));
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
          const double* ph = phi_wk + static_cast<int64_t>(word_ids[base + i]) * K;
          double p = 0.0;
          for (int k = 0; k < K; ++k) p = __dadd_rn(p, __dmul_rn(th[k], __ldg(ph + k)));
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

__global__ void k_ordered_ll(const double* __restrict__ doc_logp,
                             const int64_t* __restrict__ doc_scored, int64_t n_docs,
                             double* __restrict__ ll_out, int* __restrict__ err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double total = 0.0;
  int64_t scored = 0;
  for (int64_t d = 0; d < n_docs; ++d) {
    total = __dadd_rn(total, doc_logp[d]);
    scored += doc_scored[d];
  }
  if (scored == 0) {
    atomicOr(err, kErrNumerical);
    *ll_out = 0.0;
    return;
  }
  *ll_out = __ddiv_rn(total, static_cast<double>(scored));
}

template <int KPL>
int launch_sample_kpl(const BatchView& bv, const double* theta_batch, const double* phi_wk,
                      const double* mu, int K, double m_t, uint64_t seed, uint32_t t,
                      uint32_t sweep, int mode, unsigned long long* tc, unsigned long long* pc,
                      double* tf, double* pf, int* err, cudaStream_t st) {
  const int n_slices = (K + kWarp * KPL - 1) / (kWarp * KPL);
  const int64_t chunk = 128;
  const int64_t items = (bv.nnz + chunk - 1) / chunk;
  const int64_t threads = items * n_slices * kWarp;
  const int block = kSampleBlock;
  if (mode == kModeExpected) {
    k_sample<KPL, kModeExpected><<<grid_for(threads, block), block, 0, st>>>(
        bv, theta_batch, phi_wk, mu, K, m_t, seed, t, sweep, chunk, n_slices, tc, pc, tf, pf,
        err);
  } else {
    k_sample<KPL, kModeParity><<<grid_for(threads, block), block, 0, st>>>(
        bv, theta_batch, phi_wk, mu, K, m_t, seed, t, sweep, chunk, n_slices, tc, pc, tf, pf,
        err);
  }
  return 1;
}

constexpr size_t kEvalSmemMax = 200 * 1024;

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

int64_t deferred_record_bytes() { return static_cast<int64_t>(sizeof(Deferred)); }

int launch_sample_fast(const BatchView& bv, const double* theta_b64, const float* theta_b32,
                       const double* phi64, const float* phi32, const double* mu, int K,
                       double m_t, uint64_t seed, uint32_t t, uint32_t sweep,
                       unsigned long long* tc, unsigned long long* pc, void* deferred,
                       unsigned long long* n_deferred, int* err, cudaStream_t st) {
  if (bv.nnz == 0) return 0;
  if (K <= 32)
    return launch_fast_kpl<1>(bv, theta_b64, theta_b32, phi64, phi32, mu, K, m_t, seed, t, sweep,
                              tc, pc, deferred, n_deferred, err, st);
  if (K <= 64)
    return launch_fast_kpl<2>(bv, theta_b64, theta_b32, phi64, phi32, mu, K, m_t, seed, t, sweep,
                              tc, pc, deferred, n_deferred, err, st);
  if (K <= 128)
    return launch_fast_kpl<4>(bv, theta_b64, theta_b32, phi64, phi32, mu, K, m_t, seed, t, sweep,
                              tc, pc, deferred, n_deferred, err, st);
  return launch_fast_kpl<8>(bv, theta_b64, theta_b32, phi64, phi32, mu, K, m_t, seed, t, sweep,
                            tc, pc, deferred, n_deferred, err, st);
}

int launch_theta_from_counts(const unsigned long long* cu, const double* cf, int64_t n,
                             double m_t, double alpha, double* out, float* out32,
                             cudaStream_t st) {
  if (n == 0) return 0;
  k_theta_from_counts<<<grid_for(n, 256), 256, 0, st>>>(cu, cf, n, m_t, alpha, out, out32);
  return 1;
}

int launch_theta_persist(const unsigned long long* cu, const double* cf,
                         const int32_t* batch_docs, int64_t B, int K, double m_t, double alpha,
                         double* theta, cudaStream_t st) {
  if (B * K == 0) return 0;
  k_theta_persist<<<grid_for(B * K, 256), 256, 0, st>>>(cu, cf, batch_docs, B, K, m_t, alpha,
                                                       theta);
  return 1;
}

int launch_phi_mstep(const unsigned long long* cu, const double* cf, int64_t W, int K,
                     double m_t, double beta, double rho, double* phi_wk, float* phi32,
                     double* totals, int* err, cudaStream_t st) {
  const int64_t n = W * K;
  if (n == 0) return 0;
  if (cu)
    k_col_totals<0><<<grid_for(static_cast<int64_t>(K) * 32, 256), 256, 0, st>>>(cu, cf, W, K, m_t, beta, totals, err);
  else
    k_col_totals<1><<<grid_for(static_cast<int64_t>(K) * 32, 256), 256, 0, st>>>(cu, cf, W, K, m_t, beta, totals, err);
  k_phi_blend<<<grid_for(n, 256), 256, 0, st>>>(cu, cf, totals, n, K, m_t, beta, 1.0 - rho, rho,
                                               phi_wk, phi32);
  return 2;
}

int launch_to_f32(const double* x, int64_t n, float* y, cudaStream_t st) {
  if (n == 0) return 0;
  k_to_f32<<<grid_for(n, 256), 256, 0, st>>>(x, n, y);
  return 1;
}

int launch_phi_init(double* phi_wk, int64_t W, int K, double init_noise, uint64_t seed,
                    double* totals, cudaStream_t st) {
  const int64_t n = W * K;
  if (n == 0) return 0;
  if (!(init_noise > 0.0)) {
    k_fill<<<grid_for(n, 256), 256, 0, st>>>(phi_wk, n, 1.0 / static_cast<double>(W));
    return 1;
  }
  uint32_t k0, k1;
  stream_key(seed, make_tag(kPhiInit, 0, 0), k0, k1);
  k_phi_init_values<<<grid_for(n, 256), 256, 0, st>>>(phi_wk, W, K, init_noise, k0, k1);
  k_col_totals<2><<<grid_for(static_cast<int64_t>(K) * 32, 256), 256, 0, st>>>(nullptr, phi_wk, W, K, 1.0, 0.0, totals, nullptr);
  k_div_cols<<<grid_for(n, 256), 256, 0, st>>>(phi_wk, n, K, totals);
  return 3;
}

int launch_fill(double* p, int64_t n, double v, cudaStream_t st) {
  if (n == 0) return 0;
  k_fill<<<grid_for(n, 256), 256, 0, st>>>(p, n, v);
  return 1;
}

int launch_transpose(const double* in, int64_t rows, int64_t cols, double* out,
                     cudaStream_t st) {
  if (rows * cols == 0) return 0;
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  k_transpose<<<grid, dim3(32, 8), 0, st>>>(in, rows, cols, out);
  return 1;
}

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
  const size_t smem = static_cast<size_t>(kEvalWarps) * 2 * K * sizeof(double);
  int64_t blocks = (n_docs + kEvalWarps - 1) / kEvalWarps;
  if (smem <= kEvalSmemMax) {
    static size_t configured = 48 * 1024;
    if (smem > configured) {
      cudaFuncSetAttribute(k_eval_docs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kEvalSmemMax));
      configured = kEvalSmemMax;
    }
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
  k_ordered_ll<<<1, 32, 0, st>>>(doc_logp, doc_scored, n_docs, ll_out, err);
  return 1;
}

}  // namespace scu
