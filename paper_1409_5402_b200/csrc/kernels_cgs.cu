// kernels_cgs.cu -- the collapsed Gibbs sampler baseline (
// the paper's comparison method, cgs.cpp:11-157) on the device, draw for draw
// the reference's chain.
//
// cgs_init (cgs.cpp:11-55) is parallel: one thread per document, each cell's
// tokens drawn from its own stream (t=0, doc, word, tag(cgs_init)).
//
// cgs_sweep (cgs.cpp:57-98) is sequential BY DEFINITION: every token's
// conditional depends on the counts left by the token before it (the word's
// topic row and the topic totals are shared by all documents).  The device
// version keeps the reference's order -- documents, cells, tokens -- in one
// warp: lane = topic (K / 32 topics per lane), the document's topic row, the
// current word's row and the topic totals live in registers; per token the
// lanes form the K weights (cgs.cpp:80-85, same operations and rounding), one
// lane runs the categorical sample's sequential running sum over k
// (rng.cpp:152-179) and the whole warp finds the first k with u < cum_k by
// ballot.  A cell's uniforms (one per token, from the cell's stream
// (t=sweep, doc, word, tag(cgs_sweep))) are drawn by the lanes in parallel
// before its tokens.  This is a latency-bound chain of ~0.2 us per token on
// one SM: the method has no parallelism to give (the reason the paper's
// SAME sampler exists).
#include "kernels_common.cuh"

namespace scu {

namespace {

constexpr uint32_t kCgsInit = 4;
constexpr uint32_t kCgsSweep = 5;

// exact for 0 <= v < 2^52 (counts): no I2F.F64
__device__ __forceinline__ double small_to_double(long long v) {
  return __dsub_rn(__longlong_as_double(v | 0x4330000000000000ll), 4503599627370496.0);
}

__global__ void k_cgs_init(const int64_t* __restrict__ offsets, const int32_t* __restrict__ words,
                           const int32_t* __restrict__ counts, const int64_t* __restrict__ tok_off,
                           int64_t D, int K, uint64_t seed, int32_t* __restrict__ z,
                           int32_t* __restrict__ dt, int32_t* __restrict__ wt,
                           unsigned long long* __restrict__ tt) {
  const int64_t d = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (d >= D) return;
  for (int64_t c = offsets[d]; c < offsets[d + 1]; ++c) {
    const int32_t w = words[c];
    Stream s;
    s.init(seed, 0u, static_cast<uint32_t>(d), static_cast<uint32_t>(w), make_tag(kCgsInit, 0, 0));
    for (int64_t tok = tok_off[c]; tok < tok_off[c + 1]; ++tok) {
      const int k = static_cast<int>(s.uniform_below(static_cast<uint64_t>(K)));
      z[tok] = k;
      dt[d * K + k] += 1;  // this thread owns row d
      atomicAdd(wt + static_cast<int64_t>(w) * K + k, 1);
      atomicAdd(tt + k, 1ull);
    }
  }
}

// One warp, the whole corpus in the reference's order.  KPL topics per lane
// (lane + 32 j); wsum / cum: K doubles of shared memory each.
template <int KPL>
__global__ void __launch_bounds__(32) k_cgs_sweep(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ words,
    const int32_t* __restrict__ counts, const int64_t* __restrict__ tok_off, int64_t D, int K,
    int64_t W, double alpha, double beta, uint64_t seed, uint32_t sweep, int32_t* __restrict__ z,
    int32_t* __restrict__ dt, int32_t* __restrict__ wt, unsigned long long* __restrict__ tt,
    int* __restrict__ err) {
  extern __shared__ double sm[];
  double* wts = sm;       // K weights of the current token
  double* cum = sm + K;   // their running sums (the categorical scan's)
  const int lane = threadIdx.x;
  const double w_beta = __dmul_rn(static_cast<double>(W), beta);
  uint32_t k0, k1;
  stream_key(seed, make_tag(kCgsSweep, 0, 0), k0, k1);
  long long ttr[KPL];
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const int k = lane + 32 * j;
    ttr[j] = k < K ? static_cast<long long>(tt[k]) : 0;
  }
  for (int64_t d = 0; d < D; ++d) {
    int32_t dtr[KPL];
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int k = lane + 32 * j;
      dtr[j] = k < K ? dt[d * K + k] : 0;
    }
    for (int64_t c = offsets[d]; c < offsets[d + 1]; ++c) {
      const int32_t w = words[c];
      int32_t* wrow = wt + static_cast<int64_t>(w) * K;
      int32_t wtr[KPL];
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = lane + 32 * j;
        wtr[j] = k < K ? wrow[k] : 0;
      }
      const int64_t t0 = tok_off[c], t1 = tok_off[c + 1];
      for (int64_t tb = t0; tb < t1; tb += 32) {
        // this chunk's uniforms: token i of the cell takes the i-th uniform of
        // the stream, i.e. words 2 (i % 2), 2 (i % 2) + 1 of block i / 2
        const int64_t i = tb - t0 + lane;
        double u_mine = 0.0;
        int32_t z_mine = 0;
        if (tb + lane < t1) {
          const U4 r = philox10(U4{static_cast<uint32_t>(i >> 1), static_cast<uint32_t>(w),
                                   static_cast<uint32_t>(d), sweep},
                                k0, k1);
          u_mine = u64_to_uniform((i & 1) ? join64(r.z, r.w) : join64(r.x, r.y));
          z_mine = z[tb + lane];
        }
        const int n_here = static_cast<int>(min(static_cast<int64_t>(32), t1 - tb));
        for (int q = 0; q < n_here; ++q) {
          const int old_k = __shfl_sync(0xffffffffu, z_mine, q);
          const double u = __shfl_sync(0xffffffffu, u_mine, q);
          // remove the token (cgs.cpp:75-78), then the K weights (:80-85):
          // (dt + alpha) * (wt + beta) / (tt + W beta)
#pragma unroll
          for (int j = 0; j < KPL; ++j) {
            const int k = lane + 32 * j;
            if (k == old_k) {
              --dtr[j];
              --wtr[j];
              --ttr[j];
            }
            if (k < K)
              wts[k] = __ddiv_rn(__dmul_rn(__dadd_rn(small_to_double(dtr[j]), alpha),
                                           __dadd_rn(small_to_double(wtr[j]), beta)),
                                 __dadd_rn(small_to_double(ttr[j]), w_beta));
          }
          __syncwarp();
          // categorical_sample (rng.cpp:152-179): total and running sums in k
          // order (the same partial sums), then the first k < K - 1 with
          // u * total < cum_k; else the last index with positive weight
          if (lane == 0) {
            double s = 0.0;
#pragma unroll 8
            for (int k = 0; k < K; ++k) {
              s = __dadd_rn(s, wts[k]);
              cum[k] = s;
            }
            if (!(s > 0.0) || isinf(s)) atomicOr(err, kErrNumerical);
          }
          __syncwarp();
          const double x = __dmul_rn(u, cum[K - 1]);
          int new_k = K;
#pragma unroll
          for (int j = 0; j < KPL; ++j) {
            const int k = lane + 32 * j;
            const unsigned hit = __ballot_sync(0xffffffffu, k < K - 1 && x < cum[k]);
            if (hit && new_k == K) new_k = 32 * j + __ffs(hit) - 1;
          }
          if (new_k == K) {  // last index carrying positive weight
#pragma unroll
            for (int j = KPL - 1; j >= 0; --j) {
              const int k = lane + 32 * j;
              const unsigned pos = __ballot_sync(0xffffffffu, k < K && wts[k] > 0.0);
              if (pos && new_k == K) new_k = 32 * j + 31 - __clz(pos);
            }
            if (new_k == K) new_k = 0;
          }
#pragma unroll
          for (int j = 0; j < KPL; ++j)
            if (lane + 32 * j == new_k) {
              ++dtr[j];
              ++wtr[j];
              ++ttr[j];
            }
          if (lane == q) z_mine = new_k;
          __syncwarp();  // wts / cum are rewritten by the next token
        }
        if (tb + lane < t1) z[tb + lane] = z_mine;
      }
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const int k = lane + 32 * j;
        if (k < K) wrow[k] = wtr[j];
      }
    }
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int k = lane + 32 * j;
      if (k < K) dt[d * K + k] = dtr[j];
    }
  }
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const int k = lane + 32 * j;
    if (k < K) tt[k] = static_cast<unsigned long long>(ttr[j]);
  }
}

// cgs_model (cgs.cpp:100-129): phi word-major (W x K, the eval layout) and theta
__global__ void k_cgs_model(const int32_t* __restrict__ dt, const int32_t* __restrict__ wt,
                            const unsigned long long* __restrict__ tt, int64_t D, int64_t W, int K,
                            double alpha, double beta, double* __restrict__ phi_wk,
                            double* __restrict__ theta) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const double w_beta = __dmul_rn(static_cast<double>(W), beta);
  if (i < W * K) {
    const int k = static_cast<int>(i % K);
    const double denom = __dadd_rn(static_cast<double>(static_cast<long long>(tt[k])), w_beta);
    phi_wk[i] = __ddiv_rn(__dadd_rn(static_cast<double>(wt[i]), beta), denom);
  }
  if (theta && i < D * K) theta[i] = __dadd_rn(static_cast<double>(dt[i]), alpha);
}

}  // namespace

int launch_cgs_init(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                    const int64_t* tok_off, int64_t D, int K, uint64_t seed, int32_t* z, int32_t* dt,
                    int32_t* wt, unsigned long long* tt, cudaStream_t st) {
  if (D == 0) return 0;
  k_cgs_init<<<grid_for(D, 128), 128, 0, st>>>(offsets, words, counts, tok_off, D, K, seed, z, dt,
                                               wt, tt);
  return 1;
}

int launch_cgs_sweep(const int64_t* offsets, const int32_t* words, const int32_t* counts,
                     const int64_t* tok_off, int64_t D, int K, int64_t W, double alpha, double beta,
                     uint64_t seed, uint32_t sweep, int32_t* z, int32_t* dt, int32_t* wt,
                     unsigned long long* tt, int* err, cudaStream_t st) {
  if (D == 0) return 0;
  const size_t smem = sizeof(double) * 2 * static_cast<size_t>(K);
  if (smem > 48 * 1024) {
    static std::atomic<unsigned long long> done{0};
    smem_opt_in(k_cgs_sweep<32>, static_cast<int>(smem), done);
  }
#define SCU_CGS(KPL)                                                                       \
  k_cgs_sweep<KPL><<<1, 32, smem, st>>>(offsets, words, counts, tok_off, D, K, W, alpha, beta, \
                                        seed, sweep, z, dt, wt, tt, err)
  if (K <= 32) SCU_CGS(1);
  else if (K <= 64) SCU_CGS(2);
  else if (K <= 128) SCU_CGS(4);
  else if (K <= 256) SCU_CGS(8);
  else if (K <= 512) SCU_CGS(16);
  else SCU_CGS(32);
#undef SCU_CGS
  return 1;
}

int launch_cgs_model(const int32_t* dt, const int32_t* wt, const unsigned long long* tt, int64_t D,
                     int64_t W, int K, double alpha, double beta, double* phi_wk, double* theta,
                     cudaStream_t st) {
  const int64_t n = std::max(W * K, theta ? D * K : 0);
  if (n == 0) return 0;
  k_cgs_model<<<grid_for(n, 256), 256, 0, st>>>(dt, wt, tt, D, W, K, alpha, beta, phi_wk, theta);
  return 1;
}

}  // namespace scu
