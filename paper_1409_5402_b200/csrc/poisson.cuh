// poisson.cuh -- exact Poisson variates on the device, reference-identical.
//
//   rng.cpp:39-52   inversion by sequential search (lambda < 10)
//   rng.cpp:57-86   PTRS transformed rejection, Hormann 1993 (lambda >= 10)
//   rng.cpp:139-150 dispatch; lambda == 0 returns 0 without touching the stream
//
// Every f64 operation is written as an explicit round-to-nearest intrinsic
// (__dmul_rn / __ddiv_rn / __dadd_rn): no FMA contraction may merge them,
// because the reference is built for x86-64 baseline without FMA.  lgamma of
// integers below kLgammaTab is glibc's own value (a host-filled table); exp /
// log are CUDA libdevice (<= 1-2 ulp from glibc); a last-ulp difference
// can only flip a draw when the uniform lands inside that ulp gap (~1e-16
// per draw), see DESIGN.md "Parity".
#pragma once

#include <cstdint>

#include "philox.cuh"

namespace scu {

// Inversion for lambda in (0, 10) given the draw's first uniform u.
__device__ __forceinline__ int64_t poisson_inversion(double lambda, double u) {
  double pmf = exp(-lambda);
  double cdf = pmf;
  int64_t k = 0;
  while (u > cdf && k < 1000) {
    ++k;
    pmf = __dmul_rn(pmf, __ddiv_rn(lambda, static_cast<double>(k)));
    cdf = __dadd_rn(cdf, pmf);
  }
  return k;
}

// lgamma(k + 1) for integer k < kLgammaTab as glibc computes it (the
// reference's std::lgamma, rng.cpp:81), filled on the host per device by
// init_lgamma_table (kernels_sample.cu); larger k use libdevice lgamma.
constexpr int kLgammaTab = 4096;
__device__ double g_lgamma_int[kLgammaTab];
__device__ int g_lgamma_ready;

// PTRS for lambda >= 10, consuming the stream exactly like rng.cpp:64-85.
__device__ __noinline__ int64_t poisson_ptrs(double lambda, Stream& s) {
  const double log_lambda = log(lambda);
  const double b = __dadd_rn(0.931, __dmul_rn(2.53, sqrt(lambda)));
  const double a = __dadd_rn(-0.059, __dmul_rn(0.02483, b));
  const double inv_alpha = __dadd_rn(1.1239, __ddiv_rn(1.1328, __dadd_rn(b, -3.4)));
  const double v_r = __dadd_rn(0.9277, -__ddiv_rn(3.6224, __dadd_rn(b, -2.0)));
  for (;;) {
    const double u = __dadd_rn(s.uniform_oo(), -0.5);
    const double v = s.uniform_oo();
    const double us = __dadd_rn(0.5, -fabs(u));
    // (2a/us + b) * u + lambda + 0.43, left to right
    const double g = __dadd_rn(
        __dadd_rn(__dmul_rn(__dadd_rn(__ddiv_rn(__dmul_rn(2.0, a), us), b), u), lambda), 0.43);
    if (us >= 0.07 && v <= v_r) return static_cast<int64_t>(g);
    if (g < 0.0 || g > 9.0e18 || (us < 0.013 && v > us)) continue;
    const int64_t k = static_cast<int64_t>(g);
    const double lhs =
        log(__ddiv_rn(__dmul_rn(v, inv_alpha), __dadd_rn(__ddiv_rn(a, __dmul_rn(us, us)), b)));
    const double lg = k < kLgammaTab && g_lgamma_ready ? g_lgamma_int[k]
                                                       : lgamma(__dadd_rn(static_cast<double>(k), 1.0));
    const double rhs = __dadd_rn(__dadd_rn(-lambda, __dmul_rn(static_cast<double>(k), log_lambda)), -lg);
    if (lhs <= rhs) return k;
  }
}

// poisson_sample for a draw whose stream key is (seed, t, doc, word, tag),
// with the stream's first block already computed into b0.  The caller has
// checked lambda is finite and >= 0.
__device__ __forceinline__ int64_t poisson_from_block0(double lambda, U4 b0, uint64_t seed,
                                                       uint32_t t, uint32_t doc, uint32_t word,
                                                       uint32_t tag) {
  if (lambda == 0.0) return 0;
  if (lambda < 10.0) return poisson_inversion(lambda, u64_to_uniform(join64(b0.x, b0.y)));
  Stream s;
  s.init_with_block0(seed, t, doc, word, tag, b0, 0);
  return poisson_ptrs(lambda, s);
}

}  // namespace scu
