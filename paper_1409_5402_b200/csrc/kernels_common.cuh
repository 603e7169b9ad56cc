// kernels_common.cuh -- helpers shared by the kernel translation units
// (kernels_sample.cu, kernels_mstep.cu, kernels_eval.cu), all compiled with
// -fmad=false: every f64 expression rounds like the reference's x86-64
// (no FMA) build.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "philox.cuh"

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

}  // namespace
}  // namespace scu
