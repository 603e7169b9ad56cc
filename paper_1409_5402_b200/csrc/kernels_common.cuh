// kernels_common.cuh -- helpers shared by the kernel translation units
// (kernels_sample.cu, kernels_mstep.cu, kernels_eval.cu), all compiled with
// -fmad=false: every f64 expression rounds like the reference's x86-64
// (no FMA) build.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
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

// Dynamic shared-memory opt-in of `kernel` on the current device, once per
// device (the attribute is per device; `done` is the kernel's bitmask of
// devices already configured, updated atomically).
template <class Kernel>
inline void smem_opt_in(Kernel* kernel, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (bit) done.fetch_or(bit, std::memory_order_acq_rel);
}

inline unsigned grid_for(int64_t threads, int block) {
  return static_cast<unsigned>((threads + block - 1) / block);
}

}  // namespace
}  // namespace scu
