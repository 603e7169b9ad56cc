// philox.cuh -- counter-based Philox4x32-10 streams, host + device.
//
// Bit-level contract of the reference RNG:
//   rng.cpp:24-35   philox_block: 10 rounds, Random123 constants
//   rng.cpp:90-101  stream: counter {block, word, doc, t}, key = seed halves ^ tag*M
//   rng.cpp:110-133 u64 = first | second << 32; uniform / uniform_oo / uniform_below
//   rng.hpp:35-39   tag = purpose<<28 | (sub&0xff)<<20 | (index&0xfffff)
//
// The sampling kernels do not keep a buffered stream per draw: a draw's first
// block is one philox10() call on {0, word, doc, t}, and only the rare PTRS
// path walks further blocks through Stream.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define SCU_HD __host__ __device__ __forceinline__
#else
#define SCU_HD inline
#endif

namespace scu {

constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;

enum Purpose : uint32_t {
  kPoissonCounts = 1,
  kBatchShuffle = 2,
  kHoldoutSplit = 3,
  kEvalSplit = 6,
  kPhiInit = 8,
  kThroughput = 9,  // throughput mode's own streams (not in the reference)
  kMultinomial = 10,  // multinomial mode's own streams (not in the reference)
  kThroughputDoc = 11,  // throughput mode's per-(document, topic) draws (not in the reference)
};

SCU_HD uint32_t make_tag(uint32_t purpose, uint32_t sub, uint32_t index) {
  return (purpose << 28) | ((sub & 0xffu) << 20) | (index & 0xfffffu);
}

SCU_HD void mulhilo(uint32_t a, uint32_t b, uint32_t& lo, uint32_t& hi) {
#if defined(__CUDA_ARCH__)
  const uint64_t p = static_cast<uint64_t>(a) * b;  // one IMAD.WIDE.U32
  lo = static_cast<uint32_t>(p);
  hi = static_cast<uint32_t>(p >> 32);
#else
  const uint64_t p = static_cast<uint64_t>(a) * b;
  lo = static_cast<uint32_t>(p);
  hi = static_cast<uint32_t>(p >> 32);
#endif
}

struct U4 {
  uint32_t x, y, z, w;
};

// Ten Philox4x32 rounds; the key is bumped after every round (rng.cpp:26-33).
SCU_HD U4 philox10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t lo0, hi0, lo1, hi1;
    mulhilo(kPhiloxM0, c.x, lo0, hi0);
    mulhilo(kPhiloxM1, c.z, lo1, hi1);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return c;
}

// Stream key (rng.cpp:92-94).
SCU_HD void stream_key(uint64_t seed, uint32_t tag, uint32_t& k0, uint32_t& k1) {
  k0 = static_cast<uint32_t>(seed) ^ (tag * kPhiloxM0);
  k1 = static_cast<uint32_t>(seed >> 32) ^ (tag * kPhiloxM1);
}

SCU_HD double u64_to_uniform(uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }
SCU_HD double u64_to_uniform_oo(uint64_t x) {
  return (static_cast<double>(x >> 11) + 0.5) * 0x1.0p-53;
}
SCU_HD uint64_t join64(uint32_t lo, uint32_t hi) {
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Buffered stream with the reference's consumption order (rng.cpp:96-122).
struct Stream {
  uint32_t word, doc, t;
  uint32_t k0, k1;
  uint32_t block;
  uint32_t buf[4];
  int pos;

  SCU_HD void init(uint64_t seed, uint32_t t_, uint32_t doc_, uint32_t word_, uint32_t tag) {
    word = word_;
    doc = doc_;
    t = t_;
    stream_key(seed, tag, k0, k1);
    block = 0;
    pos = 4;
  }
  // Resume a stream whose block 0 was already generated into `b0`.
  SCU_HD void init_with_block0(uint64_t seed, uint32_t t_, uint32_t doc_, uint32_t word_,
                               uint32_t tag, U4 b0, int consumed) {
    init(seed, t_, doc_, word_, tag);
    buf[0] = b0.x;
    buf[1] = b0.y;
    buf[2] = b0.z;
    buf[3] = b0.w;
    block = 1;
    pos = consumed;
  }
  SCU_HD void refill() {
    const U4 r = philox10(U4{block, word, doc, t}, k0, k1);
    block += 1u;
    buf[0] = r.x;
    buf[1] = r.y;
    buf[2] = r.z;
    buf[3] = r.w;
    pos = 0;
  }
  SCU_HD uint32_t next_u32() {
    if (pos == 4) refill();
    return buf[pos++];
  }
  SCU_HD uint64_t next_u64() {
    const uint64_t lo = next_u32();
    const uint64_t hi = next_u32();
    return (hi << 32) | lo;
  }
  SCU_HD double uniform() { return u64_to_uniform(next_u64()); }
  SCU_HD double uniform_oo() { return u64_to_uniform_oo(next_u64()); }
  SCU_HD uint64_t uniform_below(uint64_t n) {
    const uint64_t rem = (0 - n) % n;
    for (;;) {
      const uint64_t x = next_u64();
      if (x >= rem) return (x - rem) % n;
    }
  }
};

}  // namespace scu
