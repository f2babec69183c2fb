// Philox4x64-10 (host + device), bit-compatible with the reference's
// /root/reference/proj/core/src/rng.cpp:34-47 and its RandomStream layout
// (key {seed, stream}, counter {block, substream, 0, 0}; rng.hpp:20-21).
// Every draw is a pure function of its index, so device code can evaluate
// draw #k of a stream directly (counter-indexed) instead of sequentially.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define GPK_HD __host__ __device__ __forceinline__
#else
#define GPK_HD inline
#endif

namespace gpk {

struct U64x4 {
  uint64_t v[4];
};

GPK_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = static_cast<unsigned __int128>(a) * b;
  hi = static_cast<uint64_t>(p >> 64);
  lo = static_cast<uint64_t>(p);
#endif
}

GPK_HD U64x4 philox4x64(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0, uint64_t k1) {
  for (int round = 0; round < 10; ++round) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, hi0, lo0);
    mulhilo64(0xCA5A826395121157ULL, c2, hi1, lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  U64x4 r;
  r.v[0] = c0; r.v[1] = c1; r.v[2] = c2; r.v[3] = c3;
  return r;
}

// u64 draw number `k` of RandomStream(seed, stream, substream).
GPK_HD uint64_t stream_u64(uint64_t seed, uint64_t stream, uint64_t substream, uint64_t k) {
  const U64x4 b = philox4x64(k >> 2, substream, 0, 0, seed, stream);
  return b.v[k & 3];
}

// Sequential host-side RandomStream (rng.cpp:49-126), used for the small
// draws the host keeps (RFF basis) and for cross-checks.
struct HostStream {
  uint64_t key0, key1, block = 0, sub;
  U64x4 buf{};
  int pos = 4;
  double cached = 0.0;
  bool has_cached = false;
  HostStream(uint64_t seed, uint64_t stream, uint64_t substream = 0)
      : key0(seed), key1(stream), sub(substream) {}
  uint64_t next_u64() {
    if (pos >= 4) {
      buf = philox4x64(block, sub, 0, 0, key0, key1);
      ++block;
      pos = 0;
    }
    return buf.v[pos++];
  }
};

}  // namespace gpk
