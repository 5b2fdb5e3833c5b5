// bs_rng.cuh — bit-exact restatement of the reference's random streams on
// host and device: std::mt19937_64 (the engine behind pdsim::Rng,
// rng.hpp:15-75; its output sequence is fixed by the C++ standard),
// Rng::uniform01 (rng.hpp:22) and FNV-1a (rng.hpp:77-95), plus
// probe_seed (placement.hpp:135-140).
#pragma once

#include <cstdint>

namespace bs {

#if defined(__CUDACC__)
#define BS_HD __host__ __device__ __forceinline__
#else
#define BS_HD inline
#endif

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr unsigned long long kMtMatrix = 0xB5026F5AA96619E9ull;
constexpr unsigned long long kMtUpper = 0xFFFFFFFF80000000ull;
constexpr unsigned long long kMtLower = 0x7FFFFFFFull;

// Sequential engine (host, and device threads that need a single stream).
struct Mt64 {
  unsigned long long mt[kMtN];
  int idx;

  BS_HD void seed(unsigned long long s) {
    mt[0] = s;
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    idx = kMtN;
  }

  BS_HD void twist() {
    for (int i = 0; i < kMtN; ++i) {
      const unsigned long long x = (mt[i] & kMtUpper) | (mt[(i + 1) % kMtN] & kMtLower);
      unsigned long long xa = x >> 1;
      if (x & 1ull) xa ^= kMtMatrix;
      mt[i] = mt[(i + kMtM) % kMtN] ^ xa;
    }
    idx = 0;
  }

  BS_HD static unsigned long long temper(unsigned long long x) {
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
  }

  BS_HD unsigned long long next() {
    if (idx >= kMtN) twist();
    return temper(mt[idx++]);
  }

  // Rng::uniform01 (rng.hpp:22): (engine() >> 11) * 2^-53
  BS_HD double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

BS_HD unsigned long long fnv1a64(const unsigned char* p, int len, unsigned long long h) {
  for (int i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// probe_seed (placement.hpp:135-140): FNV-1a("goodput-probe", seed) then the
// bytes of int64 k and of int replicate (little-endian, as the reference
// hashes the objects' memory).
BS_HD unsigned long long probe_seed(unsigned long long seed, long long k, int replicate) {
  const unsigned char tag[13] = {'g', 'o', 'o', 'd', 'p', 'u', 't', '-', 'p', 'r', 'o', 'b', 'e'};
  unsigned long long h = fnv1a64(tag, 13, seed);
  unsigned char kb[8], rb[4];
  for (int i = 0; i < 8; ++i) kb[i] = static_cast<unsigned char>((static_cast<unsigned long long>(k) >> (8 * i)) & 0xff);
  for (int i = 0; i < 4; ++i) rb[i] = static_cast<unsigned char>((static_cast<unsigned>(replicate) >> (8 * i)) & 0xff);
  h = fnv1a64(kb, 8, h);
  h = fnv1a64(rb, 4, h);
  return h;
}

}  // namespace bs
