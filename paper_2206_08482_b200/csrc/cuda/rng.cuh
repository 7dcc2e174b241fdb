// Counter-based randomness and bit-exact integer helpers shared by the host runtime
// and the device kernels (host+device). Every stream of randomness is a pure function of
// (seed, global env / tensor / GMI id, step, tag), so results do not depend on how envs
// are partitioned over GMIs or GPUs.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define GMI_HD __host__ __device__ __forceinline__
#else
#define GMI_HD inline
#endif

namespace gmi::rng {

enum Tag : uint32_t { kNoise = 1, kReset = 2, kEpisode = 3, kInit = 4, kPerm = 5 };

// Philox4x32-10 (Salmon et al., SC'11), Random123 round/key schedule.
GMI_HD void philox(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                   uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
#if defined(__CUDA_ARCH__)
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
    const uint64_t p0 = uint64_t(0xD2511F53u) * c0, p1 = uint64_t(0xCD9E8D57u) * c2;
    const uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0);
    const uint32_t hi1 = uint32_t(p1 >> 32), lo1 = uint32_t(p1);
#endif
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

GMI_HD void draw(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t tag, uint32_t out[4]) {
  philox(uint32_t(seed), uint32_t(seed >> 32), a, b, c, tag, out);
}

// [0,1) and (0,1] with 24-bit resolution; the products are exact in fp32.
GMI_HD float u01(uint32_t x) { return float(x >> 8) * 5.9604644775390625e-8f; }
GMI_HD float u01_open0(uint32_t x) { return float((x >> 8) + 1u) * 5.9604644775390625e-8f; }

// Keyed bijection on [0, n) (4 xorshift-multiply-add rounds on ceil(log2 n) bits,
// cycle-walked into range): the per-epoch minibatch permutation, integer-exact.
GMI_HD uint32_t perm_index(uint32_t j, uint32_t n, const uint32_t keys[4]) {
  if (n <= 1) return 0;
  uint32_t bits = 0;
  while ((uint64_t(1) << bits) < n) ++bits;
  const uint32_t mask = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  const uint32_t half = (bits + 1) / 2;
  uint32_t x = j;
  do {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      x ^= x >> half;
      x = (x * 0x9E3779B1u + keys[r]) & mask;
    }
  } while (x >= n);
  return x;
}

}  // namespace gmi::rng
