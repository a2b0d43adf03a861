// philox.cuh -- device Philox4x32-10 counter-based RNG (reading #1 of DESIGN.md).
// Written independently of the oracle; checked against the Random123 known-answer
// vectors and against the oracle's stream in tests/test_gpu_*.py.
#pragma once
#include <stdint.h>

namespace santa {

enum : uint32_t { kTagValueSampler = 1, kTagBernoulliHead = 2, kTagBernoulliGroup = 3, kTagPropTileOffset = 4, kTagFlashTileOffset = 5 };

struct Philox4 {
  uint32_t x[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                 uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  Philox4 o;
  o.x[0] = c0;
  o.x[1] = c1;
  o.x[2] = c2;
  o.x[3] = c3;
  return o;
}

// One stream = (seed, offset, tag, id, batch).  Draw i is word (i & 3) of block i >> 2.
struct PhiloxStream {
  uint32_t k0, k1, c1, c2, c3;
  __device__ __forceinline__ PhiloxStream(uint64_t seed, uint64_t offset, uint32_t tag,
                                          uint32_t id_global, uint32_t b_global)
      : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)),
        c1((tag << 24) | (id_global & 0xFFFFFFu)), c2(b_global), c3((uint32_t)offset) {}
  __device__ __forceinline__ uint32_t word(uint32_t draw) const {
    Philox4 o = philox4x32_10(draw >> 2, c1, c2, c3, k0, k1);
    const uint32_t w = draw & 3u;
    return w == 0 ? o.x[0] : (w == 1 ? o.x[1] : (w == 2 ? o.x[2] : o.x[3]));
  }
  // u = r * 2^-32 exactly representable in fp64, in [0, 1 - 2^-32]
  __device__ __forceinline__ double uniform(uint32_t draw) const {
    return (double)word(draw) * 2.3283064365386963e-10;
  }
};

// Thresholds of the three samplers, fp64 (reading #2/#3).
__device__ __forceinline__ double sample_threshold(int mode, int m, int S, const PhiloxStream& ps) {
  if (mode == 0) return ps.uniform((uint32_t)m);                        // iid
  if (mode == 1) return ((double)m + ps.uniform((uint32_t)m)) / (double)S; // stratified
  return ((double)m + ps.uniform(0u)) / (double)S;                      // systematic
}

}  // namespace santa
