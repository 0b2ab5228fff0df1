// Philox4x64-10 (Random123 constants) with numpy's counter convention:
// numpy.random.Philox pre-increments its 256-bit counter before every block,
// so raw word j of a fresh Philox(seed) is lane j % 4 of block counter j/4 + 1
// (pinned against numpy in tests/test_oracle.py and tests/test_gpu_parity.py).
#pragma once

#include <stdint.h>

namespace apmg {

__device__ __forceinline__ void philox_block(uint64_t ctr_lo, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t c0 = ctr_lo, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t lo0 = M0 * c0, hi0 = __umul64hi(M0, c0);
    const uint64_t lo1 = M1 * c2, hi1 = __umul64hi(M1, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
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

// numpy next_double: (x >> 11) * 2^-53
__device__ __forceinline__ double word_to_double(uint64_t w) {
  return double(w >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace apmg
