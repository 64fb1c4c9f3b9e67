// Philox4x32-10 (Salmon et al., SC'11), the sampling RNG of reading R17:
// key = seed, counter = (v >> 2, gidx mod 2^32, step mod 2^32, gidx >> 32), word v & 3,
// u = (word >> 8) 2^-24.  Shared by the per-node sampler (sample.cu) and the autoregressive
// decoder (ar.cu), which must draw the same uniform for the same (node, placement, step).
#pragma once
#include <stdint.h>

namespace gdp {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// the uniform of node v in placement gidx (R17)
__device__ __forceinline__ float philox_uniform(uint64_t seed, uint64_t gidx, uint64_t step, int v) {
  const uint4 w = philox4x32_10(make_uint4((unsigned)(v >> 2), (unsigned)(gidx & 0xffffffffu),
                                           (unsigned)(step & 0xffffffffu), (unsigned)(gidx >> 32)),
                                make_uint2((unsigned)(seed & 0xffffffffu), (unsigned)(seed >> 32)));
  const unsigned x = (v & 3) == 0 ? w.x : (v & 3) == 1 ? w.y : (v & 3) == 2 ? w.z : w.w;
  return (float)(x >> 8) * 5.9604644775390625e-08f;   // 2^-24
}

}  // namespace gdp
