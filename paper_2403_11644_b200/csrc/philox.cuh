// philox.cuh -- device side of the seeded counter-based input recipe (DESIGN.md "Input
// recipe"): Philox4x32-10 keyed by the seed, counter = global element index,
// Box-Muller.  Used by the generator kernels (generate.cu) and by the matrix-free dense
// pipeline (row f1), which computes A[i][i ^ x] inside phase A instead of loading it.
// Written independently of the host module ptdr_inputs/gen.c (the tests compare them).
#pragma once
#include <cstdint>

#include "engine.cuh"

namespace ptdr {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// (re, im) iid N(0,1) for (seed, idx, stream)
__device__ __forceinline__ double2 gauss_pair(u64 seed, u64 idx, unsigned stream) {
  const uint4 o = philox4x32_10(make_uint4((unsigned)idx, (unsigned)(idx >> 32), stream, 0u),
                                make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
  const u64 a = ((u64)o.y << 32) | o.x;
  const u64 b = ((u64)o.w << 32) | o.z;
  const double u1 = __dmul_rn((double)((a >> 11) + 1ull), 0x1.0p-53);
  const double u2 = __dmul_rn((double)(b >> 11), 0x1.0p-53);
  const double r = sqrt(__dmul_rn(-2.0, log(u1)));
  const double th = __dmul_rn(6.283185307179586, u2);  // (2 * M_PI) * u2
  double s, c;
  sincos(th, &s, &c);
  return make_double2(__dmul_rn(r, c), __dmul_rn(r, s));
}

}  // namespace ptdr
