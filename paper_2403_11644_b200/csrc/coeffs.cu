// coeffs.cu -- selected coefficients of a dense matrix (Algorithm 2, compute_coeff,
// PAPER.md l.302-313): alpha(x, z) = 2^-n i^{popcount(x & z)} sum_i (-1)^{popcount(i & z)}
// A[i][i ^ x] evaluated directly, O(2^n) per coefficient, one warp per requested string.
// For users who need a few coefficients (or a spot check at sizes where the full transform
// would not fit) without decomposing the whole matrix.
#include <cstdint>

#include "engine.cuh"
#include "internal.h"

namespace ptdr {

// A[i][j] at A + i * ld + (j & colmask): the dense matrix (ld = 2^n, colmask = 2^n - 1), or
// rank `rank`'s X-mask shard after the all-to-all (ld = colmask + 1 = R: A_local[i][c] =
// A[i][((i >> (n - g)) ^ rank) R + c], which holds A[i][i ^ x] at column (i ^ x) & (R - 1) for
// every x of the shard).  Strings whose X-mask is outside the shard (x & ~colmask != xbase)
// get NaN.
__global__ void __launch_bounds__(256) coeffs_kernel(const double2* __restrict__ A, int n, u64 ld, u64 colmask,
                                                     u64 xbase, const u64* __restrict__ qs, u64 count,
                                                     double2* __restrict__ out) {
  const u64 N = 1ull << n;
  const int lane = threadIdx.x & 31;
  const u64 warps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 w = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < count; w += warps) {
    const u64 q = qs[w];
    // q -> (x, z): code_l = 2 z_l + (x_l ^ z_l) (include/ptdr.h)
    u64 x = 0, z = 0;
    for (int l = 0; l < n; ++l) {
      const u64 c = (q >> (2 * l)) & 3ull;
      const u64 zl = c >> 1;
      z |= zl << l;
      x |= ((c & 1ull) ^ zl) << l;
    }
    if ((x & ~colmask) != xbase) {
      if (lane == 0) out[w] = make_double2(__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll));
      continue;
    }
    // lanes stride over i; each lane keeps a Kahan-free pairwise-ish partial sum
    double re = 0.0, im = 0.0;
    for (u64 i = (u64)lane; i < N; i += 32) {
      const double2 v = ld_stream(A + i * ld + ((i ^ x) & colmask));
      if (__popcll(i & z) & 1) { re -= v.x; im -= v.y; }
      else { re += v.x; im += v.y; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, off);
      im += __shfl_xor_sync(0xffffffffu, im, off);
    }
    if (lane == 0) {
      const double2 c = rot_ipow(make_double2(re, im), __popcll(x & z));
      const double s = ldexp(1.0, -n);
      out[w] = make_double2(c.x * s, c.y * s);
    }
  }
}

cudaError_t launch_coeffs(const double2* A, int n, int rank, int world, const uint64_t* qs, uint64_t count,
                          double2* out, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  u64 g = (count * 32 + 255) / 256;
  const u64 cap = (u64)device_sm_count() * 16;
  if (g > cap) g = cap;
  const u64 R = (1ull << n) / (u64)world;
  coeffs_kernel<<<(unsigned)g, 256, 0, st>>>(A, n, R, R - 1ull, world > 1 ? (u64)rank * R : 0ull,
                                             reinterpret_cast<const u64*>(qs), count, out);
  return cudaGetLastError();
}

}  // namespace ptdr
