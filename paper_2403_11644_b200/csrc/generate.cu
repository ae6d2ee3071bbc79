// generate.cu -- seeded counter-based input generator kernels.
//
// Device implementation of the input recipe of DESIGN.md "Input recipe"
// (Philox4x32-10 keyed by the seed, counter = global element index, Box-Muller);
// written independently of the host module ptdr_inputs/gen.c, which the tests
// use to check it (tests/test_gpu_generator.py).  The paper fixes no
// distribution ("a generic matrix, with no specific structure")
// and allows function-defined entries (l.646).
#include <cstdint>

#include "engine.cuh"
#include "internal.h"
#include "philox.cuh"

namespace ptdr {

__device__ __forceinline__ double2 dense_entry(int n, u64 seed, int variant, u64 row, u64 col) {
  const u64 N = 1ull << n;
  if (variant == 0) return gauss_pair(seed, row * N + col, 0u);
  if (variant == 1) {
    const double2 a = gauss_pair(seed, row * N + col, 0u);
    const double2 b = gauss_pair(seed, col * N + row, 0u);
    return make_double2(__dmul_rn(__dadd_rn(a.x, b.x), 0.5), __dmul_rn(__dsub_rn(a.y, b.y), 0.5));
  }
  const u64 lo = row < col ? row : col, hi = row < col ? col : row;
  return make_double2(gauss_pair(seed, lo * N + hi, 0u).x, 0.0);
}

// ||A||_F^2 partials (the right-hand side of Parseval, Theorem 1)
// fused into the generators: each block writes the sum of |a|^2 over its grid-stride
// elements to partials[blockIdx.x] (a fixed shared-memory tree, so the value is
// deterministic); the grid never exceeds kFro2Parts and the host zeroes the array first.
constexpr int kFro2Parts = 4096;

__device__ __forceinline__ void block_sum_to(double acc, double* partials) {
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
#pragma unroll
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}
__device__ __forceinline__ double abs2(double2 v) { return __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)); }

__global__ void __launch_bounds__(256) gen_dense_kernel(int n, u64 seed, int variant, u64 row0, u64 nrows,
                                                        double2* A, double* fro2) {
  const u64 N = 1ull << n;
  const u64 total = nrows * N;
  double acc = 0.0;
  for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (u64)gridDim.x * blockDim.x) {
    const double2 v = dense_entry(n, seed, variant, row0 + e / N, e % N);
    A[e] = v;
    acc += abs2(v);
  }
  if (fro2) block_sum_to(acc, fro2);
}

// Send layout of the all-to-all, split into K sub-ranges of every rank's X-masks
// ("overlap"): element (s, h, t, r', c') of [K][world][K][R'][R'],
// R' = R / K, is A[(rank K + t) R' + r'][((rank ^ h) K + (t ^ s)) R' + c'] -- the block that
// virtual rank (rank K + t) of world K sends to virtual rank (h K + s).  Sub-range s is one
// contiguous equal-split all-to-all that delivers rank h the input of
// ptdr_decompose_xshard_async(rank' = h K + s, world' = world K).  K = 1 is the plain
// column-block-major layout send[h][r][c] = A[rank R + r][(rank ^ h) R + c].
__global__ void __launch_bounds__(256) gen_sendblocks_kernel(int n, u64 seed, int rank, int world, int K,
                                                             double2* send, double* fro2) {
  const u64 N = 1ull << n;
  const u64 Rp = N / (u64)world / (u64)K;
  const u64 total = N * (N / (u64)world);
  double acc = 0.0;
  for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (u64)gridDim.x * blockDim.x) {
    const u64 cc = e % Rp, rr = (e / Rp) % Rp;
    const u64 t = (e / (Rp * Rp)) % (u64)K;
    const u64 h = (e / (Rp * Rp * (u64)K)) % (u64)world;
    const u64 sr = e / (Rp * Rp * (u64)K * (u64)world);
    const u64 row = ((u64)rank * (u64)K + t) * Rp + rr;
    const u64 col = ((((u64)rank ^ h) * (u64)K) + (t ^ sr)) * Rp + cc;
    const double2 v = gauss_pair(seed, row * N + col, 0u);
    send[e] = v;
    acc += abs2(v);
  }
  if (fro2) block_sum_to(acc, fro2);
}

__global__ void __launch_bounds__(256) gen_band_kernel(int n, u64 seed, int variant, double2* band, double* fro2) {
  const u64 N = 1ull << n;
  double acc = 0.0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (u64)gridDim.x * blockDim.x) {
    if (variant == 3) {
      const double2 v = gauss_pair(seed, i, 1u);
      band[i] = v;
      acc += abs2(v);
      continue;
    }
    const double2 m = make_double2(gauss_pair(seed, i, 1u).x, 0.0);
    const double2 up = (i + 1 < N) ? make_double2(gauss_pair(seed, i, 2u).x, 0.0) : make_double2(0.0, 0.0);
    if (variant == 6) {
      // HERMITIAN_TRIDIAGONAL storage [main | sup] of the same matrix (sub = conj(sup) implied)
      band[i] = m;
      band[N + i] = up;
      acc += abs2(m) + 2.0 * abs2(up);
      continue;
    }
    const double2 lo = (i > 0) ? make_double2(gauss_pair(seed, i - 1, 2u).x, 0.0) : make_double2(0.0, 0.0);
    band[N + i] = m;
    band[2 * N + i] = up;
    band[i] = lo;
    acc += abs2(m) + abs2(up) + abs2(lo);
  }
  if (fro2) block_sum_to(acc, fro2);
}

// Parseval's left-hand side: partials[b] = sum |x_e|^2 over block b's grid-stride elements.
__global__ void __launch_bounds__(256) sumsq_kernel(const double2* __restrict__ x, u64 count, double* partials) {
  double acc = 0.0;
  for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (u64)gridDim.x * blockDim.x)
    acc += abs2(__ldcs(x + e));
  block_sum_to(acc, partials);
}

static unsigned gen_blocks(u64 total) {
  u64 b = (total + 255) / 256;
  u64 cap = (u64)device_sm_count() * 32;
  if (cap > (u64)kFro2Parts) cap = kFro2Parts;
  return (unsigned)(b < cap ? b : cap);
}

static cudaError_t zero_parts(double* fro2, cudaStream_t st) {
  return fro2 ? cudaMemsetAsync(fro2, 0, kFro2Parts * sizeof(double), st) : cudaSuccess;
}

int fro2_partial_count() { return kFro2Parts; }

cudaError_t launch_generate_dense(int n, uint64_t seed, int variant, uint64_t row0,
                                  uint64_t nrows, double2* A, double* fro2, cudaStream_t st) {
  const u64 total = nrows << n;
  cudaError_t e = zero_parts(fro2, st);
  if (e != cudaSuccess || total == 0) return e;
  gen_dense_kernel<<<gen_blocks(total), 256, 0, st>>>(n, seed, variant, row0, nrows, A, fro2);
  return cudaGetLastError();
}

cudaError_t launch_generate_band(int n, uint64_t seed, int variant, double2* band, double* fro2,
                                 cudaStream_t st) {
  cudaError_t e = zero_parts(fro2, st);
  if (e != cudaSuccess) return e;
  gen_band_kernel<<<gen_blocks(1ull << n), 256, 0, st>>>(n, seed, variant, band, fro2);
  return cudaGetLastError();
}

cudaError_t launch_generate_sendblocks(int n, uint64_t seed, int rank, int world, int K, double2* send,
                                       double* fro2, cudaStream_t st) {
  const u64 N = 1ull << n;
  const u64 total = N * (N / (u64)world);
  cudaError_t e = zero_parts(fro2, st);
  if (e != cudaSuccess) return e;
  gen_sendblocks_kernel<<<gen_blocks(total), 256, 0, st>>>(n, seed, rank, world, K, send, fro2);
  return cudaGetLastError();
}

cudaError_t launch_sumsq(const double2* x, uint64_t count, double* partials, cudaStream_t st) {
  cudaError_t e = zero_parts(partials, st);
  if (e != cudaSuccess || count == 0) return e;
  sumsq_kernel<<<gen_blocks(count), 256, 0, st>>>(x, count, partials);
  return cudaGetLastError();
}

}  // namespace ptdr
