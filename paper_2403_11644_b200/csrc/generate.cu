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

__global__ void gen_dense_kernel(int n, u64 seed, int variant, u64 row0, u64 nrows, double2* A) {
  const u64 N = 1ull << n;
  const u64 total = nrows * N;
  for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (u64)gridDim.x * blockDim.x) {
    A[e] = dense_entry(n, seed, variant, row0 + e / N, e % N);
  }
}

__global__ void gen_sendblocks_kernel(int n, u64 seed, int rank, int world, double2* send) {
  const u64 N = 1ull << n;
  const u64 R = N / (u64)world;
  const u64 total = (u64)world * R * R;
  for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (u64)gridDim.x * blockDim.x) {
    const u64 b = e / (R * R), rr = (e / R) % R, cc = e % R;
    const u64 row = (u64)rank * R + rr;
    const u64 col = (((u64)rank ^ b) * R) + cc;
    send[e] = gauss_pair(seed, row * N + col, 0u);
  }
}

__global__ void gen_band_kernel(int n, u64 seed, int variant, double2* band) {
  const u64 N = 1ull << n;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (u64)gridDim.x * blockDim.x) {
    if (variant == 3) {
      band[i] = gauss_pair(seed, i, 1u);
      continue;
    }
    band[N + i] = make_double2(gauss_pair(seed, i, 1u).x, 0.0);
    band[2 * N + i] = (i + 1 < N) ? make_double2(gauss_pair(seed, i, 2u).x, 0.0) : make_double2(0.0, 0.0);
    band[i] = (i > 0) ? make_double2(gauss_pair(seed, i - 1, 2u).x, 0.0) : make_double2(0.0, 0.0);
  }
}

static unsigned gen_blocks(u64 total) {
  u64 b = (total + 255) / 256;
  const u64 cap = (u64)device_sm_count() * 32;
  return (unsigned)(b < cap ? b : cap);
}

cudaError_t launch_generate_dense(int n, uint64_t seed, int variant, uint64_t row0,
                                  uint64_t nrows, double2* A, cudaStream_t st) {
  const u64 total = nrows << n;
  if (total == 0) return cudaSuccess;
  gen_dense_kernel<<<gen_blocks(total), 256, 0, st>>>(n, seed, variant, row0, nrows, A);
  return cudaGetLastError();
}

cudaError_t launch_generate_band(int n, uint64_t seed, int variant, double2* band,
                                 cudaStream_t st) {
  gen_band_kernel<<<gen_blocks(1ull << n), 256, 0, st>>>(n, seed, variant, band);
  return cudaGetLastError();
}

cudaError_t launch_generate_sendblocks(int n, uint64_t seed, int rank, int world, double2* send,
                                       cudaStream_t st) {
  const u64 N = 1ull << n;
  const u64 total = N * (N / (u64)world);
  gen_sendblocks_kernel<<<gen_blocks(total), 256, 0, st>>>(n, seed, rank, world, send);
  return cudaGetLastError();
}

}  // namespace ptdr
