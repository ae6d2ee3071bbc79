// dense_launch.cuh -- host launcher template for one MODE of the dense path.
// Each dense_mode<k>.cu instantiates it for one MODE so the ~50 kernel
// instantiations compile in parallel translation units.
#pragma once
#include <atomic>
#include <mutex>

#include "dense_impl.cuh"
#include "dense_plan.h"
#include "internal.h"

namespace ptdr {

template <auto kernel>
static cudaError_t prep_kernel(int* blocks_per_sm) {
  // the shared-memory attribute once per (kernel, device); the occupancy (identical on every
  // B200) queried after it
  static std::atomic<int> cached[64];  // per device; 0 = not queried yet
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev >= 0 && dev < 64) {
    const int c = cached[dev].load(std::memory_order_relaxed);
    if (c > 0) {
      *blocks_per_sm = c;
      return cudaSuccess;
    }
  }
  err = ensure_smem_attr(reinterpret_cast<const void*>(kernel), kTileBytes);
  if (err != cudaSuccess) return err;
  int bps = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, kThreads, kTileBytes);
  if (err == cudaSuccess && bps < 1) err = cudaErrorInvalidConfiguration;
  if (err == cudaSuccess && dev >= 0 && dev < 64) cached[dev].store(bps, std::memory_order_relaxed);
  *blocks_per_sm = bps;
  return err;
}

template <int R, int M, int MODE>
static cudaError_t launch_fused(const DenseArgs& a, u64 total_tiles, cudaStream_t st) {
  constexpr auto kern = dense_fused_kernel<R, M, MODE>;
  int bps = 0;
  cudaError_t e = prep_kernel<kern>(&bps);
  if (e != cudaSuccess) return e;
  u64 grid = (u64)device_sm_count() * (u64)bps;
  if (grid > total_tiles) grid = total_tiles;
  kern<<<(unsigned)grid, kThreads, kTileBytes, st>>>(a);
  return cudaGetLastError();
}

template <int R, int MODE>
static cudaError_t launch_single(const DenseArgs& a, u64 ntiles, cudaStream_t st) {
  constexpr auto kern = dense_single_kernel<R, MODE>;
  int bps = 0;
  cudaError_t e = prep_kernel<kern>(&bps);
  if (e != cudaSuccess) return e;
  u64 grid = (u64)device_sm_count() * (u64)bps;
  const u64 all = ntiles * (a.batch ? a.batch : 1);
  if (grid > all) grid = all;
  kern<<<(unsigned)grid, kThreads, kTileBytes, st>>>(a);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_dense_mode_impl(const DenseArgs& a_in, const DensePlan& p, cudaStream_t st,
                                   int* nlaunch) {
  DenseArgs a = a_in;
  if (p.kind == 0) {
    if constexpr (MODE <= MODE_SYM_MIRROR) {
      const u64 nx = a.nchunks * 16 > (1ull << a.n) ? (1ull << a.n) : a.nchunks * 16;
      const u64 total = (nx << a.n) * (a.batch ? a.batch : 1);
      const unsigned blocks = (unsigned)((total + 255) / 256);
      dense_direct_kernel<MODE><<<blocks, 256, 0, st>>>(a, nx);
      *nlaunch += 1;
      return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
  }
  if (p.kind == 1) {
    {
      const u64 nx = a.nchunks * 16;
      *nlaunch += 1;
      switch (p.R) {
        case 6: return launch_single<6, MODE>(a, nx / (kTileElems >> 6), st);
        case 7: return launch_single<7, MODE>(a, nx / (kTileElems >> 7), st);
        case 8: return launch_single<8, MODE>(a, nx / (kTileElems >> 8), st);
        case 9: return launch_single<9, MODE>(a, nx / (kTileElems >> 9), st);
        case 10: return launch_single<10, MODE>(a, nx / (kTileElems >> 10), st);
        default: break;
      }
    }
    return cudaErrorInvalidValue;
  }
  // two-phase
  a.L = p.L;
  a.nslot = p.nslot;
  a.slot_elems = p.slot_elems;
  cudaError_t e = cudaMemsetAsync(a.ctr, 0, p.ctr_bytes, st);
  if (e != cudaSuccess) return e;
  const u64 total = a.nchunks * (u64)(p.NA + p.NB);
  *nlaunch += 1;
  switch (p.nv) {
    case 8: return launch_fused<4, 4, MODE>(a, total, st);
    case 9: return launch_fused<5, 4, MODE>(a, total, st);
    case 10: return launch_fused<6, 4, MODE>(a, total, st);
    case 11: return launch_fused<7, 4, MODE>(a, total, st);
    case 12: return launch_fused<8, 4, MODE>(a, total, st);
    case 13: return launch_fused<8, 5, MODE>(a, total, st);
    case 14: return launch_fused<8, 6, MODE>(a, total, st);
    case 15: return launch_fused<8, 7, MODE>(a, total, st);
    case 16: return launch_fused<8, 8, MODE>(a, total, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ptdr

#define PTDR_DEFINE_DENSE_MODE(MODE)                                                       \
  namespace ptdr {                                                                         \
  cudaError_t launch_dense_mode##MODE(const DenseArgs& a, const DensePlan& p, cudaStream_t st, \
                                      int* nlaunch) {                                      \
    return launch_dense_mode_impl<MODE>(a, p, st, nlaunch);                                \
  }                                                                                        \
  }
