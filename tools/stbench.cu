// stbench.cu -- developer microbenchmark (not part of libptdr): full-chip store throughput
// by store path, into an L2-resident buffer (32 MiB) and into HBM (4 GiB).
//   v2     st.global.v2.f64 (16 B per lane), 4 CTAs x 512 threads per SM
//   v4     st.global.v4.f64 (32 B per lane, sm_100 256-bit stores)
//   half   v2 with one CTA on only half of the SMs (per-SM cap vs chip cap)
//   bulk<B> cp.async.bulk.global.shared::cta of B-byte pieces from a staged SMEM tile
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stbench tools/stbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void st_v2_k(double2* buf, uint64_t n, int iters) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
      asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(buf + i), "d"((double)it), "d"((double)i) : "memory");
}

__global__ void st_v4_k(double2* buf, uint64_t n, int iters) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; 2 * i < n; i += stride)
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(buf + 2 * i), "d"((double)it), "d"((double)i),
                   "d"((double)it), "d"((double)i)
                   : "memory");
}

// one CTA per SM (big SMEM request), each CTA pushes its SMEM tile out in B-byte pieces
template <int B>
__global__ void st_bulk_k(double2* buf, uint64_t n, int iters) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int TILE = 64 * 1024;
  for (int i = threadIdx.x; i < TILE / 16; i += blockDim.x) reinterpret_cast<double2*>(sm)[i] = make_double2(i, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint64_t tiles = n * 16 / TILE;
  constexpr int PIECES = TILE / B;
  for (int it = 0; it < iters; ++it) {
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int p = threadIdx.x; p < PIECES; p += blockDim.x) {
        char* g = reinterpret_cast<char*>(buf) + t * TILE + (uint64_t)p * B;
        const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm + p * B);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(s), "n"(B)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// mixed: warps 1..nw-1 stream 16 B STG stores over bufA; warp 0 streams 16 KiB bulk stores of
// a staged SMEM tile over bufB (do the two store paths of one SM add up?)
__global__ void st_mixed_k(double2* bufA, uint64_t nA, double2* bufB, uint64_t nB, int iters, int use_bulk,
                           int use_stg) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int TILE = 64 * 1024, B = 16384;
  for (int i = threadIdx.x; i < TILE / 16; i += blockDim.x) reinterpret_cast<double2*>(sm)[i] = make_double2(i, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (!use_bulk) return;
    const uint64_t tiles = nB * 16 / TILE;
    for (int it = 0; it < iters; ++it)
      for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        if ((threadIdx.x & 31) < TILE / B) {
          const int p = threadIdx.x & 31;
          char* g = reinterpret_cast<char*>(bufB) + t * TILE + (uint64_t)p * B;
          const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm + p * B);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(s), "n"(B)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
        }
      }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    return;
  }
  if (!use_stg) return;
  const uint64_t nthr = (uint64_t)gridDim.x * (blockDim.x - 32);
  const uint64_t t0 = blockIdx.x * (uint64_t)(blockDim.x - 32) + (threadIdx.x - 32);
  for (int it = 0; it < iters; ++it)
    for (uint64_t i = t0; i < nA; i += nthr)
      asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(bufA + i), "d"((double)it), "d"((double)i) : "memory");
}

template <class F>
float best_of(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t sizes[2] = {32ull << 20, 4ull << 30};
  const char* where[2] = {"L2 32MiB", "HBM 4GiB"};
  CK(cudaFuncSetAttribute(st_bulk_k<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(st_bulk_k<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(st_bulk_k<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(st_v2_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int w = 0; w < 2; ++w) {
    const uint64_t bytes = sizes[w], n = bytes / 16;
    double2* buf;
    CK(cudaMalloc(&buf, bytes));
    const int iters = w == 0 ? 256 : 2;
    const double moved = (double)bytes * iters;
    auto rep = [&](const char* name, float ms) {
      printf("%-10s %-9s %8.3f ms  %8.1f GB/s\n", name, where[w], ms, moved / ms / 1e6);
    };
    rep("v2", best_of([&] { st_v2_k<<<sms * 4, 512>>>(buf, n, iters); }));
    rep("v4", best_of([&] { st_v4_k<<<sms * 4, 512>>>(buf, n, iters); }));
    rep("v2_1cta", best_of([&] { st_v2_k<<<sms, 1024, 200 * 1024>>>(buf, n, iters); }));
    rep("v2_halfSM", best_of([&] { st_v2_k<<<sms / 2, 1024, 200 * 1024>>>(buf, n, iters); }));
    rep("bulk512", best_of([&] { st_bulk_k<512><<<sms, 128, 200 * 1024>>>(buf, n, iters); }));
    rep("bulk2k", best_of([&] { st_bulk_k<2048><<<sms, 32, 200 * 1024>>>(buf, n, iters); }));
    rep("bulk16k", best_of([&] { st_bulk_k<16384><<<sms, 32, 200 * 1024>>>(buf, n, iters); }));
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaFree(buf));
  }

  {
    CK(cudaFuncSetAttribute(st_mixed_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    const uint64_t bytes = 32ull << 20;
    double2 *a, *b;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&b, bytes));
    const int iters = 128;
    for (int mode = 1; mode <= 3; ++mode) {
      const int ub = mode & 1, us = (mode >> 1) & 1;
      float ms = best_of([&] { st_mixed_k<<<sms, 1024, 200 * 1024>>>(a, bytes / 16, b, bytes / 16, iters, ub, us); });
      const double moved = (double)bytes * iters * (ub + us);
      printf("mixed bulk=%d stg=%d  L2 2x32MiB %8.3f ms  %8.1f GB/s total\n", ub, us, ms, moved / ms / 1e6);
    }
    CK(cudaGetLastError());
    CK(cudaFree(a));
    CK(cudaFree(b));
  }
  return 0;
}
