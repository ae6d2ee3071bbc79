// roundtrip_bench.cu -- developer microbenchmark (not part of libptdr): the memory traffic of
// the dense pipeline without its arithmetic or SMEM exchanges.  Every 64 KiB tile of a 16 GiB
// matrix is read from HBM, written to an L2-resident scratch ring, read back, and written to
// a 16 GiB output: HBM 32 GiB, L2 round trip 32 GiB, SM stores 32 GiB -- the dense path's
// per-launch traffic at n = 15.
//   copy        A -> out (no round trip; the copy roofline)
//   rt<SL>      A -> scratch (ring of SL MiB) -> out, each tile read back by the same CTA
//   rtx<SL>     the same, but a tile is read back by another CTA one grid-step later (the
//               pipeline's cross-SM hand-off; ordered by a per-tile flag)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/roundtrip_bench tools/roundtrip_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr uint64_t TE = 4096;  // elements per tile (64 KiB)

__device__ __forceinline__ double2 ldcs(const double2* p) { return __ldcs(p); }

__global__ void __launch_bounds__(256) copy_k(const double2* __restrict__ a, double2* __restrict__ out, uint64_t tiles) {
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    double2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = ldcs(a + t * TE + k * 256 + threadIdx.x);
#pragma unroll
    for (int k = 0; k < 16; ++k) __stcs(out + t * TE + k * 256 + threadIdx.x, v[k]);
  }
}

// cross = 0: read back own tile; cross = 1: read back the tile written one grid-step earlier
// by block (blockIdx.x + 1) % gridDim.x, after its flag says it is complete.
__global__ void __launch_bounds__(256) rt_k(const double2* __restrict__ a, double2* scratch, double2* __restrict__ out,
                                            uint64_t tiles, uint64_t ring_tiles, unsigned* flags, int cross) {
  uint64_t step = 0;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++step) {
    double2 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = ldcs(a + t * TE + k * 256 + threadIdx.x);
    double2* s = scratch + (t % ring_tiles) * TE;
#pragma unroll
    for (int k = 0; k < 16; ++k) s[k * 256 + threadIdx.x] = v[k];
    __syncthreads();
    if (!cross) {
      // read back coalesced, by another warp (warp w reads what warp w ^ 1 wrote)
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = __ldcg(s + k * 256 + (threadIdx.x ^ 32));
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) __stcs(out + t * TE + k * 256 + threadIdx.x, v[k]);
    } else {
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&flags[t], 1u);
      }
      // the tile another block wrote at the previous step
      if (step > 0) {
        const uint64_t src = t - gridDim.x + 1 < tiles ? t - gridDim.x + 1 : t;
        if (threadIdx.x == 0) {
          while (atomicAdd(&flags[src], 0u) == 0u) __nanosleep(32);
          __threadfence();
        }
        __syncthreads();
        const double2* r = scratch + (src % ring_tiles) * TE;
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = __ldcg(r + k * 256 + threadIdx.x);
#pragma unroll
        for (int k = 0; k < 16; ++k) __stcs(out + src * TE + k * 256 + threadIdx.x, v[k]);
      }
    }
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t n = 1ull << 30;  // elements (16 GiB)
  const uint64_t tiles = n / TE;
  double2 *a, *out, *scratch;
  unsigned* flags;
  CK(cudaMalloc(&a, n * 16));
  CK(cudaMalloc(&out, n * 16));
  CK(cudaMalloc(&scratch, 256ull << 20));
  CK(cudaMalloc(&flags, tiles * 4));
  CK(cudaMemset(a, 0, n * 16));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaMemset(flags, 0, tiles * 4);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    printf("%-22s %8.3f ms  %8.1f GB/s (32 B per element)\n", name, best, 32.0 * n / best / 1e6);
  };
  for (int cpb : {2, 4}) {
    char nm[64];
    snprintf(nm, sizeof nm, "copy  %d CTA/SM", cpb);
    run(nm, [&] { copy_k<<<sms * cpb, 256>>>(a, out, tiles); });
    for (int mib : {16, 32, 64}) {
      const uint64_t ring = ((uint64_t)mib << 20) / (TE * 16);
      snprintf(nm, sizeof nm, "rt  %2d MiB %d CTA/SM", mib, cpb);
      run(nm, [&] { rt_k<<<sms * cpb, 256>>>(a, scratch, out, tiles, ring, flags, 0); });
      snprintf(nm, sizeof nm, "rtx %2d MiB %d CTA/SM", mib, cpb);
      run(nm, [&] { rt_k<<<sms * cpb, 256>>>(a, scratch, out, tiles, ring, flags, 1); });
    }
  }
  CK(cudaGetLastError());
  return 0;
}
