// membench.cu -- developer microbenchmark (not part of libptdr): HBM cost of the access
// shapes the dense path uses, on a 2^15 x 2^15 complex128 matrix (16 GiB).
//   copy           sequential read 16 GiB + sequential write 16 GiB (the copy roofline)
//   rdseg<W>       read each row in W-element segments, window (row ^ x0) & ~(W-1), tiles of
//                  128 rows x W columns in chunk-major order (the phase-A gather shape);
//                  negligible writes
//   rdseg_wr<W,L>  the same reads + writes of the same volume in runs of L elements
//                  scattered with a large stride (the q-order epilogue shape)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int NB = 15;
constexpr uint64_t N = 1ull << NB;

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

// One tile = 128 rows x W columns; tile id t: chunk = t / (N/128), rowtile = t % (N/128).
template <int W, int L>
__global__ void rdseg_k(const double2* __restrict__ a, double2* __restrict__ out, int write) {
  const uint64_t tiles = (N / W) * (N / 128);
  double2 acc = make_double2(0, 0);
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint64_t chunk = t / (N / 128), rt = t % (N / 128);
    const uint64_t x0 = chunk * W;
    // 256 threads: each element (r, c) of the 128 x W tile, c fastest
    constexpr int E = 128 * W;
#pragma unroll 4
    for (int e = threadIdx.x; e < E; e += 256) {
      const uint64_t r = rt * 128 + e / W, c = e % W;
      const uint64_t col = ((r ^ x0) & ~(uint64_t)(W - 1)) + c;
      double2 v = __ldcs(a + r * N + col);
      if (write) {
        // element index inside the tile -> run of L consecutive elements, runs scattered:
        const uint64_t g = t * E + e;          // global element id
        const uint64_t run = g / L, off = g % L;
        // bit-reverse-ish scatter of runs: swap the low and high halves of the run index
        const uint64_t nruns = (N * N) / L;
        const int rb = 63 - __clzll(nruns);
        const int h = rb / 2;
        const uint64_t lo = run & ((1ull << h) - 1), hi = run >> h;
        const uint64_t pos = (lo << (rb - h)) | hi;
        __stcs(out + pos * L + off, v);
      } else {
        acc.x += v.x;
        acc.y += v.y;
      }
    }
  }
  if (!write && acc.x == 1.2345) out[blockIdx.x * 256 + threadIdx.x] = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
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
  double2 *a, *b;
  const size_t bytes = N * N * 16;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 0, bytes));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double gb = bytes / 1e9;
  float ms = timeit([&] { copy_k<<<sms * 8, 512>>>(a, b, N * N); });
  printf("copy                 %8.3f ms  %7.1f GB/s (r+w)\n", ms, 2 * gb / ms * 1e3);
#define RD(W)                                                                                  \
  ms = timeit([&] { rdseg_k<W, 32><<<sms * 8, 256>>>(a, b, 0); });                             \
  printf("rdseg W=%-4d          %8.3f ms  %7.1f GB/s (read)\n", W, ms, gb / ms * 1e3);
  RD(4) RD(8) RD(16) RD(32) RD(64) RD(128) RD(256)
#define RW(W, L)                                                                               \
  ms = timeit([&] { rdseg_k<W, L><<<sms * 8, 256>>>(a, b, 1); });                              \
  printf("rdseg_wr W=%-4d L=%-4d %8.3f ms  %7.1f GB/s (r+w)\n", W, L, ms, 2 * gb / ms * 1e3);
  RW(4, 16) RW(8, 16) RW(32, 16) RW(32, 32) RW(32, 64) RW(64, 32) RW(64, 64) RW(128, 64) RW(256, 256)
  CK(cudaGetLastError());
  return 0;
}
