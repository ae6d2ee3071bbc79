// mio_bench.cu -- developer microbenchmark (not part of libptdr): per-SM throughput of the
// on-chip exchange mechanisms (LDS/STS.128, SHFL, both interleaved) and the chip-wide L2
// bandwidth for an L2-resident working set (LDG/STG).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mio_bench tools/mio_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

// 16 B per lane per op, conflict-free (lane-contiguous).
__global__ void lds_k(double2* out, int mode) {
  __shared__ double2 s[2048];
  const int t = threadIdx.x;
  double2 v = make_double2(t, t);
  double a = 0;
  for (int i = 0; i < ITERS; ++i) {
    const int idx = (t + i * 32) & 2047;
    if (mode & 1) {
      s[idx] = v;
      v = s[idx ^ 32];
      v.x += 1.0;
    }
    if (mode & 2) {
      // exchange 16 B through four 32-bit shuffles
      const int m = (i & 15) + 1;
      v.x = __shfl_xor_sync(0xffffffffu, v.x, m & 31);
      v.y = __shfl_xor_sync(0xffffffffu, v.y, m & 31);
      a += v.x;
    }
  }
  if (v.x == -1.0 || a == -1.0) out[t] = v;
}

__global__ void l2_rd(const double2* __restrict__ p, size_t n, double2* out) {
  double2 acc = make_double2(0, 0);
  for (int rep = 0; rep < 8; ++rep)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + i);
      acc.x += v.x;
      acc.y += v.y;
    }
  if (acc.x == 1.2345) out[0] = acc;
}
__global__ void l2_rw(const double2* __restrict__ p, double2* q, size_t n) {
  for (int rep = 0; rep < 8; ++rep)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      __stcg(q + i, __ldcg(p + i));
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double2* o;
  cudaMalloc(&o, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"", "lds+sts.128", "shfl x2 (16B)", "both"};
  for (int mode = 1; mode <= 3; ++mode) {
    for (int warps = 8; warps <= 32; warps *= 2) {
      lds_k<<<sms, warps * 32>>>(o, mode);
      cudaEventRecord(e0);
      lds_k<<<sms, warps * 32>>>(o, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double cyc = ms * 1e-3 * clk * 1e3;  // at the max clock (approximate)
      const double warp_ops = (double)warps * ITERS;
      printf("%-14s warps/SM %2d: %8.3f ms  %6.2f cyc per warp-iteration (max-clock est)\n", names[mode], warps,
             ms, cyc / warp_ops);
    }
  }
  for (size_t mb : {16, 32, 48, 64, 96}) {
    const size_t n = (mb << 20) / 16;
    double2 *p, *q;
    cudaMalloc(&p, n * 16);
    cudaMalloc(&q, n * 16);
    cudaMemset(p, 0, n * 16);
    l2_rd<<<sms * 4, 512>>>(p, n, o);
    cudaEventRecord(e0);
    l2_rd<<<sms * 4, 512>>>(p, n, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("L2 read  %3zu MiB: %7.1f GB/s\n", mb, 8.0 * n * 16 / ms / 1e6);
    l2_rw<<<sms * 4, 512>>>(p, q, n / 2);
    cudaEventRecord(e0);
    l2_rw<<<sms * 4, 512>>>(p, q, n / 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("L2 r+w   %3zu MiB: %7.1f GB/s (read+write bytes)\n", mb, 8.0 * n * 16 / ms / 1e6);
    cudaFree(p);
    cudaFree(q);
  }
  return 0;
}
