// die_bench.cu -- developer microbenchmark (not part of libptdr): does keeping the dense
// pipeline's L2 hand-off on one die pay?
//
// 1. probe: every SM times dependent L2 loads into 64 granules of 2 KiB (L2 hit latency is
//    ~234 cycles near-die vs ~262 far-die on this part family, B300_MICROARCH.md); SMs whose
//    near/far patterns agree are on the same die.  Prints the SM -> die map.
// 2. hand-off: the roundtrip_bench traffic (64 KiB tile of a 16 GiB matrix -> L2 scratch ring
//    -> read back by ANOTHER CTA -> 16 GiB output), with the reader chosen
//      any  : from one global ticket queue (the pipeline today),
//      die  : from a per-die ticket queue (writer and reader on the same die),
//      self : the writer reads its own tile (roundtrip_bench's rt).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/die_bench tools/die_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kGran = 64;          // granules probed
constexpr int kGranU32 = 512;      // 2 KiB
constexpr int kChain = 24;         // dependent loads per granule

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned ldcg_u32(const unsigned* p) { unsigned v; asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }

__global__ void probe_k(const unsigned* buf, float* lat, int* sm_of_block) {
  if (threadIdx.x != 0) return;
  const unsigned s = smid();
  sm_of_block[blockIdx.x] = (int)s;
  for (int k = 0; k < kGran; ++k) {
    const unsigned* g = buf + (size_t)k * kGranU32 * 97;   // granules 194 KiB apart
    unsigned idx = 0;
    for (int w = 0; w < 4; ++w) idx = ldcg_u32(g + idx);   // warm (L2 resident)
    idx = 0;
    const long long t0 = clock64();
    for (int c = 0; c < kChain; ++c) idx = ldcg_u32(g + idx);
    const long long t1 = clock64();
    lat[(size_t)blockIdx.x * kGran + k] = (float)(t1 - t0 + (idx == 12345u ? 1 : 0)) / kChain;
  }
}

constexpr uint64_t TE = 4096;  // elements per tile (64 KiB)

// mode 0: self (read back own tile); 1: global queue; 2: per-die queue
__global__ void __launch_bounds__(256) handoff_k(const double2* __restrict__ a, double2* scratch, double2* __restrict__ out,
                                                 uint64_t tiles, uint64_t ring_tiles, unsigned* flags, unsigned* tickets,
                                                 const int* die_of_sm, uint64_t die0_tiles, int mode, int lag, int discard) {
  __shared__ unsigned long long s_t;
  const int die = die_of_sm[smid()];
  unsigned* tk = tickets + (mode == 2 ? die : 0);
  const uint64_t lo = (mode == 2 && die == 1) ? die0_tiles : 0;
  const uint64_t hi = (mode == 2 && die == 0) ? die0_tiles : tiles;
  const uint64_t mine = hi - lo;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_t = atomicAdd(tk, 1u);
    __syncthreads();
    const uint64_t k = s_t;
    if (k >= mine + (mode ? (uint64_t)lag : 0)) break;
    double2 v[16];
    if (k < mine) {  // write tile lo + k
      const uint64_t t = lo + k;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __ldcs(a + t * TE + j * 256 + threadIdx.x);
      double2* s = scratch + ((mode == 2 ? (uint64_t)die * ring_tiles : 0) + (k % ring_tiles)) * TE;
#pragma unroll
      for (int j = 0; j < 16; ++j) s[j * 256 + threadIdx.x] = v[j];
      __syncthreads();
      if (mode == 0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __ldcg(s + j * 256 + (threadIdx.x ^ 32));
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 16; ++j) __stcs(out + t * TE + j * 256 + threadIdx.x, v[j]);
        continue;
      }
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&flags[t], 1u);
      }
    }
    if (mode && k >= (uint64_t)lag) {  // read back tile lo + k - lag (written by another CTA)
      const uint64_t t = lo + k - lag;
      if (threadIdx.x == 0) {
        while (atomicAdd(&flags[t], 0u) == 0u) __nanosleep(32);
        __threadfence();
      }
      __syncthreads();
      const double2* r = scratch + ((mode == 2 ? (uint64_t)die * ring_tiles : 0) + ((k - lag) % ring_tiles)) * TE;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __ldcg(r + j * 256 + threadIdx.x);
      if (discard) {
        // drop the consumed scratch lines from L2 without write-back (as the pipeline does)
        __syncthreads();
        const char* rb = reinterpret_cast<const char*>(r);
        for (int d = threadIdx.x; d < (int)(TE * 16 / 128); d += 256)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(rb + (size_t)d * 128) : "memory");
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) __stcs(out + t * TE + j * 256 + threadIdx.x, v[j]);
    }
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // ---- 1. probe ------------------------------------------------------------------
  const size_t pbytes = (size_t)kGran * 97 * kGranU32 * 4;
  std::vector<unsigned> hb(pbytes / 4);
  for (size_t i = 0; i < hb.size(); ++i) hb[i] = (unsigned)(((i % kGranU32) * 37 + 101) % kGranU32);
  unsigned* dbuf;
  float* dlat;
  int* dsm;
  CK(cudaMalloc(&dbuf, pbytes));
  CK(cudaMemcpy(dbuf, hb.data(), pbytes, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dlat, (size_t)sms * kGran * 4));
  CK(cudaMalloc(&dsm, sms * 4));
  probe_k<<<sms, 32>>>(dbuf, dlat, dsm);  // one block per SM (148 blocks, all resident)
  CK(cudaDeviceSynchronize());
  std::vector<float> lat((size_t)sms * kGran);
  std::vector<int> smb(sms);
  CK(cudaMemcpy(lat.data(), dlat, lat.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(smb.data(), dsm, sms * 4, cudaMemcpyDeviceToHost));
  // classify: sign of the correlation of each block's pattern with block 0's
  std::vector<double> mean(kGran, 0.0);
  for (int b = 0; b < sms; ++b)
    for (int k = 0; k < kGran; ++k) mean[k] += lat[(size_t)b * kGran + k] / sms;
  std::vector<int> die_of_sm(sms, 0);
  int cnt[2] = {0, 0};
  double sep = 0;
  for (int b = 0; b < sms; ++b) {
    double c = 0, a0 = 0, ab = 0;
    for (int k = 0; k < kGran; ++k) {
      const double x = lat[k] - mean[k], y = lat[(size_t)b * kGran + k] - mean[k];
      c += x * y;
      a0 += x * x;
      ab += y * y;
    }
    const double r = c / sqrt(a0 * ab + 1e-30);
    const int d = r > 0 ? 0 : 1;
    die_of_sm[smb[b]] = d;
    cnt[d]++;
    sep += fabs(r) / sms;
  }
  printf("probe: die0 %d SMs, die1 %d SMs, mean |corr| %.3f\n", cnt[0], cnt[1], sep);
  printf("sm->die:");
  for (int s = 0; s < sms; ++s) printf("%d", die_of_sm[s]);
  printf("\n");
  {
    double near = 0, far = 0;
    int nn = 0, nf = 0;
    for (int b = 0; b < sms; ++b)
      for (int k = 0; k < kGran; ++k) {
        // granule k is "near" for die 0 if die-0 SMs see it faster than the mean
        const float v = lat[(size_t)b * kGran + k];
        const bool near0 = lat[k] < mean[k];
        const bool is_near = (die_of_sm[smb[b]] == 0) == near0;
        if (is_near) { near += v; ++nn; } else { far += v; ++nf; }
      }
    printf("latency near %.1f cycles, far %.1f cycles (classified)\n", near / nn, far / nf);
  }
  int* ddie;
  CK(cudaMalloc(&ddie, sms * 4));
  CK(cudaMemcpy(ddie, die_of_sm.data(), sms * 4, cudaMemcpyHostToDevice));
  // ---- 2. hand-off ---------------------------------------------------------------
  const uint64_t n = 1ull << 30;
  const uint64_t tiles = n / TE;
  double2 *a, *out, *scratch;
  unsigned *flags, *tickets;
  CK(cudaMalloc(&a, n * 16));
  CK(cudaMalloc(&out, n * 16));
  CK(cudaMalloc(&scratch, 512ull << 20));
  CK(cudaMalloc(&flags, tiles * 4));
  CK(cudaMalloc(&tickets, 64));
  CK(cudaMemset(a, 0, n * 16));
  const uint64_t die0_tiles = tiles * (uint64_t)cnt[0] / (uint64_t)sms;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, int mode, int mib, int lag, int cpb, int discard) {
    const uint64_t ring = ((uint64_t)mib << 20) / (TE * 16);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaMemset(flags, 0, tiles * 4);
      cudaMemset(tickets, 0, 64);
      cudaEventRecord(e0);
      handoff_k<<<sms * cpb, 256>>>(a, scratch, out, tiles, ring, flags, tickets, ddie, die0_tiles, mode, lag, discard);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    printf("%-6s ring %3d MiB lag %4d %d CTA/SM discard %d  %8.3f ms  %8.1f GB/s (32 B per element)\n", name, mib,
           lag, cpb, discard, best, 32.0 * n / best / 1e6);
  };
  for (int cpb : {2, 4}) {
    run("self", 0, 32, 0, cpb, 0);
    for (int lag : {sms * cpb / 2, sms * cpb, 2 * sms * cpb}) {
      const int mib = lag * 64 / 1024 * 2 + 16;   // ring covers twice the lag
      run("any", 1, mib, lag, cpb, 0);
      run("any", 1, mib, lag, cpb, 1);
      run("die", 2, mib, lag / 2, cpb, 1);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
