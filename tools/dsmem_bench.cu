// dsmem_bench.cu -- developer microbenchmark (not part of libptdr): distributed shared
// memory all-to-all bandwidth inside a thread-block cluster (16 B per lane stores to the
// other CTAs' SMEM, and cp.async.bulk SMEM->remote SMEM), cluster sizes 2..16.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_bench tools/dsmem_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int BUF = 96 * 1024;  // bytes sent per CTA per round (and received)
constexpr int ROUNDS = 200;

__global__ void st_k(int dummy) {
  extern __shared__ __align__(16) unsigned char sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), me = cl.block_rank();
  double2* src = reinterpret_cast<double2*>(sm);
  double2* dst = reinterpret_cast<double2*>(sm + BUF);
  const int per = BUF / 16 / C;  // elements to each peer
  for (int i = threadIdx.x; i < BUF / 16; i += blockDim.x) src[i] = make_double2(i, me);
  cl.sync();
  for (int r = 0; r < ROUNDS; ++r) {
    for (int i = threadIdx.x; i < BUF / 16; i += blockDim.x) {
      const int peer = (me + 1 + i / per) % C;
      double2* rd = cl.map_shared_rank(dst, peer);
      rd[me * per + (i % per)] = src[i];
    }
    cl.sync();
  }
  if (dummy == 12345) src[0] = dst[1];
}

__global__ void bulk_k(int dummy) {
  extern __shared__ __align__(128) unsigned char sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), me = cl.block_rank();
  unsigned char* src = sm;
  unsigned char* dst = sm + BUF;
  __shared__ __align__(8) uint64_t bar;
  const int per = BUF / C;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  for (int r = 0; r < ROUNDS; ++r) {
    if (threadIdx.x == 0) {
      // expect C-1 incoming chunks of `per` bytes on my barrier
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)),
                   "r"((unsigned)(per * (C - 1))));
    }
    cl.sync();
    if (threadIdx.x < C - 1) {
      const int peer = (me + 1 + threadIdx.x) % C;
      const unsigned s_local = (unsigned)__cvta_generic_to_shared(src + threadIdx.x * per);
      const unsigned d_local = (unsigned)__cvta_generic_to_shared(dst + me * per);
      const unsigned b_local = (unsigned)__cvta_generic_to_shared(&bar);
      unsigned d_remote, b_remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d_remote) : "r"(d_local), "r"(peer));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(b_remote) : "r"(b_local), "r"(peer));
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d_remote), "r"(s_local), "r"((unsigned)per), "r"(b_remote) : "memory");
    }
    if (threadIdx.x == 0) {
      const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(b), "r"((unsigned)(r & 1)));
    }
    cl.sync();
  }
  if (dummy == 12345) src[0] = dst[1];
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k = 0; k < 2; ++k) {
    auto kern = k == 0 ? st_k : bulk_k;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * BUF);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int C : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = 2 * BUF;
      int ncl = 0;
      cfg.gridDim = dim3(C);
      cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
      cfg.gridDim = dim3(ncl * C);
      cudaLaunchKernelEx(&cfg, kern, 0);
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, kern, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)ncl * C * ROUNDS * BUF * (C - 1) / C;
      printf("%s C=%2d clusters=%3d (%3d SMs): %.3f ms  %.1f GB/s total  %.1f GB/s per SM  %s\n",
             k == 0 ? "st.shared::cluster" : "cp.async.bulk     ", C, ncl, ncl * C, ms, bytes / ms / 1e6,
             bytes / ms / 1e6 / (ncl * C), cudaGetErrorString(err));
    }
  }
  return 0;
}
