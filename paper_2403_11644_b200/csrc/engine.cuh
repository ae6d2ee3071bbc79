// engine.cuh -- device building blocks of the B200 Pauli-decomposition path.
//
// The identity the path is built on: for the Pauli string
// with X-mask x and Z-mask z (bit l of x set iff sigma_l in {X,Y}, bit l of z set
// iff sigma_l in {Y,Z}), PauliComposer's arrays have the
// closed form k[j] = j ^ x and m[j] = (-1)^{popcount(j & z)}, with the phase
// (-i)^{n_Y}, n_Y = popcount(x & z) (l.184).  So Alg. 2's trace (l.308-310) for
// all strings sharing x is one Walsh-Hadamard transform:
//
//   alpha(x, z) = 2^-n * i^{popcount(x&z)} * WHT_n(v_x)[z],   v_x[i] = A[i][i ^ x]
//
// (tr(P^*A) form; equal to Tr(PA) since P is Hermitian, l.128).  Everything here
// is HBM-bound data movement plus 2n FP64 adds per element; no tensor cores.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ptdr {

typedef unsigned long long u64;

constexpr int kThreads = 256;        // CTA size of every tile kernel
constexpr int kTileElems = 4096;     // complex128 elements per tile = 64 KiB of SMEM
constexpr int kTileBytes = kTileElems * 16;

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// In-register radix-2^B Walsh-Hadamard butterflies (natural order, unnormalised):
// v[j] <- sum_k (-1)^{popcount(j & k)} v[k] over the B index bits of the slice.
template <int B>
__device__ __forceinline__ void wht_regs(double2* v) {
#pragma unroll
  for (int s = 0; s < B; ++s) {
#pragma unroll
    for (int j = 0; j < (1 << B); ++j) {
      if (!(j & (1 << s))) {
        double2 a = v[j], b = v[j | (1 << s)];
        v[j] = cadd(a, b);
        v[j | (1 << s)] = csub(a, b);
      }
    }
  }
}

// Bit l of v -> bit 2l of the result (v < 2^32).
__device__ __forceinline__ u64 spread_bits(u64 v) {
  v &= 0xFFFFFFFFull;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// q order (R5): code(sigma_l) = 2 z_l + (x_l ^ z_l)
// maps I,X,Y,Z -> 0,1,2,3 and q = sum_l code_l 4^l.  With `gshift` = n - log2(world)
// the top log2(world) bits of x are the (fixed) rank and those of z give the
// block index of the rank-local output.
__device__ __forceinline__ u64 q_offset(u64 x, u64 z, int gshift) {
  const u64 m = (1ull << gshift) - 1ull;
  return ((z >> gshift) << (2 * gshift)) | spread_bits((x ^ z) & m) | (spread_bits(z & m) << 1);
}

// i^p * w for p in Z_4 (exact: swaps and negations only).
__device__ __forceinline__ double2 rot_ipow(double2 w, int p) {
  switch (p & 3) {
    case 0: return w;
    case 1: return make_double2(-w.y, w.x);
    case 2: return make_double2(-w.x, -w.y);
    default: return make_double2(w.y, -w.x);
  }
}

// Insert a 0 bit at position t.
__device__ __forceinline__ u64 insert0(u64 v, int t) {
  const u64 lo = v & ((1ull << t) - 1ull);
  return ((v >> t) << (t + 1)) | lo;
}

// ---------------------------------------------------------------------------------
// fiber_tile<K>: one 4096-element tile = F = 4096/2^K "fibers" of length 2^K.
// Computes the length-2^K WHT of every fiber:  out(f, j) = sum_k (-1)^{j.k} in(f, k).
//   ld(f, j) -> double2   element j of fiber f       (all 16 loads of a thread are
//                                                      issued before any arithmetic)
//   st(f, j, v)           final value of element j
// Stage 1: each thread owns 2^min(K,4) consecutive j of 16/2^min(K,4) fibers, radix
// in registers.  Stage 2 (K > 4): one transpose through SMEM (S[(jh*16+jl)*F + f],
// conflict-free: lanes vary f), radix-2^(K-4) in registers.  Lanes always vary the
// fiber index fastest, so loads/stores are coalesced when consecutive fibers are
// consecutive in memory.  S must hold 4096 double2.  Caller syncs before reusing S.
// ---------------------------------------------------------------------------------
template <int K, class Ld, class St>
__device__ __forceinline__ void fiber_tile(double2* S, const Ld& ld, const St& st) {
  static_assert(K >= 1 && K <= 8, "fiber length 2..256");
  constexpr int F = kTileElems >> K;
  constexpr int R1 = K < 4 ? K : 4;
  constexpr int U1 = 1 << (4 - R1);
  const int tid = threadIdx.x;
  double2 v[16];
#pragma unroll
  for (int p = 0; p < U1; ++p) {
    const int uu = tid + kThreads * p;
    const int f = uu % F, jh = uu / F;
#pragma unroll
    for (int kk = 0; kk < (1 << R1); ++kk) v[p * (1 << R1) + kk] = ld(f, (jh << R1) + kk);
  }
#pragma unroll
  for (int p = 0; p < U1; ++p) wht_regs<R1>(&v[p * (1 << R1)]);
  if constexpr (K <= 4) {
#pragma unroll
    for (int p = 0; p < U1; ++p) {
      const int uu = tid + kThreads * p;
      const int f = uu % F, jh = uu / F;
#pragma unroll
      for (int kk = 0; kk < (1 << R1); ++kk) st(f, (jh << R1) + kk, v[p * (1 << R1) + kk]);
    }
  } else {
    {
      const int f = tid % F, jh = tid / F;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) S[(jh * 16 + kk) * F + f] = v[kk];
    }
    __syncthreads();
    constexpr int R2 = K - 4;
    constexpr int U2 = 1 << (8 - K);
#pragma unroll
    for (int p = 0; p < U2; ++p) {
      const int uu = tid + kThreads * p;
      const int f = uu % F, jl = uu / F;
      double2 w[1 << R2];
#pragma unroll
      for (int jh = 0; jh < (1 << R2); ++jh) w[jh] = S[(jh * 16 + jl) * F + f];
      wht_regs<R2>(w);
#pragma unroll
      for (int jh = 0; jh < (1 << R2); ++jh) st(f, jh * 16 + jl, w[jh]);
    }
  }
}

// fiber_tile3<K> (K = 9, 10): F = 4096 / 2^K fibres of length 2^K in three register stages
// (bits 0-3, 4-7, 8..K-1) with two SMEM exchanges; element (f, j) lives at S[j F + f], so
// lanes always run along f and then the low bits of j (conflict-free, and the loads/stores
// of consecutive lanes touch consecutive fibres).  Used for whole-vector tiles at n = 9, 10.
template <int K, class Ld, class St>
__device__ __forceinline__ void fiber_tile3(double2* S, const Ld& ld, const St& st) {
  static_assert(K == 9 || K == 10, "three-stage tile");
  constexpr int F = kTileElems >> K;
  constexpr int K3 = K - 8;        // bits of the third stage
  constexpr int U3 = 16 >> K3;     // third-stage units per thread
  const int tid = threadIdx.x;
  double2 v[16];
  {  // stage 1: bits 0-3
    const int f = tid % F, jh = tid / F;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) v[kk] = ld(f, jh * 16 + kk);
    wht_regs<4>(v);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) S[(jh * 16 + kk) * F + f] = v[kk];
  }
  __syncthreads();
  {  // stage 2: bits 4-7
    const int f = tid % F, rest = tid / F;
    const int jl = rest & 15, jt = rest >> 4;
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = S[((jt * 16 + m) * 16 + jl) * F + f];
    wht_regs<4>(v);
#pragma unroll
    for (int m = 0; m < 16; ++m) S[((jt * 16 + m) * 16 + jl) * F + f] = v[m];
  }
  __syncthreads();
  // stage 3: bits 8..K-1
#pragma unroll
  for (int p = 0; p < U3; ++p) {
    const int uu = tid + kThreads * p;
    const int f = uu % F, jlow = uu / F;
#pragma unroll
    for (int q = 0; q < (1 << K3); ++q) v[p * (1 << K3) + q] = S[(q * 256 + jlow) * F + f];
  }
#pragma unroll
  for (int p = 0; p < U3; ++p) {
    const int uu = tid + kThreads * p;
    const int f = uu % F, jlow = uu / F;
    wht_regs<K3>(&v[p * (1 << K3)]);
#pragma unroll
    for (int q = 0; q < (1 << K3); ++q) st(f, q * 256 + jlow, v[p * (1 << K3) + q]);
  }
}

// Global-memory access helpers with cache hints.
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }   // read-once input
__device__ __forceinline__ double ld_stream_re(const double2* p) { return __ldcs(reinterpret_cast<const double*>(p)); }
__device__ __forceinline__ double2 ld_l2(const double2* p) { return __ldcg(p); }       // scratch: L2 only (coherent)
__device__ __forceinline__ void st_l2(double2* p, double2 v) { __stcg(p, v); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }     // write-once output

// Inter-CTA signalling inside one persistent grid (tickets are taken in order, a
// CTA only ever waits for tiles with smaller tickets, so progress is guaranteed).
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cta_wait_counter(const unsigned* p, unsigned target) {
  if (threadIdx.x == 0) {
    while (ld_acquire(p) < target) __nanosleep(64);
  }
  __syncthreads();
}
__device__ __forceinline__ void cta_signal_counter(unsigned* p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1u);
  }
}

}  // namespace ptdr
