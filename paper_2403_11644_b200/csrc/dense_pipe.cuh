// dense_pipe.cuh -- warp-specialised TMA pipeline for the dense path (two-phase, nv >= 11).
//
// Same math as dense_impl.cuh (phase A: XOR-transpose gather + WHT over the low R index
// bits into the scratch; phase B: WHT over the high M = nv - R bits + epilogue in q
// order), organised for sm_100a:
//   * one CTA per SM; warp 0 lane 0 = producer (tickets, inter-CTA dependency checks
//     prefetched one tile ahead, TMA issue); NG consumer groups of GW warps take tiles
//     round-robin from an NS-stage SMEM ring (mbarrier full/empty pipeline);
//   * phase-A tiles (2^(R-4) row blocks of 16 x 16 complex128) arrive by 2-D TMA
//     (cp.async.bulk.tensor), phase-B tiles (one contiguous 2^LT-element block of the
//     B-tile-major scratch) by 1-D bulk copy;  HBM loads of later tiles overlap the
//     arithmetic of earlier ones;
//   * the XOR transpose happens in the SMEM read (conflict-free); the exchange between
//     the two radix-16 register stages is done in place in the stage buffer;
//   * consumed scratch lines are discarded from L2 (never written back to HBM);
//   * completion counters are bumped per warp with release atomics (no CTA barrier).
// Tile = 2^LT complex128 (LT = R + 4); a group has 2^(LT-4) threads holding 16 each.
#pragma once
#include <cudaTypedefs.h>

#include <cstdlib>
#include <numeric>
#include <mutex>

#include "dense_impl.cuh"
#include "dense_plan.h"
#include "internal.h"
#include "philox.cuh"
#include "sm100_ptx.cuh"

namespace ptdr {

// Developer diagnostics (PTDR_DIAG_BUILD=<bits>; never in the product library):
//   bit 0: phase B computes but does not store the output (isolates the read side);
//   bit 1: phase-A TMA loads come from the first 256 rows of A (L2-resident: isolates
//          the write side);
//   bit 2: no butterflies (pure data movement through the same pipeline);
//   bit 4: phase A skips its SMEM exchange (STS + LDS); bit 5: phase B skips its exchange.
#ifndef PTDR_DIAG
#define PTDR_DIAG 0
#endif
constexpr int kDiag = PTDR_DIAG;
// bit 2 (diagnostics): skip the radix butterflies (data movement only)
// bit 6 (diagnostics): output stores without the streaming hint; bit 7: output stores with
// an L2 evict-first policy (createpolicy) instead of .cs
__device__ __forceinline__ void st_out(double2* p, double2 v) {
  if constexpr ((kDiag & 64) != 0) {
    *p = v;
  } else if constexpr ((kDiag & 128) != 0) {
    st_global_hint(p, v, policy_evict_first());
  } else {
    st_stream(p, v);
  }
}
template <int B>
__device__ __forceinline__ void pwht(double2* v) {
  if constexpr ((kDiag & 4) == 0) wht_regs<B>(v);
}

// Tensor maps of the A source: one (the local matrix or shard), or one per rank's row-block
// shard in peer-pull mode (ptdr_decompose_peer_async).
constexpr int kMaxPeers = 8;
struct TmapSet {
  CUtensorMap m[kMaxPeers];
};

struct TileMeta {
  int valid, phase, tile, seq;
  unsigned chunk, slot, pad1, pad2;
};

// Completion counters are read with ld.acquire.gpu by default (the acquire half of the
// signalers' red.release; measured free); the relaxed form below is a
// developer variant.  Either way the scratch is then fetched by the TMA from L2 after
// fence.proxy.async.global.
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Debug timeline (PTDR_TRACE=1): CTA 0 records clock64 stamps of its first kTraceTiles
// tiles into a.trace[tile * 16 + field].
constexpr int kTraceTiles = 512;
// Compiled in only with -DPTDR_ENABLE_TRACE=1 (PTDR_TRACE_BUILD=1 python build.py).
#ifndef PTDR_ENABLE_TRACE
#define PTDR_ENABLE_TRACE 0
#endif
__device__ __forceinline__ void trace_stamp(unsigned long long* tr, int k, int field) {
  if constexpr (PTDR_ENABLE_TRACE) {
    if (tr != nullptr && blockIdx.x == 0 && k < kTraceTiles) tr[k * 16 + field] = clock64();
  }
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- 32-bit index arithmetic: n <= 16 so x, z < 2^16 and q < 2^32 ----------------------
__device__ __forceinline__ uint32_t spread16(uint32_t v) {
  v &= 0xFFFFu;
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__device__ __forceinline__ uint32_t q_offset32(uint32_t x, uint32_t z, int gshift) {
  const uint32_t m = (gshift >= 32) ? 0xFFFFFFFFu : ((1u << gshift) - 1u);
  const uint32_t top = (gshift >= 16) ? 0u : ((z >> gshift) << (2 * gshift));
  return top | spread16((x ^ z) & m) | (spread16(z & m) << 1);
}
// q delta of setting z bit l (code_l = 2 z_l + (x_l ^ z_l); above gshift the z bit
// indexes the rank-local block).
__device__ __forceinline__ uint32_t q_delta32(uint32_t x, int l, int gshift) {
  return (l < gshift) ? ((uint32_t)(3 - 2 * (int)((x >> l) & 1u)) << (2 * l)) : (1u << (l + gshift));
}
// Matrix layout (in-place decomposition): alpha(x, z) at z 2^n + (z ^ x); setting z bit l
// adds 2^(l+n) and flips bit l of z ^ x (+2^l if x_l = 0, -2^l if x_l = 1).  n <= 16, so
// every index fits 32 bits (mod-2^32 arithmetic handles the negative deltas).
__device__ __forceinline__ uint32_t mat_offset32(uint32_t x, uint32_t z, int n) { return (z << n) | (z ^ x); }
__device__ __forceinline__ uint32_t mat_delta32(uint32_t x, int l, int n) {
  return (1u << (l + n)) + (((x >> l) & 1u) ? (0u - (1u << l)) : (1u << l));
}
__device__ __forceinline__ uint32_t insert0_32(uint32_t v, int t) {
  const uint32_t lo = v & ((1u << t) - 1u);
  return ((v >> t) << (t + 1)) | lo;
}

// Epilogue of one thread-unit: q offset and phase of the unit's base (x, z) plus per-bit
// deltas for the NB z bits that vary over the unit's registers (compile-time subsets).
template <int NB, bool HALF>
struct EpiUnit {
  uint32_t q0, p0, Dt;
  uint32_t D[NB];
  uint32_t P[NB];
  // mat_n = 0: q order (gshift: rank-local blocks); mat_n = n: matrix layout
  __device__ __forceinline__ void init(uint32_t x, uint32_t zu, int base_pos, int t, int gshift, int mat_n) {
    const uint32_t zf = HALF ? insert0_32(zu, t) : zu;
    q0 = mat_n ? mat_offset32(x, zf, mat_n) : q_offset32(x, zf, gshift);
    p0 = __popc(x & zf);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      int l = base_pos + b;
      if (HALF) l += (l >= t) ? 1 : 0;
      D[b] = mat_n ? mat_delta32(x, l, mat_n) : q_delta32(x, l, gshift);
      P[b] = (x >> l) & 1u;
    }
    Dt = HALF ? (mat_n ? mat_delta32(x, t, mat_n) : q_delta32(x, t, gshift)) : 0u;
  }
};

// One output register: alpha = 2^-n i^p w at q (GENERAL), or the two real outputs of the
// half-length modes.  Branch-free: i^p w * scale = (p&1 ? (-w.y, w.x) : (w.x, w.y)) *
// (p&2 ? -scale : scale).
template <int MODE>
__device__ __forceinline__ void emit_one(const DenseArgs& a, uint32_t q, uint32_t p, uint32_t dt,
                                         double2 w) {
  if constexpr (MODE == MODE_INV || MODE == MODE_INVQ) {
    st_out(a.out + q, w);  // the inverse: A[i][i ^ x] = WHT(u_x)[i], no phase, no scale
  } else if constexpr (MODE == MODE_GENERAL || MODE == MODE_GEN) {
    const bool sw = (p & 1u) != 0;
    const double s = (p & 2u) ? -a.scale : a.scale;
    const double re = sw ? -w.y : w.x;
    const double im = sw ? w.x : w.y;
    if constexpr ((kDiag & 1) != 0) {
      if (re == 12345.678) st_stream(a.out + q, make_double2(re * s, im * s));  // keeps the math live
    } else {
      st_out(a.out + q, make_double2(re * s, im * s));
    }
  } else {
    // half-length modes: alpha = 2^{1-n} {Re, -Im, -Re, Im}[p mod 4] for z_t = 0 and the
    // same with p + 1 for z_t = 1 (real)
    const double s = 2.0 * a.scale;
    const uint32_t p1 = p + 1u;
    const double v0 = ((p & 1u) ? w.y : w.x) * ((((p ^ (p >> 1)) & 1u) != 0) ? -s : s);
    const double v1 = ((p1 & 1u) ? w.y : w.x) * ((((p1 ^ (p1 >> 1)) & 1u) != 0) ? -s : s);
    st_out(a.out + q, make_double2(v0, 0.0));
    st_out(a.out + (q + dt), make_double2(v1, 0.0));
  }
}

// All 2^NB registers of a unit, visited in Gray-code order so that consecutive outputs
// differ in one z bit: q and p are updated with one add each (q += +-D[b], p += +-P[b]).
template <int MODE, int NB, int I = 0>
__device__ __forceinline__ void emit_gray(const DenseArgs& a, const EpiUnit<NB, (MODE == 3 || MODE == 4)>& e,
                                          const double2* w, uint32_t q, uint32_t p) {
  if constexpr (I < (1 << NB)) {
    constexpr int J = I ^ (I >> 1);
    if constexpr (I > 0) {
      constexpr int PREV = (I - 1) ^ ((I - 1) >> 1);
      constexpr int B = __builtin_ctz(J ^ PREV);
      if constexpr ((J >> B) & 1) {
        q += e.D[B];
        p += e.P[B];
      } else {
        q -= e.D[B];
        p -= e.P[B];
      }
    }
    emit_one<MODE>(a, q, p, e.Dt, w[J]);
    emit_gray<MODE, NB, I + 1>(a, e, w, q, p);
  }
}

template <int MODE, int NB>
__device__ __forceinline__ void emit_all(const DenseArgs& a, const EpiUnit<NB, (MODE == 3 || MODE == 4)>& e,
                                         const double2* w) {
  emit_gray<MODE, NB, 0>(a, e, w, e.q0, e.p0);
}

// Ticket order of dense_impl.cuh's decode_ticket, 32-bit, NA = NB = 2^M.
__device__ __forceinline__ void decode_ticket32(uint32_t t, int M, uint32_t C, uint32_t L, int& phase,
                                                uint32_t& chunk, uint32_t& tile) {
  const uint32_t NA = 1u << M;
  const uint32_t lp1 = (L + 1u < C) ? L + 1u : C;
  const uint32_t pro = lp1 << M;
  if (t < pro) {
    phase = 0; chunk = t >> M; tile = t & (NA - 1u);
    return;
  }
  t -= pro;
  const uint32_t steady = C > L + 1u ? C - L - 1u : 0u;
  if (t < (steady << (M + 1))) {
    const uint32_t c = t >> (M + 1), o = t & (2u * NA - 1u);
    if (o < NA) { phase = 1; chunk = c; tile = o; }
    else { phase = 0; chunk = c + L + 1u; tile = o - NA; }
    return;
  }
  t -= steady << (M + 1);
  phase = 1; chunk = steady + (t >> M); tile = t & (NA - 1u);
}

// NR = 0: the radix stages exchange in place in the stage buffer, which is released after
// the exchange.  NR = 2 ("early release"): each group owns an exchange buffer of half a
// tile; the stage is released right after its first read into registers and the exchange
// runs in two rounds (exchange_rounds / xor_half_transpose below).
template <int LT, int XB, int GW, int NG, int NS, int NR = 0>
struct PipeCfg {
  static constexpr int TE = 1 << LT;          // tile elements
  static constexpr int TB = TE * 16;          // tile bytes
  static constexpr int W = 1 << XB;           // X-masks per chunk (TMA box = W rows x W cols)
  static constexpr int R = LT - XB;           // phase-A index bits (rows per phase-A tile = 2^R)
  static constexpr int GT = GW * 32;          // threads per group (= TE / 16)
  static constexpr int SIGD = 4;               // completion-signal slots per group
  // Warpgroup 0 (warps 0-3): warp 0 producer, warp 1 signaler, warps 2-3 idle; they give
  // their registers back (setmaxnreg) to the consumer warpgroups that follow.
  static constexpr int THREADS = 32 * (4 + NG * GW);
  static constexpr int CONS_THREADS = 32 * NG * GW;
  static_assert(CONS_THREADS % 128 == 0, "consumer warps form whole warpgroups");
  // The CTA's register pool is fixed at launch (THREADS x LAUNCH_REGS, LAUNCH_REGS = what
  // ptxas allocates under __launch_bounds__(THREADS, 1)); setmaxnreg.inc blocks until the
  // pool can satisfy it, so PROD_REGS x 128 + CONS_REGS x CONS_THREADS must fit in it.
  static constexpr int LAUNCH_REGS = ((65536 / THREADS) / 8) * 8 > 248 ? 248 : ((65536 / THREADS) / 8) * 8;
  static constexpr int PROD_REGS = 40;
  static constexpr int CONS_REGS_RAW = ((THREADS * LAUNCH_REGS - PROD_REGS * 128) / CONS_THREADS / 8) * 8;
  static constexpr int CONS_REGS = CONS_REGS_RAW > 248 ? 248 : CONS_REGS_RAW;
  static_assert(CONS_REGS >= LAUNCH_REGS && PROD_REGS * 128 + CONS_REGS * CONS_THREADS <= THREADS * LAUNCH_REGS,
                "register rebalancing must fit the launch-time pool");
  static constexpr int XE = NR ? TE / NR : 0;  // exchange-buffer elements per group
  static constexpr int SMEM = NS * TB + NG * XE * 16 + 2048;
  static_assert(GT * 16 == TE, "16 elements per consumer thread");
  static_assert(NR == 0 || NR == 2, "exchange rounds");
  static_assert(SMEM <= 227 * 1024, "shared memory per CTA");
};

// Fiber index of the phase-B tiles: phi encodes (u, zl) with bits [0,1]=u0,u1 [2,3]=zl0,zl1
// [4, XB+2)=u2.. [XB+2, ..)=zl2.., so 2^k consecutive fibers form a (u, zl) square of
// 4^(k/2) consecutive q (coalesced epilogue stores).

// In the matrix layout of the in-place decomposition (A[z][z ^ x]) consecutive addresses
// are consecutive X-masks of one z instead, so there the fibre index is simply
// phi = u | zl << XB: 2^XB lanes store one 2^XB x 16 B run.
template <int XB>
__device__ __forceinline__ uint32_t phi_of(uint32_t u, uint32_t zl, bool mat) {
  if (mat) return u | (zl << XB);
  return (u & 3u) | ((zl & 3u) << 2) | ((u >> 2) << 4) | ((zl >> 2) << (XB + 2));
}
template <int XB>
__device__ __forceinline__ uint32_t phi_u_of(uint32_t phi, bool mat) {
  if (mat) return phi & ((1u << XB) - 1u);
  return (phi & 3u) | (((phi >> 4) & ((1u << (XB - 2)) - 1u)) << 2);
}
template <int XB>
__device__ __forceinline__ uint32_t phi_zl_of(uint32_t phi, bool mat) {
  if (mat) return phi >> XB;
  return ((phi >> 2) & 3u) | ((phi >> (XB + 2)) << 2);
}

// ---- exchange between the two radix stages through a half-tile buffer X (early release) --
// Stage 1 leaves thread (c, a) with v[kk] = T[a][kk] (a = its row block, kk = 16 register
// indices) for the column c it owns (X-mask u in phase A, fibre f in phase B; lanes run
// along c, STR = number of columns).  Stage 2 needs, for unit p = (c, jl = a + 2^R2 p),
// the 2^R2 values T[j][jl], j < 2^R2.  With U >= 2 units per thread, the units whose jl
// falls in [8h, 8h+8) take exactly the registers v[8h..8h+8) that round h frees, so both
// rounds are compile-time register maps: on exit v[p 2^R2 + j] = T[j][a + 2^R2 p].
template <int R2, int U, int STR>
__device__ __forceinline__ void exchange_rounds(double2 (&v)[16], double2* X, int a, int c, int bar_id,
                                                int nthr) {
  static_assert(U * (1 << R2) == 16 && U >= 2, "two rounds of 8 registers");
  constexpr int PH = U / 2;  // units per round
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int kq = 0; kq < 8; ++kq) X[(a * 8 + kq) * STR + c] = v[8 * h + kq];
    named_bar_sync(bar_id, nthr);
#pragma unroll
    for (int pp = 0; pp < PH; ++pp) {
      const int jl = a + (1 << R2) * (h * PH + pp);  // in [8h, 8h+8)
#pragma unroll
      for (int jj = 0; jj < (1 << R2); ++jj) v[8 * h + pp * (1 << R2) + jj] = X[(jj * 8 + (jl - 8 * h)) * STR + c];
    }
    named_bar_sync(bar_id, nthr);
  }
}

// One unit of 16 (R2 = 4): a full 16 x 16 transpose per column through half a tile.  Entry
// (j, kk) travels in round bit3(j ^ kk), so each round every thread sends 8 and receives 8
// values; a thread whose row a has bit 3 set swaps its register halves before and after
// (warp-uniform: a = 2 warp + lane/16 or coarser).  On exit v[j] = T[j][a].
template <int STR>
__device__ __forceinline__ void xor_half_transpose(double2 (&v)[16], double2* X, int a, int c, int bar_id,
                                                   int nthr) {
  const bool b = ((a >> 3) & 1) != 0;
  auto swap_halves = [&]() {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double2 lo = v[q], hi = v[q + 8];
      v[q] = b ? hi : lo;
      v[q + 8] = b ? lo : hi;
    }
  };
  swap_halves();  // v[q] = T[a][q ^ 8b]
  const int jb = b ? 8 : 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) X[(a * 8 + q) * STR + c] = v[q];
  named_bar_sync(bar_id, nthr);
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = X[((q + jb) * 8 + (a & 7)) * STR + c];      // T[q + 8b][a]
  named_bar_sync(bar_id, nthr);
#pragma unroll
  for (int q = 0; q < 8; ++q) X[(a * 8 + q) * STR + c] = v[q + 8];
  named_bar_sync(bar_id, nthr);
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q + 8] = X[((q + 8 - jb) * 8 + (a & 7)) * STR + c];  // T[q + 8(1-b)][a]
  named_bar_sync(bar_id, nthr);
  swap_halves();  // v[j] = T[j][a]
}

// Scratch layout (per chunk slot): B-tile-major Y[tileB][ih][f], 2^LT elements per phase-B
// tile, so a phase-B tile is one contiguous bulk copy (fiber phi = tileB * FB + f).
template <int LT, int XB, int GW, int NG, int NS, int NR, int M, int MODE>
__global__ void __launch_bounds__(PipeCfg<LT, XB, GW, NG, NS, NR>::THREADS, 1)
    dense_pipe_kernel(const __grid_constant__ TmapSet maps, DenseArgs a) {
  using Cfg = PipeCfg<LT, XB, GW, NG, NS, NR>;
  constexpr int R = Cfg::R, TE = Cfg::TE, GT = Cfg::GT, W = Cfg::W;
  constexpr bool HALF = (MODE == MODE_HERM_HALF || MODE == MODE_SYM_HALF);
  constexpr int FB = TE >> M;  // phase-B fibers per tile
  constexpr int kLcm = NS * NG / std::gcd(NS, NG);
  constexpr int LFB = LT - M;
  static_assert(M >= 4 && M <= 8 && LFB <= XB + 4, "phase-B fibre length 2^4..2^8");
  static_assert(R >= XB && R - 4 >= 1 && R - 4 <= 4, "phase-A tile geometry");
  extern __shared__ __align__(1024) unsigned char smem[];
  double2* stage0 = reinterpret_cast<double2*>(smem);
  double2* xbuf = reinterpret_cast<double2*>(smem + NS * Cfg::TB);  // [NG][XE] (NR > 0)
  // full barriers per (stage, group): tile k lands in stage k % NS for group k % NG, so the
  // barrier full[s NG + g] completes once per LCM = lcm(NS, NG) tiles and a group waiting for
  // tile k can never see an older phase of it (the previous one, tile k - LCM, is its own
  // and already consumed): a plain parity wait, the warps sleep in hardware until the data
  // lands (no polling of a sequence number)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * Cfg::TB + NG * Cfg::XE * 16);
  uint64_t* empty = full + NS * NG;
  // 32-byte aligned (the producer publishes a tile's metadata with a 16-byte store)
  TileMeta* meta = reinterpret_cast<TileMeta*>(
      (reinterpret_cast<uintptr_t>(empty + NS) + 31) & ~static_cast<uintptr_t>(31));
  constexpr int SIGD = Cfg::SIGD;
  uint64_t* sigbar = reinterpret_cast<uint64_t*>(meta + NS);  // [NG][SIGD], count GW
  uint64_t* sigfree = sigbar + NG * SIGD;                       // [NG][SIGD], count 1
  unsigned** sigptr = reinterpret_cast<unsigned**>(sigfree + NG * SIGD);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t C = (uint32_t)a.nchunks;
  unsigned* ticket = a.ctr;
  unsigned* doneA = a.ctr + 1;
  unsigned* doneB = a.ctr + 1 + C;
  const uint32_t nslot = (uint32_t)a.nslot;           // a power of two (dense_plan.h)
  const uint32_t slot_mask = nslot - 1u;
  const int slot_shift = __ffsll((long long)a.slot_elems) - 1;  // slot_elems = W << nv
  const unsigned done_target = 1u << M;  // one completion signal per tile

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS * NG; ++i) mbar_init(&full[i], 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&empty[s], GW);
      meta[s].seq = -1;
    }
    for (int i = 0; i < NG * SIGD; ++i) {
      mbar_init(&sigbar[i], GW);
      mbar_init(&sigfree[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::PROD_REGS));

  // ------------------------------------------------------------------ producer
  if (warp == 0) {
    if (lane == 0) {
      for (int pm = 0; pm < (a.peer_shift ? a.npeers : 1); ++pm) prefetch_tmap(&maps.m[pm]);
      const uint64_t pol = policy_of(a.pol_a), pol_sl = policy_of(a.pol_b);
      const uint32_t total = C << (M + 1);
      // Decoded ticket: (tk, phase, chunk, tile) and its dependency counter, whose value is
      // requested (dv) one tile before it is checked.
      auto decode_into = [&](uint32_t tk, uint32_t& tkX, int& phX, uint32_t& chX, uint32_t& tlX,
                             const unsigned*& depX, unsigned& dvX) {
        tkX = tk;
        phX = 0; chX = 0; tlX = 0;
        depX = nullptr;
        dvX = 0;
        if (tk < total) {
          decode_ticket32(tk, M, C, (uint32_t)a.L, phX, chX, tlX);
          if (phX == 1) depX = &doneA[chX];
          else if (chX >= nslot) depX = &doneB[chX - nslot];
          if (depX) dvX = a.acq_fence == 2 ? ld_acquire(depX) : ld_relaxed(depX);
        }
      };
      int k = 0, ends = 0;
      // Publish one tile (or an end marker) into stage k % NS.  Returns true when all
      // groups have received their end marker.
      auto process = [&](const uint32_t& tkX, const int& phX, const uint32_t& chX,
                         const uint32_t& tlX, const unsigned* const& depX,
                         const unsigned& dvX) -> bool {
        const int s = k % NS;
        uint64_t* fullk = &full[s * NG + k % NG];
        trace_stamp(a.trace, k, 0);
        if (k >= NS) mbar_wait(&empty[s], (uint32_t)((k / NS) - 1) & 1u);
        trace_stamp(a.trace, k, 1);
        if (tkX >= total) {
          // one invalid tile per group ends the consumers
          meta[s].valid = 0;
          meta[s].seq = k;
          mbar_arrive(fullk);
          ++k;
          return ++ends == NG;
        }
        if (depX) {
          unsigned v = dvX;
          while (v < done_target) {
            __nanosleep(64);
            v = a.acq_fence == 2 ? ld_acquire(depX) : ld_relaxed(depX);
          }
          // developer variant: a fence after the wait (the acquire pattern of the PTX memory
          // model); measured 10 % slower, see launch_dense_pipe
          if (a.acq_fence == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        trace_stamp(a.trace, k, 2);
        if (PTDR_ENABLE_TRACE && a.trace && blockIdx.x == 0 && k < kTraceTiles) a.trace[k * 16 + 8] = phX;
        double2* dst = stage0 + (size_t)s * TE;
        // one 16-byte and one 4-byte shared store instead of five
        *reinterpret_cast<int4*>(&meta[s]) = make_int4(1, phX, (int)tlX, k);
        const uint32_t gch = chX, slot = chX & slot_mask;
        meta[s].chunk = gch;
        meta[s].slot = slot;
        if (phX == 0 && MODE == MODE_GEN) {
          mbar_arrive(fullk);  // matrix-free: the consumers generate the tile's entries
        } else if (phX == 0 && MODE == MODE_INVQ) {
          // inverse from q order: the W x W (X-mask low bits, z low bits) combinations of a
          // box are W^2 consecutive q (the low 2 XB bits of q): one TMA box of W^2 / 8 rows of
          // the [4^n / 8][8] view, 128-byte swizzled (launch_dense_pipe)
          mbar_arrive_expect_tx(fullk, (uint32_t)Cfg::TB);
          // zh = (tlX << (R - XB)) + rb: spread() is linear over XOR and the low R - XB bits of
          // zh are rb, so the producer spreads once per tile and adds a constant per box
          const uint32_t xh = ((uint32_t)a.x_base + (gch << XB)) >> XB;
          const uint32_t zh0 = tlX << (R - XB);
          const uint64_t b0 = spread_bits((uint64_t)(xh ^ zh0)) | (spread_bits((uint64_t)zh0) << 1);
#pragma unroll
          for (int rb = 0; rb < (1 << (R - XB)); ++rb) {
            const uint64_t qb = (b0 ^ (3ull * spread_bits((uint64_t)rb))) << (2 * XB);
            tma_load_2d(dst + rb * W * W, &maps.m[0], 0, (int)(qb >> 3), fullk, pol);
          }
        } else if (phX == 0) {
          mbar_arrive_expect_tx(fullk, (uint32_t)Cfg::TB);
          const uint32_t x0 = (uint32_t)a.x_base + (gch << XB);
          const int t = HALF ? 31 - __clz(x0) : 0;
          const uint32_t cm = (uint32_t)a.colmask & ~(uint32_t)(W - 1);
          // peer-pull: all rows of a tile lie in one rank's shard (R >= rows per tile), so
          // the tensor map and the row mask are chosen once per tile
          const CUtensorMap* tm = &maps.m[0];
          uint32_t rmask = 0xFFFFFFFFu;
          if (a.peer_shift) {
            const uint32_t r0 = (tlX << R);
            tm = &maps.m[r0 >> a.peer_shift];
            rmask = (uint32_t)a.peer_rowmask;
          }
#pragma unroll
          for (int rb = 0; rb < (1 << (R - XB)); ++rb) {
            const uint32_t iv0 = (tlX << R) + (uint32_t)rb * W;
            uint32_t row0 = HALF ? insert0_32(iv0, t) : iv0;
            if constexpr ((kDiag & 2) != 0) row0 &= 255u;
            const uint32_t col0 = (row0 ^ x0) & cm;
            tma_load_2d(dst + rb * W * W, tm, (int)(col0 * 2u), (int)(row0 & rmask), fullk, pol);
          }
        } else {
          // scratch written by other CTAs' generic stores, read by the async proxy
          fence_proxy_async_global();
          mbar_arrive_expect_tx(fullk, (uint32_t)Cfg::TB);
          const double2* src = a.scratch + ((size_t)slot << slot_shift) + ((size_t)tlX << LT);
          bulk_load(dst, src, (uint32_t)Cfg::TB, fullk, pol_sl);
        }
        trace_stamp(a.trace, k, 3);
        ++k;
        return false;
      };
      // Tickets come in pairs (one atomic per two tiles, one pair ahead), and the two
      // decoded tickets live in fixed register sets P and Q that alternate: no register
      // holding an in-flight load result is ever copied (a copy would stall on it).
      // A claimed ticket is always processed, in claim order, so this is deadlock-free.
      uint32_t tkP, chP, tlP, tkQ, chQ, tlQ;
      int phP, phQ;
      const unsigned *depP, *depQ;
      unsigned dvP, dvQ;
      // Ticket pairs from the shared counter (dynamic balance across CTAs).
      auto claim = [&]() -> uint32_t { return atomicAdd(ticket, 2u); };
      const uint32_t b0 = claim();
      decode_into(b0, tkP, phP, chP, tlP, depP, dvP);
      decode_into(b0 + 1, tkQ, phQ, chQ, tlQ, depQ, dvQ);
      uint32_t nb = (b0 + 1 < total) ? claim() : total;
      for (;;) {
        if (process(tkP, phP, chP, tlP, depP, dvP)) break;
        decode_into(nb, tkP, phP, chP, tlP, depP, dvP);
        trace_stamp(a.trace, k - 1, 9);
        if (process(tkQ, phQ, chQ, tlQ, depQ, dvQ)) break;
        decode_into(nb + 1, tkQ, phQ, chQ, tlQ, depQ, dvQ);
        trace_stamp(a.trace, k - 1, 9);
        nb = (nb + 1 < total) ? claim() : total;
        trace_stamp(a.trace, k - 1, 10);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ signaler
  // Consumers arrive (per warp, non-blocking) on sigbar after their global stores; this
  // thread turns each completed tile into one release increment of the tile's counter
  // (cumulative over the stores observed through the mbarrier, as a CTA barrier followed
  // by one thread's release would be), so no consumer warp ever waits on a memory fence.
  if (warp == 1) {
    if (lane == 0) {
      int jg[NG];
#pragma unroll
      for (int gg = 0; gg < NG; ++gg) jg[gg] = 0;
      int ended = 0;
      while (ended < NG) {
        bool progress = false;
#pragma unroll
        for (int gg = 0; gg < NG; ++gg) {
          if (jg[gg] < 0) continue;
          const int d = jg[gg] % SIGD;
          if (mbar_try_wait(&sigbar[gg * SIGD + d], (uint32_t)(jg[gg] / SIGD) & 1u)) {
            unsigned* p = sigptr[gg * SIGD + d];
            if (p == nullptr) {
              jg[gg] = -1;
              ++ended;
            } else {
              red_release_add(p, 1u);
              ++jg[gg];
            }
            mbar_arrive(&sigfree[gg * SIGD + d]);
            progress = true;
          }
        }
        if (!progress) __nanosleep(32);
      }
    }
    return;
  }
  return;  // idle warps 2-3 of warpgroup 0
  }  // warpgroup 0

  // Consumer warpgroups: take the registers warpgroup 0 released.  (The setmaxnreg must
  // head a region only consumers reach, or ptxas allocates the join at the low count.)
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Cfg::CONS_REGS));

  // ------------------------------------------------------------------ consumers
  const int g = (warp - 4) / GW;
  const int gtid = threadIdx.x - 128 - g * GT;
  const int wig = gtid >> 5;  // warp index within the group
  // per-warp completion signal of the group's j-th tile (see the signaler)
  auto fresh_lane = []() {
    int l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
  };
  auto signal = [&](int j, unsigned* counter) {
    __syncwarp();
    if (fresh_lane() == 0) {
      const int d = j % SIGD;
      if (j >= SIGD) mbar_wait(&sigfree[g * SIGD + d], (uint32_t)((j / SIGD) - 1) & 1u);
      if (wig == 0) sigptr[g * SIGD + d] = counter;
      mbar_arrive(&sigbar[g * SIGD + d]);
    }
  };
  const int bar_id = 1 + g;
  // The thread's index inside the group, re-read from %tid.x in every tile: index values
  // derived from a loop-invariant gtid were kept live across the whole loop and spilled, and
  // their per-tile local reloads queued behind the group's global stores in the LSU.
  auto fresh_gtid = [&]() {
    int t;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
    return t - 128 - g * GT;
  };
  int j = 0;
  for (int k = g;; k += NG, ++j) {
    const int s = k % NS;
    const int gtid = fresh_gtid();
    const int lane = fresh_lane();
    // tile k: stage k % NS, this group's full barrier of that stage (phase k / kLcm)
    if (gtid == 0) trace_stamp(a.trace, k, 4);
    mbar_wait(&full[s * NG + g], (uint32_t)(k / kLcm) & 1u);
    if (gtid == 0) trace_stamp(a.trace, k, 5);
    const TileMeta m = meta[s];
    if (!m.valid) {
      signal(j, nullptr);  // end marker for the signaler
      break;
    }
    double2* S = stage0 + (size_t)s * TE;
    const uint32_t chunk = m.chunk;
    double2* Y = a.scratch + ((size_t)m.slot << slot_shift);
    double2 v[16];
    if (m.phase == 0 && NR > 0) {
      // ---- phase A, early release: read the stage once, release it, exchange through X
      const int u = gtid & (W - 1), jh = gtid >> XB;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int r = jh * 16 + kk;
        v[kk] = S[r * W + ((r & (W - 1)) ^ u)];
        if (MODE == MODE_SYM_HALF) v[kk].y = 0.0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (gtid == 0) trace_stamp(a.trace, k, 6);
      pwht<4>(v);
      constexpr int R2 = R - 4;
      constexpr int UA = (W * 16) / GT;   // second-stage units per thread, 2^R2 registers each
      double2* X = xbuf + g * Cfg::XE;
      const uint64_t pol_last = policy_of(a.pol_s);
      // unit (u, jl) -> Y[tileB][ih][f]
      auto store_unit = [&](const double2* w, int jl) {
        const uint32_t phi_lo = phi_of<XB>((uint32_t)u, (uint32_t)jl, a.layout_mat != 0);
        double2* base = Y + (((phi_lo >> LFB) << LT) | ((uint32_t)m.tile << LFB) | (phi_lo & (FB - 1)));
#pragma unroll
        for (int jj = 0; jj < (1 << R2); ++jj)
          st_global_hint(base + ((size_t)jj << (XB + 4 - LFB + LT)), w[jj], pol_last);
      };
      if constexpr (UA >= 2) {
        exchange_rounds<R2, UA, W>(v, X, jh, u, bar_id, GT);
#pragma unroll
        for (int p = 0; p < UA; ++p) {
          pwht<R2>(&v[p * (1 << R2)]);
          store_unit(&v[p * (1 << R2)], jh + (1 << R2) * p);
        }
      } else {
        xor_half_transpose<W>(v, X, jh, u, bar_id, GT);
        pwht<4>(v);
        store_unit(v, jh);
      }
      signal(j, &doneA[chunk]);
      if (gtid == 0) trace_stamp(a.trace, k, 7);
    } else if (m.phase == 0) {
      // ---- phase A: v_x[i] for x = x0+u, i = tile*2^R + r, r = jh*16 + kk; the element
      //      sits in SMEM row r at column (r mod W) ^ u (XOR transpose in the read)
      {
        const int u = gtid & (W - 1), jh = gtid >> XB;
        if constexpr (MODE == MODE_GEN) {
          // matrix-free: A[i][i ^ x] from the counter-based
          // generator, bit-identical to what ptdr_generate_dense_async stores
          const u64 x = a.x_base + ((u64)m.chunk << XB) + (u64)u;
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) {
            const u64 i = ((u64)m.tile << R) + (u64)(jh * 16 + kk);
            v[kk] = gauss_pair(a.gen_seed, (i << a.n) + (i ^ x), 0u);
          }
        } else {
          if constexpr (MODE == MODE_INVQ) {
            // element (z = row r, X-mask u) is q8 = spread(r_l ^ u) | spread(r_l) << 1 =
            // spread(u) ^ 3 spread(r_l) of its box (r_l = r mod W); the swizzled box holds
            // 128-byte row q8 >> 3 with its 16-byte chunk q8 & 7 at chunk (q8 & 7) ^ (row & 7)
            const uint32_t su = (uint32_t)spread_bits((uint64_t)u);
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              const int r = jh * 16 + kk;
              const uint32_t sr = (uint32_t)spread_bits((uint64_t)(r & (W - 1)));
              const uint32_t q8 = su ^ (3u * sr);
              const uint32_t row = q8 >> 3;
              v[kk] = S[(r >> XB) * W * W + (int)((row << 3) | ((q8 ^ row) & 7u))];
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              const int r = jh * 16 + kk;
              v[kk] = S[r * W + ((r & (W - 1)) ^ u)];
              if (MODE == MODE_SYM_HALF) v[kk].y = 0.0;
            }
          }
          if constexpr (MODE == MODE_INV || MODE == MODE_INVQ) {
            // inverse: the gathered element M[z][z ^ x] = alpha(x, z) of the
            // matrix-layout coefficients enters as u_x[z] = (-i)^{popcount(x & z)} alpha(x, z)
            // (z0 has 4 zero low bits, so popcount(x & z) = popcount(x & z0) + popcount(x & kk);
            // the lanes' phases differ, so the rotation is branch-free: swap + sign bits)
            const uint32_t x = (uint32_t)a.x_base + (m.chunk << XB) + (uint32_t)u;
            const uint32_t z0 = ((uint32_t)m.tile << R) + (uint32_t)(jh * 16);
            const uint32_t p0 = 4u - (uint32_t)__popc(x & z0);
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              const uint32_t p = p0 - (uint32_t)__popc(x & (uint32_t)kk);   // (-i)^popc = i^p
              const bool sw = p & 1u;
              const unsigned long long sre = (unsigned long long)(((p + 1u) >> 1) & 1u) << 63;
              const unsigned long long sim = (unsigned long long)((p >> 1) & 1u) << 63;
              const double re = sw ? v[kk].y : v[kk].x, im = sw ? v[kk].x : v[kk].y;
              v[kk].x = __longlong_as_double((long long)((unsigned long long)__double_as_longlong(re) ^ sre));
              v[kk].y = __longlong_as_double((long long)((unsigned long long)__double_as_longlong(im) ^ sim));
            }
          }
        }
        pwht<4>(v);
        __syncwarp();  // rows of this jh are read and written only by this warp
        if constexpr ((kDiag & 16) == 0) {
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) S[(jh * 16 + kk) * W + u] = v[kk];
        }
      }
      named_bar_sync(bar_id, GT);
      constexpr int R2 = R - 4;
      constexpr int UA = (W * 16) / GT;  // (u, jl) units per thread, each 2^R2 registers
      if constexpr ((kDiag & 16) == 0) {
#pragma unroll
        for (int p = 0; p < UA; ++p) {
          const int uu = gtid + GT * p;
          const int u = uu & (W - 1), jl = uu >> XB;
#pragma unroll
          for (int j = 0; j < (1 << R2); ++j) v[p * (1 << R2) + j] = S[(j * 16 + jl) * W + u];
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (gtid == 0) trace_stamp(a.trace, k, 6);
      const uint64_t pol_last = policy_of(a.pol_s);
#pragma unroll
      for (int p = 0; p < UA; ++p) {
        const int uu = gtid + GT * p;
        const int u = uu & (W - 1), jl = uu >> XB;
        pwht<R2>(&v[p * (1 << R2)]);
        // element (u, ih = tile, zl = j*16 + jl) -> Y[tileB][ih][f]
        const uint32_t phi_lo = phi_of<XB>((uint32_t)u, (uint32_t)jl, a.layout_mat != 0);
        double2* base = Y + (((phi_lo >> LFB) << LT) | ((uint32_t)m.tile << LFB) | (phi_lo & (FB - 1)));
#pragma unroll
        for (int j = 0; j < (1 << R2); ++j)
          st_global_hint(base + ((size_t)j << (XB + 4 - LFB + LT)), v[p * (1 << R2) + j], pol_last);
      }
      signal(j, &doneA[chunk]);
      if (gtid == 0) trace_stamp(a.trace, k, 7);
    } else {
      // ---- phase B: tile Y[tileB][ih][f] = [j][f] (one contiguous 2^LT block of the
      //      scratch); WHT over j for FB fibers
      const u64 x0 = a.x_base + ((u64)chunk << XB);
      const int t = HALF ? 63 - __clzll(x0) : 0;
      const int f = gtid % FB, jh = gtid / FB;
      const double2* yt = Y + ((size_t)m.tile << LT);
      // the tile's scratch lines are dead once every thread of the group has loaded them:
      // drop them from L2 without write-back (the next writer of the slot waits for doneB
      // of this chunk).  Called after a group barrier that follows all stage-1 loads.
      auto discard_tile = [&]() {
        if (a.discard) {
          const char* yb = reinterpret_cast<const char*>(yt);
#pragma unroll
          for (int d = 0; d < Cfg::TB / 128 / GT; ++d) discard_l2(yb + ((size_t)(gtid + GT * d) << 7));
        }
      };
      if constexpr (NR > 0 && M > 4) {
        // ---- early release: read the stage once, drop the scratch lines (the TMA copy has
        //      completed), release the stage, exchange through X
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) v[kk] = S[(jh * 16 + kk) * FB + f];
        discard_tile();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (gtid == 0) trace_stamp(a.trace, k, 6);
        pwht<4>(v);
        constexpr int R2 = M - 4;
        constexpr int UB = (FB * 16) / GT;
        double2* X = xbuf + g * Cfg::XE;
        auto emit_unit = [&](const double2* w, int jl) {
          const uint32_t phi = (uint32_t)m.tile * FB + (uint32_t)f;
          EpiUnit<R2, HALF> e;
          e.init((uint32_t)x0 + phi_u_of<XB>(phi, a.layout_mat != 0), ((uint32_t)jl << R) | phi_zl_of<XB>(phi, a.layout_mat != 0), R + 4, t,
                 a.gshift, a.layout_mat ? a.n : 0);
          emit_all<MODE, R2>(a, e, w);
        };
        if constexpr (UB >= 2) {
          exchange_rounds<R2, UB, FB>(v, X, jh, f, bar_id, GT);
#pragma unroll
          for (int p = 0; p < UB; ++p) {
            pwht<R2>(&v[p * (1 << R2)]);
            emit_unit(&v[p * (1 << R2)], jh + (1 << R2) * p);
          }
        } else {
          xor_half_transpose<FB>(v, X, jh, f, bar_id, GT);
          pwht<4>(v);
          emit_unit(v, jh);
        }
        signal(j, &doneB[chunk]);
        if (gtid == 0) trace_stamp(a.trace, k, 7);
        continue;
      }
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) v[kk] = S[(jh * 16 + kk) * FB + f];
      pwht<4>(v);
      if constexpr (M == 4) {
        named_bar_sync(bar_id, GT);
        discard_tile();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const uint32_t phi = (uint32_t)m.tile * FB + (uint32_t)f;
        EpiUnit<4, HALF> e;
        e.init((uint32_t)x0 + phi_u_of<XB>(phi, a.layout_mat != 0), phi_zl_of<XB>(phi, a.layout_mat != 0), R, t, a.gshift, a.layout_mat ? a.n : 0);
        emit_all<MODE, 4>(a, e, v);
      } else {
        constexpr int R2 = M - 4;
        constexpr int UB = (FB * 16) / GT;  // (f, jl) units per thread, 2^R2 registers each
        if constexpr ((kDiag & 32) == 0) {
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) S[(jh * 16 + kk) * FB + f] = v[kk];
        }
        named_bar_sync(bar_id, GT);
        discard_tile();
        if constexpr ((kDiag & 32) == 0) {
#pragma unroll
          for (int p = 0; p < UB; ++p) {
            const int uu = gtid + GT * p;
            const int f2 = uu % FB, jl = uu / FB;
#pragma unroll
            for (int j = 0; j < (1 << R2); ++j) v[p * (1 << R2) + j] = S[(j * 16 + jl) * FB + f2];
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (gtid == 0) trace_stamp(a.trace, k, 6);
#pragma unroll
        for (int p = 0; p < UB; ++p) {
          const int uu = gtid + GT * p;
          const int f2 = uu % FB, jl = uu / FB;
          const uint32_t phi = (uint32_t)m.tile * FB + (uint32_t)f2;
          pwht<R2>(&v[p * (1 << R2)]);
          EpiUnit<R2, HALF> e;
          e.init((uint32_t)x0 + phi_u_of<XB>(phi, a.layout_mat != 0), ((uint32_t)jl << R) | phi_zl_of<XB>(phi, a.layout_mat != 0), R + 4, t,
                 a.gshift, a.layout_mat ? a.n : 0);
          emit_all<MODE, R2>(a, e, &v[p * (1 << R2)]);
        }
      }
      signal(j, &doneB[chunk]);
      if (gtid == 0) trace_stamp(a.trace, k, 7);
    }
  }
}

// ------------------------------------------------------------------ launch template
template <int LT, int XB, int GW, int NG, int NS, int NR, int M, int MODE>
static cudaError_t launch_pipe_impl(const TmapSet& map, const DenseArgs& a, cudaStream_t st) {
  using Cfg = PipeCfg<LT, XB, GW, NG, NS, NR>;
  constexpr auto kern = dense_pipe_kernel<LT, XB, GW, NG, NS, NR, M, MODE>;
  const cudaError_t err = ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg::SMEM);
  if (err != cudaSuccess) return err;
  // one persistent CTA per SM, or fewer when the caller leaves SMs to a concurrent
  // collective (DenseArgs::max_ctas; tickets are dynamic, any grid size is correct)
  int grid = device_sm_count();
  if (a.max_ctas > 0 && a.max_ctas < grid) grid = a.max_ctas;
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(map, a);
  return cudaGetLastError();
}

template <int LT, int XB, int GW, int NG, int NS, int NR, int MODE>
static cudaError_t launch_pipe_m(const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st) {
  switch (M) {
    case 4: return launch_pipe_impl<LT, XB, GW, NG, NS, NR, 4, MODE>(map, a, st);
    case 5: return launch_pipe_impl<LT, XB, GW, NG, NS, NR, 5, MODE>(map, a, st);
    case 6: return launch_pipe_impl<LT, XB, GW, NG, NS, NR, 6, MODE>(map, a, st);
    case 7: return launch_pipe_impl<LT, XB, GW, NG, NS, NR, 7, MODE>(map, a, st);
    case 8: return launch_pipe_impl<LT, XB, GW, NG, NS, NR, 8, MODE>(map, a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int LT, int XB, int GW, int NG, int NS, int NR>
static cudaError_t launch_pipe_cfg(int mode, const TmapSet& map, const DenseArgs& a, int M,
                                   cudaStream_t st) {
  switch (mode) {
    case MODE_GENERAL: return launch_pipe_m<LT, XB, GW, NG, NS, NR, MODE_GENERAL>(map, a, M, st);
    case MODE_HERM_HALF: return launch_pipe_m<LT, XB, GW, NG, NS, NR, MODE_HERM_HALF>(map, a, M, st);
    case MODE_SYM_HALF: return launch_pipe_m<LT, XB, GW, NG, NS, NR, MODE_SYM_HALF>(map, a, M, st);
    case MODE_GEN:
      // matrix-free: instantiated for the 3-stage in-place configurations only
      if constexpr (NR == 0 && LT == 12) return launch_pipe_m<LT, XB, GW, NG, NS, NR, MODE_GEN>(map, a, M, st);
      return cudaErrorInvalidValue;
    case MODE_INV:
      if constexpr (NR == 0 && LT == 12) return launch_pipe_m<LT, XB, GW, NG, NS, NR, MODE_INV>(map, a, M, st);
      return cudaErrorInvalidValue;
    case MODE_INVQ:
      if constexpr (NR == 0 && LT == 12) return launch_pipe_m<LT, XB, GW, NG, NS, NR, MODE_INVQ>(map, a, M, st);
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

#define PTDR_DEFINE_PIPE_CFG(NAME, LT, XB, GW, NG, NS, NR)                                     \
  cudaError_t NAME(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st) {     \
    return launch_pipe_cfg<LT, XB, GW, NG, NS, NR>(mode, map, a, M, st);                       \
  }

}  // namespace ptdr
