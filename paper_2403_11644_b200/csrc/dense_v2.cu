// dense_v2.cu -- warp-specialised TMA pipeline for the dense path (nv >= 12).
//
// Same math and tiling as dense_impl.cuh (phase A: XOR-transpose gather + WHT over
// the low 8 index bits into the L2-resident scratch ring; phase B: WHT over the
// high M bits + epilogue in q order), but organised for sm_100a:
//   * one CTA per SM: warp 0 = producer (tickets, inter-CTA dependency waits, TMA),
//     warps 1..16 = two consumer groups of 8 warps that take tiles alternately;
//   * phase-A input tiles (16 row blocks of 16 x 16 complex128, 64 KiB) are fetched by
//     cp.async.bulk.tensor into a 3-stage SMEM ring (mbarrier full/empty pipeline),
//     so HBM loads for tile k+2 overlap the arithmetic of tiles k and k+1;
//   * the XOR transpose happens in the SMEM read (conflict-free), the exchange between
//     the two radix-16 register stages is done in place in the same stage buffer;
//   * the epilogue computes q offsets and i^{popcount(x&z)} phases incrementally
//     (per-thread base + compile-time subset sums of per-bit deltas).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "dense_impl.cuh"
#include "dense_plan.h"
#include "internal.h"
#include "sm100_ptx.cuh"

namespace ptdr {

constexpr int kStages = 3;
constexpr int kGroupWarps = 8;
constexpr int kV2Threads = 32 * (1 + 2 * kGroupWarps);  // 544
constexpr int kV2Smem = kStages * kTileBytes + 256;

struct TileMeta {
  int valid, phase, tile, pad;
  unsigned long long chunk;
};

__device__ __forceinline__ void spin_until(const unsigned* p, unsigned target) {
  while (ld_acquire(p) < target) __nanosleep(32);
}

// 32-bit index arithmetic: n <= 16 so x, z < 2^16 and q < 2^32.
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
// q delta of setting z bit l (code_l = 2 z_l + (x_l ^ z_l); above gshift the
// z bit indexes the rank-local block).
__device__ __forceinline__ uint32_t q_delta32(uint32_t x, int l, int gshift) {
  return (l < gshift) ? ((uint32_t)(3 - 2 * (int)((x >> l) & 1u)) << (2 * l)) : (1u << (l + gshift));
}
__device__ __forceinline__ uint32_t insert0_32(uint32_t v, int t) {
  const uint32_t lo = v & ((1u << t) - 1u);
  return ((v >> t) << (t + 1)) | lo;
}

template <int NB, bool HALF>
struct EpiUnit {
  uint32_t q0;
  uint32_t p0;
  uint32_t D[NB];
  uint32_t P[NB];
  uint32_t Dt;
  __device__ __forceinline__ void init(uint32_t x, uint32_t zu, int base_pos, int t, int gshift) {
    const uint32_t zf = HALF ? insert0_32(zu, t) : zu;
    q0 = q_offset32(x, zf, gshift);
    p0 = __popc(x & zf);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      int l = base_pos + b;
      if (HALF) l += (l >= t) ? 1 : 0;
      D[b] = q_delta32(x, l, gshift);
      P[b] = (x >> l) & 1u;
    }
    if (HALF) Dt = q_delta32(x, t, gshift);
  }
};

template <int MODE, int NB, int J>
__device__ __forceinline__ void emit_reg(const DenseArgs& a, const EpiUnit<NB, (MODE >= 3)>& e,
                                         double2 w) {
  uint32_t q = e.q0;
  uint32_t p = e.p0;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (J & (1 << b)) {
      q += e.D[b];
      p += e.P[b];
    }
  }
  if constexpr (MODE == MODE_GENERAL) {
    double2 c = rot_ipow(w, (int)p);
    st_stream(a.out + q, make_double2(c.x * a.scale, c.y * a.scale));
  } else {
    const uint32_t p0 = p & 3u, p1 = (p + 1u) & 3u;
    const double s = 2.0 * a.scale;
    const double v0 = (p0 == 0) ? w.x : (p0 == 1) ? -w.y : (p0 == 2) ? -w.x : w.y;
    const double v1 = (p1 == 0) ? w.x : (p1 == 1) ? -w.y : (p1 == 2) ? -w.x : w.y;
    st_stream(a.out + q, make_double2(v0 * s, 0.0));
    st_stream(a.out + (q + e.Dt), make_double2(v1 * s, 0.0));
  }
}

template <int MODE, int NB, int J = 0>
__device__ __forceinline__ void emit_all(const DenseArgs& a, const EpiUnit<NB, (MODE >= 3)>& e,
                                         const double2* w) {
  if constexpr (J < (1 << NB)) {
    emit_reg<MODE, NB, J>(a, e, w[J]);
    emit_all<MODE, NB, J + 1>(a, e, w);
  }
}

// Ticket order of dense_impl.cuh's decode_ticket, in 32-bit arithmetic with NA = NB = 2^M.
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

// Scratch layout (per chunk slot): B-tile-major, Y[tileB][ih][f] with 4096 elements per
// phase-B tile, so that a phase-B tile is one contiguous 64 KiB bulk copy.  The fiber
// index phi = tileB * FB + f encodes (u, zl): bits [0,1]=u0,u1 [2,3]=zl0,zl1 [4,5]=u2,u3
// [6..]=zl2.. (phi_u / phi_zl in dense_impl.cuh).
template <int M, int MODE>
__global__ void __launch_bounds__(kV2Threads, 1)
    dense_v2_kernel(const __grid_constant__ CUtensorMap tmap, DenseArgs a) {
  constexpr bool HALF = (MODE == MODE_HERM_HALF || MODE == MODE_SYM_HALF);
  constexpr int FB = kTileElems >> M;  // phase-B fibers per tile
  constexpr int LFB = 12 - M;
  extern __shared__ __align__(1024) unsigned char smem[];
  double2* stage0 = reinterpret_cast<double2*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kTileBytes);
  uint64_t* empty = full + kStages;
  TileMeta* meta = reinterpret_cast<TileMeta*>(empty + kStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t C = (uint32_t)a.nchunks;
  unsigned* ticket = a.ctr;
  unsigned* doneA = a.ctr + 1;
  unsigned* doneB = a.ctr + 1 + C;
  const uint32_t nslot = (uint32_t)a.nslot;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGroupWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ------------------------------------------------------------------ producer
  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmap);
      const uint64_t pol = policy_evict_first();
      const uint32_t total = C << (M + 1);
      int tail = 0;
      // tickets are claimed one ahead so the atomic's round trip overlaps the current
      // tile's dependency wait and TMA issue (a claimed ticket is always processed next)
      uint32_t next_tk = atomicAdd(ticket, 1u);
      for (int k = 0;; ++k) {
        const int s = k % kStages;
        if (k >= kStages) mbar_wait(&empty[s], (uint32_t)((k / kStages) - 1) & 1u);
        const uint32_t tk = tail ? total : next_tk;
        if (tk < total) next_tk = atomicAdd(ticket, 1u);
        if (tk >= total) {
          meta[s].valid = 0;
          mbar_arrive(&full[s]);
          if (++tail == 2) break;
          continue;
        }
        int phase;
        uint32_t chunk, tile;
        decode_ticket32(tk, M, C, (uint32_t)a.L, phase, chunk, tile);
        if (phase == 0) {
          if (chunk >= nslot) spin_until(&doneB[chunk - nslot], 1u << M);
        } else {
          spin_until(&doneA[chunk], 1u << M);
        }
        meta[s].valid = 1;
        meta[s].phase = phase;
        meta[s].tile = (int)tile;
        meta[s].chunk = chunk;
        double2* dst = stage0 + (size_t)s * kTileElems;
        if (phase == 0) {
          mbar_arrive_expect_tx(&full[s], (uint32_t)kTileBytes);
          const u64 x0 = a.x_base + 16ull * chunk;
          const int t = HALF ? 63 - __clzll(x0) : 0;
#pragma unroll 4
          for (int rb = 0; rb < 16; ++rb) {
            const u64 iv0 = ((u64)tile << 8) + (u64)rb * 16;
            const u64 row0 = HALF ? insert0(iv0, t) : iv0;
            const u64 col0 = ((row0 ^ x0) & a.colmask) & ~15ull;
            tma_load_2d(dst + rb * 256, &tmap, (int)(col0 * 2), (int)row0, &full[s], pol);
          }
        } else {
          // scratch written by other CTAs' generic stores, read by the async proxy
          fence_proxy_async_global();
          mbar_arrive_expect_tx(&full[s], (uint32_t)kTileBytes);
          const double2* src = a.scratch + (size_t)(chunk % nslot) * a.slot_elems + ((size_t)tile << 12);
          bulk_load(dst, src, (uint32_t)kTileBytes, &full[s], pol);
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const int g = (warp - 1) / kGroupWarps;
  const int gtid = threadIdx.x - 32 - g * (32 * kGroupWarps);
  for (int k = g;; k += 2) {
    const int s = k % kStages;
    mbar_wait(&full[s], (uint32_t)(k / kStages) & 1u);
    const TileMeta m = meta[s];
    if (!m.valid) break;
    double2* S = stage0 + (size_t)s * kTileElems;
    const uint32_t chunk = (uint32_t)m.chunk;
    double2* Y = a.scratch + (size_t)(chunk % nslot) * a.slot_elems;
    double2 v[16];
    if (m.phase == 0) {
      // ---- phase A: v_x[i] for x = x0+u, i = tile*256 + jh*16 + kk (XOR transpose in SMEM)
      const int u = gtid & 15, jh = gtid >> 4;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        v[kk] = S[(jh * 16 + kk) * 16 + (kk ^ u)];
        if (MODE == MODE_SYM_HALF) v[kk].y = 0.0;
      }
      wht_regs<4>(v);
      __syncwarp();
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) S[(jh * 16 + kk) * 16 + u] = v[kk];
      named_bar_sync(1 + g, 32 * kGroupWarps);
      const int jl = gtid >> 4;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = S[(j * 16 + jl) * 16 + u];
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      wht_regs<4>(v);
      // element (u, ih = tile, zl = j*16 + jl) -> Y[tileB][ih][f]
      const uint32_t phi_lo = (uint32_t)((u & 3) | ((jl & 3) << 2) | ((u >> 2) << 4) | ((jl >> 2) << 6));
      double2* base = Y + (((phi_lo >> LFB) << 12) | ((uint32_t)m.tile << LFB) | (phi_lo & (FB - 1)));
      const uint64_t pol_last = policy_evict_last();
#pragma unroll
      for (int j = 0; j < 16; ++j) st_global_hint(base + ((size_t)j << (M - 4 + 12)), v[j], pol_last);
      named_bar_sync(1 + g, 32 * kGroupWarps);
      if (gtid == 0) {
        __threadfence();
        atomicAdd(&doneA[chunk], 1u);
      }
    } else {
      // ---- phase B: SMEM holds Y[tileB][ih][f] = [j][f]; WHT over j for FB fibers
      const u64 x0 = a.x_base + 16ull * chunk;
      const int t = HALF ? 63 - __clzll(x0) : 0;
      const int f = gtid % FB, jh = gtid / FB;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) v[kk] = S[(jh * 16 + kk) * FB + f];
      if (a.discard) {
        // the slot region of this tile is dead once in SMEM: drop it from L2 without
        // write-back (the next writer of the slot waits for doneB of this chunk)
        char* yb = reinterpret_cast<char*>(Y + ((size_t)m.tile << 12));
        discard_l2(yb + (size_t)gtid * 256);
        discard_l2(yb + (size_t)gtid * 256 + 128);
      }
      wht_regs<4>(v);
      if constexpr (M == 4) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const uint32_t phi = (uint32_t)m.tile * FB + (uint32_t)f;
        EpiUnit<4, HALF> e;
        e.init((uint32_t)x0 + (uint32_t)phi_u(phi), (uint32_t)phi_zl(phi), 8, t, a.gshift);
        emit_all<MODE, 4>(a, e, v);
      } else {
        constexpr int R2 = M - 4;
        constexpr int U2 = 1 << (8 - M);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) S[(jh * 16 + kk) * FB + f] = v[kk];
        named_bar_sync(1 + g, 32 * kGroupWarps);
#pragma unroll
        for (int p = 0; p < U2; ++p) {
          const int uu = gtid + 256 * p;
          const int f2 = uu % FB, jl = uu / FB;
#pragma unroll
          for (int j = 0; j < (1 << R2); ++j) v[p * (1 << R2) + j] = S[(j * 16 + jl) * FB + f2];
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
        for (int p = 0; p < U2; ++p) {
          const int uu = gtid + 256 * p;
          const int f2 = uu % FB, jl = uu / FB;
          const uint32_t phi = (uint32_t)m.tile * FB + (uint32_t)f2;
          wht_regs<R2>(&v[p * (1 << R2)]);
          EpiUnit<R2, HALF> e;
          e.init((uint32_t)x0 + (uint32_t)phi_u(phi), ((uint32_t)jl << 8) | (uint32_t)phi_zl(phi), 12,
                 t, a.gshift);
          emit_all<MODE, R2>(a, e, &v[p * (1 << R2)]);
        }
      }
      named_bar_sync(1 + g, 32 * kGroupWarps);
      if (gtid == 0) {
        __threadfence();
        atomicAdd(&doneB[chunk], 1u);
      }
    }
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

template <int M, int MODE>
static cudaError_t launch_v2_impl(const CUtensorMap& map, const DenseArgs& a, cudaStream_t st) {
  constexpr auto kern = dense_v2_kernel<M, MODE>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [&]() {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kV2Smem);
  });
  if (err != cudaSuccess) return err;
  kern<<<device_sm_count(), kV2Threads, kV2Smem, st>>>(map, a);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_v2_mode(const CUtensorMap& map, const DenseArgs& a, int M,
                                  cudaStream_t st) {
  switch (M) {
    case 4: return launch_v2_impl<4, MODE>(map, a, st);
    case 5: return launch_v2_impl<5, MODE>(map, a, st);
    case 6: return launch_v2_impl<6, MODE>(map, a, st);
    case 7: return launch_v2_impl<7, MODE>(map, a, st);
    case 8: return launch_v2_impl<8, MODE>(map, a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_dense_v2(int mode, const DenseArgs& a_in, const DensePlan& p, cudaStream_t st,
                            int* nlaunch) {
  if (p.kind != 2 || p.R != 8) return cudaErrorInvalidValue;
  DenseArgs a = a_in;
  a.L = p.L;
  a.nslot = p.nslot;
  a.slot_elems = p.slot_elems;
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t ncols = a.colmask + 1, nrows = 1ull << a.n;
  cuuint64_t gdim[2] = {2 * ncols, nrows};
  cuuint64_t gstride[1] = {a.ld * 16};
  cuuint32_t box[2] = {32, 16};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(a.A), gdim, gstride,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  {
    const char* nd = getenv("PTDR_NO_DISCARD");
    a.discard = (nd && nd[0] == '1') ? 0 : 1;
  }
  cudaError_t e = cudaMemsetAsync(a.ctr, 0, p.ctr_bytes, st);
  if (e != cudaSuccess) return e;
  *nlaunch += 1;
  switch (mode) {
    case MODE_GENERAL: return launch_v2_mode<MODE_GENERAL>(map, a, p.M, st);
    case MODE_HERM_HALF: return launch_v2_mode<MODE_HERM_HALF>(map, a, p.M, st);
    case MODE_SYM_HALF: return launch_v2_mode<MODE_SYM_HALF>(map, a, p.M, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ptdr
