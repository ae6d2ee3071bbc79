// band.cu -- DIAGONAL and TRIDIAGONAL paths (Sec. IV-A, l.367-465).
//
// DIAGONAL (l.369-389): only x = 0 strings ({I,Z}^n) can be nonzero and
//   alpha(0, z) = 2^-n WHT_n(d)[z]  (v_0[i] = A[i][i] = d[i]).
// TRIDIAGONAL (l.395-465): only the n+1 X-masks x_b = 2^b - 1 are nonzero.  For
//   b = t+1 >= 1, v_x[i] is nonzero only at i = h 2^{t+1} + 2^t - 1 (super-diagonal
//   S_t[h] = A[i][i+1]) and at i + 1 (sub-diagonal U_t[h] = A[i+1][i]), so with
//   P_t = WHT(S_t + U_t), M_t = WHT(S_t - U_t) (length 2^{n-t-1}),
//   zl = z mod 2^{t+1}, zh = z >> (t+1), s1 = (-1)^{popcount(z mod 2^t)}, s2 = (-1)^{z_t}:
//   alpha(x_b, z) = 2^-n i^{popcount(zl)} s1 (s1 == s2 ? P_t[zh] : M_t[zh]).
//   DESIGN.md derives this from the per-x WHT identity.
// HERMITIAN_TRIDIAGONAL: U_t = conj(S_t), so one W_t = WHT(S_t) per segment gives
//   P_t = (2 Re W_t, 0) and M_t = (0, 2 Im W_t) (herm_seg_view).
// ANTI_DIAGONAL and BAND(s) (the (2s+1)-band planner) follow further down.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "dense_plan.h"
#include "engine.cuh"
#include "sm100_ptx.cuh"
#include "internal.h"
#include "wht_passes.h"

namespace ptdr {

// Vectors of at least 2^kTopMin elements run their three top butterfly levels first (the
// z-sharded paths read them once and transform only the rank's part; see topk_pass_kernel).
// Tridiagonal segments from 2^13 on (their split is per element, and 2^10-2^11-element
// branches are whole-vector tiles: one pass); the x = 0 vector from 2^15 on (a
// topk_pass_kernel tile needs 4096 / 2^KK <= 2^(n - TB) consecutive elements per branch).
constexpr int kTopMin = 13;
constexpr int kTopMinX0 = 15;

// ---- flat WHT pass over bits [b0, b0+K) of a contiguous array ---------------------
template <int K>
struct FlatLd {
  const double2* in;
  u64 rbase;
  int b0;
  __device__ __forceinline__ double2 operator()(int f, int j) const {
    const u64 rho = rbase + (u64)f;
    const u64 e = ((rho >> b0) << (b0 + K)) | ((u64)j << b0) | (rho & ((1ull << b0) - 1ull));
    return ld_l2(in + e);
  }
};
// z-slice of a rank (z-sharded structured outputs): element e of a
// single-vector family is stored iff e >> zshift == zrank, at e - (zrank << zshift).
// zshift = 63 keeps everything (one GPU, or a workspace-targeted pass).
__device__ __forceinline__ bool in_slice(u64 e, int zshift, u64 zrank) { return (e >> zshift) == zrank; }

// Last-pass store of element e (= z of a single-vector family): scale, the phase
// i^{popcount(px & z)} of a fixed X-mask px (ANTI_DIAGONAL: px = 2^n - 1; 0 otherwise) and the
// slice filter.
__device__ __forceinline__ void store_final(double2* out, u64 e, double2 v, double scale, int zshift,
                                            u64 zrank, u64 px, u64 zoff = 0) {
  if (!in_slice(e, zshift, zrank)) return;
  if (px) v = rot_ipow(v, __popcll(px & (e + zoff)));
  st_l2(out + (e - (zrank << zshift)), make_double2(v.x * scale, v.y * scale));
}

template <int K>
struct FlatSt {
  double2* out;
  u64 rbase;
  int b0;
  double scale;
  int zshift;
  u64 zrank;
  u64 px;
  u64 zoff;
  __device__ __forceinline__ void operator()(int f, int j, double2 v) const {
    const u64 rho = rbase + (u64)f;
    const u64 e = ((rho >> b0) << (b0 + K)) | ((u64)j << b0) | (rho & ((1ull << b0) - 1ull));
    store_final(out, e, v, scale, zshift, zrank, px, zoff);
  }
};

// Pass over the 8 lowest index bits of a contiguous 4096-element tile (16 contiguous fibres
// of 256).  fiber_tile's lane order (lanes along the fibre index) would make every access
// a 4 KiB-strided 16 B request here, so this variant keeps lanes along the element index:
// thread (f = tid >> 4, jl = tid & 15) loads j = jl + 16 kk (two 256 B runs per warp
// instruction), radix-16 over kk in registers, one padded SMEM exchange
// (P(f, j) = 272 f + 17 (j >> 4) + (j & 15), conflict-free both ways), radix-16 over jl,
// and a coalesced copy-out through the same slots.
__device__ __forceinline__ int contig_slot(int f, int j) { return f * 272 + (j >> 4) * 17 + (j & 15); }
constexpr int kContigSlots = 16 * 272;
constexpr int kBandSmem = kContigSlots * 16;  // >= kTileBytes: also the fiber_tile buffer
static_assert(kBandSmem >= kTileBytes, "band tile buffer holds a full tile");

__device__ __forceinline__ void contig8_tile(double2* S, const double2* in, double2* out, u64 base,
                                             double scale, int zshift, u64 zrank, u64 px) {
  const int tid = threadIdx.x;
  double2 v[16];
  {
    const int f = tid >> 4, jl = tid & 15;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) v[kk] = ld_l2(in + base + (u64)(f * 256 + jl + 16 * kk));
    wht_regs<4>(v);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) S[contig_slot(f, jl + 16 * kk)] = v[kk];
  }
  __syncthreads();
  {
    const int f = tid >> 4, kh = tid & 15;
#pragma unroll
    for (int jl = 0; jl < 16; ++jl) v[jl] = S[contig_slot(f, jl + 16 * kh)];
    wht_regs<4>(v);
#pragma unroll
    for (int jl = 0; jl < 16; ++jl) S[contig_slot(f, jl + 16 * kh)] = v[jl];  // own slots only
  }
  __syncthreads();
  {
    const int f = tid >> 4, jl = tid & 15;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      store_final(out, base + (u64)(f * 256 + jl + 16 * kk), S[contig_slot(f, jl + 16 * kk)], scale, zshift,
                  zrank, px);
    }
  }
}

// ---- tridiagonal expansion into blocks 1..n (write-bound) ------------------------------
// Each thread writes 8 outputs of one block at z = base + lane + 32 k (512 B per warp store);
// the P/M values (reused 2^(t+1) times) come through the read-only cache.
// z-sharded (world > 1): only z in [zrank 2^zshift, (zrank+1) 2^zshift) of each block, stored
// block-major with 2^zshift outputs per block (block 0 is written by the WHT passes).
// Segment t's P/M values for zh (long segments, lam >= kTopMin: the KS kept top-bit branches
// of the rank, stored compactly, local index zh mod KS 2^(lam-3); short ones: full vectors).
struct SegView {
  const double2* P;
  const double2* M;
  u64 mask;
};
__device__ __forceinline__ SegView seg_view(const double2* PM, int n, int t, int k_keep) {
  const u64 N = 1ull << n;
  const int lam = n - t - 1;
  const double2* Pt = PM + 2 * (N - (N >> t));
  if (lam >= kTopMin) {
    const u64 len = 1ull << (lam - 3 + k_keep);
    return SegView{Pt, Pt + len, len - 1ull};
  }
  return SegView{Pt, Pt + (1ull << lam), ~0ull};
}

// HERMITIAN_TRIDIAGONAL (sub[i + 1] = conj(sup[i])): U_t = conj(S_t), so with W_t = WHT(S_t)
// P_t = W_t + conj(W_t) = (2 Re W_t, 0) and M_t = (0, 2 Im W_t) -- one WHT per segment instead
// of two, stored as S_t at PM + (2^n - 2^(n-t)) (KS branches of 2^(lam-3) for long segments).
// For an input that satisfies the relation exactly, these are bitwise the P_t / M_t of the
// general path: 2x is exact, and S + conj(S), S - conj(S) have exact +0 parts.
__device__ __forceinline__ SegView herm_seg_view(const double2* W, int n, int t, int k_keep) {
  const u64 N = 1ull << n;
  const int lam = n - t - 1;
  const double2* St = W + (N - (N >> t));
  if (lam >= kTopMin) return SegView{St, St, (1ull << (lam - 3 + k_keep)) - 1ull};
  return SegView{St, St, ~0ull};
}
template <bool HERM>
__device__ __forceinline__ double2 pm_value(const SegView& sv, bool use_p, u64 idx) {
  if constexpr (HERM) {
    const double2 w = __ldg(sv.P + idx);
    return use_p ? make_double2(2.0 * w.x, 0.0) : make_double2(0.0, 2.0 * w.y);
  } else {
    return __ldg((use_p ? sv.P : sv.M) + idx);
  }
}

template <bool HERM>
__global__ void __launch_bounds__(256) tridiag_expand_kernel(const double2* PM, double2* out, int n,
                                                             double scale, int zshift, u64 zrank, int k_keep,
                                                             int t_first) {
  const u64 N = 1ull << n;
  const u64 NL = 1ull << zshift;              // outputs per block on this rank
  const u64 z0 = zrank << zshift;
  const u64 groups = ((u64)n * NL) >> 8;      // 256 outputs per warp-group of 8 stores
  const u64 g0 = ((u64)t_first * NL) >> 8;    // blocks 1..t_first come from the fused kernel
  const int lane = threadIdx.x & 31;
  for (u64 gidx = g0 + (((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5); gidx < groups;
       gidx += ((u64)gridDim.x * blockDim.x) >> 5) {
    const u64 id0 = gidx << 8;
    const int t = (int)(id0 >> zshift);
    const SegView sv = HERM ? herm_seg_view(PM, n, t, k_keep) : seg_view(PM, n, t, k_keep);
    double2 w[8];
    int ph[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const u64 z = z0 + (id0 & (NL - 1)) + (u64)lane + 32ull * k;
      const u64 zl = z & ((2ull << t) - 1ull);
      const u64 zh = z >> (t + 1);
      const int s1 = __popcll(z & ((1ull << t) - 1ull)) & 1;
      const int s2 = (int)((z >> t) & 1ull);
      w[k] = pm_value<HERM>(sv, s1 == s2, zh & sv.mask);
      ph[k] = __popcll(zl) + 2 * s1;  // i^{popcount(zl)} * (-1)^{s1}
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool sw = (ph[k] & 1) != 0;
      const double sc = (ph[k] & 2) ? -scale : scale;
      const double re = sw ? -w[k].y : w[k].x;
      const double im = sw ? w[k].x : w[k].y;
      st_stream(out + NL + id0 + (u64)lane + 32ull * k, make_double2(re * sc, im * sc));
    }
  }
}

// Small slices (2^zshift < 256): one output per thread.
template <bool HERM>
__global__ void tridiag_expand_small_kernel(const double2* PM, double2* out, int n, double scale,
                                            int zshift, u64 zrank, int k_keep) {
  const u64 N = 1ull << n;
  const u64 NL = 1ull << zshift;
  const u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (u64)n * NL) return;
  const int t = (int)(id >> zshift);
  const u64 z = (zrank << zshift) + (id & (NL - 1));
  const SegView sv = HERM ? herm_seg_view(PM, n, t, k_keep) : seg_view(PM, n, t, k_keep);
  const u64 zl = z & ((2ull << t) - 1ull);
  const int s1 = __popcll(z & ((1ull << t) - 1ull)) & 1;
  const int s2 = (int)((z >> t) & 1ull);
  const double2 w = pm_value<HERM>(sv, s1 == s2, (z >> (t + 1)) & sv.mask);
  const int ph = __popcll(zl) + 2 * s1;
  const double2 c = rot_ipow(w, ph);
  out[NL + id] = make_double2(c.x * scale, c.y * scale);
}

// ---- multi-segment WHT passes ---------------------------------------------------------
// One launch runs pass p (index bits [8p, 8p+8)) for every segment that needs it: the x=0
// vector (main diagonal) and the tridiagonal P/M segments.  Segments with lambda <= 12 are
// transformed whole, one vector per tile, in pass 0.  Tiles of all segments are handed out
// grid-stride; each tile dispatches its fibre length K at run time.
struct SegPass {
  const double2* in;
  double2* out;
  unsigned long long first_tile;  // prefix sum of tiles over the table
  int b0;                         // first index bit of this pass
  int K;                          // bits transformed in this pass (flat tiles)
  int small;                      // 1: whole-vector WHT of 2^small_lam elements per tile
  int small_lam;
  double scale;
  int zshift;  // slice filter of the stores (63: none)
  unsigned long long zrank;
  unsigned long long px;  // X-mask phase of the last pass (0: none)
  unsigned long long zoff;  // z of element 0 (px phase)
  int fn;                 // 1: the combined near+far pass 0 of a 17..20-bit family (fn_tile)
  int fn_lam;
};
constexpr int kMaxSeg = 40;
struct SegPassTable {
  int count;
  unsigned long long total_tiles;
  SegPass s[kMaxSeg];
};

__device__ __forceinline__ void small_wht_tile(double2* S, const double2* in, double2* out, int lam,
                                               double scale, u64 e0, int zshift, u64 zrank, u64 px) {
  const int len = 1 << lam;
  for (int i = threadIdx.x; i < len; i += blockDim.x) S[i] = ld_l2(in + i);
  for (int sb = 0; sb < lam; ++sb) {
    __syncthreads();
    for (int p = threadIdx.x; p < len / 2; p += blockDim.x) {
      const int lo = p & ((1 << sb) - 1);
      const int i0 = ((p >> sb) << (sb + 1)) | lo;
      const int i1 = i0 | (1 << sb);
      const double2 a = S[i0], b = S[i1];
      S[i0] = cadd(a, b);
      S[i1] = csub(a, b);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < len; i += blockDim.x) store_final(out, e0 + (u64)i, S[i], scale, zshift, zrank, px);
}

template <int F>
__device__ __forceinline__ void fn_far(double2* S, int tid) {
  constexpr int B = 4 - F;
#pragma unroll
  for (int r = 0; r < (1 << (4 - F)); ++r) {
    const int p = tid + 256 * r;
    const int b = p >> 8, j = p & 255;
    double2 w[1 << F];
#pragma unroll
    for (int f = 0; f < (1 << F); ++f) w[f] = S[contig_slot((f << B) | b, j)];
    wht_regs<F>(w);
#pragma unroll
    for (int f = 0; f < (1 << F); ++f) S[contig_slot((f << B) | b, j)] = w[f];
  }
}

// Pass 0 of a family of 2^lam-element vectors, 17 <= lam <= 20: the 8 near bits [0, 8)
// (runs of 256, the stages of contig8_tile) and the lam - 16 far bits [16, lam) in ONE tile,
// with the 20 - lam bits above 8 as batch, so the family needs two passes instead of three
// (bits [8, 16) are the second).  Tile = 2^(lam-16) far x 2^(20-lam) batch x 256 near;
// "fibre" fb = (far << (20 - lam)) | batch holds 256 near elements at contig_slot(fb, j).
__device__ __forceinline__ void fn_tile(double2* S, const double2* in, double2* out, u64 tile, int lam) {
  const int F = lam - 16, B = 20 - lam;
  const u64 v = tile >> (lam - 12), mb = tile & ((1ull << (lam - 12)) - 1ull);
  const u64 vbase = v << lam;
  auto addr = [&](int fb, int j) -> u64 {
    const u64 f = (u64)(fb >> B), b = (u64)(fb & ((1 << B) - 1));
    return vbase + (f << 16) + (((mb << B) + b) << 8) + (u64)j;
  };
  const int tid = threadIdx.x;
  double2 v16[16];
  {  // near bits 4-7 (as contig8_tile)
    const int fb = tid >> 4, jl = tid & 15;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) v16[kk] = ld_l2(in + addr(fb, jl + 16 * kk));
    wht_regs<4>(v16);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) S[contig_slot(fb, jl + 16 * kk)] = v16[kk];
  }
  __syncthreads();
  {  // near bits 0-3
    const int fb = tid >> 4, kh = tid & 15;
#pragma unroll
    for (int jl = 0; jl < 16; ++jl) v16[jl] = S[contig_slot(fb, jl + 16 * kh)];
    wht_regs<4>(v16);
#pragma unroll
    for (int jl = 0; jl < 16; ++jl) S[contig_slot(fb, jl + 16 * kh)] = v16[jl];
  }
  __syncthreads();
  // far bits: 2^F values per (batch, near) position, 2^(4-F) positions per thread
  switch (F) {
    case 1: fn_far<1>(S, tid); break;
    case 2: fn_far<2>(S, tid); break;
    case 3: fn_far<3>(S, tid); break;
    default: fn_far<4>(S, tid); break;
  }
  __syncthreads();
  {
    const int fb = tid >> 4, jl = tid & 15;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) st_l2(out + addr(fb, jl + 16 * kk), S[contig_slot(fb, jl + 16 * kk)]);
  }
}

template <int K>
__device__ __forceinline__ void flat_tile(double2* S, const SegPass& sp, u64 local) {
  constexpr int F = kTileElems >> K;
  FlatLd<K> ld{sp.in, local * F, sp.b0};
  FlatSt<K> st{sp.out, local * F, sp.b0, sp.scale, sp.zshift, sp.zrank, sp.px, sp.zoff};
  fiber_tile<K>(S, ld, st);
}

__global__ void __launch_bounds__(kThreads, 2) seg_pass_kernel(const __grid_constant__ SegPassTable T) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  for (u64 tile = blockIdx.x; tile < T.total_tiles; tile += gridDim.x) {
    int i = 0;
    while (i + 1 < T.count && T.s[i + 1].first_tile <= tile) ++i;
    const SegPass& sp = T.s[i];
    const u64 local = tile - sp.first_tile;
    if (sp.fn) {
      fn_tile(S, sp.in, sp.out, local, sp.fn_lam);
    } else if (sp.small) {
      const u64 off = local << sp.small_lam;
      small_wht_tile(S, sp.in + off, sp.out, sp.small_lam, sp.scale, off, sp.zshift, sp.zrank, sp.px);
    } else if (sp.b0 == 0 && sp.K == 8) {
      contig8_tile(S, sp.in, sp.out, local * (u64)kTileElems, sp.scale, sp.zshift, sp.zrank, sp.px);
    } else {
      switch (sp.K) {
        case 1: flat_tile<1>(S, sp, local); break;
        case 2: flat_tile<2>(S, sp, local); break;
        case 3: flat_tile<3>(S, sp, local); break;
        case 4: flat_tile<4>(S, sp, local); break;
        case 5: flat_tile<5>(S, sp, local); break;
        case 6: flat_tile<6>(S, sp, local); break;
        case 7: flat_tile<7>(S, sp, local); break;
        default: flat_tile<8>(S, sp, local); break;
      }
    }
    __syncthreads();
  }
}

// Runs all passes for all families (at most 3 launches for lam <= 24).
cudaError_t run_families(const WhtFamily* fam, int nfam, cudaStream_t st, int* nl) {
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(seg_pass_kernel), kBandSmem);
    if (e != cudaSuccess) return e;
  }
  // whole-vector tiles for lam <= 12 (pass 0 only), else flat passes over bits [8p, 8p+8)
  auto whole = [](const WhtFamily& w) { return w.first_bit == 0 && w.lam <= 12; };
  // 17..20 bits: near bits 0-7 + far bits 16.. in pass 0 (fn_tile), bits 8-15 last
  auto fnfam = [](const WhtFamily& w) { return w.first_bit == 0 && w.lam >= 17 && w.lam <= 20; };
  int npass = 0;
  for (int f = 0; f < nfam; ++f) {
    const int need = whole(fam[f]) ? 1 : fnfam(fam[f]) ? 2 : (fam[f].lam + 7) / 8;
    npass = need > npass ? need : npass;
  }
  for (int p = 0; p < npass; ++p) {
    SegPassTable T;
    T.count = 0;
    u64 tiles = 0;
    for (int f = 0; f < nfam; ++f) {
      const WhtFamily& w = fam[f];
      if (w.count == 0) continue;
      SegPass sp{};
      if (w.lam == 0 && w.in == w.out && w.scale == 1.0) continue;  // length-1 WHT: identity
      double2* fin = w.final_out ? w.final_out : w.out;
      sp.zshift = 63;
      sp.zrank = 0;
      sp.px = 0;
      sp.zoff = 0;
      if (fnfam(w)) {
        if (p >= 2 - w.skip_last) continue;
        const bool last = p == 1;
        sp.in = p == 0 ? w.in : w.out;
        sp.out = last ? fin : w.out;
        if (p == 0) {
          sp.fn = 1;
          sp.fn_lam = w.lam;
        } else {
          sp.b0 = 8;
          sp.K = 8;
        }
        sp.scale = last ? w.scale : 1.0;
        if (last) {
          sp.zshift = w.zshift;
          sp.zrank = w.zrank;
          sp.px = w.px;
          sp.zoff = w.zoff;
        }
        sp.first_tile = tiles;
        tiles += (w.count << w.lam) / kTileElems;
      } else if (whole(w)) {
        if (p != 0) continue;
        sp.small = 1;
        sp.in = w.in;
        sp.out = fin;
        sp.small_lam = w.lam;
        sp.scale = w.scale;
        sp.zshift = w.zshift;
        sp.zrank = w.zrank;
        sp.px = w.px;
        sp.zoff = w.zoff;
        sp.first_tile = tiles;
        tiles += w.count;
      } else {
        const int b0 = 8 * p;
        if (b0 < w.first_bit || b0 >= w.lam) continue;
        const int K = (w.lam - b0) < 8 ? (w.lam - b0) : 8;
        const bool last = b0 + K >= w.lam;
        if (last && w.skip_last) continue;
        sp.in = b0 == w.first_bit ? w.in : w.out;
        sp.out = last ? fin : w.out;
        sp.b0 = b0;
        sp.K = K;
        sp.scale = last ? w.scale : 1.0;
        if (last) {
          sp.zshift = w.zshift;
          sp.zrank = w.zrank;
          sp.px = w.px;
          sp.zoff = w.zoff;
        }
        sp.first_tile = tiles;
        tiles += (w.count << w.lam) / kTileElems;
      }
      if (T.count >= kMaxSeg) return cudaErrorInvalidValue;
      T.s[T.count++] = sp;
    }
    if (T.count == 0) continue;
    T.total_tiles = tiles;
    u64 grid = (u64)device_sm_count() * 2;
    if (grid > tiles) grid = tiles;
    seg_pass_kernel<<<(unsigned)grid, kThreads, kBandSmem, st>>>(T);
    *nl += 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---- top bits first: the z-sharded structured paths -------------
// Rank r of G = 2^g GPUs needs W[r 2^(lam-g) + zl] of every long WHT.  Splitting the index
// into its top 3 bits h and the rest il, W[zt 2^(lam-3) + zl] = WHT_{lam-3}(u_zt)[zl] with
// u_zt[il] = sum_h (-1)^{popcount(h & zt)} v[h 2^(lam-3) + il]: the three butterfly levels
// over the top bits come FIRST, and a rank keeps only the branches its z bits select (the
// signed projection u_r of the SURVEY's 8(e) formula), so it reads the vector once and
// transforms 1/G of it.  The one-GPU path runs the very same levels in the same order (top
// bit first) and keeps all eight branches, so every rank's outputs are bitwise the one-GPU
// values.  Used for vectors of at least 2^kTopMin elements; shorter ones stay replicated.

// W over the TB top index bits for the kept outputs zt = (rsel << KK) | kt, kt < 2^KK,
// levels in descending bit order (bit TB-1 first: pairs (h, h + 2^(TB-1)), ...); a z bit of
// 0 takes the sum.  The TB - KK top bits are fixed by rsel: each of those levels keeps one
// branch (a select, no divergence); the last KK levels are full butterflies.  Every kept
// output is the same sequence of operations whatever KK is -- on one GPU (KK = TB) all
// 2^TB outputs share their partial sums (TB 2^(TB-1) butterflies) -- so a rank's values are
// bitwise the one-GPU values.
__device__ __forceinline__ double2 bfly(double2 a, double2 b, bool diff) { return diff ? csub(a, b) : cadd(a, b); }
// fixed level S (S >= KK) and below, compile-time unrolled (a runtime level index would
// put the array in local memory)
template <int S, int KK, int N>
__device__ __forceinline__ void topk_fixed(double2 (&c)[N], unsigned zt0) {
  if constexpr (S >= KK) {
    const bool diff = ((zt0 >> S) & 1u) != 0;  // keep branch (zt0 >> S) & 1
#pragma unroll
    for (int j = 0; j < (1 << S); ++j) c[j] = bfly(c[j], c[j + (1 << S)], diff);
    topk_fixed<S - 1, KK, N>(c, zt0);
  }
}
template <int S, int N>
__device__ __forceinline__ void topk_full(double2 (&c)[N]) {
  if constexpr (S >= 0) {  // kept bits: full butterflies in place, bit S
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if constexpr (true) {
        if ((j >> S) & 1) continue;
        const double2 x = c[j], y = c[j | (1 << S)];
        c[j] = cadd(x, y);
        c[j | (1 << S)] = csub(x, y);
      }
    }
    topk_full<S - 1, N>(c);
  }
}
template <int TB, int KK>
__device__ __forceinline__ void topk_kept(const double2 (&d)[1 << TB], unsigned rsel, double2* o) {
  double2 c[1 << TB];
#pragma unroll
  for (int h = 0; h < (1 << TB); ++h) c[h] = d[h];
  topk_fixed<TB - 1, KK, (1 << TB)>(c, rsel << KK);
  double2 k[1 << KK];
#pragma unroll
  for (int j = 0; j < (1 << KK); ++j) k[j] = c[j];
  topk_full<KK - 1, (1 << KK)>(k);
#pragma unroll
  for (int kt = 0; kt < (1 << KK); ++kt) o[kt] = k[kt];
}

// Pass 0 of a long single vector: the TB top levels, then bits 4-7 and 0-3 of il exactly as
// contig8_tile orders them.  A tile holds KS = 2^KK kept top-bit branches x IL = 4096 / KS
// consecutive il (16 fibres of 256); it reads 2^TB x IL elements (2^TB runs of IL
// contiguous, coalesced) and writes KS runs of IL: out[kt 2^(lam-TB) + il].
template <int TB, int KK>
__global__ void __launch_bounds__(kThreads, 2) topk_pass_kernel(const double2* __restrict__ in, double2* out,
                                                                int lam, unsigned rsel) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  const int L = lam - TB;
  constexpr int KS = 1 << KK;
  constexpr int IL = kTileElems >> KK;
  const u64 Q = 1ull << L;
  const u64 ntiles = Q / (u64)IL;
  const int tid = threadIdx.x;
  for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const u64 il0 = tile * (u64)IL;
    // stage 0: top levels; IPR il per thread per round (16-32 loads in flight)
    constexpr int IPR = TB == 4 ? (KK <= 1 ? 2 : 1) : 2;
    for (int m = 0; m < IL / 256; m += IPR) {
      double2 d[IPR][1 << TB];
#pragma unroll
      for (int r = 0; r < IPR; ++r)
#pragma unroll
        for (int h = 0; h < (1 << TB); ++h) {
          // a rank keeping a fraction of the branches (KK < TB) reads the band once and
          // writes little: evict-first loads keep its output L2-resident for the tail
          // (n = 24, G = 8: 0.084 -> 0.076 ms); keeping every branch, plain loads are faster
          // (99 vs 115 us)
          const double2* p = in + (u64)h * Q + il0 + (u64)(tid + 256 * (m + r));
          d[r][h] = KK < TB ? ld_stream(p) : ld_l2(p);
        }
#pragma unroll
      for (int r = 0; r < IPR; ++r) {
        double2 o[KS];
        topk_kept<TB, KK>(d[r], rsel, o);
#pragma unroll
        for (int kt = 0; kt < KS; ++kt) {
          const int e = kt * IL + tid + 256 * (m + r);
          S[contig_slot(e >> 8, e & 255)] = o[kt];
        }
      }
    }
    __syncthreads();
    double2 v[16];
    {  // bits 4-7 of il
      const int f = tid >> 4, jl = tid & 15;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) v[kk] = S[contig_slot(f, jl + 16 * kk)];
      wht_regs<4>(v);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) S[contig_slot(f, jl + 16 * kk)] = v[kk];  // own slots only
    }
    __syncthreads();
    {  // bits 0-3 of il
      const int f = tid >> 4, kh = tid & 15;
#pragma unroll
      for (int jl = 0; jl < 16; ++jl) v[jl] = S[contig_slot(f, jl + 16 * kh)];
      wht_regs<4>(v);
#pragma unroll
      for (int jl = 0; jl < 16; ++jl) S[contig_slot(f, jl + 16 * kh)] = v[jl];
    }
    __syncthreads();
    {
      const int f = tid >> 4, jl = tid & 15;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int e = f * 256 + jl + 16 * kk;
        const int kt = e / IL, il = e - kt * IL;
        st_l2(out + ((u64)kt << L) + il0 + (u64)il, S[contig_slot(f, jl + 16 * kk)]);
      }
    }
    __syncthreads();
  }
}

template <int TB, int KK>
static cudaError_t launch_topk(const double2* in, double2* out, int lam, unsigned rsel, unsigned grid,
                               cudaStream_t st) {
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(topk_pass_kernel<TB, KK>), kBandSmem);
  if (e != cudaSuccess) return e;
  topk_pass_kernel<TB, KK><<<grid, kThreads, kBandSmem, st>>>(in, out, lam, rsel);
  return cudaGetLastError();
}

// Split of the short segments (lam < kTopMin, replicated on every rank): element id =
// 2^lam - 1 + h of segment lam (t = n - 1 - lam); TRIDIAGONAL stores full P_t (2^lam) then
// M_t (2^lam), HERMITIAN_TRIDIAGONAL S_t.  Run by the tail loop of the split kernels below
// (and alone when no segment is long).
__device__ __forceinline__ void split_small_one(const double2* __restrict__ band, double2* PM, int n, u64 id,
                                                bool herm) {
  const u64 N = 1ull << n;
  const int lam = 63 - __clzll((long long)(id + 1));
  const u64 h = id + 1 - (1ull << lam);
  const int t = n - 1 - lam;
  const u64 i = (h << (t + 1)) + (1ull << t) - 1ull;
  const u64 seg = N - (N >> t);
  if (herm) {
    PM[seg + h] = ld_stream(band + N + i);  // [main | sup]
    return;
  }
  const double2 sv = ld_stream(band + 2 * N + i), uv = ld_stream(band + i + 1);
  PM[2 * seg + h] = cadd(sv, uv);
  PM[2 * seg + (1ull << lam) + h] = csub(sv, uv);
}
__device__ __forceinline__ void split_small_loop(const double2* band, double2* PM, int n, int lam_max, bool herm) {
  const u64 total = (2ull << lam_max) - 1ull;  // lam = 0 .. lam_max
  for (u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x; id < total; id += (u64)gridDim.x * blockDim.x)
    split_small_one(band, PM, n, id, herm);
}
__global__ void split_small_kernel(const double2* __restrict__ band, double2* PM, int n, int lam_max, int herm) {
  split_small_loop(band, PM, n, lam_max, herm != 0);
}

// Tridiagonal split of the long segments (lam = n - t - 1 >= kTopMin) fused with their top
// levels: for i = h 2^(n-3) + i_low with t trailing ones (t < n - 3, the same for all eight
// top blocks h), S_t[.] = sup[i] and U_t[.] = sub[i + 1] sit at segment index
// h 2^(lam-3) + hl, hl = i_low >> (t + 1), so one coalesced read of the eight blocks feeds
// the top levels of P_t = WHT(S_t + U_t) and M_t = WHT(S_t - U_t).  Layout of a long
// segment: P_t at PM + 2 seg, KS branches of 2^(lam-3) (kt major), M_t right after.
template <int KK>
__global__ void __launch_bounds__(256) tri_split_top3_kernel(const double2* __restrict__ band, double2* PM, int n,
                                                             unsigned rsel, int lam_small) {
  const u64 N = 1ull << n;
  const u64 Q = N >> 3;
  const double2* sub = band;
  const double2* sup = band + 2 * N;
  constexpr int KS = 1 << KK;
  for (u64 il = (u64)blockIdx.x * blockDim.x + threadIdx.x; il < Q - 1; il += (u64)gridDim.x * blockDim.x) {
    const int t = __ffsll((long long)~il) - 1;
    const int lam = n - t - 1;
    if (lam < kTopMin) continue;
    double2 P[8], M[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const double2 sv = ld_stream(sup + (u64)h * Q + il);
      const double2 uv = ld_stream(sub + (u64)h * Q + il + 1);
      P[h] = cadd(sv, uv);
      M[h] = csub(sv, uv);
    }
    const u64 seg = N - (N >> t);
    const int Lb = lam - 3;
    double2* Pt = PM + 2 * seg;
    double2* Mt = Pt + ((u64)KS << Lb);
    const u64 hl = il >> (t + 1);
    double2 oP[KS], oM[KS];
    topk_kept<3, KK>(P, rsel, oP);
    topk_kept<3, KK>(M, rsel, oM);
#pragma unroll
    for (int kt = 0; kt < KS; ++kt) {
      st_l2(Pt + ((u64)kt << Lb) + hl, oP[kt]);
      st_l2(Mt + ((u64)kt << Lb) + hl, oM[kt]);
    }
  }
  split_small_loop(band, PM, n, lam_small, false);
}

// HERMITIAN_TRIDIAGONAL split: S_t only (sup; the sub-diagonal is conj(sup) and not stored).
template <int KK>
__global__ void __launch_bounds__(256) htri_split_top3_kernel(const double2* __restrict__ band, double2* W, int n,
                                                              unsigned rsel, int lam_small) {
  const double2* sup = band + (1ull << n);
  const u64 N = 1ull << n;
  const u64 Q = N >> 3;
  constexpr int KS = 1 << KK;
  for (u64 il = (u64)blockIdx.x * blockDim.x + threadIdx.x; il < Q - 1; il += (u64)gridDim.x * blockDim.x) {
    const int t = __ffsll((long long)~il) - 1;
    const int lam = n - t - 1;
    if (lam < kTopMin) continue;
    double2 S[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) S[h] = ld_stream(sup + (u64)h * Q + il);
    const u64 seg = N - (N >> t);
    const int Lb = lam - 3;
    double2* St = W + seg;
    const u64 hl = il >> (t + 1);
    double2 o[KS];
    topk_kept<3, KK>(S, rsel, o);
#pragma unroll
    for (int kt = 0; kt < KS; ++kt) st_l2(St + ((u64)kt << Lb) + hl, o[kt]);
  }
  split_small_loop(band, W, n, lam_small, true);
}

// ---- L2-resident tail of a long vector family (top-bits-first x = 0 vectors) ------------
// After topk_pass_kernel the family is `nvec` branches of 2^L elements (L = lam - 4 >= 17:
// 16 MiB each at n = 24), each still needing bits [8, 16) and [16, L).  Instead of two passes
// over the whole family (each a DRAM round trip of all of it), one persistent kernel runs
// both passes branch by branch: pass 1 of branch v reads it from DRAM and leaves it in L2,
// pass 2 of v (which needs all of v's pass-1 tiles: a completion counter per branch) reads
// it back from L2 and writes the result -- one DRAM round trip instead of two.  Ticket
// order P1(0..look), P2(0), P1(look+1), P2(1), ... (decode_tail); a CTA only ever waits for
// tiles with smaller tickets, which running CTAs hold, so progress is guaranteed.  Same
// tiles, same order of operations per element as the two flat passes: bitwise identical.
struct TailArgs {
  const double2* in;  // branches after pass 0 (pass 1 runs in place on them)
  double2* out;       // final output (pass 2)
  int L, nvec, look;
  double scale;
  int zshift;
  u64 zrank, px, zoff;
  unsigned* ctr;      // [0] ticket, [1 .. nvec] pass-1 tiles done per branch
};

__device__ __forceinline__ void decode_tail(u64 t, u64 TP, u64 C, u64 look, int& phase, u64& v, u64& tile) {
  const u64 lp1 = look + 1 < C ? look + 1 : C;
  if (t < lp1 * TP) { phase = 0; v = t / TP; tile = t % TP; return; }
  t -= lp1 * TP;
  const u64 steady = C > look + 1 ? C - look - 1 : 0;
  if (t < steady * 2 * TP) {
    const u64 c = t / (2 * TP), o = t % (2 * TP);
    if (o < TP) { phase = 1; v = c; tile = o; }
    else { phase = 0; v = c + look + 1; tile = o - TP; }
    return;
  }
  t -= steady * 2 * TP;
  phase = 1;
  v = steady + t / TP;
  tile = t % TP;
}

__global__ void __launch_bounds__(kThreads, 2) tail_pipe_kernel(const __grid_constant__ TailArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  const u64 TP = (1ull << A.L) / (u64)kTileElems;  // tiles per pass per branch
  const u64 total = 2ull * (u64)A.nvec * TP;
  unsigned* doneP1 = A.ctr + 1;
  // The next ticket is claimed while the current tile runs (its atomic's latency is hidden).
  // Tickets still rise per CTA and a tile only waits for smaller tickets, so the smallest
  // unfinished ticket is always some CTA's current tile: progress is guaranteed.
  __shared__ unsigned long long s_next[2];
  if (threadIdx.x == 0) s_next[0] = atomicAdd(A.ctr, 1u);
  __syncthreads();
  u64 tk = s_next[0];
  for (int par = 0; tk < total; par ^= 1) {
    if (threadIdx.x == 0) s_next[par ^ 1] = atomicAdd(A.ctr, 1u);
    int phase;
    u64 v, tile;
    decode_tail(tk, TP, (u64)A.nvec, (u64)A.look, phase, v, tile);
    SegPass sp{};
    sp.in = A.in;
    sp.zshift = 63;
    if (phase == 0) {
      sp.out = const_cast<double2*>(A.in);
      sp.b0 = 8;
      sp.scale = 1.0;
      flat_tile<8>(S, sp, v * TP + tile);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&doneP1[v], 1u);
      }
    } else {
      if (threadIdx.x == 0) {
        while (ld_acquire(&doneP1[v]) < (unsigned)TP) __nanosleep(64);
      }
      __syncthreads();
      sp.out = A.out;
      sp.b0 = 16;
      sp.scale = A.scale;
      sp.zshift = A.zshift;
      sp.zrank = A.zrank;
      sp.px = A.px;
      sp.zoff = A.zoff;
      switch (A.L - 16) {
        case 1: flat_tile<1>(S, sp, v * TP + tile); break;
        case 2: flat_tile<2>(S, sp, v * TP + tile); break;
        case 3: flat_tile<3>(S, sp, v * TP + tile); break;
        case 4: flat_tile<4>(S, sp, v * TP + tile); break;
        case 5: flat_tile<5>(S, sp, v * TP + tile); break;
        case 6: flat_tile<6>(S, sp, v * TP + tile); break;
        case 7: flat_tile<7>(S, sp, v * TP + tile); break;
        default: flat_tile<8>(S, sp, v * TP + tile); break;
      }
    }
    __syncthreads();  // S is reused by the next tile; s_next[par ^ 1] is visible
    tk = s_next[par ^ 1];
  }
}

constexpr int kTailMinL = 17;  // branches of >= 2^17 elements (two tail passes: bits 8-15, 16..)
constexpr int kTailMaxL = 24;  // pass 2 at most 8 bits

static cudaError_t launch_tail(const WhtFamily& f, unsigned* ctr, cudaStream_t st, int* nl) {
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(tail_pipe_kernel), kBandSmem);
  if (e != cudaSuccess) return e;
  TailArgs A;
  A.in = f.in;
  A.out = f.final_out ? f.final_out : f.out;
  A.L = f.lam;
  A.nvec = (int)f.count;
  A.look = 1;
#if PTDR_DEV
  {
    const char* el = getenv("PTDR_TAIL_LOOK");
    if (el && el[0] >= '0' && el[0] <= '3') A.look = el[0] - '0';
  }
#endif
  A.scale = f.scale;
  A.zshift = f.zshift;
  A.zrank = f.zrank;
  A.px = f.px;
  A.zoff = f.zoff;
  A.ctr = ctr;
  if ((e = cudaMemsetAsync(ctr, 0, (size_t)(A.nvec + 1) * 4, st)) != cudaSuccess) return e;
  const u64 tiles = 2ull * f.count * ((1ull << f.lam) / (u64)kTileElems);
  u64 grid = (u64)device_sm_count() * 2;
  if (grid > tiles) grid = tiles;
  tail_pipe_kernel<<<(unsigned)grid, kThreads, kBandSmem, st>>>(A);
  *nl += 1;
  return cudaGetLastError();
}

// ---- tridiagonal: last P/M pass fused with the expansion (segments t <= 3) ---------------
// For a long segment t whose last WHT pass runs over bits [8, 8 + K) of the branch index (the
// 17-20-bit families after fn_tile, or a 13-16-bit family after its contig8 pass), one tile
// takes the 2^(12-K) x 2^K fibres of that pass from P_t AND from M_t, transforms both (the same
// fiber_tile arithmetic, bitwise), and writes the 2^(t+1) outputs of every one of its 4096 zh
// values straight into block t+1 -- the P/M values never go back to DRAM and the expansion
// does not read them again (n = 24: 0.96 GiB less traffic).  Blocks t >= 4 keep the separate
// expansion (a tile's output, 2^(t+1) x 64 KiB, would unbalance the grid).  One CTA per SM
// (two 64 KiB transform buffers); the next tile's 32 loads per thread are issued before the
// current tile's output loop, so load latency hides behind the stores.
constexpr int kFuseMaxT = 7;
struct FusedSeg {
  const double2* P;  // P_t branches (KS x 2^lamp), M_t follows at P + KS 2^lamp
  u64 tiles;         // KS 2^lamp / 4096
  u64 first_tile;
  int lamp;          // branch length bits
  int K;             // bits of the last pass (at bit 8)
  int t;
  int parts_log;     // work items per tile = 2^parts_log (each emits 4096 / 2^parts_log slots)
};
struct FusedArgs {
  FusedSeg s[kFuseMaxT + 1];
  int count;
  u64 total_tiles;
  double2* out;  // block 0 of the rank's output (block t+1 at out + (t+1) NL)
  u64 NL;
  double scale;
  unsigned* ticket;
};
constexpr int kFusedSmem = 2 * kTileBytes;

template <int K, bool HERM>
__device__ __forceinline__ void fused_load(const FusedSeg& sg, u64 local, double2 (&vP)[16], double2 (&vM)[16]) {
  constexpr int F = kTileElems >> K;
  const int tid = threadIdx.x;
  const int f = tid % F, jh = tid / F;
  const u64 rho = local * F + (u64)f;
  const u64 msk = (1ull << 8) - 1ull;
  const double2* M = sg.P + ((u64)sg.tiles << 12);
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    const u64 j = (u64)((jh << 4) + kk);
    const u64 e = ((rho >> 8) << (8 + K)) | (j << 8) | (rho & msk);
    vP[kk] = ld_l2(sg.P + e);
    if constexpr (!HERM) vM[kk] = ld_l2(M + e);
  }
}

// fiber_tile<K> stages on registers already loaded (K >= 5: radix 16 then 2^(K-4)); the
// final values land at S[j F + f] (in place of the exchange slots).
template <int K>
__device__ __forceinline__ void fused_transform(double2* S, double2 (&v)[16]) {
  constexpr int F = kTileElems >> K;
  const int tid = threadIdx.x;
  wht_regs<4>(v);
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
    for (int jh = 0; jh < (1 << R2); ++jh) S[(jh * 16 + jl) * F + f] = w[jh];
  }
}

// Outputs of slots [part S_p, (part + 1) S_p) of the tile (S_p = 4096 / parts).  Thread tid
// writes o = tid + 256 i: zl = o mod 2^(t+1) is fixed per thread (t <= 3), so the phase and
// the P/M choice are too; slot = j F + f maps to e = e0 + (j << 8) + f (F <= 256).
template <int K, bool HERM>
__device__ __forceinline__ void fused_emit(const FusedArgs& A, const FusedSeg& sg, u64 local, int part,
                                           const double2* SP, const double2* SM) {
  constexpr int F = kTileElems >> K;
  const int t = sg.t;
  const int tb = t + 1;
  const int sp_bits = 12 - (sg.parts_log);
  const u64 per = 1ull << (sp_bits + tb);  // outputs of this work item
  double2* blk = A.out + (u64)tb * A.NL;
  const u64 rb = local * (u64)F;
  const u64 e0 = ((rb >> 8) << (8 + K)) | (rb & 255ull);
  const int zl = threadIdx.x & ((1 << tb) - 1);
  const int s1 = __popc(zl & ((1 << t) - 1)) & 1;
  const int s2 = (zl >> t) & 1;
  const double2* src = (HERM || s1 == s2) ? SP : SM;
  const int ph = __popc(zl) + 2 * s1;
  const bool sw = (ph & 1) != 0;
  const double sc = (ph & 2) ? -A.scale : A.scale;
  double2* base = blk + (e0 << tb) + (u64)zl;
  const int slot_base = part << sp_bits;
  for (u64 o = threadIdx.x; o < per; o += kThreads) {
    const int slot = slot_base + (int)(o >> tb);
    const int f = slot & (F - 1), j = slot / F;
    double2 w = src[slot];
    if constexpr (HERM) w = s1 == s2 ? make_double2(2.0 * w.x, 0.0) : make_double2(0.0, 2.0 * w.y);
    const double re = sw ? -w.y : w.x;
    const double im = sw ? w.x : w.y;
    st_stream(base + ((((u64)j << 8) + (u64)f) << tb), make_double2(re * sc, im * sc));
  }
}

__device__ __forceinline__ int fused_seg_of(const FusedArgs& A, u64 tile) {
  int i = 0;
  while (i + 1 < A.count && A.s[i + 1].first_tile <= tile) ++i;
  return i;
}

template <bool HERM>
__device__ __forceinline__ void fused_load_any(const FusedSeg& sg, u64 local, double2 (&vP)[16], double2 (&vM)[16]) {
  switch (sg.K) {
    case 5: fused_load<5, HERM>(sg, local, vP, vM); break;
    case 6: fused_load<6, HERM>(sg, local, vP, vM); break;
    case 7: fused_load<7, HERM>(sg, local, vP, vM); break;
    default: fused_load<8, HERM>(sg, local, vP, vM); break;
  }
}
template <int K, bool HERM>
__device__ __forceinline__ void fused_transform2(double2* SP, double2* SM, double2 (&vP)[16], double2 (&vM)[16]) {
  fused_transform<K>(SP, vP);
  if constexpr (!HERM) fused_transform<K>(SM, vM);
}

template <bool HERM>
__global__ void __launch_bounds__(kThreads, 1) tri_fused_expand_kernel(const __grid_constant__ FusedArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* SP = reinterpret_cast<double2*>(smem_raw);
  double2* SM = SP + kTileElems;
  __shared__ unsigned long long s_tk;
  if (threadIdx.x == 0) s_tk = atomicAdd(A.ticket, 1u);
  __syncthreads();
  u64 item = s_tk;
  double2 vP[16], vM[16];
  if (item < A.total_tiles) {
    const FusedSeg& sg = A.s[fused_seg_of(A, item)];
    fused_load_any<HERM>(sg, (item - sg.first_tile) >> sg.parts_log, vP, vM);
  }
  while (item < A.total_tiles) {
    const FusedSeg& sg = A.s[fused_seg_of(A, item)];
    const u64 rel = item - sg.first_tile;
    const u64 local = rel >> sg.parts_log;
    const int part = (int)(rel & ((1ull << sg.parts_log) - 1ull));
    switch (sg.K) {
      case 5: fused_transform2<5, HERM>(SP, SM, vP, vM); break;
      case 6: fused_transform2<6, HERM>(SP, SM, vP, vM); break;
      case 7: fused_transform2<7, HERM>(SP, SM, vP, vM); break;
      default: fused_transform2<8, HERM>(SP, SM, vP, vM); break;
    }
    // next ticket, and its loads issued before this item's output loop
    if (threadIdx.x == 0) s_tk = atomicAdd(A.ticket, 1u);
    __syncthreads();
    const u64 next = s_tk;
    if (next < A.total_tiles) {
      const FusedSeg& sn = A.s[fused_seg_of(A, next)];
      fused_load_any<HERM>(sn, (next - sn.first_tile) >> sn.parts_log, vP, vM);
    }
    switch (sg.K) {
      case 5: fused_emit<5, HERM>(A, sg, local, part, SP, SM); break;
      case 6: fused_emit<6, HERM>(A, sg, local, part, SP, SM); break;
      case 7: fused_emit<7, HERM>(A, sg, local, part, SP, SM); break;
      default: fused_emit<8, HERM>(A, sg, local, part, SP, SM); break;
    }
    __syncthreads();  // SP / SM and s_tk are rewritten by the next item
    item = next;
  }
}

// Workspace: [P/M segments: 2 * 2^n] (TRIDIAGONAL; S segments: 2^n for
// HERMITIAN_TRIDIAGONAL) + [x = 0 vector: 2^n] (world > 1: the x = 0 intermediate when it
// does not fit the rank's output block) + [tail counters].
constexpr size_t kTailCtrBytes = 256;
static size_t seg_ws_elems(int n, int structure) {
  const size_t N = (size_t)1 << n;
  return structure == 4 ? 2 * N : structure == 6 ? N : 0;
}
size_t band_workspace_bytes(int n, int structure, int world) {
  const size_t N = (size_t)1 << n;
  size_t b = seg_ws_elems(n, structure) * 16;
  if (world > 1 && n > 12) b += N * 16;
  return b + kTailCtrBytes;
}

cudaError_t launch_band(const double2* A, double2* out, int n, int structure, void* ws, int rank,
                        int world, cudaStream_t st, int* nl) {
  const u64 N = 1ull << n;
  const double scale = ldexp(1.0, -n);
  const int g = __builtin_ctz((unsigned)world);
  const int zshift = world > 1 ? n - g : 63;
  const u64 zrank = world > 1 ? (u64)rank : 0ull;
  double2* PM = reinterpret_cast<double2*>(ws);
  double2* X0 = world > 1 ? PM + seg_ws_elems(n, structure) : nullptr;  // x = 0 scratch
  unsigned* tail_ctr = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ws) + band_workspace_bytes(n, structure, world) -
                                                   kTailCtrBytes);
  // the x = 0 family after topk_pass_kernel: its two remaining passes as the L2-resident tail
  auto tail_ok = [](const WhtFamily& f) { return f.first_bit == 8 && f.lam >= kTailMinL && f.lam <= kTailMaxL; };
  const int sms = device_sm_count();
  // top-bits-first geometry: gp of the rank's bits select branches (at most the 3 top ones),
  // the remaining g - gp bits are a slice filter of the last pass
  const int gp = g < 3 ? g : 3;
  const int k_keep = 3 - gp;
  const unsigned rsel = (unsigned)(world > 1 ? (rank >> (g - gp)) : 0);
  cudaError_t e = cudaSuccess;
  // The x = 0 family (diagonal, anti-diagonal, tridiagonal main diagonal): vector `src`,
  // output block 0 of `out` (2^n / world elements), px = X-mask phase.
  auto x0_family = [&](const double2* src, u64 px, WhtFamily& f) -> cudaError_t {
    if (n >= kTopMinX0) {
      // top levels + bits 0-7 in one pass into the rank's kept branches (the top 4 bits from
      // n = 16 on: 16 branches of 2^(n-4), short enough for the L2-resident tail; 3 at
      // n = 15), then bits 8.. of the branches; ranks beyond the top TB bits filter their
      // slice in the last pass
      const int TB = n >= 16 ? 4 : 3;
      const int gx = g < TB ? g : TB;
      const int kx = TB - gx;
      const unsigned rx = (unsigned)(world > 1 ? (rank >> (g - gx)) : 0);
      double2* mid = (g <= TB) ? out : X0;
      u64 tiles = ((N >> TB) / (u64)(kTileElems >> kx));
      u64 grid = (u64)sms * 2;
      if (grid > tiles) grid = tiles;
      const unsigned gr = (unsigned)grid;
      if (TB == 4) {
        switch (kx) {
          case 4: e = launch_topk<4, 4>(src, mid, n, rx, gr, st); break;
          case 3: e = launch_topk<4, 3>(src, mid, n, rx, gr, st); break;
          case 2: e = launch_topk<4, 2>(src, mid, n, rx, gr, st); break;
          case 1: e = launch_topk<4, 1>(src, mid, n, rx, gr, st); break;
          default: e = launch_topk<4, 0>(src, mid, n, rx, gr, st); break;
        }
      } else {
        switch (kx) {
          case 3: e = launch_topk<3, 3>(src, mid, n, rx, gr, st); break;
          case 2: e = launch_topk<3, 2>(src, mid, n, rx, gr, st); break;
          case 1: e = launch_topk<3, 1>(src, mid, n, rx, gr, st); break;
          default: e = launch_topk<3, 0>(src, mid, n, rx, gr, st); break;
        }
      }
      if (e != cudaSuccess) return e;
      *nl += 1;
      f = WhtFamily{mid, mid, n - TB, 1ull << kx, scale};
      f.first_bit = 8;
      f.final_out = out;
      f.zshift = g > TB ? n - g : 63;
      f.zrank = g > TB ? (u64)(rank & ((1 << (g - TB)) - 1)) : 0ull;
      f.zoff = (u64)rx << (n - gx);
      f.px = px;
      return cudaSuccess;
    }
    // short vectors: every rank runs the whole transform; only the last pass stores, and
    // only the rank's slice
    f = WhtFamily{src, world > 1 && n > 12 ? X0 : out, n, 1, scale};
    f.final_out = out;
    f.zshift = zshift;
    f.zrank = zrank;
    f.px = px;
    return cudaSuccess;
  };
  if (structure == 3 || structure == 5) {
    // DIAGONAL: x = 0.  ANTI_DIAGONAL: v_x[i] = A[i][i ^ (2^n - 1)] = a[i] is
    // nonzero only for x = 2^n - 1, so alpha(2^n - 1, z) = 2^-n i^{popcount(z)} WHT(a)[z].
    WhtFamily f;
    if ((e = x0_family(A, structure == 5 ? N - 1 : 0ull, f)) != cudaSuccess) return e;
    if (tail_ok(f)) return launch_tail(f, tail_ctr, st, nl);
    return run_families(&f, 1, st, nl);
  }
  // TRIDIAGONAL: A = [sub | main | sup]; HERMITIAN_TRIDIAGONAL: A = [main | sup], the
  // sub-diagonal conj(sup) implied (one WHT per segment, see herm_seg_view).
  const bool herm = structure == 6;
  const double2* mainv = herm ? A : A + N;
  const u64 segmul = herm ? 1 : 2;  // P_t and M_t, or S_t
  // Block 0 (x = 0, WHT(main) scaled) first: its passes stream the main diagonal through L2,
  // so running them before the split keeps the split's output L2-resident for the segment
  // passes that follow.
  WhtFamily fam[kMaxSeg];
  int nf = 0;
  if ((e = x0_family(mainv, 0ull, fam[nf])) != cudaSuccess) return e;
  if (tail_ok(fam[nf])) {
    if ((e = launch_tail(fam[nf], tail_ctr, st, nl)) != cudaSuccess) return e;
  } else {
    ++nf;
  }
  // Segments t with lam = n - t - 1 >= kTopMin: fused split + top levels (the rank's branches
  // only); shorter ones: plain split, replicated.
  const int lam_small = n - 1 < kTopMin - 1 ? n - 1 : kTopMin - 1;
  if (n - 1 >= kTopMin) {
    // long segments + (tail loop) the short ones, one launch
    u64 blocks = ((N >> 3) + 255) / 256;
    if (blocks > (u64)sms * 16) blocks = (u64)sms * 16;
    const unsigned b = (unsigned)blocks;
    if (herm) {
      switch (k_keep) {
        case 3: htri_split_top3_kernel<3><<<b, 256, 0, st>>>(A, PM, n, rsel, lam_small); break;
        case 2: htri_split_top3_kernel<2><<<b, 256, 0, st>>>(A, PM, n, rsel, lam_small); break;
        case 1: htri_split_top3_kernel<1><<<b, 256, 0, st>>>(A, PM, n, rsel, lam_small); break;
        default: htri_split_top3_kernel<0><<<b, 256, 0, st>>>(A, PM, n, rsel, lam_small); break;
      }
    } else {
      switch (k_keep) {
        case 3: tri_split_top3_kernel<3><<<b, 256, 0, st>>>(A, PM, n, rsel, lam_small); break;
        case 2: tri_split_top3_kernel<2><<<b, 256, 0, st>>>(A, PM, n, rsel, lam_small); break;
        case 1: tri_split_top3_kernel<1><<<b, 256, 0, st>>>(A, PM, n, rsel, lam_small); break;
        default: tri_split_top3_kernel<0><<<b, 256, 0, st>>>(A, PM, n, rsel, lam_small); break;
      }
    }
  } else {
    u64 total = (2ull << lam_small) - 1ull;
    u64 blocks = (total + 255) / 256;
    if (blocks > (u64)sms * 32) blocks = (u64)sms * 32;
    split_small_kernel<<<(unsigned)blocks, 256, 0, st>>>(A, PM, n, lam_small, herm ? 1 : 0);
  }
  *nl += 1;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // blocks t+1: P_t / M_t (or S_t).  Segments t < tf run their last pass inside the fused
  // expansion.
  const int zs = world > 1 ? zshift : n;
  const u64 NL = 1ull << zs;
  FusedArgs FA{};
  int tf = 0;
  if (g <= 3 && NL >= 256) {
    for (int t = 0; t <= kFuseMaxT && t < n; ++t) {
      const int lam = n - t - 1, lamp = lam - 3;
      if (lam < kTopMin || lamp < 13 || lamp > 20) break;
      FusedSeg& sg = FA.s[tf];
      sg.P = PM + segmul * (N - (N >> t));
      sg.tiles = ((u64)1 << (lamp + k_keep)) / (u64)kTileElems;
      sg.lamp = lamp;
      sg.K = lamp - 8 < 8 ? lamp - 8 : 8;
      sg.t = t;
      sg.parts_log = t > 1 ? t - 1 : 0;  // <= 256 KiB of output per work item
      ++tf;
    }
  }
  for (int t = 0; t < n; ++t) {
    const int lam = n - t - 1;
    double2* base = PM + segmul * (N - (N >> t));
    if (lam >= kTopMin) {
      WhtFamily f{base, base, lam - 3, segmul << k_keep, 1.0};  // [P then M] or S branches
      f.first_bit = 0;
      f.skip_last = t < tf ? 1 : 0;
      fam[nf++] = f;
    } else {
      fam[nf++] = WhtFamily{base, base, lam, segmul, 1.0};
    }
  }
  if ((e = run_families(fam, nf, st, nl)) != cudaSuccess) return e;
  if (tf > 0) {
    // largest outputs per tile first (t descending) for the dynamic tickets
    FusedArgs B = FA;
    u64 first = 0;
    for (int i = 0; i < tf; ++i) {
      B.s[i] = FA.s[tf - 1 - i];
      B.s[i].first_tile = first;
      first += B.s[i].tiles << B.s[i].parts_log;
    }
    B.count = tf;
    B.total_tiles = first;
    B.out = out;
    B.NL = NL;
    B.scale = scale;
    B.ticket = tail_ctr + 63;
    if ((e = cudaMemsetAsync(B.ticket, 0, 4, st)) != cudaSuccess) return e;
    const void* kf = herm ? reinterpret_cast<const void*>(tri_fused_expand_kernel<true>)
                          : reinterpret_cast<const void*>(tri_fused_expand_kernel<false>);
    if ((e = ensure_smem_attr(kf, kFusedSmem)) != cudaSuccess) return e;
    u64 grid = (u64)sms;
    if (grid > first) grid = first;
    if (herm) tri_fused_expand_kernel<true><<<(unsigned)grid, kThreads, kFusedSmem, st>>>(B);
    else tri_fused_expand_kernel<false><<<(unsigned)grid, kThreads, kFusedSmem, st>>>(B);
    *nl += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  {
    const u64 total = (u64)n * NL;
    if (NL >= 256) {
      u64 blocks = (total / 8 + 255) / 256;
      if (blocks > (u64)sms * 16) blocks = (u64)sms * 16;
      if (herm) tridiag_expand_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(PM, out, n, scale, zs, zrank, k_keep, tf);
      else tridiag_expand_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(PM, out, n, scale, zs, zrank, k_keep, tf);
    } else {
      const unsigned b = (unsigned)((total + 255) / 256);
      if (herm) tridiag_expand_small_kernel<true><<<b, 256, 0, st>>>(PM, out, n, scale, zs, zrank, k_keep);
      else tridiag_expand_small_kernel<false><<<b, 256, 0, st>>>(PM, out, n, scale, zs, zrank, k_keep);
    }
    *nl += 1;
    e = cudaGetLastError();
  }
  return e;
}


// =====================================================================================
// BAND(s): (2s+1)-band matrices (Table I l.500-518).
//
// Input diags[d + s][i] = A[i][i + d], d in [-s, s].  For an X-mask x with top bit t,
// v_x[i] = A[i][i ^ x] with i ^ x - i = x - 2 (i & x) (the high bits of i above t are
// unchanged), so v_x[i] != 0 only if m = i & x satisfies |x - 2m| <= s, a condition on the
// low t+1 bits l of i alone.  Writing i = h 2^{t+1} + l:
//   WHT_n(v_x)[z] = sum_{l in L_x} (-1)^{popcount(l & z_lo)} W_{x,l}[z_hi],
//   W_{x,l} = WHT_{n-t-1}(h -> D_{x - 2(l & x)}[h 2^{t+1} + l]),
// z_lo = z mod 2^{t+1}, z_hi = z >> (t+1), and alpha(x, z) = 2^-n i^{popcount(x & z)}
// WHT_n(v_x)[z].  L_x = {m | f : m subset of x, |x - 2m| <= s, f subset of the zero bits of
// x below t+1}.  x is in the support X_s iff L_x is non-empty; that forces
// x >= 2^{t+1} - s, so at most s candidates per top bit (|X_s| = s n - c(s), Table I).
// The tridiagonal path is s = 1 with the two segments folded into P/M; x = 0 is the main
// diagonal (t = -1, one segment of length 2^n).
// =====================================================================================
struct BandBlockDev {
  unsigned long long x;
  int t;      // top bit of x (-1 for x = 0)
  int nL;     // segments of this block
  int first;  // index into the segment-reference list
  int pad;
};
struct BandSegRef {
  unsigned long long l;
  unsigned long long off;  // element offset of W_{x,l} in the segment storage
};

struct BandPlan {
  int n = 0, s = 0;
  std::vector<BandBlockDev> blocks;
  std::vector<BandSegRef> refs;
  std::vector<int> seg_d, seg_t, seg_lam;  // per segment (same order as refs)
  std::vector<int> fam_lam;                // families: lam and their [first, count) in refs
  std::vector<int> fam_count;
  std::vector<unsigned long long> fam_off;  // storage offset of each family
  unsigned long long seg_elems = 0;
  size_t table_bytes = 0, ws_bytes = 0;
};

static bool band_member(unsigned long long x, int s) {
  // exists m subset of x with |x - 2m| <= s
  const long long lo = ((long long)x - s + 1) / 2 > 0 ? ((long long)x - s + 1) / 2 : 0;
  const long long hi = ((long long)x + s) / 2;
  for (long long m = lo; m <= hi && m <= (long long)x; ++m)
    if (((unsigned long long)m & ~x) == 0ull && std::llabs((long long)x - 2 * m) <= s) return true;
  return false;
}

static BandPlan make_band_plan(int n, int s) {
  BandPlan p;
  p.n = n;
  p.s = s;
  struct Seg { unsigned long long x, l; int t, d, lam, block; };
  std::vector<Seg> segs;
  auto add_block = [&](unsigned long long x, int t) {
    BandBlockDev b{};
    b.x = x;
    b.t = t;
    b.first = 0;
    b.nL = 0;
    const int lam = n - t - 1;
    const int blk = (int)p.blocks.size();
    if (t < 0) {
      segs.push_back({0ull, 0ull, -1, 0, n, blk});
      b.nL = 1;
    } else {
      const unsigned long long F = (~x) & ((2ull << t) - 1ull);  // free bits
      const long long lo = ((long long)x - s + 1) / 2 > 0 ? ((long long)x - s + 1) / 2 : 0;
      for (long long m = lo; m <= ((long long)x + s) / 2 && m <= (long long)x; ++m) {
        if (((unsigned long long)m & ~x) != 0ull || std::llabs((long long)x - 2 * m) > s) continue;
        // every submask f of F
        unsigned long long f = 0;
        for (;;) {
          segs.push_back({x, (unsigned long long)m | f, t, (int)((long long)x - 2 * m), lam, blk});
          ++b.nL;
          if (f == F) break;
          f = (f - F) & F;  // next submask in increasing order
        }
      }
    }
    p.blocks.push_back(b);
  };
  add_block(0ull, -1);
  for (int t = 0; t < n; ++t) {
    const unsigned long long top = 1ull << t, hi = (2ull << t) - 1ull;
    const unsigned long long lo = (hi + 1 > (unsigned long long)s && hi + 1 - s > top) ? hi + 1 - s : top;
    for (unsigned long long x = lo; x <= hi; ++x)
      if (band_member(x, s)) add_block(x, t);
  }
  // storage grouped by lam (one WHT family per length), refs in block order
  std::vector<int> order(segs.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return segs[a].lam > segs[b].lam; });
  std::vector<unsigned long long> off(segs.size());
  unsigned long long cur = 0;
  for (size_t k = 0; k < order.size(); ++k) {
    const Seg& sg = segs[order[k]];
    if (p.fam_lam.empty() || p.fam_lam.back() != sg.lam) {
      p.fam_lam.push_back(sg.lam);
      p.fam_off.push_back(cur);
      p.fam_count.push_back(0);
    }
    ++p.fam_count.back();
    off[order[k]] = cur;
    cur += 1ull << sg.lam;
  }
  p.seg_elems = cur;
  // refs grouped per block (segments were appended block by block)
  int first = 0;
  for (size_t bi = 0; bi < p.blocks.size(); ++bi) {
    p.blocks[bi].first = first;
    first += p.blocks[bi].nL;
  }
  p.refs.resize(segs.size());
  p.seg_d.resize(segs.size());
  p.seg_t.resize(segs.size());
  p.seg_lam.resize(segs.size());
  for (size_t k = 0; k < segs.size(); ++k) {
    p.refs[k] = BandSegRef{segs[k].l, off[k]};
    p.seg_d[k] = segs[k].d;
    p.seg_t[k] = segs[k].t;
    p.seg_lam[k] = segs[k].lam;
  }
  const size_t tb = p.blocks.size() * sizeof(BandBlockDev) + p.refs.size() * sizeof(BandSegRef) +
                    segs.size() * sizeof(int4) + (size_t)n * (s > 0 ? s : 1) * sizeof(int);
  p.table_bytes = (tb + 255) / 256 * 256;
  p.ws_bytes = p.table_bytes + (size_t)p.seg_elems * 16;
  return p;
}

// Gather: seg[h] = diags[d + s][h 2^{t+1} + l] for every segment; one thread per element.
// gat[k] = {t, d, lam, unused} per segment (segment order = refs order).
__global__ void band_gather_kernel(const double2* diags, int n, int s, const BandSegRef* refs,
                                   const int4* gat, int nseg, double2* segs) {
  const u64 N = 1ull << n;
  for (int k = blockIdx.y; k < nseg; k += gridDim.y) {
    const int4 g = gat[k];
    const u64 len = 1ull << g.z;
    const u64 l = refs[k].l;
    const int sh = g.x + 1;  // t + 1 (0 for x = 0)
    const double2* D = diags + (u64)(g.y + s) * N;
    double2* dst = segs + refs[k].off;
    for (u64 h = (u64)blockIdx.x * blockDim.x + threadIdx.x; h < len; h += (u64)gridDim.x * blockDim.x)
      dst[h] = ld_stream(D + ((h << sh) | l));
  }
}

// Gather in diagonal order: every stored band element A[i][i+d] belongs to exactly one
// segment -- x = i ^ (i+d), l = i mod 2^{t+1}, h = i >> (t+1) -- so each diagonal is read
// once, coalesced (the per-segment gather above reads a 32 B sector per element).
// xblock[t * s + e] = block index of x = 2^{t+1} - 1 - e (-1 if x is not in the support).
__global__ void band_gather_diag_kernel(const double2* diags, int n, int s, const BandBlockDev* blocks,
                                        const BandSegRef* refs, const int* xblock, double2* segs) {
  const u64 N = 1ull << n;
  const u64 total = (u64)(2 * s + 1) * N;
  for (u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x; id < total; id += (u64)gridDim.x * blockDim.x) {
    const int d = (int)(id >> n) - s;
    const u64 i = id & (N - 1);
    const long long j = (long long)i + d;
    if (j < 0 || j >= (long long)N) continue;
    const double2 v = ld_stream(diags + id);
    if (d == 0) {  // x = 0: block 0, one segment of length 2^n
      segs[refs[blocks[0].first].off + i] = v;
      continue;
    }
    const u64 x = i ^ (u64)j;
    const int t = 63 - __clzll(x);
    const u64 e = ((2ull << t) - 1ull) - x;
    const BandBlockDev B = blocks[xblock[t * s + (int)e]];
    const u64 l = i & ((2ull << t) - 1ull);
    for (int k = 0; k < B.nL; ++k) {
      const BandSegRef r = refs[B.first + k];
      if (r.l == l) {
        segs[r.off + (i >> (t + 1))] = v;
        break;
      }
    }
  }
}

// Gather with the top three butterfly levels first (n >= kTopMin + 1): thread (d, il) reads the
// eight rows i_h = h 2^(n-3) + il of diagonal d (coalesced along il).  When il + d stays inside
// [0, 2^(n-3)) the eight elements share x = il ^ (il + d) and l, and sit at segment indices
// h 2^(lam-3) + (il >> (t+1)): for a long segment (lam >= kTopMin) they are combined by the
// top three levels of its WHT right here (topk_kept, as the tridiagonal split) and stored as
// eight branches of 2^(lam-3) -- the branch-major result of the remaining passes is the natural
// output order, so the expansion is unchanged -- and a long family needs one pass less (n = 24,
// s = 2: two passes instead of three).  Short segments and boundary rows are scattered as
// band_gather_diag_kernel does.
__device__ __forceinline__ const BandSegRef* band_find_ref(const BandBlockDev& B, const BandSegRef* refs, u64 l) {
  for (int k = 0; k < B.nL; ++k)
    if (refs[B.first + k].l == l) return &refs[B.first + k];
  return nullptr;
}
__global__ void __launch_bounds__(256) band_gather_top3_kernel(const double2* diags, int n, int s,
                                                               const BandBlockDev* blocks, const BandSegRef* refs,
                                                               const int* xblock, double2* segs) {
  const u64 N = 1ull << n;
  const u64 Q = N >> 3;
  const u64 Q4 = N >> 4;
  // ids [0, 2s Q): the off-diagonals (d = -s..-1, 1..s); [2s Q, 2s Q + Q4): the main diagonal
  // (x = 0: one segment of 2^n, its top FOUR levels here -> 16 branches of 2^(n-4), so it
  // needs two passes like the rest)
  const u64 total = (u64)(2 * s) * Q + Q4;
  for (u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x; id < total; id += (u64)gridDim.x * blockDim.x) {
    if (id >= (u64)(2 * s) * Q) {
      const u64 il = id - (u64)(2 * s) * Q;
      const double2* D = diags + (u64)s * N;
      double2 w[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) w[h] = ld_stream(D + (u64)h * Q4 + il);
      const BandSegRef r = refs[blocks[0].first];
      double2 o[16];
      topk_kept<4, 4>(w, 0u, o);
#pragma unroll
      for (int kt = 0; kt < 16; ++kt) segs[r.off + ((u64)kt << (n - 4)) + il] = o[kt];
      continue;
    }
    const int di = (int)(id / Q);
    const int d = di < s ? di - s : di - s + 1;
    const u64 il = id - (u64)di * Q;
    const double2* D = diags + (u64)(d + s) * N;
    double2 v[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) v[h] = ld_stream(D + (u64)h * Q + il);
    const long long jl = (long long)il + d;
    if (jl >= 0 && jl < (long long)Q) {
      const u64 x = il ^ (u64)jl;
      const int t = 63 - __clzll(x);
      const int lam = n - t - 1;
      if (lam >= kTopMin) {
        const u64 e = ((2ull << t) - 1ull) - x;
        const BandBlockDev B = blocks[xblock[t * s + (int)e]];
        const BandSegRef* r = band_find_ref(B, refs, il & ((2ull << t) - 1ull));
        if (r) {
          double2 o[8];
          topk_kept<3, 3>(v, 0u, o);
          const u64 hl = il >> (t + 1);
#pragma unroll
          for (int kt = 0; kt < 8; ++kt) segs[r->off + ((u64)kt << (lam - 3)) + hl] = o[kt];
        }
        continue;
      }
    }
    // short segments / rows whose + d crosses a top-block boundary: one element each
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const u64 i = (u64)h * Q + il;
      const long long j = (long long)i + d;
      if (j < 0 || j >= (long long)N) continue;
      const u64 x = i ^ (u64)j;
      const int t = 63 - __clzll(x);
      const u64 e = ((2ull << t) - 1ull) - x;
      const BandBlockDev B = blocks[xblock[t * s + (int)e]];
      const BandSegRef* r = band_find_ref(B, refs, i & ((2ull << t) - 1ull));
      if (r) segs[r->off + (i >> (t + 1))] = v[h];
    }
  }
}

// One segment's contribution to a lane's 8 outputs z = z0 + 32 j (z0 = base + lane, base a
// multiple of 256, so bits 5-7 of z0 are zero).  Wg = W + (base >> SH): the sample of output z
// is Wg[(lane + 32 j) >> SH], which for SH >= 5 does not depend on the lane, so only 256 >> SH
// distinct values (one for SH >= 8) are loaded instead of one per output.  The signs
// (-1)^{popcount(lm & z)} = (-1)^{popcount(lm & z0)} (-1)^{popcount(((lm >> 5) & 7) & j)} come
// from one byte-table lookup per segment (bit j of T), and are applied as fma(+-1, w, acc):
// exactly acc +- w.
#ifndef PTDR_BAND_PF
#define PTDR_BAND_PF 1
#endif
constexpr int kBandPrefetchDist = PTDR_BAND_PF;  // groups ahead (grid strides) for the L1 prefetch

template <int SH>
__device__ __forceinline__ void band_accum(const double2* __restrict__ Wg, unsigned z0, unsigned lane, unsigned lm,
                                           double (&re)[8], double (&im)[8]) {
  constexpr int D = SH >= 8 ? 1 : (SH >= 5 ? (256 >> SH) : 8);  // loads per lane
  double2 w[D];
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const unsigned idx = SH >= 5 ? (unsigned)m : ((lane + 32u * m) >> SH);
#if defined(PTDR_DIAG) && (PTDR_DIAG & 8)
    w[m] = make_double2((double)(size_t)Wg, (double)idx);  // diagnostics: no W loads
#else
    w[m] = __ldg(Wg + idx);
#endif
  }
  // byte m of {0x963C5AF0 : 0x66CCAA00} has bit j = parity(m & j)
  const unsigned T = __byte_perm(0x66CCAA00u, 0x963C5AF0u, (lm >> 5) & 7u) ^ (0u - (__popc(lm & z0) & 1u));
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double2 v = w[SH >= 8 ? 0 : (SH >= 5 ? (j >> (SH - 5)) : j)];
    const double sg = __hiloint2double((int)(((T << (31 - j)) & 0x80000000u) | 0x3ff00000u), 0);
    re[j] = fma(sg, v.x, re[j]);
    im[j] = fma(sg, v.y, im[j]);
  }
}

// NL segments with one sample each (block shift >= 8): all loads first, then the signed sums.
template <int NL>
__device__ __forceinline__ void band_accum_single(const BandSegRef* __restrict__ rf, const double2* Wb,
                                                  unsigned lomask, unsigned z0, double (&re)[8], double (&im)[8]) {
  double2 wk[NL];
  unsigned lmk[NL];
#pragma unroll
  for (int kk = 0; kk < NL; ++kk) {
    const unsigned long long rl = __ldg(&rf[kk].l), roff = __ldg(&rf[kk].off);
    lmk[kk] = (unsigned)rl & lomask;
#if defined(PTDR_DIAG) && (PTDR_DIAG & 8)
    wk[kk] = make_double2((double)roff, 1.0);
#else
    wk[kk] = __ldg(Wb + roff);
#endif
  }
#pragma unroll
  for (int kk = 0; kk < NL; ++kk) {
    const unsigned lm = lmk[kk];
    const unsigned T = __byte_perm(0x66CCAA00u, 0x963C5AF0u, (lm >> 5) & 7u) ^ (0u - (__popc(lm & z0) & 1u));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double sg = __hiloint2double((int)(((T << (31 - j)) & 0x80000000u) | 0x3ff00000u), 0);
      re[j] = fma(sg, wk[kk].x, re[j]);
      im[j] = fma(sg, wk[kk].y, im[j]);
    }
  }
}

// Expansion: out[b][z] = 2^-n i^{popcount(x_b & z)} sum_k (-1)^{popcount(l_k & z_lo)} W_k[z_hi].
// Every warp produces 256 consecutive outputs of one block, 8 per lane (z = base + lane + 32 j),
// so each store instruction writes 512 B.  Warps walk the output in address order (group g =
// 256 consecutive outputs of block g >> (n-8)), like the tridiagonal expansion: the chip's
// write front stays within a few tens of MiB, which keeps HBM row-buffer locality (a grid with
// one CTA row per block spreads the front over all blocks and ran 2.5x slower).  The kernel is
// issue-bound rather than load-bound (a version without any W loads wrote at 6.4 TB/s, and an
// L2 prefetch of the next group's W ranges changed nothing), so the per-output work is
// integer-light: shift-specialised loads, table-driven signs, and an i^p phase applied with
// sign-bit arithmetic on the scale.
__global__ void __launch_bounds__(256, 2) band_expand_kernel(const BandBlockDev* blocks, const BandSegRef* refs,
                                                             const double2* segs, int nblocks, int n,
                                                             double scale, double2* out) {
  const u64 N = 1ull << n;
  const unsigned lane = threadIdx.x & 31;
  const int gshift = n - 8;  // groups per block = 2^(n-8); z < 2^28 fits 32 bits
  const u64 groups = (u64)nblocks << gshift;
  const int scale_hi = __double2hiint(scale), scale_lo = __double2loint(scale);
  for (u64 gi = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gi < groups;
       gi += ((u64)gridDim.x * blockDim.x) >> 5) {
    const int b = (int)(gi >> gshift);
    const unsigned xb = (unsigned)__ldg(&blocks[b].x);
    const int bt = __ldg(&blocks[b].t), nL = __ldg(&blocks[b].nL), first = __ldg(&blocks[b].first);
    const int sh = bt + 1;
    const unsigned lomask = (1u << sh) - 1u;
    const unsigned z0 = ((unsigned)(gi & ((1ull << gshift) - 1ull)) << 8) + lane;
    {
      // L1 prefetch of the W samples of a later group of this warp: its loads then hit L1 instead
      // of waiting an L2 / DRAM round trip (lane kk: segment kk's sample, or lines of it)
      const u64 gn = gi + kBandPrefetchDist * (((u64)gridDim.x * blockDim.x) >> 5);
      if (gn < groups) {
        const int bn = (int)(gn >> gshift);
        const int shn = __ldg(&blocks[bn].t) + 1, nLn = __ldg(&blocks[bn].nL), fn = __ldg(&blocks[bn].first);
        const unsigned zb = (unsigned)(gn & ((1ull << gshift) - 1ull)) << 8;
        if (shn >= 8) {
          if ((int)lane < nLn) prefetch_l1(segs + __ldg(&refs[fn + (int)lane].off) + (zb >> shn));
        } else {
          const unsigned cnt = 256u >> shn;  // samples per segment, 8 per 128 B line
          for (int kk = 0; kk < nLn; ++kk)
            if (lane * 8u < cnt) prefetch_l1(segs + __ldg(&refs[fn + kk].off) + (zb >> shn) + lane * 8u);
        }
      }
    }
    double re[8], im[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { re[j] = 0.0; im[j] = 0.0; }
    int k = 0;
    if (sh >= 8) {
      // one sample per segment: issue all of them (up to 8) before using any, so a group
      // waits one memory latency instead of one per segment (exact counts: no predicated-off
      // work for the common 2-4 segments)
      const double2* Wb = segs + ((z0 - lane) >> sh);
      switch (nL < 8 ? nL : 8) {
        case 0: break;
        case 1: band_accum_single<1>(refs + first, Wb, lomask, z0, re, im); break;
        case 2: band_accum_single<2>(refs + first, Wb, lomask, z0, re, im); break;
        case 3: band_accum_single<3>(refs + first, Wb, lomask, z0, re, im); break;
        case 4: band_accum_single<4>(refs + first, Wb, lomask, z0, re, im); break;
        case 5: band_accum_single<5>(refs + first, Wb, lomask, z0, re, im); break;
        case 6: band_accum_single<6>(refs + first, Wb, lomask, z0, re, im); break;
        case 7: band_accum_single<7>(refs + first, Wb, lomask, z0, re, im); break;
        default: band_accum_single<8>(refs + first, Wb, lomask, z0, re, im); break;
      }
      k = 8;
    }
    for (; k < nL; ++k) {
      const unsigned long long rl = __ldg(&refs[first + k].l), roff = __ldg(&refs[first + k].off);
      const double2* Wg = segs + roff + ((z0 - lane) >> sh);
      const unsigned lm = (unsigned)rl & lomask;
      switch (sh < 8 ? sh : 8) {
        case 0: band_accum<0>(Wg, z0, lane, lm, re, im); break;
        case 1: band_accum<1>(Wg, z0, lane, lm, re, im); break;
        case 2: band_accum<2>(Wg, z0, lane, lm, re, im); break;
        case 3: band_accum<3>(Wg, z0, lane, lm, re, im); break;
        case 4: band_accum<4>(Wg, z0, lane, lm, re, im); break;
        case 5: band_accum<5>(Wg, z0, lane, lm, re, im); break;
        case 6: band_accum<6>(Wg, z0, lane, lm, re, im); break;
        case 7: band_accum<7>(Wg, z0, lane, lm, re, im); break;
        default: band_accum<8>(Wg, z0, lane, lm, re, im); break;
      }
    }
    double2* ob = out + (u64)b * N;
    const unsigned p0 = (unsigned)__popc(xb & z0), mx = (xb >> 5) & 7u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      // i^p (re + i im): p odd swaps the parts; Re is negated for p in {1, 2}, Im for p in {2, 3}
      const unsigned p = (p0 + (unsigned)__popc(mx & (unsigned)j)) & 3u;
      const bool odd = (p & 1u) != 0;
      const double a = odd ? im[j] : re[j], c = odd ? re[j] : im[j];
      const double sa = __hiloint2double(scale_hi ^ (int)(((p ^ (p >> 1)) & 1u) << 31), scale_lo);
      const double sc = __hiloint2double(scale_hi ^ (int)((p & 2u) << 30), scale_lo);
      st_stream(ob + z0 + 32u * j, make_double2(a * sa, c * sc));
    }
  }
}

// n < 8 (fewer than 256 outputs per block): one output per thread.
__global__ void band_expand_small_kernel(const BandBlockDev* blocks, const BandSegRef* refs, const double2* segs,
                                         int nblocks, int n, double scale, double2* out) {
  const u64 N = 1ull << n;
  for (u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x; id < (u64)nblocks * N;
       id += (u64)gridDim.x * blockDim.x) {
    const BandBlockDev B = blocks[id >> n];
    const u64 z = id & (N - 1);
    const int sh = B.t + 1;
    const u64 zlo = z & ((1ull << sh) - 1ull), zhi = z >> sh;
    double re = 0.0, im = 0.0;
    for (int k = 0; k < B.nL; ++k) {
      const BandSegRef r = refs[B.first + k];
      const double2 w = segs[r.off + zhi];
      if (__popcll(r.l & zlo) & 1) { re -= w.x; im -= w.y; }
      else { re += w.x; im += w.y; }
    }
    const double2 c = rot_ipow(make_double2(re, im), __popcll(B.x & z));
    out[id] = make_double2(c.x * scale, c.y * scale);
  }
}

static bool band_args_ok(int n, int s) { return n >= 1 && n <= 28 && s >= 0 && s <= 64 && (1ll << n) > s; }

size_t band_s_xmask_count(int n, int s) {
  if (!band_args_ok(n, s)) return 0;
  return make_band_plan(n, s).blocks.size();
}
int band_s_xmasks(int n, int s, unsigned long long* xs, size_t cap) {
  if (!band_args_ok(n, s)) return -1;
  BandPlan p = make_band_plan(n, s);
  if (cap < p.blocks.size()) return -2;
  for (size_t i = 0; i < p.blocks.size(); ++i) xs[i] = p.blocks[i].x;
  return (int)p.blocks.size();
}
size_t band_s_workspace_bytes(int n, int s) {
  if (!band_args_ok(n, s)) return (size_t)-1;
  return make_band_plan(n, s).ws_bytes;
}

// Device tables of a (n, s) plan, staged once per process in pinned host memory: the
// per-call upload is then a truly asynchronous copy from a buffer that outlives every
// launch (graph-capturable), instead of a pageable copy that synchronises the stream
// (ADVICE r01).  Entries are immutable once built; the cache holds one table per (n, s).
struct BandTables {
  BandPlan plan;
  void* pinned = nullptr;
  size_t xb_off = 0;
};
static const BandTables* band_tables(int n, int s, cudaError_t* err) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, BandTables*> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find({n, s});
  if (it != cache.end()) return it->second;
  BandTables* T = new BandTables();
  T->plan = make_band_plan(n, s);
  const BandPlan& p = T->plan;
  const int nseg = (int)p.refs.size(), nb = (int)p.blocks.size();
  if ((*err = cudaHostAlloc(&T->pinned, p.table_bytes, cudaHostAllocPortable)) != cudaSuccess) {
    delete T;
    return nullptr;
  }
  char* host = reinterpret_cast<char*>(T->pinned);
  memset(host, 0, p.table_bytes);
  memcpy(host, p.blocks.data(), nb * sizeof(BandBlockDev));
  memcpy(host + nb * sizeof(BandBlockDev), p.refs.data(), nseg * sizeof(BandSegRef));
  std::vector<int4> gat(nseg);
  for (int k = 0; k < nseg; ++k) gat[k] = make_int4(p.seg_t[k], p.seg_d[k], p.seg_lam[k], 0);
  memcpy(host + nb * sizeof(BandBlockDev) + nseg * sizeof(BandSegRef), gat.data(), nseg * sizeof(int4));
  // x -> block table for the diagonal-order gather
  const int sw = s > 0 ? s : 1;
  std::vector<int> xb((size_t)n * sw, -1);
  for (int bi = 0; bi < nb; ++bi) {
    const BandBlockDev& B = p.blocks[bi];
    if (B.t < 0) continue;
    const unsigned long long e = ((2ull << B.t) - 1ull) - B.x;
    if (e < (unsigned long long)sw) xb[(size_t)B.t * sw + e] = bi;
  }
  T->xb_off = nb * sizeof(BandBlockDev) + nseg * sizeof(BandSegRef) + nseg * sizeof(int4);
  memcpy(host + T->xb_off, xb.data(), xb.size() * sizeof(int));
  cache[{n, s}] = T;
  return T;
}

cudaError_t launch_band_s(const double2* diags, int n, int s, double2* out, void* ws, cudaStream_t st,
                          int* nl) {
  cudaError_t e = cudaSuccess;
  const BandTables* T = band_tables(n, s, &e);
  if (!T) return e;
  const BandPlan& p = T->plan;
  const int nseg = (int)p.refs.size(), nb = (int)p.blocks.size();
  char* base = reinterpret_cast<char*>(ws);
  BandBlockDev* dblocks = reinterpret_cast<BandBlockDev*>(base);
  BandSegRef* drefs = reinterpret_cast<BandSegRef*>(base + nb * sizeof(BandBlockDev));
  int4* dgat = reinterpret_cast<int4*>(base + nb * sizeof(BandBlockDev) + nseg * sizeof(BandSegRef));
  double2* segs = reinterpret_cast<double2*>(base + p.table_bytes);
  const int* dxb = reinterpret_cast<const int*>(base + T->xb_off);
  e = cudaMemcpyAsync(base, T->pinned, p.table_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  const int sms = device_sm_count();
  const bool top3 = s >= 1 && n - 1 >= kTopMin;
  if (top3) {
    const u64 total = ((u64)(2 * s) << (n - 3)) + (1ull << (n - 4));
    u64 g = (total + 255) / 256;
    if (g > (u64)sms * 16) g = (u64)sms * 16;
    band_gather_top3_kernel<<<(unsigned)g, 256, 0, st>>>(diags, n, s, dblocks, drefs, dxb, segs);
    *nl += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  } else if (s >= 1) {
    const u64 total = (u64)(2 * s + 1) << n;
    u64 g = (total + 255) / 256;
    if (g > (u64)sms * 16) g = (u64)sms * 16;
    band_gather_diag_kernel<<<(unsigned)g, 256, 0, st>>>(diags, n, s, dblocks, drefs, dxb, segs);
    *nl += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  } else {
    dim3 grid((unsigned)(sms * 4 > 1 ? sms * 4 : 1), (unsigned)(nseg < 65535 ? nseg : 65535));
    band_gather_kernel<<<grid, 256, 0, st>>>(diags, n, s, drefs, dgat, nseg, segs);
    *nl += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // WHT of every segment, in place (one family per length)
  std::vector<WhtFamily> fam;
  for (size_t f = 0; f < p.fam_lam.size(); ++f) {
    // long segments after the top-levels gather: 8 branches of 2^(lam-3) each (x = 0, the only
    // segment of 2^n elements: 16 branches of 2^(n-4))
    const int tb = !(top3 && p.fam_lam[f] >= kTopMin) ? 0 : p.fam_lam[f] == n ? 4 : 3;
    fam.push_back(WhtFamily{segs + p.fam_off[f], segs + p.fam_off[f], p.fam_lam[f] - tb,
                            (u64)p.fam_count[f] << tb, 1.0});
  }
  for (size_t f0 = 0; f0 < fam.size(); f0 += kMaxSeg) {
    const int cnt = (int)(fam.size() - f0 < (size_t)kMaxSeg ? fam.size() - f0 : kMaxSeg);
    if ((e = run_families(fam.data() + f0, cnt, st, nl)) != cudaSuccess) return e;
  }
  {
    const u64 N = 1ull << n;
    if (n >= 8) {
      u64 g = (((u64)nb << (n - 8)) + 7) / 8;
      if (g > (u64)sms * 16) g = (u64)sms * 16;
      band_expand_kernel<<<(unsigned)g, 256, 0, st>>>(dblocks, drefs, segs, nb, n, ldexp(1.0, -n), out);
    } else {
      u64 g = ((u64)nb * N + 255) / 256;
      if (g > (u64)sms * 16) g = (u64)sms * 16;
      band_expand_small_kernel<<<(unsigned)g, 256, 0, st>>>(dblocks, drefs, segs, nb, n, ldexp(1.0, -n), out);
    }
    *nl += 1;
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace ptdr
