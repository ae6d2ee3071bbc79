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
#include "engine.cuh"
#include "internal.h"

namespace ptdr {

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

template <int K>
struct FlatSt {
  double2* out;
  u64 rbase;
  int b0;
  double scale;
  int zshift;
  u64 zrank;
  __device__ __forceinline__ void operator()(int f, int j, double2 v) const {
    const u64 rho = rbase + (u64)f;
    const u64 e = ((rho >> b0) << (b0 + K)) | ((u64)j << b0) | (rho & ((1ull << b0) - 1ull));
    if (in_slice(e, zshift, zrank)) st_l2(out + (e - (zrank << zshift)), make_double2(v.x * scale, v.y * scale));
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
                                             double scale, int zshift, u64 zrank) {
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
      const double2 w = S[contig_slot(f, jl + 16 * kk)];
      const u64 e = base + (u64)(f * 256 + jl + 16 * kk);
      if (in_slice(e, zshift, zrank)) st_l2(out + (e - (zrank << zshift)), make_double2(w.x * scale, w.y * scale));
    }
  }
}

// ---- tridiagonal split: (S_t, U_t) -> (S_t + U_t, S_t - U_t) compacted per t --------
// One thread per super-diagonal index i (coalesced reads of sup[i] and sub[i+1]): i has t
// trailing ones, b_h = i with h = i >> (t+1), S_t[h] = sup[i], U_t[h] = sub[i+1].
__global__ void tridiag_split_kernel(const double2* band, double2* PM, int n) {
  const u64 N = 1ull << n;
  const double2* sub = band;
  const double2* sup = band + 2 * N;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < N - 1;
       i += (u64)gridDim.x * blockDim.x) {
    const int t = __ffsll((long long)~i) - 1;  // trailing ones of i (i < N-1 so t <= n-1)
    const int lam = n - t - 1;
    const u64 seg = N - (N >> t);
    const u64 h = i >> (t + 1);
    const double2 s = ld_stream(sup + i);
    const double2 u = ld_stream(sub + i + 1);
    PM[2 * seg + h] = cadd(s, u);
    PM[2 * seg + (1ull << lam) + h] = csub(s, u);
  }
}

// ---- tridiagonal expansion into blocks 1..n (write-bound) ------------------------------
// Each thread writes 8 outputs of one block at z = base + lane + 32 k (512 B per warp store);
// the P/M values (reused 2^(t+1) times) come through the read-only cache.
// z-sharded (world > 1): only z in [zrank 2^zshift, (zrank+1) 2^zshift) of each block, stored
// block-major with 2^zshift outputs per block (block 0 is written by the WHT passes).
__global__ void __launch_bounds__(256) tridiag_expand_kernel(const double2* PM, double2* out, int n,
                                                             double scale, int zshift, u64 zrank) {
  const u64 N = 1ull << n;
  const u64 NL = 1ull << zshift;              // outputs per block on this rank
  const u64 z0 = zrank << zshift;
  const u64 groups = ((u64)n * NL) >> 8;      // 256 outputs per warp-group of 8 stores
  const int lane = threadIdx.x & 31;
  for (u64 gidx = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gidx < groups;
       gidx += ((u64)gridDim.x * blockDim.x) >> 5) {
    const u64 id0 = gidx << 8;
    const int t = (int)(id0 >> zshift);
    const int lam = n - t - 1;
    const u64 seg = N - (N >> t);
    const double2* Pt = PM + 2 * seg;
    const double2* Mt = Pt + (1ull << lam);
    double2 w[8];
    int ph[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const u64 z = z0 + (id0 & (NL - 1)) + (u64)lane + 32ull * k;
      const u64 zl = z & ((2ull << t) - 1ull);
      const u64 zh = z >> (t + 1);
      const int s1 = __popcll(z & ((1ull << t) - 1ull)) & 1;
      const int s2 = (int)((z >> t) & 1ull);
      w[k] = __ldg(((s1 == s2) ? Pt : Mt) + zh);
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
__global__ void tridiag_expand_small_kernel(const double2* PM, double2* out, int n, double scale,
                                            int zshift, u64 zrank) {
  const u64 N = 1ull << n;
  const u64 NL = 1ull << zshift;
  const u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (u64)n * NL) return;
  const int t = (int)(id >> zshift);
  const u64 z = (zrank << zshift) + (id & (NL - 1));
  const int lam = n - t - 1;
  const u64 seg = N - (N >> t);
  const u64 zl = z & ((2ull << t) - 1ull);
  const int s1 = __popcll(z & ((1ull << t) - 1ull)) & 1;
  const int s2 = (int)((z >> t) & 1ull);
  const double2 w = PM[2 * seg + (s1 == s2 ? 0ull : (1ull << lam)) + (z >> (t + 1))];
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
};
constexpr int kMaxSeg = 40;
struct SegPassTable {
  int count;
  unsigned long long total_tiles;
  SegPass s[kMaxSeg];
};

__device__ __forceinline__ void small_wht_tile(double2* S, const double2* in, double2* out, int lam,
                                               double scale, u64 e0, int zshift, u64 zrank) {
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
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const double2 v = S[i];
    const u64 e = e0 + (u64)i;
    if (in_slice(e, zshift, zrank)) st_l2(out + (e - (zrank << zshift)), make_double2(v.x * scale, v.y * scale));
  }
}

template <int K>
__device__ __forceinline__ void flat_tile(double2* S, const SegPass& sp, u64 local) {
  constexpr int F = kTileElems >> K;
  FlatLd<K> ld{sp.in, local * F, sp.b0};
  FlatSt<K> st{sp.out, local * F, sp.b0, sp.scale, sp.zshift, sp.zrank};
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
    if (sp.small) {
      const u64 off = local << sp.small_lam;
      small_wht_tile(S, sp.in + off, sp.out, sp.small_lam, sp.scale, off, sp.zshift, sp.zrank);
    } else if (sp.b0 == 0 && sp.K == 8) {
      contig8_tile(S, sp.in, sp.out, local * (u64)kTileElems, sp.scale, sp.zshift, sp.zrank);
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

// A vector family for the pass planner: `count` contiguous vectors of 2^lam elements.
struct WhtFamily {
  const double2* in;  // input of pass 0
  double2* out;       // output of every pass but the last (later passes in place)
  int lam;
  u64 count;
  double scale;       // applied on the last pass
  double2* final_out = nullptr;  // output of the last pass (nullptr: `out`, in place)
  int zshift = 63;               // slice filter of the last pass (single-vector families)
  u64 zrank = 0;
};

// Runs all passes for all families (at most 3 launches for lam <= 24).
static cudaError_t run_families(const WhtFamily* fam, int nfam, cudaStream_t st, int* nl) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(seg_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kBandSmem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  int maxlam = 0;
  for (int f = 0; f < nfam; ++f) maxlam = fam[f].lam > maxlam ? fam[f].lam : maxlam;
  const int npass = maxlam <= 12 ? 1 : (maxlam + 7) / 8;
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
      if (w.lam <= 12) {
        if (p != 0) continue;
        sp.small = 1;
        sp.in = w.in;
        sp.out = fin;
        sp.small_lam = w.lam;
        sp.scale = w.scale;
        sp.zshift = w.zshift;
        sp.zrank = w.zrank;
        sp.first_tile = tiles;
        tiles += w.count;
      } else {
        const int b0 = 8 * p;
        if (b0 >= w.lam) continue;
        const int K = (w.lam - b0) < 8 ? (w.lam - b0) : 8;
        const bool last = b0 + K >= w.lam;
        sp.in = p == 0 ? w.in : w.out;
        sp.out = last ? fin : w.out;
        sp.b0 = b0;
        sp.K = K;
        sp.scale = last ? w.scale : 1.0;
        if (last) {
          sp.zshift = w.zshift;
          sp.zrank = w.zrank;
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

// Workspace: [P/M segments: 2 * 2^n] (TRIDIAGONAL) + [x = 0 vector: 2^n] (world > 1: the
// passes before the last run on a full-length copy; only the last one writes the slice).
size_t band_workspace_bytes(int n, int structure, int world) {
  const size_t N = (size_t)1 << n;
  size_t b = structure == 4 ? 2 * N * 16 : 0;
  if (world > 1 && n > 12) b += N * 16;
  return b;
}

cudaError_t launch_band(const double2* A, double2* out, int n, int structure, void* ws, int rank,
                        int world, cudaStream_t st, int* nl) {
  const u64 N = 1ull << n;
  const double scale = ldexp(1.0, -n);
  const int g = __builtin_ctz((unsigned)world);
  const int zshift = world > 1 ? n - g : 63;
  const u64 zrank = world > 1 ? (u64)rank : 0ull;
  double2* PM = reinterpret_cast<double2*>(ws);
  double2* X0 = world > 1 ? PM + (structure == 4 ? 2 * N : 0) : nullptr;  // full-length x=0 scratch
  // the x = 0 family (main diagonal): in place on `out` on one GPU; on a full-length
  // workspace copy with a slice-writing last pass when z-sharded
  auto x0_family = [&](const double2* src) {
    WhtFamily f{src, world > 1 && n > 12 ? X0 : out, n, 1, scale};
    f.final_out = out;
    f.zshift = zshift;
    f.zrank = zrank;
    return f;
  };
  if (structure == 3) {
    WhtFamily f = x0_family(A);
    return run_families(&f, 1, st, nl);
  }
  // TRIDIAGONAL: A = [sub | main | sup]
  const int sms = device_sm_count();
  cudaError_t e;
  {
    u64 blocks = (N + 255) / 256;
    if (blocks > (u64)sms * 32) blocks = (u64)sms * 32;
    tridiag_split_kernel<<<(unsigned)blocks, 256, 0, st>>>(A, PM, n);
    *nl += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // block 0 (x = 0): WHT(main) scaled; blocks t+1: P_t / M_t (two vectors of 2^(n-t-1))
  WhtFamily fam[kMaxSeg];
  int nf = 0;
  fam[nf++] = x0_family(A + N);
  for (int t = 0; t < n; ++t) {
    const int lam = n - t - 1;
    const u64 seg = N - (N >> t);
    fam[nf++] = WhtFamily{PM + 2 * seg, PM + 2 * seg, lam, 2, 1.0};
  }
  if ((e = run_families(fam, nf, st, nl)) != cudaSuccess) return e;
  {
    const int zs = world > 1 ? zshift : n;
    const u64 NL = 1ull << zs;
    const u64 total = (u64)n * NL;
    if (NL >= 256) {
      u64 blocks = (total / 8 + 255) / 256;
      if (blocks > (u64)sms * 16) blocks = (u64)sms * 16;
      tridiag_expand_kernel<<<(unsigned)blocks, 256, 0, st>>>(PM, out, n, scale, zs, zrank);
    } else {
      tridiag_expand_small_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(PM, out, n, scale, zs,
                                                                                 zrank);
    }
    *nl += 1;
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace ptdr
