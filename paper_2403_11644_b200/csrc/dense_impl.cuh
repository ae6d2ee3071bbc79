// dense_impl.cuh -- kernels of the dense path (GENERAL / HERMITIAN / REAL_SYMMETRIC).
//
// Two-phase fused persistent kernel:
//   phase A tile  = XOR-transpose gather of v_x[i] = A[i][i ^ x] for 16 X-masks
//                   (x0..x0+15) x 2^R consecutive i (16-row x 16-column aligned
//                   blocks, 256 B coalesced row segments), then the WHT over the
//                   low R bits of i  ->  scratch Y[ih][zl][u]   (L2-resident ring)
//   phase B tile  = WHT over the high M bits of i for 4096/2^M (u, zl) fibers,
//                   then the epilogue alpha = 2^-n i^{popcount(x&z)} W stored in
//                   q order as 512 B contiguous runs.
// Tiles are handed out by an in-order ticket counter; a phase-B tile of chunk c
// waits for the NA phase-A tiles of chunk c, a phase-A tile of chunk c waits for
// the phase-B tiles of chunk c - nslot (ring reuse).  Phase A of chunk c+L is
// ticketed before phase B of chunk c so that waits are rare.
#pragma once
#include "engine.cuh"

namespace ptdr {

// MODE: 0 GENERAL, 1 HERMITIAN mirrored (full-length vectors built from the upper
// triangle), 2 REAL_SYMMETRIC mirrored, 3 HERMITIAN half-length, 4 REAL_SYMMETRIC
// half-length.  See DESIGN.md "Hermitian / real-symmetric path".
enum { MODE_GENERAL = 0, MODE_HERM_MIRROR = 1, MODE_SYM_MIRROR = 2, MODE_HERM_HALF = 3, MODE_SYM_HALF = 4,
       MODE_GEN = 8 /* matrix-free GENERAL (pipeline only): entries generated in phase A */,
       MODE_INV = 9 /* inverse transform from the matrix layout (pipeline only, see dense_pipe.cuh) */,
       MODE_INVQ = 10 /* inverse transform from q order (pipeline only) */ };

struct DenseArgs {
  const double2* A;
  double2* out;
  double2* scratch;
  unsigned* ctr;       // [0] ticket, [1 .. C] phase-A done, [C+1 .. 2C] phase-B done
  u64 ld;              // row pitch of A (elements)
  u64 colmask;         // column index mask (2^n - 1, or R - 1 for an X-mask shard)
  u64 x_base;          // X-mask of chunk 0 of this launch
  u64 nchunks;
  u64 slot_elems;
  int n;               // qubits (scale 2^-n)
  int nv;              // bits of the transformed vectors
  int gshift;          // n - log2(world)
  int L;
  int nslot;
  int discard;         // pipeline: discard consumed scratch lines from L2 (no write-back)
  int pol_a, pol_s, pol_b;  // pipeline L2 policies (policy_of codes): A loads, scratch stores,
                            //   scratch loads
  int peer_shift;      // peer-pull mode (> 0): row i lives in shard i >> peer_shift
  u64 peer_rowmask;    //   at local row i & peer_rowmask
  int npeers;          //   shards (host side: tensor maps are built from peer_ptrs)
  const double2* peer_ptrs[8];
  u64 gen_seed;        // MODE_GEN: seed of the counter-based generator
  u64 batch;           // batched small-n launches (direct / whole-vector kernels): matrices,
  u64 bstride_in;      //   element stride between consecutive inputs
  u64 bstride_out;     //   and between consecutive outputs (0 batch = 1)
  u64 rows_valid;      // zero padding: rows / columns of A actually stored;
  u64 cols_valid;      // 0 = all (the TMA tensor map fills the rest with zeros)
  unsigned long long* trace;  // pipeline debug timeline (nullptr unless PTDR_TRACE=1)
  double scale;        // 2^-n
  int layout_mat;      // output layout: 0 = q order at q_offset(x, z, gshift); 1 = matrix
                       //   layout out[z 2^n + (z ^ x)] (the in-place decomposition)
  int max_ctas;        // pipeline grid cap (0: one CTA per SM)
  int acq_fence;       // pipeline dependency waits: 2 ld.acquire.gpu (default); developer
                       //   variants 0 relaxed read, 1 relaxed + fence.acq_rel.gpu
};

// Output index of coefficient (x, z).  The matrix layout puts alpha(x, z) where A[z][z ^ x]
// was: the X-masks of a chunk occupy exactly the elements the chunk reads, so the pipeline
// can overwrite A in place (ptdr_decompose_inplace_async, R12).
__device__ __forceinline__ u64 out_index(const DenseArgs& a, u64 x, u64 z) {
  return a.layout_mat ? ((z << a.n) | (z ^ x)) : q_offset(x, z, a.gshift);
}

// ---- loads: v_x[i] for the MODE -------------------------------------------------
template <int MODE>
__device__ __forceinline__ double2 load_v(const DenseArgs& a, u64 row, u64 x) {
  const u64 col = (row ^ x) & a.colmask;
  if constexpr (MODE == MODE_GENERAL || MODE == MODE_HERM_HALF) {
    return ld_stream(a.A + row * a.ld + col);
  } else if constexpr (MODE == MODE_SYM_HALF) {
    return make_double2(ld_stream_re(a.A + row * a.ld + col), 0.0);
  } else {
    // mirrored: read only the upper triangle (row <= col) and the diagonal's real part
    if (row < col) {
      double2 e = ld_stream(a.A + row * a.ld + col);
      if (MODE == MODE_SYM_MIRROR) e.y = 0.0;
      return e;
    } else if (row > col) {
      double2 e = ld_stream(a.A + col * a.ld + row);
      e.y = (MODE == MODE_SYM_MIRROR) ? 0.0 : -e.y;
      return e;
    } else {
      return make_double2(ld_stream_re(a.A + row * a.ld + row), 0.0);
    }
  }
}

// ---- epilogue: alpha(x, z) = 2^-n i^{popcount(x&z)} W, stored at q(x, z) ------------
// For the half-length modes W' is the WHT of the half vector (index bit t removed):
// W(z) = 2 Re W'(z') if popcount(x&z) even, 2i Im W'(z') if odd, so
// alpha = 2^{1-n} * {Re, -Im, -Re, Im}[popcount(x&z) mod 4] (real).  DESIGN.md.
template <int MODE>
__device__ __forceinline__ void emit(const DenseArgs& a, u64 x, u64 zv, double2 w, int t) {
  if constexpr (MODE == MODE_GENERAL) {
    double2 c = rot_ipow(w, __popcll(x & zv));
    c.x *= a.scale;
    c.y *= a.scale;
    st_stream(a.out + out_index(a, x, zv), c);
  } else if constexpr (MODE == MODE_HERM_MIRROR || MODE == MODE_SYM_MIRROR) {
    double2 c = rot_ipow(w, __popcll(x & zv));
    st_stream(a.out + out_index(a, x, zv), make_double2(c.x * a.scale, 0.0));
  } else {
    const u64 z0 = insert0(zv, t);
    const u64 z1 = z0 | (1ull << t);
    const int p0 = __popcll(x & z0) & 3;
    const double s = 2.0 * a.scale;
    const double sel0 = (p0 == 0) ? w.x : (p0 == 1) ? -w.y : (p0 == 2) ? -w.x : w.y;
    const int p1 = (p0 + 1) & 3;
    const double sel1 = (p1 == 0) ? w.x : (p1 == 1) ? -w.y : (p1 == 2) ? -w.x : w.y;
    st_stream(a.out + out_index(a, x, z0), make_double2(sel0 * s, 0.0));
    st_stream(a.out + out_index(a, x, z1), make_double2(sel1 * s, 0.0));
  }
}

template <int MODE>
__device__ __forceinline__ int top_bit_for(u64 x0) {
  if constexpr (MODE == MODE_HERM_HALF || MODE == MODE_SYM_HALF) return 63 - __clzll(x0);
  else return 0;
}

// ---- phase A functors -----------------------------------------------------------
template <int R, int MODE>
struct LoadA {
  const DenseArgs* a;
  u64 x0, ihbase;
  int t;
  __device__ __forceinline__ double2 operator()(int f, int j) const {
    const u64 iv = ((ihbase + (u64)(f >> 4)) << R) | (u64)j;
    u64 row = iv;
    if constexpr (MODE == MODE_HERM_HALF || MODE == MODE_SYM_HALF) row = insert0(iv, t);
    return load_v<MODE>(*a, row, x0 + (u64)(f & 15));
  }
};

template <int R>
struct StoreScratch {
  double2* Y;
  u64 ihbase;
  __device__ __forceinline__ void operator()(int f, int j, double2 v) const {
    const u64 ih = ihbase + (u64)(f >> 4);
    st_l2(Y + ((((ih << R) | (u64)j) << 4) | (u64)(f & 15)), v);
  }
};

// ---- phase B functors: fiber phi -> (u, zl); bits [0,1]=u0,u1 [2,3]=zl0,zl1
//      [4,5]=u2,u3 [6..]=zl2.. so that 16 consecutive fibers form a 4x4 (x,z) square,
//      i.e. 16 consecutive q (256 B) ------------------------------------------------
__device__ __forceinline__ int phi_u(u64 phi) { return (int)((phi & 3) | (((phi >> 4) & 3) << 2)); }
__device__ __forceinline__ u64 phi_zl(u64 phi) { return ((phi >> 2) & 3) | ((phi >> 6) << 2); }

template <int R>
struct LoadB {
  const double2* Y;
  u64 phibase;
  __device__ __forceinline__ double2 operator()(int f, int j) const {
    const u64 phi = phibase + (u64)f;
    return ld_l2(Y + (((((u64)j << R) | phi_zl(phi)) << 4) | (u64)phi_u(phi)));
  }
};

template <int R, int MODE>
struct StoreB {
  const DenseArgs* a;
  u64 x0, phibase;
  int t;
  __device__ __forceinline__ void operator()(int f, int j, double2 v) const {
    const u64 phi = phibase + (u64)f;
    emit<MODE>(*a, x0 + (u64)phi_u(phi), ((u64)j << R) | phi_zl(phi), v, t);
  }
};

// ---- single-phase functors (nv in {6,7}: one tile holds whole vectors) ---------------
template <int MODE>
struct LoadS {
  const DenseArgs* a;
  u64 xfirst;
  int t;  // half-length modes: index bit removed (top bit of the tile's X-masks)
  __device__ __forceinline__ double2 operator()(int f, int j) const {
    u64 row = (u64)j;
    if constexpr (MODE == MODE_HERM_HALF || MODE == MODE_SYM_HALF) row = insert0(row, t);
    return load_v<MODE>(*a, row, xfirst + (u64)f);
  }
};
template <int MODE>
struct StoreS {
  const DenseArgs* a;
  u64 xfirst;
  int t;
  __device__ __forceinline__ void operator()(int f, int j, double2 v) const {
    emit<MODE>(*a, xfirst + (u64)f, (u64)j, v, t);
  }
};

// ---- ticket decode ----------------------------------------------------------------
// Order: A(0..L), then for c = 0..: B(c), A(c+L+1), ..., then the remaining B's.
__device__ __forceinline__ void decode_ticket(u64 t, int NA, int NB, u64 C, int L, int& phase,
                                              u64& chunk, int& tile) {
  const u64 lp1 = (u64)L + 1 < C ? (u64)L + 1 : C;
  const u64 pro = lp1 * (u64)NA;
  if (t < pro) { phase = 0; chunk = t / NA; tile = (int)(t % NA); return; }
  t -= pro;
  const u64 P = (u64)NA + (u64)NB;
  const u64 steady = C > (u64)L + 1 ? C - (u64)L - 1 : 0;
  if (t < steady * P) {
    const u64 c = t / P, o = t % P;
    if (o < (u64)NB) { phase = 1; chunk = c; tile = (int)o; }
    else { phase = 0; chunk = c + L + 1; tile = (int)(o - NB); }
    return;
  }
  t -= steady * P;
  phase = 1;
  chunk = steady + t / NB;
  tile = (int)(t % NB);
}

template <int R, int M, int MODE>
__global__ void __launch_bounds__(kThreads, 2) dense_fused_kernel(DenseArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  __shared__ unsigned long long s_ticket;
  constexpr int FA = kTileElems >> R;   // phase-A fibers per tile (16 u x FA/16 ih)
  constexpr int FB = kTileElems >> M;   // phase-B fibers per tile
  const int NA = 1 << (R + M - 8);
  const int NB = NA;
  const u64 C = a.nchunks;
  const u64 total = C * (u64)(NA + NB);
  unsigned* ticket = a.ctr;
  unsigned* doneA = a.ctr + 1;
  unsigned* doneB = a.ctr + 1 + C;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    const u64 tk = s_ticket;
    if (tk >= total) break;
    int phase, tile;
    u64 chunk;
    decode_ticket(tk, NA, NB, C, a.L, phase, chunk, tile);
    const u64 x0 = a.x_base + 16ull * chunk;
    const int t = top_bit_for<MODE>(x0);
    double2* Y = a.scratch + (chunk % (u64)a.nslot) * a.slot_elems;
    if (phase == 0) {
      if (chunk >= (u64)a.nslot) cta_wait_counter(&doneB[chunk - a.nslot], (unsigned)NB);
      const u64 ihbase = (u64)tile * (FA / 16);
      LoadA<R, MODE> ld{&a, x0, ihbase, t};
      StoreScratch<R> st{Y, ihbase};
      fiber_tile<R>(S, ld, st);
      cta_signal_counter(&doneA[chunk]);
    } else {
      cta_wait_counter(&doneA[chunk], (unsigned)NA);
      const u64 phibase = (u64)tile * FB;
      LoadB<R> ld{Y, phibase};
      StoreB<R, MODE> st{&a, x0, phibase, t};
      fiber_tile<M>(S, ld, st);
      cta_signal_counter(&doneB[chunk]);
    }
  }
}

template <int R, int MODE>
__global__ void __launch_bounds__(kThreads, 2) dense_single_kernel(DenseArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  constexpr int F = kTileElems >> R;
  const u64 nx = a.nchunks * 16;
  const u64 ntiles = nx / F;
  const u64 nb = a.batch ? a.batch : 1;
  for (u64 tg = blockIdx.x; tg < ntiles * nb; tg += gridDim.x) {
    const u64 b = tg / ntiles, tile = tg - b * ntiles;
    DenseArgs ab = a;  // matrix b of a batch
    ab.A += b * a.bstride_in;
    ab.out += b * a.bstride_out;
    const u64 xfirst = a.x_base + tile * F;
    // the F X-masks of a tile share their top bit (tiles are F-aligned, x_base a power of
    // two >= F in the half-length modes)
    const int t = top_bit_for<MODE>(xfirst);
    LoadS<MODE> ld{&ab, xfirst, t};
    StoreS<MODE> st{&ab, xfirst, t};
    if constexpr (R <= 8) fiber_tile<R>(S, ld, st);
    else fiber_tile3<R>(S, ld, st);
    __syncthreads();
  }
}

// Direct evaluation for nv <= 5 (at most 32 terms per coefficient): thread per (x, z).
template <int MODE>
__global__ void dense_direct_kernel(DenseArgs a0, u64 nx) {
  const u64 N = 1ull << a0.n;
  const u64 gid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 per = nx * N;
  if (gid >= per * (a0.batch ? a0.batch : 1)) return;
  const u64 b = gid / per, id = gid - b * per;
  DenseArgs a = a0;
  a.A += b * a0.bstride_in;
  a.out += b * a0.bstride_out;
  const u64 x = a.x_base + id / N, z = id % N;
  double2 s = make_double2(0.0, 0.0);
  for (u64 i = 0; i < N; ++i) {
    const double2 v = load_v<MODE>(a, i, x);
    if (__popcll(i & z) & 1) s = csub(s, v);
    else s = cadd(s, v);
  }
  emit<MODE>(a, x, z, s, 0);
}

}  // namespace ptdr
