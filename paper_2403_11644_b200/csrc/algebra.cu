// algebra.cu -- decomposition algebra on q-ordered coefficient arrays (Sec. IV-B,
// l.521-627) and the inverse transform A = sum_P alpha_P P (l.116-121).  SURVEY 8(f) f3.
//
// All arrays are device complex128 in q order (include/ptdr.h): the leftmost letter is the
// most significant base-4 digit, so a new leftmost qubit (direct sum, block diagonal,
// Hermitian augmentation) makes the output four blocks of 4^n, one per leading letter.
//
// Inverse transform.  For a string (x, z), P[i][i ^ x] = (-i)^{popcount(x & z)}
// (-1)^{popcount(i & z)} (PauliComposer closed form, l.184-208), so
//   A[i][i ^ x] = sum_z alpha(x, z) P[i][i ^ x] = WHT_n(u_x)[i],
//   u_x[z] = (-i)^{popcount(x & z)} alpha(x, z),
// i.e. the forward path run backwards: q order -> x-major rows with the conjugate phase
// (q2x), a WHT over z per row (wht_passes.h), then the XOR scatter V[x][i] -> A[i][i ^ x].
#include <cstdint>

#include "engine.cuh"
#include "sm100_ptx.cuh"
#include "internal.h"
#include "wht_passes.h"

namespace ptdr {

// bit l of v -> bit l of the result from the even bits of q (compact) -- 64-bit
__device__ __forceinline__ u64 compact_even(u64 q) {
  q &= 0x5555555555555555ull;
  q = (q | (q >> 1)) & 0x3333333333333333ull;
  q = (q | (q >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  q = (q | (q >> 4)) & 0x00FF00FF00FF00FFull;
  q = (q | (q >> 8)) & 0x0000FFFF0000FFFFull;
  q = (q | (q >> 16)) & 0x00000000FFFFFFFFull;
  return q;
}

// ---- q order -> x-major rows U[x][z] = (-i)^{popcount(x & z)} alpha[q(x, z)] ------------
// Tile = 4096 consecutive q = all (x_lo6, z_lo6) for fixed high digits: coalesced 64 KiB
// read into SMEM, then 1 KiB runs along z per row.
__global__ void __launch_bounds__(256) q2x_kernel(const double2* __restrict__ c, double2* __restrict__ U,
                                                  int n) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  const u64 N = 1ull << n;
  const u64 tiles = (N * N) >> 12;
  for (u64 tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const u64 q0 = tile << 12;
#pragma unroll 4
    for (int k = threadIdx.x; k < 4096; k += 256) S[k] = ld_stream(c + q0 + k);
    __syncthreads();
    const u64 zh = compact_even(q0 >> 13), xh = compact_even(q0 >> 12) ^ zh;  // digits >= 6
#pragma unroll 4
    for (int k = threadIdx.x; k < 4096; k += 256) {
      const u64 xl = (u64)(k >> 6), zl = (u64)(k & 63);
      const u64 ql = spread_bits(xl ^ zl) | (spread_bits(zl) << 1);
      const u64 x = (xh << 6) | xl, z = (zh << 6) | zl;
      const double2 v = rot_ipow(S[ql], 4 - (__popcll(x & z) & 3));  // (-i)^p = i^{-p}
      st_l2(U + x * N + z, v);
    }
    __syncthreads();
  }
}

__global__ void q2x_small_kernel(const double2* __restrict__ c, double2* __restrict__ U, int n) {
  const u64 N = 1ull << n;
  for (u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x; id < N * N; id += (u64)gridDim.x * blockDim.x) {
    const u64 x = id >> n, z = id & (N - 1);
    const u64 q = spread_bits(x ^ z) | (spread_bits(z) << 1);
    U[id] = rot_ipow(c[q], 4 - (__popcll(x & z) & 3));
  }
}

// ---- XOR scatter A[i][i ^ x] = V[x][i] --------------------------------------------------
// Aligned 32 x 32 tiles: rows x0.. of V along i (512 B runs) -> rows i0.. of A over the
// aligned column window (i0 ^ x0) + [0, 32) (a lane permutation of a 512 B run).
__global__ void __launch_bounds__(256) xscatter_kernel(const double2* __restrict__ V, double2* __restrict__ A,
                                                       int n) {
  __shared__ double2 T[32 * 33];
  const u64 N = 1ull << n;
  const u64 tpr = N >> 5;  // tiles per row
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (u64 tile = blockIdx.x; tile < tpr * tpr; tile += gridDim.x) {
    const u64 x0 = (tile / tpr) << 5, i0 = (tile % tpr) << 5;
#pragma unroll
    for (int a = w; a < 32; a += 8) T[a * 33 + lane] = ld_stream(V + (x0 + a) * N + i0 + lane);
    __syncthreads();
    const u64 cw = i0 ^ x0;
#pragma unroll
    for (int b = w; b < 32; b += 8) {
      // lane = a: A[i0 + b][cw + (b ^ a)] = V[x0 + a][i0 + b]
      st_stream(A + (i0 + b) * N + cw + (u64)(b ^ lane), T[lane * 33 + b]);
    }
    __syncthreads();
  }
}

__global__ void xscatter_small_kernel(const double2* __restrict__ V, double2* __restrict__ A, int n) {
  const u64 N = 1ull << n;
  for (u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x; id < N * N; id += (u64)gridDim.x * blockDim.x) {
    const u64 x = id >> n, i = id & (N - 1);
    A[i * N + (i ^ x)] = V[id];
  }
}

// ---- two-pass inverse (9 <= n <= 16): 32 B of HBM traffic per coefficient per pass ---------
// Pass 1: a tile = 16 X-masks (x bits 0-3) x 256 Z-masks (z bits 0-7) with the other bits
// fixed; in q order that is 16 runs of 256 consecutive coefficients (one run per value of z
// bits 4-7), read coalesced.  Conjugate phase, WHT over z bits 0-7 per X-mask (the contig8
// register/SMEM scheme), stored as U[x >> 5][z][x & 31] (32 X-masks contiguous, so pass 2
// reads 512 B runs).  Pass 2: fibres = (32 consecutive X-masks) x (Z-masks with equal low 8
// bits), WHT over z bits 8..n-1, then the XOR scatter A[i][i ^ x] with i = z: for one i the
// 32 X-masks hit one aligned 32-column window (512 B per warp store).
__device__ __forceinline__ int inv_slot(int f, int j) { return f * 273 + (j >> 4) * 17 + (j & 15); }
constexpr int kInvSmem = 16 * 273 * 16;

// Tiles stream through a ring of kInvStages SMEM buffers filled by the bulk-copy (TMA) engine:
// a tile's 16 runs are 16 contiguous 4 KiB copies completing on the buffer's mbarrier, issued
// two tiles ahead, so the loads of the next tiles are in flight while the current tile is
// transformed and stored (one CTA per SM).  The first WHT stage reads the raw q-order copy
// (its element for (x bits 0-3 = f, z bits 0-7 = jl + 16 kk) sits at kk * 256 + qlo(f, jl)),
// applies the conjugate phase, and after a barrier writes the padded transpose layout into
// the same buffer.  (Register loads with two CTAs per SM: 8.9 ms at n = 15; 16 B cp.async
// into a double buffer: 12.7 ms.)
constexpr int kInvStages = 3;
constexpr int kInvGroups = 2;  // 256-thread groups per CTA, each transforming its own tiles

__global__ void __launch_bounds__(256 * kInvGroups, 1) inv_pass1_kernel(const double2* __restrict__ c,
                                                                        double2* __restrict__ U, int n) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double2* Tb = reinterpret_cast<double2*>(smem_raw);
  constexpr int TE = kInvSmem / 16;  // elements per buffer (padded layout; the raw copy uses 4096)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + kInvStages * kInvSmem);
  // tag[b] = the tile sequence number last issued into buffer b: the two groups consume a
  // buffer alternately, so a parity wait alone could match the previous occupant's phase
  volatile int* tag = reinterpret_cast<volatile int*>(full + kInvStages);
  const u64 N = 1ull << n;
  const u64 xtiles = N >> 4;
  const u64 tiles = xtiles * (N >> 8);
  const int g = threadIdx.x >> 8, tid = threadIdx.x & 255;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kInvStages; ++b) {
      mbar_init(&full[b], 1);
      tag[b] = -1;
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  // CTA-local tile sequence it = 0, 1, 2, ...: tile blockIdx.x + it * gridDim.x, buffer
  // it % kInvStages, transformed by group it % kInvGroups.  The first warp of the group that
  // finishes tile it refills its buffer with tile it + kInvStages (lane 0 arms the barrier,
  // lanes 0-15 copy the 16 runs).
  auto issue = [&](int it) {
    const u64 t = blockIdx.x + (u64)it * gridDim.x;
    if (t >= tiles) return;
    const int b = it % kInvStages;
    const u64 xt = (t % xtiles) << 4, zt = (t / xtiles) << 8;
    if (tid == 0) {
      fence_proxy_async_smem();  // the buffer was last written by generic stores
      mbar_arrive_expect_tx(&full[b], 4096u * 16u);
      tag[b] = it;
    }
    __syncwarp();
    if (tid < 16) {
      const u64 zr = zt | ((u64)tid << 4);
      bulk_load(Tb + (size_t)b * TE + tid * 256, c + (spread_bits(xt ^ zr) | (spread_bits(zr) << 1)), 4096u, &full[b],
                pol);
    }
  };
  if (threadIdx.x < 32)
    for (int it = 0; it < kInvStages; ++it) issue(it);
  const int bar = 1 + g;
  const int f = tid >> 4, jl = tid & 15;
  const int qlo = (int)(spread_bits((u64)(f ^ jl)) | (spread_bits((u64)jl) << 1));
  for (int it = g;; it += kInvGroups) {
    const u64 tile = blockIdx.x + (u64)it * gridDim.x;
    if (tile >= tiles) break;
    const int b = it % kInvStages;
    while (tag[b] != it) __nanosleep(20);
    mbar_wait(&full[b], (uint32_t)(it / kInvStages) & 1u);
    double2* T = Tb + (size_t)b * TE;
    const u64 xt = (tile % xtiles) << 4, zt = (tile / xtiles) << 8;
    double2 v[16];
    {
      const u64 x = xt | (u64)f;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const u64 z = zt | ((u64)kk << 4) | (u64)jl;
        v[kk] = rot_ipow(T[kk * 256 + qlo], 4 - (__popcll(x & z) & 3));
      }
      wht_regs<4>(v);
      named_bar_sync(bar, 256);  // every raw element is read before the padded layout overwrites it
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) T[inv_slot(f, jl + 16 * kk)] = v[kk];
    }
    named_bar_sync(bar, 256);
    {
      const int kh = tid & 15;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = T[inv_slot(f, j + 16 * kh)];
      wht_regs<4>(v);
#pragma unroll
      for (int j = 0; j < 16; ++j) T[inv_slot(f, j + 16 * kh)] = v[j];
    }
    named_bar_sync(bar, 256);
    {
      const int fo = tid & 15, jg = tid >> 4;
      const u64 xo = xt + (u64)fo;
#pragma unroll 4
      for (int kk = 0; kk < 16; ++kk) {
        const int j = jg + 16 * kk;
        st_stream(U + ((((xo >> 5) << n) + zt + (u64)j) << 5) + (xo & 31ull), T[inv_slot(fo, j)]);
      }
    }
    named_bar_sync(bar, 256);  // buffer b is free: refill it with tile it + kInvStages
    if (tid < 32) issue(it + kInvStages);
  }
}

template <int K>
struct InvLd {
  const double2* U;
  u64 xbase, zbase;
  int n, xw;
  __device__ __forceinline__ double2 operator()(int f, int j) const {
    const u64 x = xbase + (u64)(f % xw), z = zbase + (u64)(f / xw) + ((u64)j << 8);
    return ld_stream(U + ((((x >> 5) << n) + z) << 5) + (x & 31ull));
  }
};
template <int K>
struct InvSt {
  double2* A;
  u64 xbase, zbase;
  int n, xw;
  __device__ __forceinline__ void operator()(int f, int j, double2 v) const {
    const u64 x = xbase + (u64)(f % xw), z = zbase + (u64)(f / xw) + ((u64)j << 8);
    st_stream(A + (z << n) + (z ^ x), v);  // A[i][i ^ x], i = z
  }
};

template <int K>
__global__ void __launch_bounds__(kThreads, 2) inv_pass2_kernel(const double2* __restrict__ U, double2* __restrict__ A,
                                                               int n) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  constexpr int F = kTileElems >> K;
  constexpr int XW = F < 32 ? F : 32;  // X-masks per tile
  constexpr int ZS = F / XW;           // low-z values per tile
  const u64 N = 1ull << n;
  const u64 xtiles = N / XW, ztiles = 256 / ZS;
  for (u64 tile = blockIdx.x; tile < xtiles * ztiles; tile += gridDim.x) {
    const u64 xbase = (tile % xtiles) * XW, zbase = (tile / xtiles) * ZS;
    InvLd<K> ld{U, xbase, zbase, n, XW};
    InvSt<K> st{A, xbase, zbase, n, XW};
    fiber_tile<K>(S, ld, st);
    __syncthreads();
  }
}

template <int K>
static cudaError_t launch_inv_pass2(const double2* U, double2* A, int n, cudaStream_t st) {
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(inv_pass2_kernel<K>), kTileBytes);
    if (e != cudaSuccess) return e;
  }
  u64 tiles = (1ull << (2 * n)) / kTileElems;
  u64 g = (u64)device_sm_count() * 2;
  if (g > tiles) g = tiles;
  inv_pass2_kernel<K><<<(unsigned)g, kThreads, kTileBytes, st>>>(U, A, n);
  return cudaGetLastError();
}

size_t reconstruct_workspace_bytes(int n) { return (size_t)16 << (2 * n); }

cudaError_t launch_reconstruct(const double2* c, int n, double2* A, void* ws, cudaStream_t st, int* nl) {
  const u64 N = 1ull << n;
  double2* U = reinterpret_cast<double2*>(ws);
  const int sms = device_sm_count();
  cudaError_t e;
  if (n >= 9 && n <= 16) {
    constexpr int smem = kInvStages * kInvSmem + 64;
    if ((e = ensure_smem_attr(reinterpret_cast<const void*>(inv_pass1_kernel), smem)) != cudaSuccess) return e;
    u64 g = (N * N) >> 12;
    if (g > (u64)sms) g = (u64)sms;
    inv_pass1_kernel<<<(unsigned)g, 256 * kInvGroups, smem, st>>>(c, U, n);
    *nl += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *nl += 1;
    switch (n - 8) {
      case 1: return launch_inv_pass2<1>(U, A, n, st);
      case 2: return launch_inv_pass2<2>(U, A, n, st);
      case 3: return launch_inv_pass2<3>(U, A, n, st);
      case 4: return launch_inv_pass2<4>(U, A, n, st);
      case 5: return launch_inv_pass2<5>(U, A, n, st);
      case 6: return launch_inv_pass2<6>(U, A, n, st);
      case 7: return launch_inv_pass2<7>(U, A, n, st);
      default: return launch_inv_pass2<8>(U, A, n, st);
    }
  }
  if (n >= 6) {
    if ((e = ensure_smem_attr(reinterpret_cast<const void*>(q2x_kernel), 65536)) != cudaSuccess) return e;
    u64 g = (N * N) >> 12;
    if (g > (u64)sms * 3) g = (u64)sms * 3;
    q2x_kernel<<<(unsigned)g, 256, 65536, st>>>(c, U, n);
  } else {
    q2x_small_kernel<<<(unsigned)((N * N + 255) / 256), 256, 0, st>>>(c, U, n);
  }
  *nl += 1;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  WhtFamily f{U, U, n, N, 1.0};
  if ((e = run_families(&f, 1, st, nl)) != cudaSuccess) return e;
  if (n >= 5) {
    u64 g = (N >> 5) * (N >> 5);
    if (g > (u64)sms * 8) g = (u64)sms * 8;
    xscatter_kernel<<<(unsigned)g, 256, 0, st>>>(U, A, n);
  } else {
    xscatter_small_kernel<<<(unsigned)((N * N + 255) / 256), 256, 0, st>>>(U, A, n);
  }
  *nl += 1;
  return cudaGetLastError();
}

// ---- linear combination (l.570-577): out = mu x + nu y ----------------------------------
__global__ void axpby_kernel(double2* out, double2 mu, const double2* x, double2 nu, const double2* y, u64 count) {
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x) {
    const double2 a = ld_stream(x + i), b = ld_stream(y + i);
    st_stream(out + i, make_double2(mu.x * a.x - mu.y * a.y + nu.x * b.x - nu.y * b.y,
                                    mu.x * a.y + mu.y * a.x + nu.x * b.y + nu.y * b.x));
  }
}

// ---- block diagonal diag(A_0 .. A_{2^k - 1}) (l.524-568; k = 1 is the direct sum) --------
// sum_j |j><j| (x) A_j with |j><j| = 2^-k sum_zt (-1)^{popcount(j & zt)} Z^zt: the output
// string with leading k letters in {I, Z} (Z-mask zt) and tail s has coefficient
// 2^-k WHT_k(j -> alpha_j[s])[zt]; leading strings containing X or Y are 0.
template <int K>
__global__ void block_diag_kernel(const double2* blocks, u64 count, double2* out) {
  constexpr int B = 1 << K;
  const double scale = 1.0 / B;
  for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (u64)gridDim.x * blockDim.x) {
    double2 v[B];
#pragma unroll
    for (int j = 0; j < B; ++j) v[j] = ld_stream(blocks + (u64)j * count + q);
    wht_regs<K>(v);
    // leading digits: digit_l = 3 z_l (I or Z); every other leading string is zero
#pragma unroll
    for (int t = 0; t < (B * B); ++t) {
      // t = leading q digits (base 4, K digits)
      int zt = 0;
      bool iz = true;
#pragma unroll
      for (int l = 0; l < K; ++l) {
        const int d = (t >> (2 * l)) & 3;
        if (d == 1 || d == 2) iz = false;
        zt |= (d == 3 ? 1 : 0) << l;
      }
      const double2 w = iz ? make_double2(v[zt].x * scale, v[zt].y * scale) : make_double2(0.0, 0.0);
      st_stream(out + (u64)t * count + q, w);
    }
  }
}

// ---- Hermitian augmentation [[0, A^*], [A, 0]] = X (x) Re A + Y (x) Im A (l.590-627) ----
// leading X: Re alpha (real), leading Y: Im alpha (real), leading I and Z: 0.
__global__ void herm_augment_kernel(const double2* a, u64 count, double2* out) {
  for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (u64)gridDim.x * blockDim.x) {
    const double2 v = ld_stream(a + q);
    st_stream(out + q, make_double2(0.0, 0.0));
    st_stream(out + count + q, make_double2(v.x, 0.0));
    st_stream(out + 2 * count + q, make_double2(v.y, 0.0));
    st_stream(out + 3 * count + q, make_double2(0.0, 0.0));
  }
}

static unsigned grid_for(u64 count) {
  u64 g = (count + 255) / 256;
  const u64 cap = (u64)device_sm_count() * 16;
  return (unsigned)(g > cap ? cap : (g ? g : 1));
}

cudaError_t launch_axpby(double2* out, double2 mu, const double2* x, double2 nu, const double2* y, u64 count,
                         cudaStream_t st) {
  axpby_kernel<<<grid_for(count), 256, 0, st>>>(out, mu, x, nu, y, count);
  return cudaGetLastError();
}

cudaError_t launch_block_diag(const double2* blocks, int n, int k, double2* out, cudaStream_t st) {
  const u64 count = 1ull << (2 * n);
  const unsigned g = grid_for(count);
  switch (k) {
    case 1: block_diag_kernel<1><<<g, 256, 0, st>>>(blocks, count, out); break;
    case 2: block_diag_kernel<2><<<g, 256, 0, st>>>(blocks, count, out); break;
    case 3: block_diag_kernel<3><<<g, 256, 0, st>>>(blocks, count, out); break;
    case 4: block_diag_kernel<4><<<g, 256, 0, st>>>(blocks, count, out); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_herm_augment(const double2* a, int n, double2* out, cudaStream_t st) {
  const u64 count = 1ull << (2 * n);
  herm_augment_kernel<<<grid_for(count), 256, 0, st>>>(a, count, out);
  return cudaGetLastError();
}

}  // namespace ptdr
