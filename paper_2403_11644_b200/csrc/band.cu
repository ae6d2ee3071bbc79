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
template <int K>
struct FlatSt {
  double2* out;
  u64 rbase;
  int b0;
  double scale;
  __device__ __forceinline__ void operator()(int f, int j, double2 v) const {
    const u64 rho = rbase + (u64)f;
    const u64 e = ((rho >> b0) << (b0 + K)) | ((u64)j << b0) | (rho & ((1ull << b0) - 1ull));
    st_l2(out + e, make_double2(v.x * scale, v.y * scale));
  }
};

template <int K>
__global__ void __launch_bounds__(kThreads, 2) wht_pass_kernel(const double2* in, double2* out,
                                                               u64 ntiles, int b0, double scale) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  constexpr int F = kTileElems >> K;
  for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    FlatLd<K> ld{in, tile * F, b0};
    FlatSt<K> st{out, tile * F, b0, scale};
    fiber_tile<K>(S, ld, st);
    __syncthreads();
  }
}

template <int K>
static cudaError_t launch_pass(const double2* in, double2* out, u64 total, int b0, double scale,
                               cudaStream_t st) {
  static bool attr_done = false;  // idempotent attribute set; benign race
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(wht_pass_kernel<K>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const u64 ntiles = total / kTileElems;
  u64 grid = (u64)device_sm_count() * 2;
  if (grid > ntiles) grid = ntiles;
  wht_pass_kernel<K><<<(unsigned)grid, kThreads, kTileBytes, st>>>(in, out, ntiles, b0, scale);
  return cudaGetLastError();
}

static cudaError_t launch_pass_k(int K, const double2* in, double2* out, u64 total, int b0,
                                 double scale, cudaStream_t st) {
  switch (K) {
    case 4: return launch_pass<4>(in, out, total, b0, scale, st);
    case 5: return launch_pass<5>(in, out, total, b0, scale, st);
    case 6: return launch_pass<6>(in, out, total, b0, scale, st);
    case 7: return launch_pass<7>(in, out, total, b0, scale, st);
    case 8: return launch_pass<8>(in, out, total, b0, scale, st);
    default: return cudaErrorInvalidValue;
  }
}

// WHT over the low `lambda` bits (lambda >= 13) of `total` contiguous elements
// (a batch of total/2^lambda vectors), in -> out (out may equal in), scaled.
static cudaError_t run_passes(const double2* in, double2* out, u64 total, int lambda,
                              double scale, cudaStream_t st, int* nl) {
  const int np = (lambda + 7) / 8;
  int b0 = 0;
  for (int p = 0; p < np; ++p) {
    const int K = (lambda - b0) / (np - p);
    cudaError_t e = launch_pass_k(K, p == 0 ? in : out, out, total, b0,
                                  p == np - 1 ? scale : 1.0, st);
    if (e != cudaSuccess) return e;
    *nl += 1;
    b0 += K;
  }
  return cudaSuccess;
}

// ---- small WHTs (length <= 4096) entirely in SMEM, one CTA per vector --------------
// mode 0: one vector of length 2^lam at in/out offset 0, scaled.
// mode 1: tridiagonal P/M segments t = tmin + blockIdx.x/2 of a size-2^n problem,
//         in place in `out` (the PM workspace), unscaled.
__global__ void __launch_bounds__(kThreads) wht_small_kernel(const double2* in, double2* out,
                                                             int mode, int n, int lam_or_tmin,
                                                             double scale) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* S = reinterpret_cast<double2*>(smem_raw);
  int lam;
  u64 off;
  if (mode == 0) {
    lam = lam_or_tmin;
    off = 0;
  } else {
    const int t = lam_or_tmin + (int)(blockIdx.x >> 1);
    lam = n - t - 1;
    const u64 N = 1ull << n;
    off = 2ull * (N - (N >> t)) + ((u64)(blockIdx.x & 1) << lam);
    in = out;
  }
  const int len = 1 << lam;
  for (int i = threadIdx.x; i < len; i += blockDim.x) S[i] = ld_l2(in + off + i);
  for (int s = 0; s < lam; ++s) {
    __syncthreads();
    for (int p = threadIdx.x; p < len / 2; p += blockDim.x) {
      const int lo = p & ((1 << s) - 1);
      const int i0 = ((p >> s) << (s + 1)) | lo;
      const int i1 = i0 | (1 << s);
      const double2 a = S[i0], b = S[i1];
      S[i0] = cadd(a, b);
      S[i1] = csub(a, b);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const double2 v = S[i];
    out[off + i] = make_double2(v.x * scale, v.y * scale);
  }
}

static cudaError_t launch_small(const double2* in, double2* out, int mode, int n, int arg,
                                double scale, unsigned blocks, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(wht_small_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  wht_small_kernel<<<blocks, kThreads, kTileBytes, st>>>(in, out, mode, n, arg, scale);
  return cudaGetLastError();
}

// out[0..2^n) = 2^-n WHT(in[0..2^n))
static cudaError_t wht_vector(const double2* in, double2* out, int n, cudaStream_t st, int* nl) {
  const double scale = ldexp(1.0, -n);
  if (n <= 12) {
    *nl += 1;
    return launch_small(in, out, 0, n, n, scale, 1, st);
  }
  return run_passes(in, out, 1ull << n, n, scale, st, nl);
}

// ---- tridiagonal split: (S_t, U_t) -> (S_t + U_t, S_t - U_t) compacted per t --------
__global__ void tridiag_split_kernel(const double2* band, double2* PM, int n) {
  const u64 N = 1ull << n;
  const double2* sub = band;
  const double2* sup = band + 2 * N;
  for (u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x; e < N - 1;
       e += (u64)gridDim.x * blockDim.x) {
    const int t = __clzll(~(e << (64 - n)));  // leading ones of the n-bit e
    const int lam = n - t - 1;
    const u64 seg = N - (N >> t);
    const u64 h = e - seg;
    const u64 b = (h << (t + 1)) + (1ull << t) - 1ull;
    const double2 s = sup[b];
    const double2 u = sub[b + 1];
    PM[2 * seg + h] = cadd(s, u);
    PM[2 * seg + (1ull << lam) + h] = csub(s, u);
  }
}

// ---- tridiagonal expansion into blocks 1..n ----------------------------------------
__global__ void tridiag_expand_kernel(const double2* PM, double2* out, int n, double scale) {
  const u64 N = 1ull << n;
  const u64 total = (u64)n * N;
  for (u64 id = (u64)blockIdx.x * blockDim.x + threadIdx.x; id < total;
       id += (u64)gridDim.x * blockDim.x) {
    const int t = (int)(id >> n);
    const u64 z = id & (N - 1);
    const int lam = n - t - 1;
    const u64 seg = N - (N >> t);
    const u64 zl = z & ((2ull << t) - 1ull);
    const u64 zh = z >> (t + 1);
    const int s1 = __popcll(z & ((1ull << t) - 1ull)) & 1;
    const int s2 = (int)((z >> t) & 1ull);
    double2 w = ld_l2(PM + 2 * seg + (s1 == s2 ? 0ull : (1ull << lam)) + zh);
    if (s1) w = make_double2(-w.x, -w.y);
    const double2 c = rot_ipow(w, __popcll(zl));
    st_stream(out + N + id, make_double2(c.x * scale, c.y * scale));
  }
}

size_t band_workspace_bytes(int n, int structure) {
  if (structure == 4) return (size_t)2 * ((size_t)1 << n) * 16;  // P/M segments
  return 0;
}

cudaError_t launch_band(const double2* A, double2* out, int n, int structure, void* ws,
                        cudaStream_t st, int* nl) {
  const u64 N = 1ull << n;
  if (structure == 3) return wht_vector(A, out, n, st, nl);
  // TRIDIAGONAL: A = [sub | main | sup]
  cudaError_t e = wht_vector(A + N, out, n, st, nl);  // block 0 (x = 0)
  if (e != cudaSuccess) return e;
  double2* PM = reinterpret_cast<double2*>(ws);
  const int sms = device_sm_count();
  {
    u64 blocks = (N + 255) / 256;
    if (blocks > (u64)sms * 16) blocks = (u64)sms * 16;
    tridiag_split_kernel<<<(unsigned)blocks, 256, 0, st>>>(A, PM, n);
    *nl += 1;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  int tmin = n - 13 > 0 ? n - 13 : 0;  // segments with lambda = n-t-1 <= 12 done in SMEM
  for (int t = 0; t < tmin; ++t) {
    const int lam = n - t - 1;
    const u64 seg = N - (N >> t);
    e = run_passes(PM + 2 * seg, PM + 2 * seg, 2ull << lam, lam, 1.0, st, nl);
    if (e != cudaSuccess) return e;
  }
  e = launch_small(nullptr, PM, 1, n, tmin, 1.0, (unsigned)(2 * (n - tmin)), st);
  *nl += 1;
  if (e != cudaSuccess) return e;
  {
    const u64 total = (u64)n * N;
    u64 blocks = (total + 255) / 256;
    if (blocks > (u64)sms * 32) blocks = (u64)sms * 32;
    tridiag_expand_kernel<<<(unsigned)blocks, 256, 0, st>>>(PM, out, n, ldexp(1.0, -n));
    *nl += 1;
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace ptdr
