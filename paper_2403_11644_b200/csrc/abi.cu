// abi.cu -- the C ABI of libptdr.so (include/ptdr.h): validation, workspace
// layout and dispatch to the kernels.  No torch types, no exceptions across the ABI.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <string>

#include "../../include/ptdr.h"
#include "../../include/ptdr_debug.h"
#include "dense_impl.cuh"
#include "dense_plan.h"
#include "internal.h"

namespace ptdr {

static thread_local std::string g_last_error;
static thread_local int g_last_launches = 0;

static std::atomic<int> g_sm_count[64] = {};

int device_sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = g_sm_count[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    g_sm_count[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device), raised again if
// a later launch of the same kernel asks for more.
cudaError_t ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  int& have = done[{fn, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

static ptdr_status fail(ptdr_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
static ptdr_status cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return PTDR_ECUDA;
}
// error reporting for plan.cu (same thread-local error string)
ptdr_status plan_fail(ptdr_status s, const char* msg) { return fail(s, msg); }
ptdr_status plan_cuda_fail(cudaError_t e, const char* where) { return cuda_fail(e, where); }

static bool is_dense(int s) { return s >= PTDR_GENERAL && s <= PTDR_REAL_SYMMETRIC; }
static bool is_band(int s) {
  return s == PTDR_DIAGONAL || s == PTDR_TRIDIAGONAL || s == PTDR_ANTI_DIAGONAL || s == PTDR_HERMITIAN_TRIDIAGONAL;
}
static bool is_tri(int s) { return s == PTDR_TRIDIAGONAL || s == PTDR_HERMITIAN_TRIDIAGONAL; }
static bool valid_n(int n, int s) {
  if (is_dense(s)) return n >= 1 && n <= 16;
  if (is_band(s)) return n >= 1 && n <= 28;
  return false;
}


// Dense-path kernel selection.  The product library always takes the default pipeline
// configuration (dense_plan.h kPipeDefault).  Developer builds (PTDR_DEV=1: build.py with
// PTDR_DEV_BUILD / PTDR_TRACE_BUILD / PTDR_DIAG_BUILD) also read PTDR_DENSE_V1=1 (force the
// dense_impl.cuh kernels) and PTDR_PIPE_CFG=<k> (another dense_pipe configuration).
static int pipe_choice() {
#if PTDR_DEV
  // read once (thread-safe static initialisation)
  static const int v = []() {
    const char* e1 = getenv("PTDR_DENSE_V1");
    const char* ec = getenv("PTDR_PIPE_CFG");
    if (e1 && e1[0] == '1') return kPipeNone;
    if (ec && ec[0] >= '1' && ec[0] <= '0' + kPipeCfgCount) return ec[0] - '0';
    return kPipeDefault;
  }();
  return v;
#else
  return kPipeDefault;
#endif
}

static bool pipe_mode(int mode) {
  return mode == MODE_GENERAL || mode == MODE_HERM_HALF || mode == MODE_SYM_HALF;
}

static DensePlan plan_for(int mode, int nv, uint64_t x_count) {
  return make_dense_plan(nv, x_count, pipe_mode(mode) ? pipe_choice() : kPipeNone, kSingleMax);
}
// The workspace is the max over every kernel choice the library can make (developer
// builds: every configuration) so that the size never depends on a switch.
static size_t plan_ws(int nv, uint64_t x_count) {
  size_t m = 0;
  for (int cfg = kPipeNone; cfg <= kPipeCfgCount; ++cfg)
    for (int smax : {7, kSingleMax}) {
      if (!pipe_cfg_built(cfg)) continue;
      const size_t b = make_dense_plan(nv, x_count, cfg, smax).ws_bytes();
      if (b > m) m = b;
    }
  return m;
}

// X-masks handled by the mirrored launch of HERMITIAN / REAL_SYMMETRIC (n >= 9): the first
// chunk of the half-length launch must start at a power of two >= its chunk width.
static uint64_t herm_mirror_width(int n, int hmode) {
  const uint64_t N = 1ull << n;
  const DensePlan hp = plan_for(hmode, n - 1, N - 32);
  return hp.W;
}

// Workspace of the dense path = max over the launches of one call.
static size_t dense_ws(int n, int s, int world) {
  const uint64_t N = 1ull << n;
  if (s == PTDR_GENERAL) return plan_ws(n, world > 1 ? N / (uint64_t)world : N);
  if (n <= 8) return plan_ws(n, N);
  size_t m = 0;
  for (uint64_t w : {16ull, 32ull}) {
    const size_t a = plan_ws(n, w), b = plan_ws(n - 1, N - w);
    if (a > m) m = a;
    if (b > m) m = b;
  }
  return m;
}

static ptdr_status launch_mode(int mode, const DenseArgs& a, const DensePlan& p, cudaStream_t st,
                               int* nl) {
  cudaError_t e;
  if (p.pipe_cfg != kPipeNone) {
    e = launch_dense_pipe(mode, a, p, st, nl);
    if (e != cudaSuccess) return cuda_fail(e, "dense pipeline kernel launch");
    return PTDR_OK;
  }
  switch (mode) {
    case MODE_GENERAL: e = launch_dense_mode0(a, p, st, nl); break;
    case MODE_HERM_MIRROR: e = launch_dense_mode1(a, p, st, nl); break;
    case MODE_SYM_MIRROR: e = launch_dense_mode2(a, p, st, nl); break;
    case MODE_HERM_HALF: e = launch_dense_mode3(a, p, st, nl); break;
    default: e = launch_dense_mode4(a, p, st, nl); break;
  }
  if (e != cudaSuccess) return cuda_fail(e, "dense kernel launch");
  return PTDR_OK;
}

static DenseArgs base_args(const double2* A, double2* out, int n, void* ws) {
  DenseArgs a{};
  a.A = A;
  a.out = out;
  a.n = n;
  a.ld = 1ull << n;
  a.colmask = (1ull << n) - 1ull;
  a.gshift = n;
  a.scale = std::ldexp(1.0, -n);
  a.ctr = reinterpret_cast<unsigned*>(ws);
  return a;
}

static ptdr_status run_dense(const double2* A, int n, int s, double2* out, void* ws,
                             cudaStream_t st, int* nl, uint64_t lda = 0, uint64_t m = 0,
                             uint64_t batch = 0, int layout_mat = 0) {
  const uint64_t N = 1ull << n;
  auto batched = [&](DenseArgs& a) {
    a.batch = batch;
    a.bstride_in = N * N;
    a.bstride_out = N * N;
    a.layout_mat = layout_mat;
  };
  if (s == PTDR_GENERAL || n <= 8) {
    const int mode = s == PTDR_GENERAL ? MODE_GENERAL
                     : s == PTDR_HERMITIAN ? MODE_HERM_MIRROR : MODE_SYM_MIRROR;
    DensePlan p = plan_for(mode, n, N);
    DenseArgs a = base_args(A, out, n, ws);
    batched(a);
    if (m) {  // zero-padded view (TMA pipeline only, see ptdr_decompose_padded_async)
      a.ld = lda;
      a.rows_valid = m;
      a.cols_valid = m;
    }
    a.nv = n;
    a.x_base = 0;
    a.nchunks = p.nchunks;
    a.scratch = reinterpret_cast<double2*>(reinterpret_cast<char*>(ws) + p.ctr_bytes);
    return launch_mode(mode, a, p, st, nl);
  }
  // HERMITIAN / REAL_SYMMETRIC, n >= 9: X-masks below the half-length launch's chunk width
  // on full-length mirrored vectors, the rest on half-length vectors.
  const int hmode = s == PTDR_HERMITIAN ? MODE_HERM_HALF : MODE_SYM_HALF;
  const uint64_t w = herm_mirror_width(n, hmode);
  {
    DensePlan p = plan_for(MODE_HERM_MIRROR, n, w);
    DenseArgs a = base_args(A, out, n, ws);
    batched(a);
    a.nv = n;
    a.x_base = 0;
    a.nchunks = p.nchunks;
    a.scratch = reinterpret_cast<double2*>(reinterpret_cast<char*>(ws) + p.ctr_bytes);
    ptdr_status r = launch_mode(s == PTDR_HERMITIAN ? MODE_HERM_MIRROR : MODE_SYM_MIRROR, a, p, st, nl);
    if (r != PTDR_OK) return r;
  }
  {
    DensePlan p = plan_for(hmode, n - 1, N - w);
    DenseArgs a = base_args(A, out, n, ws);
    batched(a);
    a.nv = n - 1;
    a.x_base = w;
    a.nchunks = p.nchunks;
    a.scratch = reinterpret_cast<double2*>(reinterpret_cast<char*>(ws) + p.ctr_bytes);
    return launch_mode(hmode, a, p, st, nl);
  }
}

// The inverse transform on the dense pipeline (MODE_INV from the matrix layout, MODE_INVQ from
// q order): the forward kernel with the phase (-i)^{popcount(x & z)} applied on input, no
// scale, and the matrix-layout store A[i][i ^ x] (dense_pipe.cuh).  Sizes with the pipeline only.
static bool inv_pipe(int n) {
  const DensePlan p = plan_for(MODE_GENERAL, n, 1ull << n);
  return p.pipe_cfg != kPipeNone && p.kind == 2;
}
static ptdr_status run_inverse_pipe(int mode, const double2* src, int n, double2* out, void* ws, cudaStream_t st,
                                    int* nl) {
  const DensePlan p = plan_for(MODE_GENERAL, n, 1ull << n);
  DenseArgs a = base_args(src, out, n, ws);
  a.scale = 1.0;
  a.layout_mat = 1;
  a.nv = n;
  a.x_base = 0;
  a.nchunks = p.nchunks;
  a.scratch = reinterpret_cast<double2*>(reinterpret_cast<char*>(ws) + p.ctr_bytes);
  return launch_mode(mode, a, p, st, nl);
}

static bool overlaps(const void* a, size_t abytes, const void* b, size_t bbytes) {
  const uintptr_t a0 = (uintptr_t)a, b0 = (uintptr_t)b;
  return a0 < b0 + bbytes && b0 < a0 + abytes;
}

}  // namespace ptdr

using namespace ptdr;

extern "C" {

int ptdr_version(void) { return 1; }

int ptdr_debug_trace_copy(void* host, size_t bytes) { return debug_trace_copy(host, bytes); }

int ptdr_max_n(int structure) {
  if (is_dense(structure)) return 16;
  if (is_band(structure)) return 28;
  return 0;
}

size_t ptdr_input_count(int n, int s) {
  if (!valid_n(n, s)) return 0;
  const size_t N = (size_t)1 << n;
  if (is_dense(s)) return N * N;
  return s == PTDR_TRIDIAGONAL ? 3 * N : s == PTDR_HERMITIAN_TRIDIAGONAL ? 2 * N : N;
}

size_t ptdr_output_count(int n, int s) {
  if (!valid_n(n, s)) return 0;
  const size_t N = (size_t)1 << n;
  if (is_dense(s)) return N * N;
  return is_tri(s) ? (size_t)(n + 1) * N : N;
}

size_t ptdr_workspace_bytes(int n, int s, int world) {
  if (!valid_n(n, s) || world < 1 || (world & (world - 1))) return (size_t)-1;
  if (world > 1) {
    const int g = __builtin_ctz((unsigned)world);
    if (s == PTDR_GENERAL) {
      if (n - g < 4) return (size_t)-1;
    } else if (is_band(s)) {
      if (g > n) return (size_t)-1;
    } else {
      return (size_t)-1;
    }
  }
  if (is_dense(s)) return dense_ws(n, s, world);
  return band_workspace_bytes(n, s, world);
}

const char* ptdr_status_string(int status) {
  switch (status) {
    case PTDR_OK: return "PTDR_OK";
    case PTDR_EINVAL: return "PTDR_EINVAL";
    case PTDR_EUNSUPPORTED: return "PTDR_EUNSUPPORTED";
    case PTDR_ENOMEM: return "PTDR_ENOMEM";
    case PTDR_ECUDA: return "PTDR_ECUDA";
    default: return "PTDR_UNKNOWN";
  }
}

const char* ptdr_last_error(void) { return g_last_error.c_str(); }

int ptdr_last_launch_count(void) { return g_last_launches; }

ptdr_status ptdr_decompose_async(const ptdr_c128* A, int n, int structure, ptdr_c128* out,
                                 void* workspace, size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  if (!valid_n(n, structure)) return fail(PTDR_EINVAL, "invalid n or structure");
  if (!A || !out) return fail(PTDR_EINVAL, "null A or out");
  if (((uintptr_t)A & 15) || ((uintptr_t)out & 15)) return fail(PTDR_EINVAL, "A/out not 16-byte aligned");
  const size_t need = ptdr_workspace_bytes(n, structure, 1);
  if (need > 0) {
    if (!workspace) return fail(PTDR_ENOMEM, "workspace required");
    if ((uintptr_t)workspace & 255) return fail(PTDR_EINVAL, "workspace not 256-byte aligned");
  }
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  const size_t inb = ptdr_input_count(n, structure) * 16, outb = ptdr_output_count(n, structure) * 16;
  if (overlaps(A, inb, out, outb)) return fail(PTDR_EUNSUPPORTED, "out overlaps A");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int nl = 0;
  ptdr_status r;
  if (is_dense(structure)) {
    r = run_dense(reinterpret_cast<const double2*>(A), n, structure, reinterpret_cast<double2*>(out),
                  workspace, st, &nl);
  } else {
    cudaError_t e = launch_band(reinterpret_cast<const double2*>(A), reinterpret_cast<double2*>(out), n,
                                structure, workspace, 0, 1, st, &nl);
    r = e == cudaSuccess ? PTDR_OK : cuda_fail(e, "band kernel launch");
  }
  g_last_launches = nl;
  return r;
}

ptdr_status ptdr_decompose_xshard_ex_async(const ptdr_c128* A_local, int n, int rank, int world,
                                           ptdr_c128* out_local, void* workspace, size_t ws_bytes,
                                           int max_ctas, void* stream) {
  g_last_launches = 0;
  if (world < 1 || (world & (world - 1))) return fail(PTDR_EINVAL, "world must be a power of two");
  if (rank < 0 || rank >= world) return fail(PTDR_EINVAL, "rank out of range");
  if (!valid_n(n, PTDR_GENERAL)) return fail(PTDR_EINVAL, "invalid n");
  const int g = __builtin_ctz((unsigned)world);
  if (n - g < 4) return fail(PTDR_EINVAL, "need n - log2(world) >= 4");
  if (!A_local || !out_local) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)A_local & 15) || ((uintptr_t)out_local & 15)) return fail(PTDR_EINVAL, "misaligned");
  const size_t need = ptdr_workspace_bytes(n, PTDR_GENERAL, world);
  if (need > 0 && (!workspace || ((uintptr_t)workspace & 255)))
    return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  const uint64_t N = 1ull << n, R = N >> g;
  if (overlaps(A_local, N * R * 16, out_local, N * R * 16)) return fail(PTDR_EUNSUPPORTED, "out overlaps A");
  DensePlan p = plan_for(MODE_GENERAL, n, R);
  DenseArgs a = base_args(reinterpret_cast<const double2*>(A_local), reinterpret_cast<double2*>(out_local),
                          n, workspace);
  a.ld = R;
  a.colmask = R - 1;
  a.gshift = n - g;
  a.nv = n;
  a.x_base = (uint64_t)rank * R;
  a.nchunks = p.nchunks;
  a.scratch = reinterpret_cast<double2*>(reinterpret_cast<char*>(workspace) + p.ctr_bytes);
  a.max_ctas = max_ctas > 0 ? max_ctas : 0;
  int nl = 0;
  ptdr_status r = launch_mode(MODE_GENERAL, a, p, reinterpret_cast<cudaStream_t>(stream), &nl);
  g_last_launches = nl;
  return r;
}

ptdr_status ptdr_decompose_xshard_async(const ptdr_c128* A_local, int n, int rank, int world,
                                        ptdr_c128* out_local, void* workspace, size_t ws_bytes,
                                        void* stream) {
  return ptdr_decompose_xshard_ex_async(A_local, n, rank, world, out_local, workspace, ws_bytes, 0, stream);
}

// ---- matrix-free input ------------------------------------
// GENERAL entries from the counter-based generator (variant 0),
// produced inside phase A of the pipeline: A is never stored.  world > 1: rank's X-mask
// shard (output layout of ptdr_decompose_xshard_async), no communication at all.
static bool generated_pipe(int n, int world) {
  const uint64_t R = (1ull << n) / (uint64_t)world;
  const DensePlan p = plan_for(MODE_GENERAL, n, R);
  return p.kind == 2 && p.pipe_cfg != kPipeNone && (p.pipe_cfg == 1 || p.pipe_cfg == 4);
}

size_t ptdr_generated_workspace_bytes(int n, int world) {
  if (!valid_n(n, PTDR_GENERAL) || world < 1 || (world & (world - 1)) || (uint64_t)world > (1ull << n))
    return (size_t)-1;
  if (world > 1) return generated_pipe(n, world) ? ptdr_workspace_bytes(n, PTDR_GENERAL, world) : (size_t)-1;
  if (generated_pipe(n, 1)) return ptdr_workspace_bytes(n, PTDR_GENERAL, 1);
  // small n: the matrix is generated into the workspace, then decomposed as stored
  return ((((size_t)16 << (2 * n)) + 255) / 256) * 256 + ptdr_workspace_bytes(n, PTDR_GENERAL, 1);
}

ptdr_status ptdr_decompose_generated_async(int n, uint64_t seed, int rank, int world, ptdr_c128* out_local,
                                           void* workspace, size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  const size_t need = ptdr_generated_workspace_bytes(n, world);
  if (need == (size_t)-1)
    return fail(PTDR_EINVAL, "invalid n / world (world > 1 needs n - log2(world) >= 11)");
  if (rank < 0 || rank >= world) return fail(PTDR_EINVAL, "rank out of range");
  if (!out_local || ((uintptr_t)out_local & 15)) return fail(PTDR_EINVAL, "null or misaligned out");
  if (need > 0 && (!workspace || ((uintptr_t)workspace & 255)))
    return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int g = __builtin_ctz((unsigned)world);
  const uint64_t N = 1ull << n, R = N >> g;
  if (!generated_pipe(n, world)) {  // world == 1, small n
    const size_t ab = ((((size_t)16 << (2 * n)) + 255) / 256) * 256;
    double2* A = reinterpret_cast<double2*>(workspace);
    cudaError_t e = launch_generate_dense(n, seed, 0, 0, N, A, nullptr, st);
    if (e != cudaSuccess) return cuda_fail(e, "generator launch");
    ptdr_status r = ptdr_decompose_async(reinterpret_cast<const ptdr_c128*>(A), n, PTDR_GENERAL, out_local,
                                         reinterpret_cast<char*>(workspace) + ab, ws_bytes - ab, stream);
    g_last_launches += 1;
    return r;
  }
  DensePlan p = plan_for(MODE_GENERAL, n, R);
  DenseArgs a = base_args(reinterpret_cast<const double2*>(out_local), reinterpret_cast<double2*>(out_local), n,
                          workspace);  // A unused (no loads); any valid address for the tensor map
  a.ld = N;
  a.colmask = N - 1;
  a.gshift = n - g;
  a.nv = n;
  a.x_base = (uint64_t)rank * R;
  a.nchunks = p.nchunks;
  a.scratch = reinterpret_cast<double2*>(reinterpret_cast<char*>(workspace) + p.ctr_bytes);
  a.gen_seed = seed;
  int nl = 0;
  ptdr_status r = launch_mode(MODE_GEN, a, p, st, &nl);
  g_last_launches = nl;
  return r;
}

// ---- fused exchange: peer-pull X-mask decomposition --------------------
ptdr_status ptdr_decompose_peer_async(const ptdr_c128* const* shards, int n, int rank, int world,
                                      ptdr_c128* out_local, void* workspace, size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  if (world < 2 || world > 8 || (world & (world - 1))) return fail(PTDR_EINVAL, "world must be 2, 4 or 8");
  if (rank < 0 || rank >= world) return fail(PTDR_EINVAL, "rank out of range");
  if (!valid_n(n, PTDR_GENERAL)) return fail(PTDR_EINVAL, "invalid n");
  if (!shards || !out_local) return fail(PTDR_EINVAL, "null pointer");
  const int g = __builtin_ctz((unsigned)world);
  const uint64_t N = 1ull << n, R = N >> g;
  for (int r = 0; r < world; ++r)
    if (!shards[r] || ((uintptr_t)shards[r] & 15)) return fail(PTDR_EINVAL, "null or misaligned shard pointer");
  if ((uintptr_t)out_local & 15) return fail(PTDR_EINVAL, "misaligned out");
  DensePlan p = plan_for(MODE_GENERAL, n, R);
  if (p.kind != 2 || p.pipe_cfg == kPipeNone || R < 128)
    return fail(PTDR_EUNSUPPORTED, "peer-pull needs the TMA pipeline: n - log2(world) >= 11");
  const size_t need = ptdr_workspace_bytes(n, PTDR_GENERAL, world);
  if (need > 0 && (!workspace || ((uintptr_t)workspace & 255)))
    return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  DenseArgs a = base_args(reinterpret_cast<const double2*>(shards[rank]), reinterpret_cast<double2*>(out_local),
                          n, workspace);
  a.ld = N;                 // shard rows are full matrix rows
  a.colmask = N - 1;
  a.gshift = n - g;
  a.nv = n;
  a.x_base = (uint64_t)rank * R;
  a.nchunks = p.nchunks;
  a.scratch = reinterpret_cast<double2*>(reinterpret_cast<char*>(workspace) + p.ctr_bytes);
  a.peer_shift = n - g;
  a.peer_rowmask = R - 1;
  a.npeers = world;
  for (int r = 0; r < world; ++r) a.peer_ptrs[r] = reinterpret_cast<const double2*>(shards[r]);
  int nl = 0;
  ptdr_status st = launch_mode(MODE_GENERAL, a, p, reinterpret_cast<cudaStream_t>(stream), &nl);
  g_last_launches = nl;
  return st;
}

size_t ptdr_ipc_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

ptdr_status ptdr_ipc_get_handle(const void* dev_ptr, void* handle, uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(PTDR_EINVAL, "null pointer");
  // the handle names the whole allocation: report where dev_ptr sits inside it
  static const PFN_memGetAddressRange range_fn = []() -> PFN_memGetAddressRange {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<PFN_memGetAddressRange>(fp);
  }();
  if (!range_fn) return fail(PTDR_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(PTDR_EINVAL, "dev_ptr is not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return PTDR_OK;
}

ptdr_status ptdr_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(PTDR_EINVAL, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return PTDR_OK;
}

ptdr_status ptdr_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return PTDR_OK;
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return PTDR_OK;
}

ptdr_status ptdr_decompose_zshard_async(const ptdr_c128* band, int n, int structure, int rank, int world,
                                        ptdr_c128* out_local, void* workspace, size_t ws_bytes,
                                        void* stream) {
  g_last_launches = 0;
  if (!is_band(structure))
    return fail(PTDR_EINVAL, "z-sharding is for DIAGONAL / TRIDIAGONAL / ANTI_DIAGONAL / HERMITIAN_TRIDIAGONAL");
  if (!valid_n(n, structure)) return fail(PTDR_EINVAL, "invalid n");
  if (world < 1 || (world & (world - 1))) return fail(PTDR_EINVAL, "world must be a power of two");
  if ((uint64_t)world > (1ull << n)) return fail(PTDR_EINVAL, "world > 2^n");
  if (rank < 0 || rank >= world) return fail(PTDR_EINVAL, "rank out of range");
  if (!band || !out_local) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)band & 15) || ((uintptr_t)out_local & 15)) return fail(PTDR_EINVAL, "misaligned");
  const size_t need = ptdr_workspace_bytes(n, structure, world);
  if (need > 0 && (!workspace || ((uintptr_t)workspace & 255)))
    return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  const size_t inb = ptdr_input_count(n, structure) * 16, outb = ptdr_output_count(n, structure) * 16 / world;
  if (overlaps(band, inb, out_local, outb)) return fail(PTDR_EUNSUPPORTED, "out overlaps the band");
  int nl = 0;
  cudaError_t e = launch_band(reinterpret_cast<const double2*>(band), reinterpret_cast<double2*>(out_local), n,
                              structure, workspace, rank, world, reinterpret_cast<cudaStream_t>(stream), &nl);
  g_last_launches = nl;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "band kernel launch");
}

size_t ptdr_band_xmask_count(int n, int s) { return band_s_xmask_count(n, s); }

ptdr_status ptdr_band_xmasks(int n, int s, uint64_t* xs, size_t cap) {
  if (!xs) return fail(PTDR_EINVAL, "null xs");
  const int r = band_s_xmasks(n, s, reinterpret_cast<unsigned long long*>(xs), cap);
  if (r == -1) return fail(PTDR_EINVAL, "invalid n or s");
  if (r == -2) return fail(PTDR_EINVAL, "xs capacity smaller than ptdr_band_xmask_count");
  return PTDR_OK;
}

size_t ptdr_band_workspace_bytes(int n, int s) { return band_s_workspace_bytes(n, s); }

ptdr_status ptdr_decompose_band_async(const ptdr_c128* diags, int n, int s, ptdr_c128* out, void* workspace,
                                      size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  const size_t cnt = band_s_xmask_count(n, s);
  if (cnt == 0) return fail(PTDR_EINVAL, "invalid n or s (need 1 <= n <= 28, 0 <= s <= 64, s < 2^n)");
  if (!diags || !out) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)diags & 15) || ((uintptr_t)out & 15)) return fail(PTDR_EINVAL, "misaligned");
  const size_t need = band_s_workspace_bytes(n, s);
  if (!workspace || ((uintptr_t)workspace & 255)) return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  const size_t N = (size_t)1 << n;
  if (overlaps(diags, (2 * (size_t)s + 1) * N * 16, out, cnt * N * 16)) return fail(PTDR_EUNSUPPORTED, "out overlaps the band");
  if (overlaps(workspace, need, out, cnt * N * 16) || overlaps(workspace, need, diags, (2 * (size_t)s + 1) * N * 16))
    return fail(PTDR_EINVAL, "workspace overlaps an operand");
  int nl = 0;
  cudaError_t e = launch_band_s(reinterpret_cast<const double2*>(diags), n, s, reinterpret_cast<double2*>(out),
                                workspace, reinterpret_cast<cudaStream_t>(stream), &nl);
  g_last_launches = nl;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "band(s) kernel launch");
}

// ---- algebra and inverse transform (algebra.cu) ---------------------------------------
size_t ptdr_reconstruct_workspace_bytes(int n) {
  if (n < 1 || n > 16) return (size_t)-1;
  if (inv_pipe(n)) return plan_ws(n, 1ull << n);
  return reconstruct_workspace_bytes(n);
}

ptdr_status ptdr_reconstruct_async(const ptdr_c128* coeffs, int n, ptdr_c128* A, void* workspace,
                                   size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  if (n < 1 || n > 16) return fail(PTDR_EINVAL, "invalid n (1..16)");
  if (!coeffs || !A || !workspace) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)coeffs & 15) || ((uintptr_t)A & 15) || ((uintptr_t)workspace & 255))
    return fail(PTDR_EINVAL, "misaligned pointer");
  const size_t nb = (size_t)16 << (2 * n);
  const size_t need = ptdr_reconstruct_workspace_bytes(n);
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  if (overlaps(coeffs, nb, A, nb) || overlaps(workspace, need, A, nb) || overlaps(workspace, need, coeffs, nb))
    return fail(PTDR_EUNSUPPORTED, "coeffs, A and workspace must be disjoint");
  int nl = 0;
  if (inv_pipe(n)) {
    const ptdr_status r = run_inverse_pipe(MODE_INVQ, reinterpret_cast<const double2*>(coeffs), n,
                                           reinterpret_cast<double2*>(A), workspace,
                                           reinterpret_cast<cudaStream_t>(stream), &nl);
    g_last_launches = nl;
    return r;
  }
  cudaError_t e = launch_reconstruct(reinterpret_cast<const double2*>(coeffs), n, reinterpret_cast<double2*>(A),
                                     workspace, reinterpret_cast<cudaStream_t>(stream), &nl);
  g_last_launches = nl;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "reconstruct launch");
}

ptdr_status ptdr_axpby_async(ptdr_c128* out, double mu_re, double mu_im, const ptdr_c128* x, double nu_re,
                             double nu_im, const ptdr_c128* y, size_t count, void* stream) {
  g_last_launches = 0;
  if (!out || !x || !y) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)out | (uintptr_t)x | (uintptr_t)y) & 15) return fail(PTDR_EINVAL, "misaligned pointer");
  if (count == 0) return PTDR_OK;
  cudaError_t e = launch_axpby(reinterpret_cast<double2*>(out), make_double2(mu_re, mu_im),
                               reinterpret_cast<const double2*>(x), make_double2(nu_re, nu_im),
                               reinterpret_cast<const double2*>(y), count, reinterpret_cast<cudaStream_t>(stream));
  g_last_launches = 1;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "axpby launch");
}

ptdr_status ptdr_block_diag_async(const ptdr_c128* blocks, int n, int k, ptdr_c128* out, void* stream) {
  g_last_launches = 0;
  if (n < 1 || k < 1 || k > 4 || n + k > 16) return fail(PTDR_EINVAL, "need n >= 1, 1 <= k <= 4, n + k <= 16");
  if (!blocks || !out) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)blocks | (uintptr_t)out) & 15) return fail(PTDR_EINVAL, "misaligned pointer");
  const size_t in_b = ((size_t)16 << (2 * n)) << k, out_b = (size_t)16 << (2 * (n + k));
  if (overlaps(blocks, in_b, out, out_b)) return fail(PTDR_EUNSUPPORTED, "out overlaps the blocks");
  cudaError_t e = launch_block_diag(reinterpret_cast<const double2*>(blocks), n, k, reinterpret_cast<double2*>(out),
                                    reinterpret_cast<cudaStream_t>(stream));
  g_last_launches = 1;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "block_diag launch");
}

ptdr_status ptdr_hermitian_augment_async(const ptdr_c128* coeffs, int n, ptdr_c128* out, void* stream) {
  g_last_launches = 0;
  if (n < 1 || n > 15) return fail(PTDR_EINVAL, "need 1 <= n <= 15");
  if (!coeffs || !out) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)coeffs | (uintptr_t)out) & 15) return fail(PTDR_EINVAL, "misaligned pointer");
  if (overlaps(coeffs, (size_t)16 << (2 * n), out, (size_t)64 << (2 * n)))
    return fail(PTDR_EUNSUPPORTED, "out overlaps the input");
  cudaError_t e = launch_herm_augment(reinterpret_cast<const double2*>(coeffs), n, reinterpret_cast<double2*>(out),
                                      reinterpret_cast<cudaStream_t>(stream));
  g_last_launches = 1;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "hermitian_augment launch");
}

// ---- zero padding -------------------------------------------------------
__global__ void pad_copy_kernel(const double2* __restrict__ A, uint64_t m, uint64_t lda, int n,
                                double2* __restrict__ P) {
  const uint64_t N = 1ull << n;
  for (uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; id < N * N;
       id += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = id >> n, j = id & (N - 1);
    P[id] = (i < m && j < m) ? A[i * lda + j] : make_double2(0.0, 0.0);
  }
}

static int padded_n(uint64_t m) {
  int n = 1;
  while ((1ull << n) < m && n < 63) ++n;
  return n;
}
// GENERAL with the TMA pipeline reads the stored block in place (out-of-bounds boxes are
// zero-filled); every other case copies into a zero-padded 2^n x 2^n workspace buffer.
static bool padded_in_place(int n, int structure) {
  return structure == PTDR_GENERAL && plan_for(MODE_GENERAL, n, 1ull << n).pipe_cfg != kPipeNone &&
         plan_for(MODE_GENERAL, n, 1ull << n).kind == 2;
}

// Bytes of the zero-padded copy that precedes the decomposition whenever the stored block
// cannot be read in place.  The size function does not know the row pitch, so it covers
// every pitch: an exact m = 2^n with lda != m also takes the copy.
static size_t pad_copy_bytes(int n) { return ((((size_t)16 << (2 * n)) + 255) / 256) * 256; }

size_t ptdr_padded_workspace_bytes(uint64_t m, int structure) {
  if (m < 1 || !is_dense(structure)) return (size_t)-1;
  const int n = padded_n(m);
  if (n > 16) return (size_t)-1;
  const size_t base = ptdr_workspace_bytes(n, structure, 1);
  if (padded_in_place(n, structure)) return base;
  return pad_copy_bytes(n) + base;
}

ptdr_status ptdr_decompose_padded_async(const ptdr_c128* A, uint64_t m, uint64_t lda, int structure,
                                        ptdr_c128* out, void* workspace, size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  if (!is_dense(structure)) return fail(PTDR_EINVAL, "zero padding is for the dense structures");
  if (m < 1) return fail(PTDR_EINVAL, "m must be >= 1 (an empty matrix has no decomposition)");
  if (lda < m) return fail(PTDR_EINVAL, "lda < m");
  const int n = padded_n(m);
  if (n > 16) return fail(PTDR_EINVAL, "m > 65536");
  if (!A || !out) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)A & 15) || ((uintptr_t)out & 15)) return fail(PTDR_EINVAL, "misaligned pointer");
  const size_t need = ptdr_padded_workspace_bytes(m, structure);
  if (need > 0 && (!workspace || ((uintptr_t)workspace & 255)))
    return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  const size_t inb = ((m - 1) * lda + m) * 16, outb = (size_t)16 << (2 * n);
  if (overlaps(A, inb, out, outb)) return fail(PTDR_EUNSUPPORTED, "out overlaps A");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool exact = (1ull << n) == m;
  if (exact && lda == m) return ptdr_decompose_async(A, n, structure, out, workspace, ws_bytes, stream);
  int nl = 0;
  ptdr_status r;
  if (padded_in_place(n, structure)) {
    r = run_dense(reinterpret_cast<const double2*>(A), n, structure, reinterpret_cast<double2*>(out), workspace, st,
                  &nl, lda, m);
  } else {
    const size_t pad_b = pad_copy_bytes(n);
    if (!workspace || ws_bytes < pad_b + ptdr_workspace_bytes(n, structure, 1))
      return fail(PTDR_ENOMEM, "workspace too small for the zero-padded copy");
    double2* P = reinterpret_cast<double2*>(workspace);
    const uint64_t N = 1ull << n;
    uint64_t g = (N * N + 255) / 256;
    if (g > (uint64_t)device_sm_count() * 16) g = (uint64_t)device_sm_count() * 16;
    pad_copy_kernel<<<(unsigned)g, 256, 0, st>>>(reinterpret_cast<const double2*>(A), m, lda, n, P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pad copy launch");
    r = ptdr_decompose_async(reinterpret_cast<const ptdr_c128*>(P), n, structure, out,
                             reinterpret_cast<char*>(workspace) + pad_b, ws_bytes - pad_b, stream);
    nl = 1 + g_last_launches;
  }
  g_last_launches = nl;
  return r;
}

// ---- in-place decomposition (BASELINE configs[4] "n=16 ... at 1 GPU in-place") --------
// Output in the matrix layout A[z][z ^ x] = alpha(x, z).  Every kernel that reads all of an
// X-mask's XOR-diagonal S_x = {(i, i ^ x)} before writing its coefficients -- and writes
// them only into S_x -- runs in place: the pipeline and the v1 two-phase kernels per chunk
// (phase B of a chunk starts after all its phase-A tiles), the whole-vector tiles per tile.
// Only the direct kernel (one thread per coefficient, n <= 5) would race; there the
// coefficients go through a workspace copy first (16 4^n bytes, at most 16 KiB).
static bool inplace_via_copy(int n) { return n <= 5; }

size_t ptdr_inplace_workspace_bytes(int n, int structure) {
  if (!is_dense(structure) || !valid_n(n, structure)) return (size_t)-1;
  const size_t base = ptdr_workspace_bytes(n, structure, 1);
  return inplace_via_copy(n) ? pad_copy_bytes(n) + base : base;
}

__global__ void q_to_matrix_layout_kernel(const double2* __restrict__ Q, int n, double2* __restrict__ M) {
  const uint64_t N = 1ull << n;
  for (uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; id < N * N;
       id += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = id >> n, z = id & (N - 1);
    M[(z << n) | (z ^ x)] = Q[q_offset(x, z, n)];
  }
}

ptdr_status ptdr_decompose_inplace_async(ptdr_c128* A, int n, int structure, void* workspace, size_t ws_bytes,
                                         void* stream) {
  g_last_launches = 0;
  if (!is_dense(structure)) return fail(PTDR_EINVAL, "in-place decomposition is for the dense structures");
  if (!valid_n(n, structure)) return fail(PTDR_EINVAL, "invalid n (1..16)");
  if (!A || ((uintptr_t)A & 15)) return fail(PTDR_EINVAL, "null or misaligned A");
  const size_t need = ptdr_inplace_workspace_bytes(n, structure);
  if (need > 0 && (!workspace || ((uintptr_t)workspace & 255)))
    return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  if (need > 0 && overlaps(workspace, need, A, (size_t)16 << (2 * n)))
    return fail(PTDR_EINVAL, "workspace overlaps A");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double2* a = reinterpret_cast<double2*>(A);
  int nl = 0;
  ptdr_status r;
  if (inplace_via_copy(n)) {
    double2* Q = reinterpret_cast<double2*>(workspace);
    const size_t cb = pad_copy_bytes(n);
    r = run_dense(a, n, structure, Q, reinterpret_cast<char*>(workspace) + cb, st, &nl);
    if (r != PTDR_OK) return r;
    const uint64_t total = 1ull << (2 * n);
    q_to_matrix_layout_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(Q, n, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "layout kernel launch");
    nl += 1;
  } else {
    r = run_dense(a, n, structure, a, workspace, st, &nl, 0, 0, 0, 1);
  }
  g_last_launches = nl;
  return r;
}

ptdr_status ptdr_decompose_matrix_layout_async(const ptdr_c128* A, int n, int structure, ptdr_c128* out,
                                               void* workspace, size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  if (!is_dense(structure)) return fail(PTDR_EINVAL, "the matrix layout is for the dense structures");
  if (!valid_n(n, structure)) return fail(PTDR_EINVAL, "invalid n (1..16)");
  if (!A || !out || ((uintptr_t)A & 15) || ((uintptr_t)out & 15)) return fail(PTDR_EINVAL, "null or misaligned pointer");
  if (overlaps(A, (size_t)16 << (2 * n), out, (size_t)16 << (2 * n)))
    return fail(PTDR_EUNSUPPORTED, "out overlaps A (use ptdr_decompose_inplace_async)");
  const size_t need = ptdr_inplace_workspace_bytes(n, structure);
  if (need > 0 && (!workspace || ((uintptr_t)workspace & 255)))
    return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double2* a = reinterpret_cast<const double2*>(A);
  double2* o = reinterpret_cast<double2*>(out);
  int nl = 0;
  ptdr_status r;
  if (inplace_via_copy(n)) {
    double2* Q = reinterpret_cast<double2*>(workspace);
    r = run_dense(a, n, structure, Q, reinterpret_cast<char*>(workspace) + pad_copy_bytes(n), st, &nl);
    if (r != PTDR_OK) return r;
    const uint64_t total = 1ull << (2 * n);
    q_to_matrix_layout_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(Q, n, o);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "layout kernel launch");
    nl += 1;
  } else {
    r = run_dense(a, n, structure, o, workspace, st, &nl, 0, 0, 0, 1);
  }
  g_last_launches = nl;
  return r;
}

// ---- inverse transform from the matrix layout ------------------------
// v_x = WHT_n(u_x), u_x[z] = (-i)^{popcount(x & z)} alpha(x, z), A[i][i ^ x] = v_x[i]: the
// forward pipeline with the phase moved from the epilogue into phase A (MODE_INV).  The input
// M[z][z ^ x] = alpha(x, z) and the output share every XOR-diagonal, so it runs in place.
// Sizes without the pipeline permute to q order in the workspace and call the q-order inverse.
__global__ void matrix_layout_to_q_kernel(const double2* __restrict__ M, int n, double2* __restrict__ Q) {
  const uint64_t N = 1ull << n;
  for (uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; id < N * N;
       id += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = id >> n, z = id & (N - 1);
    Q[q_offset(x, z, n)] = M[(z << n) | (z ^ x)];
  }
}

size_t ptdr_reconstruct_matrix_layout_workspace_bytes(int n) {
  if (n < 1 || n > 16) return (size_t)-1;
  if (inv_pipe(n)) return plan_ws(n, 1ull << n);
  return pad_copy_bytes(n) + reconstruct_workspace_bytes(n);
}

ptdr_status ptdr_reconstruct_matrix_layout_async(const ptdr_c128* M, int n, ptdr_c128* A, void* workspace,
                                                 size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  if (n < 1 || n > 16) return fail(PTDR_EINVAL, "invalid n (1..16)");
  if (!M || !A || ((uintptr_t)M & 15) || ((uintptr_t)A & 15)) return fail(PTDR_EINVAL, "null or misaligned pointer");
  const size_t need = ptdr_reconstruct_matrix_layout_workspace_bytes(n);
  if (!workspace || ((uintptr_t)workspace & 255)) return fail(PTDR_EINVAL, "workspace missing or not 256-byte aligned");
  if (ws_bytes < need) return fail(PTDR_ENOMEM, "workspace too small");
  const size_t nb = (size_t)16 << (2 * n);
  if (M != A && overlaps(M, nb, A, nb)) return fail(PTDR_EUNSUPPORTED, "A partially overlaps M (in place needs A == M)");
  if (overlaps(workspace, need, A, nb) || overlaps(workspace, need, M, nb))
    return fail(PTDR_EINVAL, "workspace overlaps M or A");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double2* m = reinterpret_cast<const double2*>(M);
  double2* a_out = reinterpret_cast<double2*>(A);
  int nl = 0;
  if (inv_pipe(n)) {
    const ptdr_status r = run_inverse_pipe(MODE_INV, m, n, a_out, workspace, st, &nl);
    g_last_launches = nl;
    return r;
  }
  double2* Q = reinterpret_cast<double2*>(workspace);
  const uint64_t total = 1ull << (2 * n);
  uint64_t g = (total + 255) / 256;
  if (g > (uint64_t)device_sm_count() * 16) g = (uint64_t)device_sm_count() * 16;
  matrix_layout_to_q_kernel<<<(unsigned)g, 256, 0, st>>>(m, n, Q);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "layout kernel launch");
  e = launch_reconstruct(Q, n, a_out, reinterpret_cast<char*>(workspace) + pad_copy_bytes(n), st, &nl);
  g_last_launches = 1 + nl;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "reconstruct launch");
}

// ---- selected coefficients (Algorithm 2 per string) ------------------------------------
ptdr_status ptdr_coefficients_async(const ptdr_c128* A, int n, const uint64_t* qs, uint64_t count,
                                    ptdr_c128* out, void* stream) {
  g_last_launches = 0;
  if (n < 1 || n > 16) return fail(PTDR_EINVAL, "invalid n (1..16)");
  if (count == 0) return PTDR_OK;
  if (!A || !qs || !out) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)A & 15) || ((uintptr_t)out & 15) || ((uintptr_t)qs & 7)) return fail(PTDR_EINVAL, "misaligned");
  cudaError_t e = launch_coeffs(reinterpret_cast<const double2*>(A), n, 0, 1, qs, count,
                                reinterpret_cast<double2*>(out), reinterpret_cast<cudaStream_t>(stream));
  g_last_launches = 1;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "coefficients launch");
}

ptdr_status ptdr_coefficients_xshard_async(const ptdr_c128* A_local, int n, int rank, int world, const uint64_t* qs,
                                           uint64_t count, ptdr_c128* out, void* stream) {
  g_last_launches = 0;
  if (n < 1 || n > 16) return fail(PTDR_EINVAL, "invalid n (1..16)");
  if (world < 1 || (world & (world - 1)) || (uint64_t)world > (1ull << n)) return fail(PTDR_EINVAL, "invalid world");
  if (rank < 0 || rank >= world) return fail(PTDR_EINVAL, "rank out of range");
  if (count == 0) return PTDR_OK;
  if (!A_local || !qs || !out) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)A_local & 15) || ((uintptr_t)out & 15) || ((uintptr_t)qs & 7)) return fail(PTDR_EINVAL, "misaligned");
  cudaError_t e = launch_coeffs(reinterpret_cast<const double2*>(A_local), n, rank, world, qs, count,
                                reinterpret_cast<double2*>(out), reinterpret_cast<cudaStream_t>(stream));
  g_last_launches = 1;
  return e == cudaSuccess ? PTDR_OK : cuda_fail(e, "coefficients launch");
}

// ---- batched small matrices -----------------------------------------------------------
ptdr_status ptdr_decompose_batched_async(const ptdr_c128* A, int n, int structure, uint64_t batch,
                                         ptdr_c128* out, void* stream) {
  g_last_launches = 0;
  if (!is_dense(structure)) return fail(PTDR_EINVAL, "batched decomposition is for the dense structures");
  if (n < 1 || n > kSingleMax) return fail(PTDR_EINVAL, "batched decomposition needs 1 <= n <= 10");
  if (batch == 0) return PTDR_OK;  // empty batch: nothing to read or write (pointers may be null)
  if (!A || !out) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)A & 15) || ((uintptr_t)out & 15)) return fail(PTDR_EINVAL, "misaligned pointer");
  const size_t bytes = ((size_t)16 << (2 * n)) * batch;
  if (overlaps(A, bytes, out, bytes)) return fail(PTDR_EUNSUPPORTED, "out overlaps A");
  {
    // every launch of the call must be a direct or whole-vector kernel (no workspace)
    const uint64_t N = 1ull << n;
    bool two_phase;
    if (structure == PTDR_GENERAL || n <= 8) {
      const int mode = structure == PTDR_GENERAL ? MODE_GENERAL
                       : structure == PTDR_HERMITIAN ? MODE_HERM_MIRROR : MODE_SYM_MIRROR;
      two_phase = plan_for(mode, n, N).kind == 2;
    } else {
      const int hmode = structure == PTDR_HERMITIAN ? MODE_HERM_HALF : MODE_SYM_HALF;
      const uint64_t w = herm_mirror_width(n, hmode);
      two_phase = plan_for(MODE_HERM_MIRROR, n, w).kind == 2 || plan_for(hmode, n - 1, N - w).kind == 2;
    }
    if (two_phase) return fail(PTDR_EUNSUPPORTED, "this n would need the two-phase pipeline");
  }
  int nl = 0;
  ptdr_status r = run_dense(reinterpret_cast<const double2*>(A), n, structure, reinterpret_cast<double2*>(out), nullptr,
                            reinterpret_cast<cudaStream_t>(stream), &nl, 0, 0, batch);
  g_last_launches = nl;
  return r;
}

ptdr_status ptdr_decompose(const ptdr_c128* A, int n, int structure, ptdr_c128* out) {
  if (!valid_n(n, structure)) return fail(PTDR_EINVAL, "invalid n or structure");
  const size_t need = ptdr_workspace_bytes(n, structure, 1);
  void* ws = nullptr;
  cudaError_t e;
  if (need > 0 && (e = cudaMalloc(&ws, need)) != cudaSuccess) {
    cudaGetLastError();
    return fail(PTDR_ENOMEM, std::string("cudaMalloc workspace: ") + cudaGetErrorString(e));
  }
  ptdr_status r = ptdr_decompose_async(A, n, structure, out, ws, need, nullptr);
  const int nl = g_last_launches;
  e = cudaDeviceSynchronize();
  if (ws) cudaFree(ws);
  g_last_launches = nl;
  if (r != PTDR_OK) return r;
  if (e != cudaSuccess) return cuda_fail(e, "ptdr_decompose sync");
  return PTDR_OK;
}

ptdr_status ptdr_decompose_host(const ptdr_c128* A_host, int n, int structure,
                                ptdr_c128* out_host) {
  if (!valid_n(n, structure)) return fail(PTDR_EINVAL, "invalid n or structure");
  if (!A_host || !out_host) return fail(PTDR_EINVAL, "null host pointer");
  const size_t inb = ptdr_input_count(n, structure) * 16;
  const size_t outb = ptdr_output_count(n, structure) * 16;
  const size_t need = ptdr_workspace_bytes(n, structure, 1);
  cudaStream_t st;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
  void *dA = nullptr, *dO = nullptr, *ws = nullptr;
  ptdr_status r = PTDR_OK;
  int nl = 0;
  do {
    if ((e = cudaMallocAsync(&dA, inb, st)) != cudaSuccess ||
        (e = cudaMallocAsync(&dO, outb, st)) != cudaSuccess ||
        (need > 0 && (e = cudaMallocAsync(&ws, need, st)) != cudaSuccess)) {
      r = fail(PTDR_ENOMEM, std::string("device allocation: ") + cudaGetErrorString(e));
      cudaGetLastError();
      break;
    }
    if ((e = cudaMemcpyAsync(dA, A_host, inb, cudaMemcpyHostToDevice, st)) != cudaSuccess) {
      r = cuda_fail(e, "H2D copy");
      break;
    }
    r = ptdr_decompose_async(reinterpret_cast<const ptdr_c128*>(dA), n, structure,
                             reinterpret_cast<ptdr_c128*>(dO), ws, need, st);
    nl = g_last_launches;
    if (r != PTDR_OK) break;
    if ((e = cudaMemcpyAsync(out_host, dO, outb, cudaMemcpyDeviceToHost, st)) != cudaSuccess) {
      r = cuda_fail(e, "D2H copy");
      break;
    }
  } while (0);
  if (dA) cudaFreeAsync(dA, st);
  if (dO) cudaFreeAsync(dO, st);
  if (ws) cudaFreeAsync(ws, st);
  e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  g_last_launches = nl;
  if (r == PTDR_OK && e != cudaSuccess) r = cuda_fail(e, "ptdr_decompose_host sync");
  return r;
}

size_t ptdr_fro2_partial_count(void) { return (size_t)fro2_partial_count(); }

static bool fro2_ok(const double* p) { return p == nullptr || ((uintptr_t)p & 7) == 0; }

ptdr_status ptdr_generate_dense_async(int n, uint64_t seed, int variant, uint64_t row0,
                                      uint64_t nrows, ptdr_c128* A, double* fro2_partials, void* stream) {
  g_last_launches = 0;
  if (n < 1 || n > 16 || variant < 0 || variant > 2) return fail(PTDR_EINVAL, "invalid n or variant");
  if (!A || ((uintptr_t)A & 15)) return fail(PTDR_EINVAL, "null or misaligned A");
  if (!fro2_ok(fro2_partials)) return fail(PTDR_EINVAL, "misaligned fro2_partials");
  if (row0 + nrows > (1ull << n)) return fail(PTDR_EINVAL, "rows out of range");
  cudaError_t e = launch_generate_dense(n, seed, variant, row0, nrows, reinterpret_cast<double2*>(A),
                                        fro2_partials, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "generator launch");
  g_last_launches = nrows ? 1 : 0;
  return PTDR_OK;
}

ptdr_status ptdr_generate_band_async(int n, uint64_t seed, int variant, ptdr_c128* band,
                                     double* fro2_partials, void* stream) {
  g_last_launches = 0;
  if (n < 1 || n > 28 || (variant != 3 && variant != 4 && variant != 6)) return fail(PTDR_EINVAL, "invalid n or variant");
  if (!band || ((uintptr_t)band & 15)) return fail(PTDR_EINVAL, "null or misaligned band");
  if (!fro2_ok(fro2_partials)) return fail(PTDR_EINVAL, "misaligned fro2_partials");
  cudaError_t e = launch_generate_band(n, seed, variant, reinterpret_cast<double2*>(band), fro2_partials,
                                       reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "generator launch");
  g_last_launches = 1;
  return PTDR_OK;
}

ptdr_status ptdr_generate_sendblocks_async(int n, uint64_t seed, int rank, int world, int subranges,
                                           ptdr_c128* send, double* fro2_partials, void* stream) {
  g_last_launches = 0;
  if (n < 1 || n > 16 || world < 1 || (world & (world - 1)) || rank < 0 || rank >= world ||
      (uint64_t)world > (1ull << n))
    return fail(PTDR_EINVAL, "invalid n / rank / world");
  if (subranges < 1 || (subranges & (subranges - 1)) || (uint64_t)world * (uint64_t)subranges > (1ull << n))
    return fail(PTDR_EINVAL, "subranges must be a power of two with world * subranges <= 2^n");
  if (!send || ((uintptr_t)send & 15)) return fail(PTDR_EINVAL, "null or misaligned send buffer");
  if (!fro2_ok(fro2_partials)) return fail(PTDR_EINVAL, "misaligned fro2_partials");
  cudaError_t e = launch_generate_sendblocks(n, seed, rank, world, subranges, reinterpret_cast<double2*>(send),
                                             fro2_partials, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "generator launch");
  g_last_launches = 1;
  return PTDR_OK;
}

ptdr_status ptdr_sumsq_async(const ptdr_c128* x, uint64_t count, double* partials, void* stream) {
  g_last_launches = 0;
  if ((!x && count) || !partials) return fail(PTDR_EINVAL, "null pointer");
  if (((uintptr_t)x & 15) || ((uintptr_t)partials & 7)) return fail(PTDR_EINVAL, "misaligned pointer");
  cudaError_t e = launch_sumsq(reinterpret_cast<const double2*>(x), count, partials,
                               reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "sumsq launch");
  g_last_launches = count ? 1 : 0;
  return PTDR_OK;
}

}  // extern "C"
