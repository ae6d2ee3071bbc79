// dense_pipe.cu -- host side of the dense pipeline kernel (dense_pipe.cuh): tensor map,
// configuration dispatch and the debug timeline buffer.  Kernel instantiations live in
// dense_pipe_c<k>.cu (one configuration per translation unit).
#include "dense_pipe.cuh"

namespace ptdr {

cudaError_t pipe_cfg1(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st);
cudaError_t pipe_cfg4(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st);
#if PTDR_DEV
// developer-only configurations (dense_plan.h pipe_cfg_built; DESIGN.md section 7 sweeps)
cudaError_t pipe_cfg2(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st);
cudaError_t pipe_cfg3(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st);
cudaError_t pipe_cfg5(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st);
cudaError_t pipe_cfg6(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st);
cudaError_t pipe_cfg7(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st);
cudaError_t pipe_cfg8(int mode, const TmapSet& map, const DenseArgs& a, int M, cudaStream_t st);
#endif

#if PTDR_ENABLE_TRACE
static unsigned long long* g_trace = nullptr;
static unsigned long long* debug_trace_buffer() {
  // developer timeline (trace build, PTDR_TRACE=1): allocated once, thread-safe
  static std::once_flag once;
  std::call_once(once, []() {
    const char* e = getenv("PTDR_TRACE");
    if (e && e[0] == '1' && cudaMalloc(&g_trace, (size_t)kTraceTiles * 16 * 8) != cudaSuccess) g_trace = nullptr;
  });
  return g_trace;
}
int debug_trace_copy(void* host, size_t bytes) {
  if (!g_trace) return -1;
  const size_t n = bytes < (size_t)kTraceTiles * 16 * 8 ? bytes : (size_t)kTraceTiles * 16 * 8;
  if (cudaDeviceSynchronize() != cudaSuccess) return -2;
  return cudaMemcpy(host, g_trace, n, cudaMemcpyDeviceToHost) == cudaSuccess ? (int)n : -3;
}
#else
static unsigned long long* debug_trace_buffer() { return nullptr; }
int debug_trace_copy(void*, size_t) { return -1; }
#endif
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

cudaError_t launch_dense_pipe(int mode, const DenseArgs& a_in, const DensePlan& p, cudaStream_t st,
                              int* nlaunch) {
  if (p.kind != 2 || p.pipe_cfg == 0) return cudaErrorInvalidValue;
  DenseArgs a = a_in;
  a.L = p.L;
#if PTDR_DEV
  {
    // developer override of the look-ahead.  Liveness needs L + 1 <= nslot (phase A of
    // chunk c waits for phase B of chunk c - nslot, whose tickets follow A(c - nslot + L + 1)),
    // so the override is clamped to nslot - 1.
    const char* el = getenv("PTDR_L");
    if (el && atoi(el) > 0) a.L = atoi(el);
    if (a.L > p.nslot - 1) a.L = p.nslot - 1 > 1 ? p.nslot - 1 : 1;
  }
#endif
  a.nslot = p.nslot;
#if PTDR_DEV
  {
    // developer override of the scratch ring (a power of two <= the planned slots; the
    // workspace holds p.nslot slots): a short ring reuses L2-resident lines
    const char* es = getenv("PTDR_NSLOT");
    const int v = es ? atoi(es) : 0;
    if (v >= 2 && v <= p.nslot && (v & (v - 1)) == 0) a.nslot = v;
    if (a.L > a.nslot - 1) a.L = a.nslot - 1;
  }
#endif
  a.slot_elems = p.slot_elems;
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  TmapSet map;
  const cuuint32_t W = (cuuint32_t)p.W;
  cuuint32_t box[2] = {2 * W, W};  // W complex128 x W rows
  cuuint32_t estr[2] = {1, 1};
  auto encode = [&](CUtensorMap* m, const double2* base, cuuint64_t ncols, cuuint64_t nrows) {
    cuuint64_t gdim[2] = {2 * ncols, nrows};
    cuuint64_t gstride[1] = {a.ld * 16};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(base), gdim, gstride, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUresult r = CUDA_SUCCESS;
  if (mode == MODE_INVQ) {
    // q-ordered coefficients viewed as [4^n / 8 rows][8 complex128 = 128 B]: a box of W^2
    // consecutive q is W^2 / 8 rows; the 128-byte swizzle spreads a phase-A read (16 lanes
    // along the X-mask, fixed z) over all eight 16-byte slots of a bank row
    if (W * W % 8 != 0) return cudaErrorInvalidValue;
    const cuuint64_t rows = (1ull << (2 * a.n)) / 8ull;
    cuuint64_t gdim[2] = {16, rows};
    cuuint64_t gstride[1] = {128};
    cuuint32_t qbox[2] = {16, W * W / 8};
    r = enc(&map.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(a.A), gdim, gstride, qbox, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (a.peer_shift) {
    // peer-pull: one map per rank's row-block shard [R rows][2^n columns] (row pitch a.ld)
    if (a.npeers < 1 || a.npeers > kMaxPeers) return cudaErrorInvalidValue;
    for (int g = 0; g < a.npeers && r == CUDA_SUCCESS; ++g)
      r = encode(&map.m[g], a.peer_ptrs[g], a.colmask + 1, a.peer_rowmask + 1);
  } else {
    // zero padding: the tensor map covers only the stored rows_valid x
    // cols_valid block; TMA fills every out-of-bounds element of a box with zeros.
    const cuuint64_t ncols = a.cols_valid ? a.cols_valid : a.colmask + 1;
    const cuuint64_t nrows = a.rows_valid ? a.rows_valid : 1ull << a.n;
    r = encode(&map.m[0], a.A, ncols, nrows);
  }
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  {
    // L2 policies of A loads / scratch stores / scratch loads: f n n, measured (DESIGN.md
    // section 7): scratch stores with evict_normal beat evict_last by ~3 % (8.02-8.09 vs
    // 8.31-8.34 ms at n = 15); A must stay evict_first.  Consumed scratch lines are
    // discarded from L2.
    a.discard = 1;
    a.pol_a = 0;
    a.pol_s = 1;
    a.pol_b = 1;
#if PTDR_DEV
    // developer overrides: PTDR_NO_DISCARD=1, PTDR_POL = three letters of f n l u
    // (evict_first / normal / last / unchanged)
    const char* nd = getenv("PTDR_NO_DISCARD");
    if (nd && nd[0] == '1') a.discard = 0;
    const char* pe = getenv("PTDR_POL");
    if (pe && strlen(pe) >= 3) {
      auto code = [](char c) { return c == 'n' ? 1 : c == 'l' ? 2 : c == 'u' ? 3 : 0; };
      a.pol_a = code(pe[0]);
      a.pol_s = code(pe[1]);
      a.pol_b = code(pe[2]);
    }
#endif
  }
  // Acquire side of the dependency waits: the producer reads the completion
  // counters with ld.acquire.gpu, which synchronises with the signalers' red.release, then
  // fence.proxy.async orders the async-proxy bulk copy of the scratch after it.  Measured
  // (DESIGN.md section 7): free at n = 15/16 (7.84-7.93 vs 7.99-8.08 ms relaxed), while a
  // fence.acq_rel.gpu after each wait costs 10 %; developer builds can switch between the
  // forms (PTDR_ACQ = 0 relaxed, 1 fence, 2 ld.acquire).
  a.acq_fence = 2;
#if PTDR_DEV
  {
    const char* ea = getenv("PTDR_ACQ");
    if (ea && ea[0] >= '0' && ea[0] <= '2') a.acq_fence = ea[0] - '0';
  }
#endif
  cudaError_t e = cudaMemsetAsync(a.ctr, 0, p.ctr_bytes, st);
  if (e != cudaSuccess) return e;
  a.trace = debug_trace_buffer();
  if (a.trace) {
    e = cudaMemsetAsync(a.trace, 0, (size_t)kTraceTiles * 16 * 8, st);
    if (e != cudaSuccess) return e;
  }
  *nlaunch += 1;
  switch (p.pipe_cfg) {
    case 1: return pipe_cfg1(mode, map, a, p.M, st);
    case 4: return pipe_cfg4(mode, map, a, p.M, st);
#if PTDR_DEV
    case 2: return pipe_cfg2(mode, map, a, p.M, st);
    case 3: return pipe_cfg3(mode, map, a, p.M, st);
    case 5: return pipe_cfg5(mode, map, a, p.M, st);
    case 6: return pipe_cfg6(mode, map, a, p.M, st);
    case 7: return pipe_cfg7(mode, map, a, p.M, st);
    case 8: return pipe_cfg8(mode, map, a, p.M, st);
#endif
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ptdr
