// internal.h -- declarations shared by the translation units of libptdr.so.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ptdr {

struct DenseArgs;
struct DensePlan;

int device_sm_count();  // SMs of the current device (cached per device)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `fn` on the current device, once per
// (function, device), thread-safe (a function attribute is per device context).
cudaError_t ensure_smem_attr(const void* fn, int bytes);

cudaError_t launch_dense_mode0(const DenseArgs& a, const DensePlan& p, cudaStream_t st, int* nl);
cudaError_t launch_dense_mode1(const DenseArgs& a, const DensePlan& p, cudaStream_t st, int* nl);
cudaError_t launch_dense_mode2(const DenseArgs& a, const DensePlan& p, cudaStream_t st, int* nl);
cudaError_t launch_dense_mode3(const DenseArgs& a, const DensePlan& p, cudaStream_t st, int* nl);
cudaError_t launch_dense_mode4(const DenseArgs& a, const DensePlan& p, cudaStream_t st, int* nl);

cudaError_t launch_dense_pipe(int mode, const DenseArgs& a, const DensePlan& p, cudaStream_t st,
                              int* nl);

int debug_trace_copy(void* host, size_t bytes);

// band paths (band.cu)
size_t band_workspace_bytes(int n, int structure, int world);
cudaError_t launch_band(const double2* A, double2* out, int n, int structure, void* ws, int rank,
                        int world, cudaStream_t st, int* nl);

// BAND(s) (band.cu)
size_t band_s_xmask_count(int n, int s);
int band_s_xmasks(int n, int s, unsigned long long* xs, size_t cap);
size_t band_s_workspace_bytes(int n, int s);
cudaError_t launch_band_s(const double2* diags, int n, int s, double2* out, void* ws, cudaStream_t st,
                          int* nl);

// algebra and inverse transform (algebra.cu)
size_t reconstruct_workspace_bytes(int n);
cudaError_t launch_reconstruct(const double2* c, int n, double2* A, void* ws, cudaStream_t st, int* nl);
cudaError_t launch_axpby(double2* out, double2 mu, const double2* x, double2 nu, const double2* y,
                         unsigned long long count, cudaStream_t st);
cudaError_t launch_block_diag(const double2* blocks, int n, int k, double2* out, cudaStream_t st);
cudaError_t launch_herm_augment(const double2* a, int n, double2* out, cudaStream_t st);

// selected coefficients (coeffs.cu)
cudaError_t launch_coeffs(const double2* A, int n, int rank, int world, const uint64_t* qs, uint64_t count,
                          double2* out, cudaStream_t st);

// generators (generate.cu); fro2: nullable device array of fro2_partial_count() doubles
int fro2_partial_count();
cudaError_t launch_generate_dense(int n, uint64_t seed, int variant, uint64_t row0,
                                  uint64_t nrows, double2* A, double* fro2, cudaStream_t st);
cudaError_t launch_generate_band(int n, uint64_t seed, int variant, double2* band, double* fro2,
                                 cudaStream_t st);
cudaError_t launch_generate_sendblocks(int n, uint64_t seed, int rank, int world, int K, double2* send,
                                       double* fro2, cudaStream_t st);
cudaError_t launch_sumsq(const double2* x, uint64_t count, double* partials, cudaStream_t st);

}  // namespace ptdr
