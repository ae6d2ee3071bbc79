// plan.cu -- host-memory streaming plan (include/ptdr.h, "Host plans").
//
// A plan owns `depth` slots of device buffers (A, out, workspace) for one (n, structure)
// and three streams: host->device copies, kernels, device->host copies.  Call k uses slot
// k % depth; its H2D waits for the slot's previous D2H, its kernels wait for its H2D, its
// D2H waits for its kernels.  With depth 2 the H2D of call k+1 overlaps the D2H of call k
// (PCIe is full duplex), so a stream of matrices moves at the bidirectional copy rate.
// Every step of the decomposition runs in the kernels behind ptdr_decompose_async.
#include <cuda_runtime.h>

#include <new>
#include <string>

#include "../../include/ptdr.h"

namespace ptdr {
ptdr_status plan_fail(ptdr_status s, const char* msg);
ptdr_status plan_cuda_fail(cudaError_t e, const char* where);
}  // namespace ptdr

using ptdr::plan_cuda_fail;
using ptdr::plan_fail;

constexpr int kMaxDepth = 4;

struct ptdr_plan_s {
  int n = 0, structure = 0, depth = 0, device = 0;
  size_t in_bytes = 0, out_bytes = 0, ws_bytes = 0;
  void* dA[kMaxDepth] = {};
  void* dO[kMaxDepth] = {};
  void* ws[kMaxDepth] = {};
  cudaEvent_t h2d_done[kMaxDepth] = {}, comp_done[kMaxDepth] = {}, d2h_done[kMaxDepth] = {};
  bool slot_used[kMaxDepth] = {};
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  unsigned long long calls = 0;
  int launches = 0;
};

static void plan_release(ptdr_plan_s* p) {
  for (int s = 0; s < kMaxDepth; ++s) {
    if (p->dA[s]) cudaFree(p->dA[s]);
    if (p->dO[s]) cudaFree(p->dO[s]);
    if (p->ws[s]) cudaFree(p->ws[s]);
    if (p->h2d_done[s]) cudaEventDestroy(p->h2d_done[s]);
    if (p->comp_done[s]) cudaEventDestroy(p->comp_done[s]);
    if (p->d2h_done[s]) cudaEventDestroy(p->d2h_done[s]);
  }
  if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
  if (p->s_comp) cudaStreamDestroy(p->s_comp);
  if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
  delete p;
}

extern "C" {

ptdr_status ptdr_plan_create(int n, int structure, int depth, ptdr_plan* out_plan) {
  if (!out_plan) return plan_fail(PTDR_EINVAL, "null plan pointer");
  *out_plan = nullptr;
  if (depth < 1 || depth > kMaxDepth) return plan_fail(PTDR_EINVAL, "depth must be in [1, 4]");
  const size_t in_count = ptdr_input_count(n, structure);
  if (in_count == 0) return plan_fail(PTDR_EINVAL, "invalid n or structure");
  ptdr_plan_s* p = new (std::nothrow) ptdr_plan_s;
  if (!p) return plan_fail(PTDR_ENOMEM, "host allocation of the plan");
  p->n = n;
  p->structure = structure;
  p->depth = depth;
  p->in_bytes = in_count * 16;
  p->out_bytes = ptdr_output_count(n, structure) * 16;
  p->ws_bytes = ptdr_workspace_bytes(n, structure, 1);
  cudaError_t e = cudaGetDevice(&p->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_comp, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking);
  for (int s = 0; s < depth && e == cudaSuccess; ++s) {
    e = cudaMalloc(&p->dA[s], p->in_bytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->dO[s], p->out_bytes);
    if (e == cudaSuccess && p->ws_bytes > 0) e = cudaMalloc(&p->ws[s], p->ws_bytes);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->h2d_done[s], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->comp_done[s], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->d2h_done[s], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    plan_release(p);
    return e == cudaErrorMemoryAllocation ? plan_fail(PTDR_ENOMEM, "device allocation of the plan buffers")
                                          : plan_cuda_fail(e, "ptdr_plan_create");
  }
  *out_plan = p;
  return PTDR_OK;
}

ptdr_status ptdr_plan_decompose_host_async(ptdr_plan p, const ptdr_c128* A_host, ptdr_c128* out_host) {
  if (!p) return plan_fail(PTDR_EINVAL, "null plan");
  if (!A_host || !out_host) return plan_fail(PTDR_EINVAL, "null host pointer");
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != p->device)
    return plan_fail(PTDR_EINVAL, "plan used on a device other than the one it was created on");
  const int s = (int)(p->calls % (unsigned long long)p->depth);
  cudaError_t e = cudaSuccess;
  // the slot's buffers are free once its previous D2H has finished
  if (p->slot_used[s]) e = cudaStreamWaitEvent(p->s_h2d, p->d2h_done[s], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(p->dA[s], A_host, p->in_bytes, cudaMemcpyHostToDevice, p->s_h2d);
  if (e == cudaSuccess) e = cudaEventRecord(p->h2d_done[s], p->s_h2d);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_comp, p->h2d_done[s], 0);
  if (e != cudaSuccess) return plan_cuda_fail(e, "plan H2D");
  ptdr_status r = ptdr_decompose_async(reinterpret_cast<const ptdr_c128*>(p->dA[s]), p->n, p->structure,
                                       reinterpret_cast<ptdr_c128*>(p->dO[s]), p->ws[s], p->ws_bytes,
                                       p->s_comp);
  if (r != PTDR_OK) return r;
  p->launches = ptdr_last_launch_count();
  e = cudaEventRecord(p->comp_done[s], p->s_comp);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_d2h, p->comp_done[s], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_host, p->dO[s], p->out_bytes, cudaMemcpyDeviceToHost, p->s_d2h);
  if (e == cudaSuccess) e = cudaEventRecord(p->d2h_done[s], p->s_d2h);
  if (e != cudaSuccess) return plan_cuda_fail(e, "plan D2H");
  p->slot_used[s] = true;
  ++p->calls;
  return PTDR_OK;
}

ptdr_status ptdr_plan_wait(ptdr_plan p) {
  if (!p) return plan_fail(PTDR_EINVAL, "null plan");
  cudaError_t e = cudaStreamSynchronize(p->s_h2d);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->s_comp);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->s_d2h);
  if (e != cudaSuccess) return plan_cuda_fail(e, "ptdr_plan_wait");
  return PTDR_OK;
}

int ptdr_plan_launch_count(ptdr_plan p) { return p ? p->launches : 0; }

ptdr_status ptdr_plan_destroy(ptdr_plan p) {
  if (!p) return PTDR_OK;
  cudaError_t e = cudaStreamSynchronize(p->s_h2d);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->s_comp);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->s_d2h);
  plan_release(p);
  if (e != cudaSuccess) return plan_cuda_fail(e, "ptdr_plan_destroy");
  return PTDR_OK;
}

}  // extern "C"
