// wht_passes.h -- multi-pass batched Walsh-Hadamard transforms over contiguous vector
// families (band.cu): used by the band paths and the inverse transform (algebra.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ptdr {

// A vector family for the pass planner: `count` contiguous vectors of 2^lam elements.
struct WhtFamily {
  const double2* in;  // input of pass 0
  double2* out;       // output of every pass but the last (later passes in place)
  int lam;
  unsigned long long count;
  double scale;       // applied on the last pass
  double2* final_out = nullptr;  // output of the last pass (nullptr: `out`, in place)
  int zshift = 63;               // slice filter of the last pass (single-vector families)
  unsigned long long zrank = 0;
  unsigned long long px = 0;                    // X-mask phase i^{popcount(px & z)} of the last pass
  int first_bit = 0;             // bits below first_bit are already transformed (a multiple of 8:
                                 //   the family starts at pass first_bit / 8 and never uses the
                                 //   whole-vector tiles)
  unsigned long long zoff = 0;   // z of element 0 of the last pass's output (the px phase uses z)
  int skip_last = 0;             // 1: the last pass runs elsewhere (fused into a consumer kernel)
};

constexpr int kMaxFamilies = 40;  // per run_families call

// Runs every pass of every family (at most 3 launches for vectors of <= 2^24 elements).
cudaError_t run_families(const WhtFamily* fam, int nfam, cudaStream_t st, int* nl);

}  // namespace ptdr
