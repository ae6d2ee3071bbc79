// dense_plan.h -- host-side tiling plan of the dense (GENERAL / HERMITIAN /
// REAL_SYMMETRIC) path.  Pure integer arithmetic shared by the launcher and by
// ptdr_workspace_bytes() so that the workspace size is a deterministic function
// of (n, structure, world).
#pragma once
#include <cstddef>
#include <cstdint>

namespace ptdr {

// nv = number of index bits of the transformed vectors (n, or n-1 for the
// half-length Hermitian/real-symmetric vectors).
//   nv <= 5   : direct kernel (one thread per coefficient)
//   nv in 6,7 : single-phase tiles (whole vector in one tile)
//   nv >= 8   : two phases: phase A transforms the low R index bits (gather fused),
//               phase B the high M bits (+ epilogue); x-chunks of 16 X-masks flow
//               through an L2-resident scratch ring of `nslot` chunk slots.
struct DensePlan {
  int nv = 0;
  int kind = 0;        // 0 direct, 1 single, 2 two-phase
  int R = 0, M = 0;    // bits in phase A / phase B
  int NA = 0, NB = 0;  // tiles per chunk in phase A / B (two-phase)
  int L = 0;           // look-ahead (chunks of phase A issued ahead of phase B)
  int nslot = 0;       // scratch ring slots
  uint64_t nchunks = 0;
  uint64_t slot_elems = 0;  // complex128 elements per scratch slot
  size_t ctr_bytes = 0;
  size_t scratch_bytes = 0;
  size_t ws_bytes() const { return ctr_bytes + scratch_bytes; }
};

constexpr int kNominalResidentCtas = 296;  // 148 SMs x 2 CTAs; fixes L deterministically

inline DensePlan make_dense_plan(int nv, uint64_t nchunks) {
  DensePlan p;
  p.nv = nv;
  p.nchunks = nchunks;
  if (nv <= 5) { p.kind = 0; return p; }
  if (nv <= 7) { p.kind = 1; p.R = nv; p.M = 0; return p; }
  p.kind = 2;
  if (nv <= 11) { p.R = nv - 4; p.M = 4; }
  else { p.R = 8; p.M = nv - 8; }
  p.NA = 1 << (nv - 8);
  p.NB = 1 << (nv - 8);
  int period = p.NA + p.NB;
  int L = (3 * kNominalResidentCtas + 2 * period - 1) / (2 * period);  // ceil(1.5*ctas/period)
  if (L < 1) L = 1;
  if (L > 64) L = 64;
  p.L = L;
  uint64_t ns = (uint64_t)L + 2;
  if (ns > nchunks) ns = nchunks;
  p.nslot = (int)ns;
  p.slot_elems = (uint64_t)16 << nv;
  p.ctr_bytes = ((4 * (1 + 2 * nchunks)) + 255) / 256 * 256;
  p.scratch_bytes = (size_t)p.nslot * p.slot_elems * 16;
  return p;
}

}  // namespace ptdr
