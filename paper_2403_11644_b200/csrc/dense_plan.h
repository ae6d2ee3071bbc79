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
  bool v2 = false;     // warp-specialised TMA kernel (dense_v2.cu) instead of dense_impl.cuh
  uint64_t nchunks = 0;
  uint64_t slot_elems = 0;  // complex128 elements per scratch slot
  size_t ctr_bytes = 0;
  size_t scratch_bytes = 0;
  size_t ws_bytes() const { return ctr_bytes + scratch_bytes; }
};

// Tiles resident at once on a B200 (fixes L deterministically, independent of the device):
// v1 = 148 SMs x 2 CTAs; v2 = 148 SMs x 3 pipeline stages.
constexpr int kNominalResidentCtas = 296;
constexpr int kNominalResidentV2 = 592;  // 148 SMs x (3 stages + 1 ticket claimed ahead)
constexpr uint64_t kV2ScratchBudget = 2ull << 30;  // bytes of scratch slots for the v2 kernel

// v2_ok: the caller's MODE can run on the TMA kernel (GENERAL or half-length modes).
inline DensePlan make_dense_plan(int nv, uint64_t nchunks, bool v2_ok = false) {
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
  p.v2 = v2_ok && p.R == 8;
  const int resident = p.v2 ? kNominalResidentV2 : kNominalResidentCtas;
  int period = p.NA + p.NB;
  int L = (3 * resident + 2 * period - 1) / (2 * period);  // ceil(1.5*resident/period)
  if (L < 1) L = 1;
  if (L > 64) L = 64;
  p.L = L;
  // Scratch slots.  A phase-A tile of chunk c waits until phase B of chunk c - nslot has
  // drained the slot; with ~`resident` tickets in flight that wait is rare only if
  // nslot >= L + 1 + resident/period.  v2 takes many more slots (capped by a byte budget):
  // consumed slots are discarded from L2, so only the live ~L chunks occupy L2 and the
  // extra slots cost HBM capacity, not bandwidth.
  uint64_t ns = (uint64_t)L + 2;
  if (p.v2) {
    const uint64_t slot_bytes = ((uint64_t)16 << nv) * 16;
    uint64_t budget = kV2ScratchBudget / slot_bytes;
    const uint64_t need = 2ull * (uint64_t)L + 2ull + (uint64_t)(resident / period);
    if (budget < need) budget = need;
    ns = budget;
  }
  if (ns > nchunks) ns = nchunks;
  p.nslot = (int)ns;
  p.slot_elems = (uint64_t)16 << nv;
  p.ctr_bytes = ((4 * (1 + 2 * nchunks)) + 255) / 256 * 256;
  p.scratch_bytes = (size_t)p.nslot * p.slot_elems * 16;
  return p;
}

}  // namespace ptdr
