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
  int pipe_cfg = 0;    // 0: dense_impl.cuh kernels; else a dense_pipe.cu configuration
  uint64_t nchunks = 0;
  uint64_t slot_elems = 0;  // complex128 elements per scratch slot
  size_t ctr_bytes = 0;
  size_t scratch_bytes = 0;
  size_t ws_bytes() const { return ctr_bytes + scratch_bytes; }
};

// dense_pipe.cu configurations: tile 2^LT elements, GW warps per group, NG groups, NS stages.
enum { kPipeNone = 0, kPipeCfg12 = 1 /* 12,8,2,3 */, kPipeCfg11x4 = 2 /* 11,4,4,6 */,
       kPipeCfg11x3 = 3 /* 11,4,3,6 */ };
inline int pipe_lt(int cfg) { return cfg == kPipeCfg12 ? 12 : 11; }
inline int pipe_stages(int cfg) { return cfg == kPipeCfg12 ? 3 : 6; }

// Tiles resident at once on a B200 (fixes L deterministically, independent of the device).
constexpr int kNominalSMs = 148;
constexpr int kNominalResidentCtas = 296;          // v1: 148 SMs x 2 CTAs
constexpr uint64_t kPipeScratchBudget = 2ull << 30;  // bytes of scratch slots for the pipeline

// pipe_cfg: requested dense_pipe.cu configuration (0 = v1 kernels).  Falls back to v1 when
// the phase split does not fit the configuration (M = nv - (LT-4) must be in [4, 8]).
inline DensePlan make_dense_plan(int nv, uint64_t nchunks, int pipe_cfg = kPipeNone) {
  DensePlan p;
  p.nv = nv;
  p.nchunks = nchunks;
  if (nv <= 5) { p.kind = 0; return p; }
  if (nv <= 7) { p.kind = 1; p.R = nv; p.M = 0; return p; }
  p.kind = 2;
  if (pipe_cfg != kPipeNone) {
    const int R = pipe_lt(pipe_cfg) - 4;
    if (nv - R < 4 || nv - R > 8) pipe_cfg = kPipeNone;
  }
  p.pipe_cfg = pipe_cfg;
  int resident;
  if (pipe_cfg != kPipeNone) {
    p.R = pipe_lt(pipe_cfg) - 4;
    p.M = nv - p.R;
    resident = kNominalSMs * pipe_stages(pipe_cfg);
  } else {
    if (nv <= 11) { p.R = nv - 4; p.M = 4; }
    else { p.R = 8; p.M = nv - 8; }
    resident = kNominalResidentCtas;
  }
  p.NA = 1 << p.M;
  p.NB = 1 << p.M;
  const int period = p.NA + p.NB;
  int L = (3 * resident + 2 * period - 1) / (2 * period);  // ceil(1.5*resident/period)
  if (L < 1) L = 1;
  if (L > 64) L = 64;
  p.L = L;
  // Scratch slots.  A phase-A tile of chunk c waits until phase B of chunk c - nslot has
  // drained the slot; with ~`resident` tickets in flight that wait is rare only if
  // nslot >= L + 1 + resident/period.  The pipeline takes many more slots (capped by a
  // byte budget): consumed slots are discarded from L2, so only the live ~L chunks occupy
  // L2 and the extra slots cost HBM capacity, not bandwidth.
  uint64_t ns = (uint64_t)L + 2;
  if (pipe_cfg != kPipeNone) {
    const uint64_t slot_bytes = ((uint64_t)16 << nv) * 16;
    uint64_t budget = kPipeScratchBudget / slot_bytes;
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
