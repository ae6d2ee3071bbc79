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
//               phase B the high M bits (+ epilogue); x-chunks of W X-masks (16 in the
//               default pipeline configuration) flow through an L2-resident scratch ring
//               of `nslot` chunk slots.
struct DensePlan {
  int nv = 0;
  int kind = 0;        // 0 direct, 1 single, 2 two-phase
  int R = 0, M = 0;    // bits in phase A / phase B
  int NA = 0, NB = 0;  // tiles per chunk in phase A / B (two-phase)
  int L = 0;           // look-ahead (chunks of phase A issued ahead of phase B)
  int nslot = 0;       // scratch ring slots
  int pipe_cfg = 0;    // 0: dense_impl.cuh kernels; else a dense_pipe.cuh configuration
  int W = 16;          // X-masks per chunk
  uint64_t nchunks = 0;
  uint64_t slot_elems = 0;  // complex128 elements per scratch slot
  size_t ctr_bytes = 0;
  size_t scratch_bytes = 0;
  size_t ws_bytes() const { return ctr_bytes + scratch_bytes; }
};

// dense_pipe.cuh configurations (dense_pipe_c<k>.cu): tile 2^LT elements, chunk width 2^XB,
// GW warps per group, NG groups, NS stages, NR exchange rounds (0: in-place exchange in the
// stage; 2/4: early stage release with a per-group exchange buffer of 2^LT/NR elements).
struct PipeGeom {
  int LT, XB, GW, NG, NS, NR;
};
constexpr int kPipeNone = 0;
constexpr int kPipeCfgCount = 8;
// Developer builds (PTDR_DEV=1, build.py) compile every configuration and read the
// PTDR_* environment switches; the product library has configurations 1 and 4 only (the
// default and its n = 11 fallback) and reads no environment variable.
#ifndef PTDR_DEV
#define PTDR_DEV 0
#endif
inline bool pipe_cfg_built(int cfg) { return PTDR_DEV || cfg == kPipeNone || cfg == 1 || cfg == 4; }
inline PipeGeom pipe_geom(int cfg) {
  switch (cfg) {
    case 1: return {12, 4, 8, 2, 3, 0};
    case 2: return {11, 4, 4, 4, 6, 0};
    case 3: return {11, 4, 4, 3, 6, 0};
    case 4: return {12, 5, 8, 2, 3, 0};
    case 5: return {11, 5, 4, 3, 6, 0};
    case 6: return {12, 5, 8, 2, 2, 2};
    case 7: return {11, 4, 4, 4, 4, 2};
    case 8: return {12, 4, 8, 2, 2, 2};
    default: return {0, 4, 0, 0, 0, 0};
  }
}
// Preferred configuration: 16-wide chunks (256 B row windows, 256-row phase-A tiles).  With
// the look-ahead sized by live scratch bytes and evict-normal scratch stores it beats the
// 32-wide configuration 4 by 1-5 % at n = 12..15 and on the Hermitian / real-symmetric
// paths (`profiles/r01/sweep_cfg_final.txt`).
constexpr int kPipeDefault = 1;
// Fallback of a configuration that does not fit (nv, x_count): the same pipeline style with
// the other chunk width (configuration 1 needs nv >= 12; n = 11 runs configuration 4).
inline int pipe_fallback(int cfg) {
  if (pipe_geom(cfg).NR) return cfg == 8 ? 6 : 8;
  return cfg == 1 ? 4 : 1;
}

// Tiles resident at once on a B200 (fixes L deterministically, independent of the device).
constexpr int kNominalSMs = 148;
constexpr int kNominalResidentCtas = 296;            // v1: 148 SMs x 2 CTAs
constexpr uint64_t kPipeScratchBudget = 2ull << 30;  // bytes of scratch slots for the pipeline

inline bool pipe_fits(int cfg, int nv, uint64_t x_count) {
  if (cfg == kPipeNone) return false;
  const PipeGeom g = pipe_geom(cfg);
  const int R = g.LT - g.XB, M = nv - R;
  return M >= 4 && M <= 8 && (g.LT - M) <= g.XB + 4 && x_count % (1ull << g.XB) == 0 &&
         x_count >= (1ull << g.XB);
}

// Plan for one launch transforming vectors of 2^nv elements for x_count X-masks.
// pipe_cfg: requested dense_pipe configuration (0 = v1 kernels); falls back when it does
// not fit (phase-B length M = nv - (LT - XB) must be in [4, 8], x_count a multiple of the
// chunk width).
// Whole-vector (single-phase) tiles for nv <= kSingleMax: a 4096-element tile holds
// 4096 / 2^nv complete vectors (n = 10: 4 X-masks), one pass over HBM and no inter-CTA
// dependencies -- at these sizes the two-phase pipeline is latency-bound.
constexpr int kSingleMax = 10;

inline DensePlan make_dense_plan(int nv, uint64_t x_count, int pipe_cfg = kPipeNone,
                                 int single_max = kSingleMax) {
  DensePlan p;
  p.nv = nv;
  if (nv <= 5) { p.kind = 0; p.nchunks = x_count >= 16 ? x_count / 16 : 1; return p; }
  if (nv <= single_max) {
    if (x_count % (4096u >> nv) == 0 && x_count >= 16) {
      p.kind = 1; p.R = nv; p.M = 0; p.nchunks = x_count / 16; return p;
    }
    if (nv <= 7) { p.kind = 0; p.nchunks = x_count >= 16 ? x_count / 16 : 1; return p; }  // tiny shards
  }
  p.kind = 2;
  if (pipe_cfg != kPipeNone && !pipe_fits(pipe_cfg, nv, x_count))
    pipe_cfg = pipe_fits(pipe_fallback(pipe_cfg), nv, x_count) ? pipe_fallback(pipe_cfg) : kPipeNone;
  p.pipe_cfg = pipe_cfg;
  int resident;
  if (pipe_cfg != kPipeNone) {
    const PipeGeom g = pipe_geom(pipe_cfg);
    p.W = 1 << g.XB;
    p.R = g.LT - g.XB;
    p.M = nv - p.R;
    resident = kNominalSMs * g.NS;
  } else {
    p.W = 16;
    if (nv <= 11) { p.R = nv - 4; p.M = 4; }
    else { p.R = 8; p.M = nv - 8; }
    resident = kNominalResidentCtas;
  }
  p.nchunks = x_count / (uint64_t)p.W;
  const uint64_t nchunks = p.nchunks;
  p.NA = 1 << p.M;
  p.NB = 1 << p.M;
  const int period = p.NA + p.NB;
  int L = (3 * resident + 2 * period - 1) / (2 * period);  // ceil(1.5*resident/period)
  if (pipe_cfg != kPipeNone) {
    // TMA pipeline: look ahead as far as ~40 MiB of live partials (L2-resident scratch)
    // allows; measured optimum at n = 12..16 and Hermitian n = 13.
    const uint64_t slot_bytes = ((uint64_t)p.W << nv) * 16;
    const uint64_t lmax = (40ull << 20) / slot_bytes;
    L = (int)(lmax < 2 ? 2 : (lmax > 64 ? 64 : lmax));
  }
  if (L < 1) L = 1;
  if (L > 64) L = 64;
  p.L = L;
  // Scratch slots.  A phase-A tile of chunk c waits until phase B of chunk c - nslot has
  // drained the slot; with ~`resident` tickets in flight that wait is rare only if
  // nslot >= L + 1 + resident/period.  The pipeline takes many more slots (capped by a
  // byte budget): consumed slots are discarded from L2, so only the live ~L chunks occupy
  // L2 and the extra slots cost HBM capacity, not bandwidth.
  uint64_t ns = (uint64_t)L + 2;
  p.slot_elems = (uint64_t)p.W << nv;
  if (pipe_cfg != kPipeNone) {
    const uint64_t slot_bytes = p.slot_elems * 16;
    uint64_t budget = kPipeScratchBudget / slot_bytes;
    const uint64_t need = 2ull * (uint64_t)L + 2ull + (uint64_t)(resident / period);
    if (budget < need) budget = need;
    ns = budget;
  }
  if (ns > nchunks) ns = nchunks;
  if (pipe_cfg != kPipeNone) {
    // a power of two, so the pipeline maps chunks to slots with a mask (its single producer
    // thread is on the critical path: no integer division per tile)
    uint64_t p2 = 1;
    while (p2 < ns) p2 <<= 1;
    ns = p2;
  }
  p.nslot = (int)ns;
  p.ctr_bytes = ((4 * (1 + 2 * nchunks)) + 255) / 256 * 256;
  p.scratch_bytes = (size_t)p.nslot * p.slot_elems * 16;
  return p;
}

}  // namespace ptdr
