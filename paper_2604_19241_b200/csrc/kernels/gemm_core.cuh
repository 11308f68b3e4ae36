// Persistent, warp-specialised tcgen05 grouped-GEMM engine for sm_100a.
//
// One CTA per SM (256 threads):
//   warp 0      TMA producer      (one elected lane)
//   warp 1      UMMA issuer       (one elected lane; tcgen05.mma cta_group::1, 128x256x16)
//   warp 2      TMEM owner        (alloc / dealloc 512 columns = 2 accumulators)
//   warp 3      task scheduler    (lane 0 claims task ids from the global cursor)
//   warps 4..7  epilogue          (tcgen05.ld 32x32b -> registers -> mode-specific epilogue)
//
// Operands are staged by TMA with 128-byte swizzle into a 4-stage ring
// (A 128x64, B 256x64 bf16 per stage). Either operand may be K-major (rows of
// the contraction) or MN-major (the contraction is the row index of the
// global tensor), which is how the transposed GroupGEMM of the weight
// gradient reads token-major activations without a transpose pass.
//
// Task ids come from a global atomic cursor and are forwarded to the other
// roles through a 2-deep shared-memory ring, so the same engine serves as the
// compute role of the MegaKernels (task space [pre | tiles | post], claimed in
// that order -- PAPER.md:169-189, Listing 1 :457-484).
#pragma once
#include "ptx.cuh"

namespace eplab_dev {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int ACC_STAGES = 2;
constexpr int RING = 4;
constexpr int GEMM_THREADS = 256;
constexpr uint32_t A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr uint32_t B_STAGE_BYTES = BN * BK * 2;  // 32 KB
constexpr uint32_t TMEM_COLS = 512;
constexpr int TASK_STOP = -1;

// One GEMM tile task. Meaning of the fields per mode is documented at each
// mode's producer/epilogue.
struct alignas(16) TileDesc {
  int e;      // local expert
  int m0;     // first row of A / of the row-indexed outputs (wgrad: output row)
  int n0;     // output column start
  int rows;   // valid rows (<= BM) (wgrad: unused)
  int kb0;    // wgrad: first token row of the expert segment
  int nkb;    // number of 64-wide K blocks
  int pad0, pad1;
};

constexpr int STAGES_MAX = 6;  // the CTA-pair engine runs 6 stages of 32 KB
struct GemmSmem {
  uint64_t full[STAGES_MAX];
  uint64_t empty[STAGES_MAX];
  uint64_t tfull[ACC_STAGES];
  uint64_t tempty[ACC_STAGES];
  uint64_t rfull[RING];
  uint64_t rempty[RING];
  unsigned long long tstart[8];
  TileDesc ring_td[RING];
  int ring[RING];
  uint32_t tmem_base;
  int bcast;
  int pend[2];      // CTA pair: first non-pre task id of each CTA (leader's copy)
  int post_ids[4];  // CTA pair: claimed non-tile ids to hand out after the GEMM phase
  int post_n;
  // CTA pair, Modes with a release warp: the epilogue warps queue each finished tile here and warp
  // 2 publishes it (fence + scoreboard updates) off the epilogue's critical path
  uint64_t rq_full[4];   // 4 arrivals: the four epilogue warps queued the tile
  uint64_t rq_empty[4];  // 1 arrival: the release warp published it
  TileDesc rq_td[4];
  // CTA pair, Modes with an epilogue input ring (GU_RING): two TMA-completion barriers per epilogue
  // warp for its two input buffers
  uint64_t gbar[8];
  // comm role (runs before the CTA enters the GEMM roles; reuses the stage buffers)
  uint64_t cbar[48];      // one mbarrier per bulk-copy slot
  uint32_t cphase[4];     // per issuer: parity bit per owned slot (carried across comm tasks)
  int cpos[48];           // round position of the item held by each slot
  int crel[4][64];        // per issuer: round position by load sequence (release ring)
  int citem[256];         // per-round item metadata
  int cslot[256];
  int cdst[256];
};

// Epilogue staging: per epilogue warp three 32x32 bf16 tiles (64 B rows, 64B-swizzled) that the
// warp's elected lane writes out with TMA bulk-tensor stores.
constexpr uint32_t EPI_TILE_BYTES = 32 * 64;
constexpr uint32_t EPI_WARP_BYTES = 3 * EPI_TILE_BYTES;
constexpr uint32_t EPI_BYTES = 4 * EPI_WARP_BYTES;
constexpr uint32_t TILES_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES);
constexpr uint32_t GEMM_SMEM_BYTES =
    1024 /*align slack*/ + TILES_BYTES + EPI_BYTES + sizeof(GemmSmem) + 64;

__device__ __forceinline__ uint8_t* smem_aligned(uint8_t* raw) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
}

}  // namespace eplab_dev
