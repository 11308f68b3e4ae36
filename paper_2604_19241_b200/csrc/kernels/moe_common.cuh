// Shared device-side structures of the EP-MoE data path.
//
// HBM layout per rank (one process per GPU):
//   symmetric region (same layout on every rank, peers write into it over NVLink):
//     recv_x   [M_cap][H]   bf16  expert-sorted token rows (fwd dispatch target)
//     recv_dy  [M_cap][H]   bf16  expert-sorted dY rows    (bwd dispatch target)
//     meta     [M_cap]      SlotMeta: return address (src rank, t*k+j), gate weight, relay source
//     slot_flag[M_cap]      u32 epoch: slot metadata (and, for primaries, the row) landed
//     rg_cnt   [2 ph][2 par][RG_cap] u32 rows landed per 128-row rowgroup (dispatch scoreboard)
//     rep      [T_max*k][H] bf16  combine replica slots at the source (fwd)
//     rep_dx   [T_max*k][H] bf16  combine replica slots at the source (bwd)
//     tok_cnt  [2 ph][2 par][T_max] u32 replica column-tiles landed per source token
//     cnt_all  [W][E]       i32   AllGather of per-expert counts (Alg. 1 line 3)
//     cnt_flag [W]          u32   epoch flags of cnt_all rows
//     dgp      [T_max*k][F/256] f32  gate-gradient partials <dY W_down, h> per down-dgrad column
//                                    tile, written by the expert rank, summed by the source's reduce
//   local region: GU [M_cap][2F], Hact [M_cap][F], dGU [M_cap][2F], HW [M_cap][F] bf16,
//     plan arrays (per source entry: dst slot / offset / local index; schedule), per-expert
//     receive geometry and tile prefixes.
// Expert segments in recv_* start at 128-aligned rows ("padding-free" tiles with aligned
// bases, SURVEY.md §7 hard part 4); within a segment the order is the reference's global
// (src, t, j) order (token_map.cpp:55-106), so rowgroup id = slot >> 7.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

namespace eplab_dev {

constexpr int MAX_WORLD = 8;
constexpr int MAX_EXPERTS = 512;
constexpr int PLAN_CHUNK = 2048;  // routing entries per planning CTA

struct SlotMeta {
  int src;      // source rank
  int rep;      // t * topk + j at the source
  float w;      // gate weight of (t, j)
  int primary;  // relay source slot (-1: this slot received the row itself)
};

struct SymPtrs {
  __nv_bfloat16* recv_x;
  __nv_bfloat16* recv_dy;
  SlotMeta* meta;
  uint32_t* slot_flag;
  uint32_t* rg_cnt;
  __nv_bfloat16* rep;
  __nv_bfloat16* rep_dx;
  uint32_t* tok_cnt;
  int* cnt_all;
  uint32_t* cnt_flag;
  float* dgp;  // [T_max*k][F/256] gate-gradient partials at the source, one per down-dgrad column tile
};

struct Peers {
  SymPtrs p[MAX_WORLD];
};

// Static dimensions of one context.
struct Dims {
  int H, F, E, epr, topk, world, rank;
  int T_max;
  int M_cap;   // receive rows capacity (multiple of 128)
  int RG_cap;  // M_cap / 128
};

// Per-plan device arrays (local region), written by the planning kernels.
struct PlanDev {
  int n_tok;                // tokens this rank sends
  const int* topk_ids;      // [T*k] caller's routing (device)
  const float* gate_w;      // [T*k]
  int* hist;                // [nchunks][E] -> chunk bases after the global pass
  int* counts;              // [E] C_exp of this rank
  int* send_base;           // [E] flat destination slot base of my copies to expert e
  int* o_all;               // [E] O_all[dst][e_loc][me] for global expert e (Alg. 1 base_off)
  int* bucket_base;         // [E] schedule position base of expert e (priority order)
  int* dst_slot;            // [T*k] flat slot on the destination rank
  int* offset;              // [T*k] Alg. 1 final_idx (bit-exact with the reference)
  int* sched;               // [T*k] entry index in priority order (token_map.cpp:108-126)
  // receive side (this rank as expert host), per local expert
  int* rt_all;              // [W*epr] recv_totals of every rank (token_map.cpp:71-74)
  int* sb_all_ref;          // [W*epr] reference recv_segment_base (unaligned, :75-82)
  int* sb_all;              // [W*epr] 128-aligned segment bases (the layout actually used)
  int* mblocks;             // [epr] 128-row blocks (= rowgroups) per local expert
  int* mblock_pre;          // [epr+1] prefix of mblocks (tile t of a GEMM with nb column
                            //   blocks belongs to expert e iff mblock_pre[e]*nb <= t < ..[e+1]*nb)
  int* mpair_pre;           // [epr+1] prefix of ceil(mblocks/2) (256-row CTA-pair tiles)
  int* scalars;             // [0]=M_used rows (aligned), [1]=n_rowgroups, [2]=recv total
};

// Tensor maps travel as one __grid_constant__ kernel parameter: m[0..3] operand loads,
// m[4..7] epilogue stores (box 32x32, 64B swizzle).
struct TmaSet {
  CUtensorMap m[8];
};

// Device timeline record (one per task): %globaltimer interval, SM, role, task id.
struct TimelineRec {
  unsigned long long t0, t1;
  uint32_t sm_role;  // smid | role << 16
  int task;
  uint32_t pad[2];
};
enum : uint32_t { ROLE_COMM = 0, ROLE_RELAY = 1, ROLE_COMP = 2, ROLE_REDUCE = 3 };

struct Timeline {
  TimelineRec* rec;
  int* count;
  int cap;
};


struct MkArgs {
  Dims d;
  Peers peers;
  PlanDev p;
  const __nv_bfloat16* x;       // [T][H] source rows
  const __nv_bfloat16* dy;      // [T][H]
  const __nv_bfloat16* w_up;    // [epr][2F][H]
  const __nv_bfloat16* w_down;  // [epr][H][F]
  __nv_bfloat16* y;             // [T][H]
  __nv_bfloat16* dx;            // [T][H]
  float* dgate;                 // [T*k]
  __nv_bfloat16* dw_up;         // [epr][2F][H]
  __nv_bfloat16* dw_down;       // [epr][H][F]
  __nv_bfloat16* gu;            // [M_cap][2F]
  __nv_bfloat16* hact;          // [M_cap][F]
  __nv_bfloat16* dgu;           // [M_cap][2F]
  __nv_bfloat16* hw;            // [M_cap][F]
  uint32_t* wg_cnt;             // [epr][F/256] down-dgrad tiles done (zeroed per bwd call)
  int* cursor;
  int* err;
  const uint32_t* epoch_dev;    // device iteration counter (>= 1), advanced by plan_global_kernel
  int n_disp, n_relay, n_red;
  unsigned long long timeout_ns;
  Timeline tl;
  int dbg;  // debug bits (experiments only, results wrong): 2/4 = skip dgrad epilogue TMA stores /
            // staging, 16 = skip the saved g, u loads of the dgrad epilogue, 64 = no reduce,
            // 128 = per-rowgroup relay timeline
  int pair;  // 1: CTA-pair (cta_group::2) engine
  int* comm_cursor;  // [2] u64 round counter of the comm pool (zeroed per launch with cursor)
  unsigned* red_cursor;    // reduce chunk counter (zeroed per launch with cursor)
  unsigned* relay_cursor;  // relay rowgroup counter (zeroed per launch with cursor)
  int spare_warps;  // bit 0: the GEMM CTAs' spare warps join the comm pool (warp split),
                    // bit 1: ... and the backward combine's reduce pool
  int comm_bulk;
  int rgp, tngp, tngp_d;  // CTA-pair raster groups: 256-row blocks per NT group, 256-row output
                          // blocks per TN group (up weight gradient / down weight gradient)
  int pdl;  // launched with programmatic dependent launch (the whole device is this rank's: the CTAs
            // start as the previous MegaKernel's exit, set up, then wait for its completion)
  // Unfused baseline: the same GroupGEMM tiles with every collective removed --
  // the rows were scattered into the receive layout before the launch (NCCL all-to-all), so no
  // scoreboard wait; the combine epilogues write each replica row to ret[ret_pos[slot]] (the
  // return all-to-all's send buffer) instead of pushing it to the source.
  int unfused;
  __nv_bfloat16* ret;
  const int* ret_pos;
  float* ret_dgp;  // unfused: gate-gradient partials [n_recv][F/256] in the return all-to-all's order
};

}  // namespace eplab_dev
