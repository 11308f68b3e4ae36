// The warp-specialised role loop of the grouped-GEMM engine (see gemm_core.cuh).
// Mode supplies, per tile: operand majors, TMA coordinates, an optional wait before
// the loads (scoreboard), the epilogue and a tile-done hook.
#pragma once
#include "gemm_core.cuh"
#include "moe_common.cuh"

#include <type_traits>
#include <utility>

namespace eplab_dev {

// A Mode with `static constexpr bool SPARE = true` gives the engine's otherwise idle warps work
// through `Mode::spare(args, timeline, stop)` (the MegaKernels' comm warp split). `stop` tells a
// worker that may quit early when the GEMM phase is over: every tile id has been claimed.
template <class M, class = void>
struct has_spare : std::false_type {};
template <class M>
struct has_spare<M, std::void_t<decltype(M::SPARE)>> : std::bool_constant<M::SPARE> {};
struct SpareStop {
  const int* cursor;  // the MegaKernel's task cursor
  int tile_hi;        // first id past the tiles
  __device__ __forceinline__ bool tiles_claimed() const {
    return *reinterpret_cast<const volatile int*>(cursor) >= tile_hi;
  }
};
template <class Mode, class Args, class TL>
__device__ __forceinline__ void call_spare(const Args& a, const TL& tl, const SpareStop& stop) {
  if constexpr (has_spare<Mode>::value) Mode::spare(a, tl, stop);
}
// A Mode with `static constexpr bool RELEASE_AFTER = true` publishes a tile's results in
// `Mode::epilogue_release(args, tile, row)`, called after the epilogue has handed the TMEM
// accumulator back to the MMA issuer: the release fence (system scope at EP>1) then overlaps the
// next tile's main loop instead of holding the accumulator.
template <class M, class = void>
struct has_release_after : std::false_type {};
template <class M>
struct has_release_after<M, std::void_t<decltype(M::RELEASE_AFTER)>> : std::bool_constant<M::RELEASE_AFTER> {};
template <class Mode, class Args>
__device__ __forceinline__ void call_release_after(const Args& a, const TileDesc& td, int r) {
  if constexpr (has_release_after<Mode>::value) Mode::epilogue_release(a, td, r);
}

// A Mode with `static constexpr bool RELEASE_WARP = true` (CTA-pair engine) has its tiles published
// by warp 2 instead of the epilogue warps: `Mode::wants_release(args, tile)` selects the tiles and
// `Mode::release_tile(args, tile, lane)` publishes one (a warp-wide job).
template <class M, class = void>
struct has_release_warp : std::false_type {};
template <class M>
struct has_release_warp<M, std::void_t<decltype(M::RELEASE_WARP)>> : std::bool_constant<M::RELEASE_WARP> {};
template <class Mode, class Args>
__device__ __forceinline__ void call_release_tile(const Args& a, const TileDesc& td, int lane) {
  if constexpr (has_release_warp<Mode>::value) Mode::release_tile(a, td, lane);
}

// Debug bits of the Mode's Args (MkArgs::dbg), 0 for argument types without them. Experiments only
// (eplab_set_option("dbg", ...)): 256 = the producer skips the B operand loads (wrong results; measures
// what the B operand traffic costs, the bound on TMA-multicast savings).
template <class A, class = void>
struct has_dbg : std::false_type {};
template <class A>
struct has_dbg<A, std::void_t<decltype(std::declval<A>().dbg)>> : std::true_type {};
template <class A>
__device__ __forceinline__ int dbg_bits(const A& a) {
  if constexpr (has_dbg<A>::value) return a.dbg;
  return 0;
}

__device__ __forceinline__ void timeline_push(const Timeline& tl, unsigned long long t0,
                                              unsigned long long t1, uint32_t role, int task) {
  if (!tl.rec) return;
  const int i = atomicAdd(tl.count, 1);
  if (i < tl.cap) {
    TimelineRec r;
    r.t0 = t0;
    r.t1 = t1;
    r.sm_role = smid() | (role << 16);
    r.task = task;
    r.pad[0] = r.pad[1] = 0;
    tl.rec[i] = r;
  }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Called once per CTA after barriers/TMEM are set up. `first` is the first tile
// task (already claimed by the CTA while it resolved pre-tasks). Returns the first
// claimed id beyond [tile_lo, tile_hi) so the caller can continue with post-tasks.
template <class Mode>
__device__ int gemm_roles(const typename Mode::Args& args, const TmaSet& tm, uint8_t* tiles_smem,
                          GemmSmem* S, int first, int tile_lo, int tile_hi,
                          int* __restrict__ cursor, const Timeline& tl) {
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  uint8_t* sA = tiles_smem;
  uint8_t* sB = tiles_smem + STAGES * A_STAGE_BYTES;

  if (has_spare<Mode>::value && warp == 2) {
    call_spare<Mode>(args, tl, SpareStop{cursor, tile_hi});  // the TMEM owner is idle between allocation and teardown
  } else if (warp == 3) {
    // ---------------- scheduler: claims tile ids, decodes them and resolves their scoreboard
    // dependencies (Mode::before_loads) ahead of the producer; stops at the first non-tile id
    if (lane == 0) {
      int id = first;
      for (int it = 0;; ++it) {
        const int slot = it % RING;
        const bool is_tile = id >= tile_lo && id < tile_hi;
        TileDesc td{};
        if (is_tile) {
          td = Mode::tile(args, id - tile_lo);
          Mode::before_loads(args, td);
        }
        mbar_wait(&S->rempty[slot], ((it / RING) & 1) ^ 1);
        S->ring[slot] = is_tile ? id - tile_lo : TASK_STOP;
        S->ring_td[slot] = td;
        mbar_arrive(&S->rfull[slot]);
        if (!is_tile) {
          S->bcast = id;
          break;
        }
        id = atomicAdd(cursor, 1);
      }
    }
  } else if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      for (int i = 0; i < 8; ++i) tma_prefetch_desc(&tm.m[i]);
      uint32_t stage = 0, phase = 0;
      for (int it = 0;; ++it) {
        const int slot = it % RING;
        mbar_wait(&S->rfull[slot], (it / RING) & 1);
        const int t = S->ring[slot];
        const TileDesc td = S->ring_td[slot];
        mbar_arrive(&S->rempty[slot]);
        if (t == TASK_STOP) break;
        fence_proxy_async_global();  // scoreboard acquired by the scheduler -> async-proxy reads
        S->tstart[it & 7] = globaltimer();
        for (int kb = 0; kb < td.nkb; ++kb) {
          mbar_wait(&S->empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&S->full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
          uint8_t* a = sA + stage * A_STAGE_BYTES;
          uint8_t* b = sB + stage * B_STAGE_BYTES;
          Mode::load_a(args, tm, &S->full[stage], a, td, kb);
          Mode::load_b(args, tm, &S->full[stage], b, td, kb);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer
    if (lane == 0) {
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      uint32_t stage = 0, phase = 0;
      for (int it = 0;; ++it) {
        const int slot = it % RING;
        mbar_wait(&S->rfull[slot], (it / RING) & 1);
        const int t = S->ring[slot];
        const TileDesc td = S->ring_td[slot];
        mbar_arrive(&S->rempty[slot]);
        if (t == TASK_STOP) break;
        const int amn = Mode::a_mn(td), bmn = Mode::b_mn(td);
        const uint32_t idesc = make_idesc(BM, BN, amn, bmn);
        const uint32_t acc = it & 1;
        mbar_wait(&S->tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = S->tmem_base + acc * BN;
        for (int kb = 0; kb < td.nkb; ++kb) {
          mbar_wait(&S->full[stage], phase);
          tc_fence_after();
          const uint32_t as = a0 + stage * A_STAGE_BYTES;
          const uint32_t bs = b0 + stage * B_STAGE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = amn ? make_sdesc(as + k * 2048, 8192, 1024)
                                    : make_sdesc(as + k * 32, 16, 1024);
            const uint64_t bd = bmn ? make_sdesc(bs + k * 2048, 8192, 1024)
                                    : make_sdesc(bs + k * 32, 16, 1024);
            umma_bf16(d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&S->empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&S->tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp q owns TMEM lanes / tile rows [32q, 32q+32)
    const int q = warp & 3;
    const int r = q * 32 + (int)lane;
    for (int it = 0;; ++it) {
      const int slot = it % RING;
      mbar_wait(&S->rfull[slot], (it / RING) & 1);
      const int t = S->ring[slot];
      const TileDesc td = S->ring_td[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&S->rempty[slot]);
      if (t == TASK_STOP) {
        if (lane == 0) tma_store_wait<0>();  // outstanding epilogue stores before teardown
        break;
      }
      Mode::epilogue_prefetch(args, td, r);
      const uint32_t acc = it & 1;
      mbar_wait(&S->tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = S->tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      Mode::epilogue(args, tm, td, taddr, r, tiles_smem + TILES_BYTES + q * EPI_WARP_BYTES);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S->tempty[acc]);
      call_release_after<Mode>(args, td, r);
      if (Mode::HAS_TILE_DONE || tl.rec) {
        epi_bar();  // all four epilogue warps finished this tile's stores
        if (warp == 4 && lane == 0) {
          if (Mode::HAS_TILE_DONE) Mode::tile_done(args, td);
          timeline_push(tl, S->tstart[it & 7], globaltimer(), ROLE_COMP, t + tile_lo);
        }
      }
    }
  }
  __syncthreads();
  return S->bcast;
}

// Barrier + TMEM setup shared by every kernel built on the engine.
__device__ __forceinline__ void gemm_setup(GemmSmem* S) {
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&S->full[i], 1);
      mbar_init(&S->empty[i], 1);
    }
    for (int i = 0; i < ACC_STAGES; ++i) {
      mbar_init(&S->tfull[i], 1);
      mbar_init(&S->tempty[i], 4);
    }
    for (int i = 0; i < RING; ++i) {
      mbar_init(&S->rfull[i], 1);
      mbar_init(&S->rempty[i], 6);  // producer + mma + 4 epilogue warps
    }
    for (int i = 0; i < 48; ++i) mbar_init(&S->cbar[i], 1);
    for (int i = 0; i < 4; ++i) S->cphase[i] = 0;
    S->bcast = TASK_STOP;
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&S->tmem_base, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

__device__ __forceinline__ void gemm_teardown(GemmSmem* S) {
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((threadIdx.x >> 5) == 2) tmem_dealloc(S->tmem_base, TMEM_COLS);
}

// Row-chunk helpers used by epilogues: 32 fp32 accumulators of one row.
// tcgen05.ld / wait::ld are .sync.aligned: the warp must be converged, which the divergent
// per-row code (live rows, predicated loads) around the call sites does not guarantee by itself.
__device__ __forceinline__ void acc_chunk(uint32_t taddr, int chunk, float (&v)[32]) {
  uint32_t r[32];
  __syncwarp();
  tmem_ld32(taddr + chunk * 32, r);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void store_row_bf16_32(__nv_bfloat16* dst, const float (&v)[32]) {
  int4* d = reinterpret_cast<int4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int4 w;
    w.x = (int)pack_bf16(v[8 * i + 0], v[8 * i + 1]);
    w.y = (int)pack_bf16(v[8 * i + 2], v[8 * i + 3]);
    w.z = (int)pack_bf16(v[8 * i + 4], v[8 * i + 5]);
    w.w = (int)pack_bf16(v[8 * i + 6], v[8 * i + 7]);
    d[i] = w;
  }
}

__device__ __forceinline__ void store_zero_32(__nv_bfloat16* dst) {
  int4* d = reinterpret_cast<int4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] = make_int4(0, 0, 0, 0);
}

// 32 bf16 from global (4 x 16 B) into fp32.
__device__ __forceinline__ void load_row_bf16_32(const __nv_bfloat16* src, float (&v)[32]) {
  const int4* s = reinterpret_cast<const int4*>(src);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int4 w = s[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __bfloat1622float2(h[k]);
      v[8 * i + 2 * k] = f.x;
      v[8 * i + 2 * k + 1] = f.y;
    }
  }
}


// ---------------------------------------------------------------- staged TMA-store epilogue
// Row r (0..31) of a warp's 32x32 bf16 staging tile, 64B-swizzled (16 B chunk c of row r lives at
// chunk c ^ ((r >> 1) & 3)) so the 32 lanes' 16 B stores hit distinct bank groups.
__device__ __forceinline__ void stage_row(uint8_t* buf, int r, const float (&v)[32]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    int4 w;
    w.x = (int)pack_bf16(v[8 * c + 0], v[8 * c + 1]);
    w.y = (int)pack_bf16(v[8 * c + 2], v[8 * c + 3]);
    w.z = (int)pack_bf16(v[8 * c + 4], v[8 * c + 5]);
    w.w = (int)pack_bf16(v[8 * c + 6], v[8 * c + 7]);
    *reinterpret_cast<int4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) = w;
  }
}
// Same, from 16 packed bf16x2 words.
__device__ __forceinline__ void stage_row_packed(uint8_t* buf, int r, const uint32_t (&p)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    *reinterpret_cast<int4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) =
        make_int4((int)p[4 * c], (int)p[4 * c + 1], (int)p[4 * c + 2], (int)p[4 * c + 3]);
}
__device__ __forceinline__ void stage_zero_row(uint8_t* buf, int r) {
#pragma unroll
  for (int c = 0; c < 4; ++c) *reinterpret_cast<int4*>(buf + r * 64 + (c << 4)) = make_int4(0, 0, 0, 0);
}
// Before refilling the warp's staging tiles: the previous TMA stores must have read them.
__device__ __forceinline__ void stage_acquire(uint32_t lane) {
  if (lane == 0) tma_store_wait_read<0>();
  __syncwarp();
}
// After filling: make generic-proxy smem writes visible to the TMA engine.
__device__ __forceinline__ void stage_release() {
  fence_proxy_async();
  __syncwarp();
}

}  // namespace eplab_dev
