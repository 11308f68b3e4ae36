// CTA-pair (cta_group::2) variant of the grouped-GEMM engine.
//
// A cluster of two CTAs on one TPC computes 256 x 256 tiles: CTA r stages rows
// [128r, 128r+128) of A and columns [128r, 128r+128) of B (32 KB per stage and CTA, 6 stages),
// the leader (rank 0) issues tcgen05.mma.cta_group::2 (M=256, N=256, K=16) which reads both
// CTAs' shared memory and accumulates rows [128r, ..) into CTA r's TMEM. Versus the single-CTA
// engine every B tile is fetched once per pair instead of twice and the pipeline is 6 deep.
//
// Roles (per CTA, 256 threads):  warp 0 TMA producer (both CTAs), warp 1 MMA issuer (leader),
// warp 2 TMEM owner (both, cta_group::2 allocation), warp 3 scheduler (leader: claims task ids,
// decodes tiles, resolves scoreboard waits, writes the tile into both CTAs' rings over DSMEM),
// warps 4-7 epilogue (both, each on its own 128 rows).
// Barrier ownership: full[s] (leader, 2 arrivals + tx of both CTAs), empty[s] (each CTA, one
// multicast MMA commit), tfull[a] (each CTA, multicast commit), tempty[a] (leader, 8 epilogue
// warps), rfull[q] (each CTA, leader's scheduler), rempty[q] (leader, 6 local + 5 remote).
#pragma once
#include "gemm_engine.cuh"

namespace eplab_dev {

constexpr int P_STAGES = 6;
constexpr uint32_t P_HALF_BYTES = 128 * BK * 2;  // 16 KB: one CTA's A rows or B columns
constexpr uint32_t P_STAGE_BYTES = 2 * P_HALF_BYTES;
static_assert(P_STAGES * P_STAGE_BYTES == TILES_BYTES, "pair stages reuse the single-CTA smem map");

// A Mode may run fewer operand stages (`static constexpr int PAIR_STAGES`): stage s of A stays at
// half s and of B at half P_STAGES + s, so the last A half and the last B half (16 KB each) are
// free for the epilogue's input ring (`static constexpr bool GU_RING = true`): 8 KB per epilogue
// warp, two 4 KB buffers the warp fills with TMA loads of the rows its epilogue reads
// (Mode::epilogue_issue before the accumulator wait, Mode::epilogue_ring consumes them).
template <class M, class = void>
struct pair_stages : std::integral_constant<int, P_STAGES> {};
template <class M>
struct pair_stages<M, std::void_t<decltype(M::PAIR_STAGES)>> : std::integral_constant<int, M::PAIR_STAGES> {};
template <class M, class = void>
struct has_gu_ring : std::false_type {};
template <class M>
struct has_gu_ring<M, std::void_t<decltype(M::GU_RING)>> : std::bool_constant<M::GU_RING> {};
struct EpiRing {
  uint8_t* buf;    // 2 x 4 KB
  uint64_t* bar;   // 2 barriers
};

__device__ __forceinline__ void gemm_setup_pair(GemmSmem* S, uint32_t rank) {
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < P_STAGES; ++i) {
      mbar_init(&S->full[i], 2);  // leader's expect_tx arrival + the peer's arrival
      mbar_init(&S->empty[i], 1);
    }
    for (int i = 0; i < ACC_STAGES; ++i) {
      mbar_init(&S->tfull[i], 1);
      mbar_init(&S->tempty[i], 8);  // 4 epilogue warps per CTA
    }
    for (int i = 0; i < RING; ++i) {
      mbar_init(&S->rfull[i], 1);
      mbar_init(&S->rempty[i], 11);  // leader: producer, mma, 4 epi; peer: producer, 4 epi
    }
    for (int i = 0; i < 48; ++i) mbar_init(&S->cbar[i], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&S->gbar[i], 1);
    for (int i = 0; i < 4; ++i) {
      S->cphase[i] = 0;
      mbar_init(&S->rq_full[i], 4);
      mbar_init(&S->rq_empty[i], 1);
    }
    S->bcast = TASK_STOP;
    fence_mbar_init();
  }
  __syncthreads();  // thread 0's writes (S->bcast shares a 16-byte word with S->tmem_base) before the allocation
  if (warp == 2) tmem_alloc_pair(&S->tmem_base, TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
}

__device__ __forceinline__ void gemm_teardown_pair(GemmSmem* S) {
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if ((threadIdx.x >> 5) == 2) tmem_dealloc_pair(S->tmem_base, TMEM_COLS);
}

// Both CTAs call this after exchanging their first non-pre task ids into the leader's
// S->pend[0..1] (ascending). Afterwards the leader's S->post_ids[0..S->post_n) hold the claimed
// ids that are not tiles (to be handed out by the caller).
template <class Mode>
__device__ void gemm_roles_pair(const typename Mode::Args& args, const TmaSet& tm,
                                uint8_t* tiles_smem, GemmSmem* S, int tile_lo, int tile_hi,
                                int* __restrict__ cursor, const Timeline& tl, uint32_t rank,
                                const Watchdog& wd = Watchdog{}) {
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id();
  uint8_t* sA = tiles_smem;
  uint8_t* sB = tiles_smem + P_STAGES * P_HALF_BYTES;
  const bool leader = rank == 0;
  constexpr int NST = pair_stages<Mode>::value;
  static_assert(NST <= P_STAGES && (!has_gu_ring<Mode>::value || NST < P_STAGES), "epilogue ring needs a free stage");

  // spare warps: warp 2 (TMEM owner, idle between allocation and teardown) of both CTAs and the
  // non-leader's warps 1 and 3 (the leader alone issues MMAs and schedules)
  const bool spare = warp == 2 || (!leader && (warp == 1 || warp == 3));
  constexpr bool kRelWarp = has_release_warp<Mode>::value;
  if (kRelWarp && warp == 2) {
    // ---------------- release warp (both CTAs): publishes the tiles the epilogue warps queue --
    // the system/gpu-scope fence waits for the tile's stores to complete, which would otherwise
    // stall the epilogue warps for the next accumulator (Qwen3 fwd combine: 30 % of the span)
    for (int it = 0;; ++it) {
      const int slot = it & 3;
      mbar_wait(&S->rq_full[slot], (it >> 2) & 1);  // acquire (CTA): the four warps' stores
      const TileDesc td = S->rq_td[slot];
      if (td.rows < 0) break;
      call_release_tile<Mode>(args, td, (int)lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S->rq_empty[slot]);
    }
  } else if (has_spare<Mode>::value && spare) {
    call_spare<Mode>(args, tl, SpareStop{cursor, tile_hi});
  } else if (warp == 3) {
    if (leader && lane == 0) {
      // ---------------- scheduler (leader)
      int np = 0;
      S->post_n = 0;
      if (S->pend[1] < S->pend[0]) {
        const int t0 = S->pend[0];
        S->pend[0] = S->pend[1];
        S->pend[1] = t0;
      }
      for (int it = 0;; ++it) {
        const int slot = it % RING;
        int id;
        if (np < 2) {
          id = S->pend[np++];
        } else {
          id = atomicAdd(cursor, 1);
        }
        const bool is_tile = id >= tile_lo && id < tile_hi;
        if (!is_tile) {  // pending ids are ascending: a later pending id is not a tile either
          S->post_ids[S->post_n++] = id;
          if (np < 2) S->post_ids[S->post_n++] = S->pend[np++];
        }
        TileDesc td{};
        if (is_tile) {
          td = Mode::tile_pair(args, id - tile_lo);
          Mode::before_loads_pair(args, td);
        }
        mbar_wait_cluster_wd(&S->rempty[slot], ((it / RING) & 1) ^ 1, wd, 40);
        const int rv = is_tile ? id - tile_lo : TASK_STOP;
        S->ring[slot] = rv;
        S->ring_td[slot] = td;
        // the peer's ring slot over DSMEM, then release both rfull barriers (cluster scope)
        const uint32_t peer_ring = mapa_shared(smem_u32(&S->ring[slot]), 1);
        const uint32_t peer_td = mapa_shared(smem_u32(&S->ring_td[slot]), 1);
        st_cluster_u32(peer_ring, (uint32_t)rv);
        const int4* tdv = reinterpret_cast<const int4*>(&td);
        st_cluster_v4(peer_td, tdv[0]);
        st_cluster_v4(peer_td + 16, tdv[1]);
        fence_acq_rel_cluster();  // the descriptor stores before the peer's rfull arrival
        mbar_arrive_cluster(mapa_shared(smem_u32(&S->rfull[slot]), 0));
        mbar_arrive_cluster(mapa_shared(smem_u32(&S->rfull[slot]), 1));
        if (!is_tile) break;
      }
    }
  } else if (warp == 0) {
    // ---------------- TMA producer (both CTAs)
    if (lane == 0) {
      for (int i = 0; i < 8; ++i) tma_prefetch_desc(&tm.m[i]);
      const bool skip_b = (dbg_bits(args) & 256) != 0;  // experiment: no B traffic (results wrong)
      const uint32_t rempty0 = mapa_shared(smem_u32(&S->rempty[0]), 0);
      uint32_t stage = 0, phase = 0;
      for (int it = 0;; ++it) {
        const int slot = it % RING;
        mbar_wait_cluster_wd(&S->rfull[slot], (it / RING) & 1, wd, 41);
        const int t = S->ring[slot];
        const TileDesc td = S->ring_td[slot];
        mbar_arrive_cluster(rempty0 + slot * 8);
        if (t == TASK_STOP) break;
        fence_proxy_async_global();
        if (leader) S->tstart[it & 7] = globaltimer();
        for (int kb = 0; kb < td.nkb; ++kb) {
          mbar_wait_wd(&S->empty[stage], phase ^ 1, wd, 42);
          const uint32_t full0 = mapa_shared(smem_u32(&S->full[stage]), 0);
          if (leader)
            mbar_arrive_expect_tx(&S->full[stage], skip_b ? P_STAGE_BYTES : 2 * P_STAGE_BYTES);
          else
            mbar_arrive_cluster(full0);
          Mode::load_a_pair(args, tm, full0, sA + stage * P_HALF_BYTES, td, kb, rank);
          if (!skip_b) Mode::load_b_pair(args, tm, full0, sB + stage * P_HALF_BYTES, td, kb, rank);
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer (leader)
    if (leader && lane == 0) {
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      uint32_t stage = 0, phase = 0;
      // stall accounting of the MMA issuer (timeline on): waiting for a tile (scheduler /
      // scoreboard), for a free accumulator (epilogue), for operands (producer)
      const bool acct = tl.rec != nullptr;
      unsigned long long w_tile = 0, w_acc = 0, w_ops = 0, t_begin = acct ? globaltimer() : 0, tw = 0;
      // per tile type (td.pad1: 0 = NT tiles, 1 = transposed weight-gradient tiles): main-loop time
      // (first operand wait to the last commit) and its operand waits
      unsigned long long ty_loop[2] = {0, 0}, ty_ops[2] = {0, 0}, tl0 = 0;
      for (int it = 0;; ++it) {
        const int slot = it % RING;
        if (acct) tw = globaltimer();
        mbar_wait_cluster_wd(&S->rfull[slot], (it / RING) & 1, wd, 43);
        if (acct) w_tile += globaltimer() - tw;
        const int t = S->ring[slot];
        const TileDesc td = S->ring_td[slot];
        mbar_arrive(&S->rempty[slot]);
        if (t == TASK_STOP) break;
        const int amn = Mode::a_mn(td), bmn = Mode::b_mn(td);
        const uint32_t idesc = make_idesc(2 * BM, BN, amn, bmn);
        const uint32_t acc = it & 1;
        if (acct) tw = globaltimer();
        mbar_wait_cluster_wd(&S->tempty[acc], ((it >> 1) & 1) ^ 1, wd, 44);
        if (acct) w_acc += globaltimer() - tw;
        tc_fence_after();
        const uint32_t d = S->tmem_base + acc * BN;
        const int ty = td.pad1 ? 1 : 0;
        if (acct) tl0 = globaltimer();
        for (int kb = 0; kb < td.nkb; ++kb) {
          if (acct) tw = globaltimer();
          mbar_wait_wd(&S->full[stage], phase, wd, 45);
          if (acct) {
            const unsigned long long dw = globaltimer() - tw;
            w_ops += dw;
            ty_ops[ty] += dw;
          }
          tc_fence_after();
          const uint32_t as = a0 + stage * P_HALF_BYTES;
          const uint32_t bs = b0 + stage * P_HALF_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = amn ? make_sdesc(as + k * 2048, 8192, 1024)
                                    : make_sdesc(as + k * 32, 16, 1024);
            const uint64_t bd = bmn ? make_sdesc(bs + k * 2048, 8192, 1024)
                                    : make_sdesc(bs + k * 32, 16, 1024);
            umma_bf16_pair(d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit_pair(&S->empty[stage]);
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&S->tfull[acc]);
        if (acct) ty_loop[ty] += globaltimer() - tl0;
      }
      if (acct) {  // three records per CTA pair, durations = the stall totals (task -9001..-9003)
        timeline_push(tl, t_begin, t_begin + w_tile, ROLE_COMP, -9001);
        timeline_push(tl, t_begin, t_begin + w_acc, ROLE_COMP, -9002);
        timeline_push(tl, t_begin, t_begin + w_ops, ROLE_COMP, -9003);
        for (int y = 0; y < 2; ++y) {  // -9031/-9032: main-loop time per type, -9033/-9034: its operand waits
          timeline_push(tl, t_begin, t_begin + ty_loop[y], ROLE_COMP, -9031 - y);
          timeline_push(tl, t_begin, t_begin + ty_ops[y], ROLE_COMP, -9033 - y);
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): this CTA's 128 rows of the 256-row tile
    const int q = warp & 3;
    const int r = q * 32 + (int)lane;
    EpiRing ring{nullptr, &S->gbar[2 * q]};
    if constexpr (has_gu_ring<Mode>::value)  // warps 0, 1: free A half; warps 2, 3: free B half
      ring.buf = tiles_smem + (q < 2 ? NST : P_STAGES + NST) * P_HALF_BYTES + (q & 1) * 8192;
    const uint32_t rempty0 = mapa_shared(smem_u32(&S->rempty[0]), 0);
    const uint32_t tempty0 = mapa_shared(smem_u32(&S->tempty[0]), 0);
    // stall accounting of epilogue warp 0 (timeline on): waiting for the accumulator (MMA), the
    // epilogue itself (TMEM -> registers -> stores), the release after the accumulator hand-back
    const bool acct = tl.rec != nullptr && q == 0;
    unsigned long long e_wait = 0, e_epi = 0, e_rel = 0, e_begin = acct ? globaltimer() : 0, tw = 0;
    int rq_it = 0;  // tiles queued for the release warp (the same sequence in all four warps)
    auto queue_release = [&](const TileDesc& h) {
      const int s = rq_it & 3;
      mbar_wait(&S->rq_empty[s], ((rq_it >> 2) & 1) ^ 1);
      if (q == 0 && lane == 0) S->rq_td[s] = h;
      __syncwarp();  // every lane's pushed rows precede the arrival (release, CTA scope)
      if (lane == 0) mbar_arrive(&S->rq_full[s]);
      ++rq_it;
    };
    for (int it = 0;; ++it) {
      const int slot = it % RING;
      mbar_wait_cluster_wd(&S->rfull[slot], (it / RING) & 1, wd, 46);
      const int t = S->ring[slot];
      const TileDesc td = S->ring_td[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(rempty0 + slot * 8);
      if (t == TASK_STOP) {
        if (lane == 0) tma_store_wait<0>();
        if constexpr (kRelWarp) {
          TileDesc stop{};
          stop.rows = -1;
          queue_release(stop);
        }
        break;
      }
      const TileDesc half = Mode::half_of(td, rank);
      const bool work = Mode::half_has_work(half);
      if (work) Mode::epilogue_prefetch(args, half, r);
      if constexpr (has_gu_ring<Mode>::value) {
        if (work) Mode::epilogue_issue(args, tm, half, (int)lane, q, ring);
      }
      const uint32_t acc = it & 1;
      if (acct) tw = globaltimer();
      mbar_wait_wd(&S->tfull[acc], (it >> 1) & 1, wd, 47);
      tc_fence_after();
      if (acct) {
        const unsigned long long now = globaltimer();
        e_wait += now - tw;
        tw = now;
      }
      const uint32_t taddr = S->tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      if constexpr (has_gu_ring<Mode>::value) {
        if (work) Mode::epilogue_ring(args, tm, half, taddr, r, tiles_smem + TILES_BYTES + q * EPI_WARP_BYTES, ring);
      } else {
        if (work) Mode::epilogue(args, tm, half, taddr, r, tiles_smem + TILES_BYTES + q * EPI_WARP_BYTES);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
      if (acct) {
        const unsigned long long now = globaltimer();
        e_epi += now - tw;
        tw = now;
      }
      if constexpr (kRelWarp) {
        if (work && Mode::wants_release(args, half)) queue_release(half);
      } else {
        if (work) call_release_after<Mode>(args, half, r);
      }
      if (acct) {
        __syncwarp();
        e_rel += globaltimer() - tw;
      }
      if (Mode::HAS_TILE_DONE || tl.rec) {
        epi_bar();
        if (warp == 4 && lane == 0) {
          if (Mode::HAS_TILE_DONE && work) Mode::tile_done(args, half);
          if (leader) timeline_push(tl, S->tstart[it & 7], globaltimer(), ROLE_COMP, t + tile_lo);
        }
      }
    }
    if (acct && lane == 0) {  // three records per CTA, durations = the totals (task -9004..-9006)
      timeline_push(tl, e_begin, e_begin + e_wait, ROLE_COMP, -9004);
      timeline_push(tl, e_begin, e_begin + e_epi, ROLE_COMP, -9005);
      timeline_push(tl, e_begin, e_begin + e_rel, ROLE_COMP, -9006);
    }
  }
  __syncthreads();
}

}  // namespace eplab_dev
