// The EP-MoE MegaKernels, forward and backward, on the tcgen05 engine.
//
// Each kernel is persistent (one 256-thread CTA per SM). A CTA claims task ids from one
// global cursor; the id space is linearised [pre | tiles | post] and claimed in that order,
// so producers are always claimed before the consumers that wait on them (the deadlock
// argument of types.cpp:55-67 / sim.cpp:547-551; Listing 1 :457-484).
//
//   fwd_dispatch_gemm  : [comm n_disp | relay n_relay | up-GEMM tiles (+SwiGLU)]
//   fwd_gemm_combine   : [down-GEMM tiles (epilogue pushes replicas to the source) | reduce n_red]
//   bwd_dispatch_gemm  : [comm n_disp (dY, gate grad) | relay | down-dgrad tiles (+SwiGLU bwd)
//                         | down-wgrad tiles (transposed GroupGEMM)]
//   bwd_gemm_combine   : [up-dgrad tiles (push dX replicas) | up-wgrad tiles | reduce n_red]
//
// Communication roles (the unified AllGather/AllToAll primitive):
//   relay off (n_relay = 0, AllToAll style): a comm warp writes every (t, j) replica row
//     straight into the destination slot and bumps the destination rowgroup counter with
//     red.release.sys;
//   relay on (AllGather style, sim.cpp:384-441): only the first (token, dst) item in
//     priority order crosses NVLink; the sender writes the slot metadata of every replica
//     and releases per-slot epoch flags; relay workers on the destination copy duplicates
//     from the primary slot in HBM and count their rowgroups.
// The comp tile waits for its rowgroup counter (ld.acquire.sys), fences the async proxy and
// only then lets TMA read the rows: the token-granular scoreboard of Eq. 2.
#include <cuda_runtime.h>

#include "gemm_engine.cuh"
#include "gemm_pair.cuh"
#include "moe_common.cuh"

#ifndef EPLAB_ENGINE_WD
#define EPLAB_ENGINE_WD 0
#endif

namespace eplab_dev {

// Iteration number of the running MegaKernel, read once per CTA from the device epoch counter
// (advanced by the planning kernel), so a captured CUDA graph of a whole step replays correctly;
// parity = epoch & 1 selects the scoreboard counters' double buffer.
__shared__ uint32_t sh_epoch;
#define EPOCH(a) (sh_epoch)
#define PAR(a) ((int)(sh_epoch & 1u))
__device__ __forceinline__ void load_epoch(const MkArgs& a) {
  if (threadIdx.x == 0) sh_epoch = *reinterpret_cast<const volatile uint32_t*>(a.epoch_dev);
  __syncthreads();
}


// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t* rg_counter(const SymPtrs& s, const Dims& d, int ph, int par,
                                                int g) {
  return s.rg_cnt + (size_t)(ph * 2 + par) * d.RG_cap + g;
}
__device__ __forceinline__ uint32_t* tok_counter(const SymPtrs& s, const Dims& d, int ph, int par,
                                                 int t) {
  return s.tok_cnt + (size_t)(ph * 2 + par) * d.T_max + t;
}

// Spin until *p >= target (acquire at system scope); the %globaltimer watchdog turns a
// protocol bug into error 3 instead of a hung GPU.
__device__ __forceinline__ void report_timeout(int* err, int site, uint32_t target, uint32_t seen,
                                               int where) {
  if (atomicCAS(err, 0, 3) == 0) {
    err[1] = site;
    err[2] = (int)target;
    err[3] = (int)seen;
    err[4] = where;
  }
}
// Once any watchdog has fired (err[0] != 0) every later wait gives up at once, so a protocol
// failure costs one timeout, not one per waiting tile.
__device__ __forceinline__ bool aborted(const int* err) {
  return *reinterpret_cast<const volatile int*>(err) != 0;
}
__device__ __forceinline__ void wait_geq_sys(const uint32_t* p, uint32_t target,
                                             unsigned long long timeout, int* err, int site = 0,
                                             int where = 0) {
  if (ld_acquire_sys(p) >= target) return;
  const unsigned long long t0 = globaltimer();
  uint32_t v;
  while ((v = ld_acquire_sys(p)) < target) {
    if (aborted(err)) return;
    if (globaltimer() - t0 > timeout) {
      report_timeout(err, site, target, v, where);
      return;
    }
  }
}
__device__ __forceinline__ void wait_eq_sys(const uint32_t* p, uint32_t want,
                                            unsigned long long timeout, int* err, int site = 0,
                                            int where = 0) {
  if (ld_acquire_sys(p) == want) return;
  const unsigned long long t0 = globaltimer();
  uint32_t v;
  while ((v = ld_acquire_sys(p)) != want) {
    if (aborted(err)) return;
    if (globaltimer() - t0 > timeout) {
      report_timeout(err, site, want, v, where);
      return;
    }
  }
}

// Entry check of every MegaKernel: the planner aborted this iteration (routing checks, receive
// capacity of any rank, count-exchange timeout: p.scalars[3]) or an earlier kernel's watchdog fired
// (sticky until eplab_check). Nothing of the iteration is read or written -- in particular no row
// is pushed into a peer's symmetric buffers.
__device__ __forceinline__ bool iteration_aborted(const MkArgs& a) {
  return *reinterpret_cast<const volatile int*>(a.p.scalars + 3) != 0 || aborted(a.err);
}

// Local expert of a global 128-row block index g (binary search over mblock_pre).
__device__ __forceinline__ int expert_of_block(const PlanDev& p, int epr, long long g) {
  int lo = 0, hi = epr - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((long long)p.mblock_pre[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// NT tile t of a GEMM with `nb` column blocks over the receive layout, rasterised in groups
// of G row blocks (column-major inside a group) so a group's A rows and the weight panel
// stay resident in L2.
constexpr int RASTER_G = 16;
__device__ __forceinline__ void decode_nt(const Dims& d, const PlanDev& p, int t, int nb, int& e,
                                          int& mblk, int& nblk) {
  e = expert_of_block(p, d.epr, (long long)t / nb);
  const int local = t - p.mblock_pre[e] * nb;
  const int mbs = p.mblocks[e];
  const int g = local / (RASTER_G * nb);
  const int gsz = min(RASTER_G, mbs - g * RASTER_G);
  const int r = local - g * RASTER_G * nb;
  nblk = r / gsz;
  mblk = g * RASTER_G + r % gsz;
}

__device__ __forceinline__ TileDesc nt_tile(const Dims& d, const PlanDev& p, int t, int nb,
                                            int bn_cols, int nkb) {
  int e, mb, nbk;
  decode_nt(d, p, t, nb, e, mb, nbk);
  TileDesc td;
  const int ge = d.rank * d.epr + e;
  td.e = e;
  td.m0 = p.sb_all[ge] + mb * BM;
  td.rows = min(BM, p.rt_all[ge] - mb * BM);
  td.n0 = nbk * bn_cols;
  td.kb0 = 0;
  td.nkb = nkb;
  td.pad0 = nbk;
  td.pad1 = 0;
  return td;
}

// Transposed (weight-gradient) tile t: output [NO][KO] per expert in BM x BN tiles, rasterised
// in groups of 8 output row blocks with the column blocks outer inside a group, so the ~148
// tiles in flight touch 8 A panels and ~18 B panels (each panel = all of the expert's rows).
constexpr int TN_G = 8;
__device__ __forceinline__ TileDesc tn_tile(const Dims& d, const PlanDev& p, int t, int NO, int KO) {
  const int mb = NO / BM, nb = KO / BN, per_e = mb * nb;
  TileDesc td;
  td.e = t / per_e;
  const int l = t - td.e * per_e;
  const int g = l / (TN_G * nb);
  const int gsz = min(TN_G, mb - g * TN_G);
  const int r = l - g * TN_G * nb;
  td.m0 = (g * TN_G + r % gsz) * BM;
  td.n0 = (r / gsz) * BN;
  const int ge = d.rank * d.epr + td.e;
  td.kb0 = p.sb_all[ge];
  td.nkb = p.mblocks[td.e] * (BM / BK);
  td.rows = BM;
  td.pad0 = td.n0 / BN;
  td.pad1 = 1;  // transposed tile
  return td;
}

// CTA-pair tiles: 256 token rows (two 128-row blocks of one expert; the second may be empty
// when the expert has an odd number of blocks) x column block, grouped raster of 8 pairs.
constexpr int RASTER_GP = 8;  // default raster group (MkArgs.rgp / EPLAB_RGP override)
__device__ __forceinline__ int expert_of_pair(const PlanDev& p, int epr, long long g) {
  int lo = 0, hi = epr - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((long long)p.mpair_pre[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}
__device__ __forceinline__ TileDesc nt_tile_pair(const Dims& d, const PlanDev& p, int t, int nb,
                                                 int bn_cols, int nkb, int G = RASTER_GP) {
  const int e = expert_of_pair(p, d.epr, (long long)t / nb);
  const int local = t - p.mpair_pre[e] * nb;
  const int mps = p.mpair_pre[e + 1] - p.mpair_pre[e];
  const int g = local / (G * nb);
  const int gsz = min(G, mps - g * G);
  const int r = local - g * G * nb;
  const int nbk = r / gsz, mp = g * G + r % gsz;
  TileDesc td;
  const int ge = d.rank * d.epr + e;
  td.e = e;
  td.m0 = p.sb_all[ge] + mp * 2 * BM;
  td.rows = min(2 * BM, p.rt_all[ge] - mp * 2 * BM);
  td.n0 = nbk * bn_cols;
  td.kb0 = 0;
  td.nkb = nkb;
  td.pad0 = nbk;
  td.pad1 = 0;
  return td;
}
constexpr int TN_GP = 4;
__device__ __forceinline__ TileDesc tn_tile_pair(const Dims& d, const PlanDev& p, int t, int NO,
                                                 int KO, int G = TN_GP) {
  const int mb = NO / (2 * BM), nb = KO / BN, per_e = mb * nb;
  TileDesc td;
  td.e = t / per_e;
  const int l = t - td.e * per_e;
  const int g = l / (G * nb);
  const int gsz = min(G, mb - g * G);
  const int r = l - g * G * nb;
  td.m0 = (g * G + r % gsz) * 2 * BM;
  td.n0 = (r / gsz) * BN;
  const int ge = d.rank * d.epr + td.e;
  td.kb0 = p.sb_all[ge];
  td.nkb = p.mblocks[td.e] * (BM / BK);
  td.rows = 2 * BM;
  td.pad0 = td.n0 / BN;
  td.pad1 = 1;
  return td;
}
__device__ __forceinline__ TileDesc half_tile(const TileDesc& td, uint32_t rank) {
  TileDesc h = td;
  h.m0 = td.m0 + BM * (int)rank;
  h.rows = td.pad1 ? BM : max(0, min(BM, td.rows - BM * (int)rank));
  return h;
}
// scoreboard wait of an NT pair tile: both 128-row blocks (the second only if it has rows)
__device__ __forceinline__ void wait_pair_rows(const MkArgs& a, int ph, const TileDesc& td, int site) {
  if (a.unfused) return;  // rows scattered before the launch
  const SymPtrs& me = a.peers.p[a.d.rank];
  const int g = td.m0 >> 7;
  wait_geq_sys(rg_counter(me, a.d, ph, PAR(a), g), (uint32_t)min(BM, td.rows), a.timeout_ns, a.err, site, g);
  if (td.rows > BM)
    wait_geq_sys(rg_counter(me, a.d, ph, PAR(a), g + 1), (uint32_t)(td.rows - BM), a.timeout_ns, a.err, site,
                 g + 1);
}

__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// Even split of n into parts (sim.cpp:151-161).
__device__ __forceinline__ void even_slice(long long n, int parts, int i, long long& lo,
                                           long long& hi) {
  const long long base = n / parts, rem = n % parts;
  lo = i * base + (i < rem ? i : rem);
  hi = lo + base + (i < rem ? 1 : 0);
}

// ------------------------------------------------------------------ comm role
// Row copy with U independent 16-byte loads in flight per lane (Guideline 7 / 13).
template <int U>
__device__ __forceinline__ void warp_copy_row(int4* __restrict__ dst, const int4* __restrict__ src,
                                              int vecs, int lane) {
  int c = lane;
  for (; c + (U - 1) * 32 < vecs; c += U * 32) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_nc_v4(src + c + u * 32);
#pragma unroll
    for (int u = 0; u < U; ++u) dst[c + u * 32] = v[u];
  }
  for (; c < vecs; c += 32) dst[c] = ld_nc_v4(src + c);
}


// Comm role. The rows of a slice of the priority-ordered send schedule (token_map.cpp:108-126)
// are moved by the TMA bulk-copy engine: one elected thread streams them global -> smem slot ->
// destination slot (a peer's symmetric receive buffer over NVLink, or the local one), keeping
// NSLOT rows in flight through the CTA's (idle during this phase) GEMM stage buffers. A row's
// scoreboard release (rowgroup counter, or per-slot flags for the relay) is issued only after its
// bulk store has completed. ph = 0 forward (x rows), 1 backward (dY rows; warps 1..7 meanwhile
// fold the gate gradient <dY_t, o_{t,j}> of every item of the slice).
// One issuer (lane 0 of warp `iss`) of the comm role: rows p = iss, iss + ISS, ... of the round
// through its NS = NSLOT / ISS slots. A single issuing thread is limited to ~0.55 us per row
// (tools/bulk_copy_probe.cu), so ISS independent issuers share the CTA's slots.
template <int NSLOT, int ISS>
__device__ void comm_pipeline(const MkArgs& a, int ph, GemmSmem* S, uint8_t* sbuf, int cnt, int iss) {
  constexpr int NS = NSLOT / ISS;            // slots owned by this issuer
  constexpr int L = NS / 2;                  // loads run L rows ahead of stores
  constexpr uint32_t SLOT = 196608 / NSLOT;  // bytes per slot
  const Dims& d = a.d;
  const int k = d.topk, H = d.H;
  const uint32_t row_bytes = (uint32_t)H * 2;
  const __nv_bfloat16* src_base = ph == 0 ? a.x : a.dy;
  const int slot0 = iss * NS;
  int* crel = S->crel[iss];
  uint32_t par = S->cphase[iss];
  int n_loaded = 0, n_stored = 0, n_released = 0;
  // Publish items [n_released, upto) whose bulk stores have completed: one async-proxy fence and
  // one system-scope release fence for the batch, then relaxed scoreboard updates (the fence +
  // relaxed-store release pattern), rowgroup counts aggregated over consecutive items.
  auto release_upto = [&](int upto) {
    if (n_released >= upto) return;
    fence_proxy_async_global();
    fence_acq_rel_sys();
    uint32_t* cur = nullptr;
    uint32_t run = 0;
    for (; n_released < upto; ++n_released) {
      const int pp = crel[n_released & 63];
      const SymPtrs& P = a.peers.p[S->cdst[pp]];
      const int slot = S->cslot[pp];
      if (a.n_relay > 0) {
        st_relaxed_sys(P.slot_flag + slot, EPOCH(a) * 2 + ph);
      } else {
        uint32_t* c = rg_counter(P, d, ph, PAR(a), slot >> 7);
        if (c != cur) {
          if (cur) red_relaxed_sys_add(cur, run);
          cur = c;
          run = 0;
        }
        ++run;
      }
    }
    if (cur) red_relaxed_sys_add(cur, run);
  };
  for (int p = iss; p < cnt + ISS; p += ISS) {
    if (p < cnt && S->cdst[p] >= 0) {
      const int q = n_loaded, slot = slot0 + q % NS;
      if (q >= NS) {  // slot reuse: the stores of items <= q - NS must be complete
        tma_store_wait<NS - L - 1>();
        if (q - NS + 1 - n_released >= 16) release_upto(q - NS + 1);  // <= 64 pending
      }
      mbar_arrive_expect_tx(&S->cbar[slot], row_bytes);
      bulk_load(sbuf + slot * SLOT, src_base + (size_t)(S->citem[p] / k) * H, row_bytes, &S->cbar[slot]);
      S->cpos[slot] = p;
      crel[q & 63] = p;
      ++n_loaded;
    }
    while (n_stored < n_loaded && (n_loaded - n_stored > L || p >= cnt)) {
      const int ls = n_stored % NS, slot = slot0 + ls, pp = S->cpos[slot];
      mbar_wait(&S->cbar[slot], (par >> ls) & 1u);
      par ^= 1u << ls;
      const SymPtrs& P = a.peers.p[S->cdst[pp]];
      bulk_store((ph == 0 ? P.recv_x : P.recv_dy) + (size_t)S->cslot[pp] * H, sbuf + slot * SLOT,
                 row_bytes);
      tma_store_commit();
      ++n_stored;
    }
  }
  tma_store_wait<0>();
  release_upto(n_loaded);
  S->cphase[iss] = par;
}

// Comm role (default mover): a pool of 32-item rounds of the priority-ordered send schedule
// (token_map.cpp:108-126), claimed in order from one atomic round counter by every comm
// worker -- the 8 warps of each comm CTA (SM split, n_disp) and the spare warps of the GEMM
// CTAs (warp split: warp 2 of both CTAs of a pair, warps 1 and 3 of the non-leader CTA). A
// warp moves its round with 16-byte loads/stores, CNR rows in flight (CNR x 8 x 16 B per lane). Then
// it releases the round: one system-scope fence, relaxed rowgroup counter updates aggregated per
// counter (relay off) or per-slot epoch flags (relay on).
constexpr int CROUNDS = 128;
#ifndef EPLAB_CNR
#define EPLAB_CNR 4
#endif
constexpr int CNR = EPLAB_CNR;  // rows in flight per comm warp
__device__ void comm_round_warp(const MkArgs& a, int ph, long long r) {
  const Dims& d = a.d;
  const int k = d.topk, vecs = d.H / 8, me = d.rank;
  const int lane = threadIdx.x & 31;
  const long long n = (long long)a.p.n_tok * k;
  // Super-rounds of CROUNDS rounds x 32 items: round g of a super-round takes the items
  // g, g + CROUNDS, g + 2 CROUNDS, ... so the CROUNDS warps working a super-round move its
  // schedule front to back together -- the first 128-row rowgroup (the first GEMM tiles' rows)
  // lands after one row copy instead of after a whole round.
  const long long sr = r / CROUNDS, g = r - sr * CROUNDS;
  const long long idx = sr * CROUNDS * 32 + g + (long long)lane * CROUNDS;
  // experiment (dbg 2048 + timeline): cycles per section of the round (metadata, copies, release)
  const bool sect = (a.dbg & 2048) && a.tl.rec && lane == 0;
  long long cs[5] = {0, 0, 0, 0, 0}, ct = sect ? clock64() : 0;
  const unsigned long long gt0 = sect ? globaltimer() : 0;
  auto mark = [&](int i) {
    if (sect) {
      const long long nw = clock64();
      cs[i] += nw - ct;
      ct = nw;
    }
  };
  int item = -1, slot = 0, dst = -1;  // dst < 0: the row does not travel from here
  if (idx < n) {
    const int i = a.p.sched[idx];
    const int t = i / k;
    const int e = a.p.topk_ids[i];
    const int dr = e / d.epr, el = e - dr * d.epr;
    slot = a.p.dst_slot[i];
    int prim_j = -1, best = el;
    if (a.n_relay > 0)  // relay on: the first (token, dst) replica in priority order travels
      for (int jj = 0; jj < k; ++jj) {
        const int e2 = a.p.topk_ids[t * k + jj];
        if (e2 / d.epr == dr && e2 - dr * d.epr < best) {
          best = e2 - dr * d.epr;
          prim_j = jj;
        }
      }
    const SymPtrs& P = a.peers.p[dr];
    const int prim_slot = prim_j >= 0 ? a.p.dst_slot[t * k + prim_j] : -1;
    if (ph == 0) P.meta[slot] = SlotMeta{me, i, a.p.gate_w[i], prim_slot};
    // a duplicate's flag means "metadata valid"; the relay copies it after the primary's flag
    if (prim_slot >= 0) st_release_sys(P.slot_flag + slot, EPOCH(a) * 2 + ph);
    item = i;
    dst = prim_slot >= 0 ? -1 : dr;
  }
  if (sect) asm volatile("" ::"r"(item), "r"(slot), "r"(dst));
  __syncwarp();
  mark(0);
  const int4* src_base = reinterpret_cast<const int4*>(ph == 0 ? a.x : a.dy);
  auto dst_row = [&](int dr, int sl) {
    const SymPtrs& P = a.peers.p[dr];
    return reinterpret_cast<int4*>(ph == 0 ? P.recv_x : P.recv_dy) + (size_t)sl * vecs;
  };
  // Release copied rows (fence + relaxed updates): after the first two
  // copies of the round (the super-round's warps then complete its first rowgroups together)
  // and at the end of the round (more frequent releases cost comm throughput: Qwen3's dY comm
  // tasks 770 -> 873 us with a release every 8 rows).
  unsigned done = 0, copied = 0;  // items released / items copied (lane bits)
  int n_copies = 0;
  auto release = [&]() {
    const unsigned rel = copied & ~done;
    if (!rel) return;
    __syncwarp();
    mark(1);
    if (d.world == 1)
      fence_acq_rel_gpu();  // one GPU: every reader is on this device
    else
      fence_acq_rel_sys();
    const bool mine = (rel >> lane) & 1u;
    if (a.n_relay > 0) {
      if (mine) st_relaxed_sys(a.peers.p[dst].slot_flag + slot, EPOCH(a) * 2 + ph);
    } else {
      uint32_t* ctr = mine ? rg_counter(a.peers.p[dst], d, ph, PAR(a), slot >> 7) : nullptr;
      const unsigned mm = __match_any_sync(0xffffffffu, (unsigned long long)ctr);
      if (ctr && lane == __ffs(mm) - 1) red_relaxed_sys_add(ctr, (uint32_t)__popc(mm));
    }
    done |= rel;
    __syncwarp();
    mark(2);
  };
  auto progress = [&]() {
    if (n_copies <= CNR) release();
  };
  // x rows (forward) and dY rows (backward) alike: a pure row copy, CNR rows in flight. (The gate
  // gradient is no longer folded here: the down-dgrad epilogue has <dY W_down, h> per row in
  // registers, so the comm warps no longer read the o replica rows -- a third of the backward
  // dispatch's bytes.)
  {
    // experiment: dbg 512 skips the row copies (rows of the previous identical step stay in place)
    unsigned m = (a.dbg & 512) ? 0u : __ballot_sync(0xffffffffu, dst >= 0);
    if (a.dbg & 512) copied = __ballot_sync(0xffffffffu, dst >= 0);
    while (m) {
      // up to CNR rows per pass, CNR x 8 x 16 B loads in flight per lane (the copy is
      // latency-bound: bytes in flight per warp set its rate)
      int4* dp[CNR];
      const int4* sp[CNR];
      int nr = 0;
#pragma unroll
      for (int q = 0; q < CNR; ++q) {
        const int qq = m ? __ffs(m) - 1 : -1;
        if (m) m &= m - 1;
        const int src_q = qq < 0 ? 0 : qq;
        const int it_ = __shfl_sync(0xffffffffu, item, src_q);
        const int sl_ = __shfl_sync(0xffffffffu, slot, src_q);
        const int ds_ = __shfl_sync(0xffffffffu, dst, src_q);
        sp[q] = qq < 0 ? nullptr : src_base + (size_t)(it_ / k) * vecs;
        dp[q] = qq < 0 ? nullptr : dst_row(ds_, sl_);
        if (qq >= 0) {
          copied |= 1u << qq;
          ++nr;
        }
      }
      for (int c = lane; c < vecs; c += 256) {
        int4 v[CNR][8];
#pragma unroll
        for (int q = 0; q < CNR; ++q)
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (q < nr && c + 32 * u < vecs) v[q][u] = ld_nc_v4(sp[q] + c + 32 * u);
        if (sect) {  // section accounting: wait for every load of the pass, then time the stores
          uint32_t z = 0;
#pragma unroll
          for (int q = 0; q < CNR; ++q)
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (q < nr && c + 32 * u < vecs) z ^= (uint32_t)v[q][u].x;
          asm volatile("" ::"r"(z));
          mark(3);
        }
#pragma unroll
        for (int q = 0; q < CNR; ++q)
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (q < nr && c + 32 * u < vecs) dp[q][c + 32 * u] = v[q][u];
        mark(4);
      }
      n_copies += nr;
      progress();
    }
  }
  release();
  if (sect)
    for (int i = 0; i < 5; ++i) timeline_push(a.tl, gt0, gt0 + (unsigned long long)cs[i], ROLE_COMM, -9021 - i);
}

// A comm worker warp: claim rounds until the pool is empty. Returns the number of rounds moved.
__device__ int comm_rounds(const MkArgs& a, int ph) {
  // whole super-rounds (the last may be partly empty: items beyond n are skipped)
  const long long n_items = (long long)a.p.n_tok * a.d.topk;
  const long long n_rounds = (n_items + 32 * CROUNDS - 1) / (32 * CROUNDS) * CROUNDS;
  const int lane = threadIdx.x & 31;
  int done = 0;
  for (;;) {
    long long r = 0;
    if (lane == 0) r = atomicAdd(reinterpret_cast<unsigned long long*>(a.comm_cursor), 1ull);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (r >= n_rounds) break;
    comm_round_warp(a, ph, r);
    ++done;
  }
  return done;
}

__device__ void comm_task(const MkArgs& a, int task, int ph, GemmSmem* S, uint8_t* sbuf) {
  if (!a.comm_bulk) {  // every warp of the comm CTA drains the round pool
    comm_rounds(a, ph);
    return;
  }
  const Dims& d = a.d;
  const int k = d.topk, H = d.H, me = d.rank;
  const long long n = (long long)a.p.n_tok * k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool relay_on = a.n_relay > 0;
  // Rounds of 256 schedule items are dealt round-robin to the comm tasks, so all comm CTAs move
  // through the priority order front to back together and the first rowgroups (the first GEMM
  // tiles' inputs) land after ~1/n_disp of the single-slice time.
  for (long long b0 = (long long)task * GEMM_THREADS; b0 < n; b0 += (long long)a.n_disp * GEMM_THREADS) {
    const long long hi = n;
    const int cnt = (hi - b0) < GEMM_THREADS ? (int)(hi - b0) : GEMM_THREADS;
    // ---- parallel metadata: one thread per item. Writes the destination slot's return
    // address (forward) and, relay on, publishes duplicate slots right away: their flag means
    // "metadata valid", the relay then waits for the primary slot's flag before copying.
    if ((int)threadIdx.x < cnt) {
      const int i = a.p.sched[b0 + threadIdx.x];
      const int t = i / k;
      const int e = a.p.topk_ids[i];
      const int dst = e / d.epr, el = e - dst * d.epr;
      const int slot = a.p.dst_slot[i];
      int prim_j = -1, best = el;
      if (relay_on)
        for (int jj = 0; jj < k; ++jj) {
          const int e2 = a.p.topk_ids[t * k + jj];
          if (e2 / d.epr == dst && e2 - dst * d.epr < best) {
            best = e2 - dst * d.epr;
            prim_j = jj;
          }
        }
      const SymPtrs& P = a.peers.p[dst];
      const int prim_slot = prim_j >= 0 ? a.p.dst_slot[t * k + prim_j] : -1;
      if (ph == 0) P.meta[slot] = SlotMeta{me, i, a.p.gate_w[i], prim_slot};
      if (prim_slot >= 0) st_release_sys(P.slot_flag + slot, EPOCH(a) * 2 + ph);
      S->citem[threadIdx.x] = i;
      S->cslot[threadIdx.x] = slot;
      S->cdst[threadIdx.x] = prim_slot >= 0 ? -1 : dst;
    }
    __syncthreads();
    // bulk-copy engine mover (EPLAB_COMM=bulk; the round-1 default, kept for comparison:
    // 436 / 747 us vs 386 / 645 us for the Qwen3 fwd / bwd comm tasks, profiles/r01_comm_movers.txt)
    const int n_iss = H <= 4096 ? 4 : 2;  // 14 KB rows: 2 issuers x 6 slots
    if (warp < n_iss) {  // issuer warps
      if (lane == 0) {
        if (H <= 2048)
          comm_pipeline<48, 4>(a, ph, S, sbuf, cnt, warp);
        else if (H <= 4096)
          comm_pipeline<24, 4>(a, ph, S, sbuf, cnt, warp);
        else
          comm_pipeline<12, 2>(a, ph, S, sbuf, cnt, warp);
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ relay role
// Relay workers (relay on; sim.cpp:418-441) are a pool of destination
// rowgroups claimed in order by warps -- the n_relay relay CTAs' 8 warps and, after the comm
// pool is drained, the GEMM CTAs' spare warps. A warp takes a whole rowgroup: each lane polls the
// metadata flags of its slots (and, for duplicates, the primary slot's row flag), the warp copies
// every duplicate from its primary slot in HBM (two rows in flight), then publishes the rowgroup
// count (sim.cpp:601-618).
__device__ void relay_rowgroup(const MkArgs& a, int ph, int g) {
  const Dims& d = a.d;
  const SymPtrs& me = a.peers.p[d.rank];
  const int lane = threadIdx.x & 31;
  const uint32_t flagv = EPOCH(a) * 2 + ph;
  const int4* recv = reinterpret_cast<const int4*>(ph == 0 ? me.recv_x : me.recv_dy);
  int4* recv_w = reinterpret_cast<int4*>(ph == 0 ? me.recv_x : me.recv_dy);
  const int vecs = d.H / 8;
  const int el = expert_of_block(a.p, d.epr, g);
  const int ge = d.rank * d.epr + el;
  const int rows = min(BM, a.p.rt_all[ge] - (g - a.p.mblock_pre[el]) * BM);
  for (int r0 = 0; r0 < rows; r0 += 32) {
    const int s = g * BM + r0 + lane;
    const bool live = r0 + lane < rows;
    int prim = -1;
    // lane-parallel waits: metadata flag of my slot, then (duplicate) the primary's row flag
    const unsigned long long t0 = globaltimer();
    bool ok = !live;
    while (!__all_sync(0xffffffffu, ok)) {
      if (!ok) {
        if (prim < 0 && ld_acquire_sys(me.slot_flag + s) == flagv) {
          prim = me.meta[s].primary;  // >= 0: a duplicate -- wait for its primary's row
          ok = prim < 0;
        }
        if (prim >= 0 && ld_acquire_sys(me.slot_flag + prim) == flagv) ok = true;
      }
      const bool late = globaltimer() - t0 > a.timeout_ns;
      if (__any_sync(0xffffffffu, aborted(a.err) || late)) {  // warp-uniform exit
        if (late && !ok) report_timeout(a.err, 10 + ph, flagv, 0, s);
        return;
      }
      // back off between polls: hundreds of lanes spinning on acquire loads starve the comm
      // rounds and GEMM producers sharing L2 (measured: EP=2 relay dispatch 7 ms -> <1 ms)
      if (!__all_sync(0xffffffffu, ok)) __nanosleep(200);
    }
    unsigned m = __ballot_sync(0xffffffffu, live && prim >= 0);
    while (m) {
      const int qa = __ffs(m) - 1;
      m &= m - 1;
      const int qb = m ? __ffs(m) - 1 : qa;
      if (m) m &= m - 1;
      const bool two = qb != qa;
      const int pa = __shfl_sync(0xffffffffu, prim, qa), pb = __shfl_sync(0xffffffffu, prim, qb);
      const int4* sa = recv + (size_t)pa * vecs;
      const int4* sb = recv + (size_t)pb * vecs;
      int4* da = recv_w + (size_t)(g * BM + r0 + qa) * vecs;
      int4* db = recv_w + (size_t)(g * BM + r0 + qb) * vecs;
      for (int c = lane; c < vecs; c += 256) {
        int4 va[8], vb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c + 32 * u < vecs) {
            va[u] = sa[c + 32 * u];
            if (two) vb[u] = sb[c + 32 * u];
          }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c + 32 * u < vecs) {
            da[c + 32 * u] = va[u];
            if (two) db[c + 32 * u] = vb[u];
          }
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    red_release_gpu_add(rg_counter(me, d, ph, PAR(a), g), (uint32_t)rows);
  }
}

// A relay worker warp: claim rowgroups until the pool is empty. Returns the number handled.
__device__ int relay_rowgroups(const MkArgs& a, int ph) {
  const int n_rg = a.p.scalars[1];
  const int lane = threadIdx.x & 31;
  int done = 0;
  for (;;) {
    int g = 0;
    if (lane == 0) g = (int)atomicAdd(a.relay_cursor, 1u);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= n_rg) break;
    const unsigned long long t0 = globaltimer();
    relay_rowgroup(a, ph, g);
    if (lane == 0 && (a.dbg & 128)) timeline_push(a.tl, t0, globaltimer(), ROLE_RELAY, 100000 + g);
    ++done;
  }
  return done;
}

__device__ void relay_task(const MkArgs& a, int, int ph) { relay_rowgroups(a, ph); }

// ------------------------------------------------------------------ reduce role
// Top-k completeness barrier, then the reference's canonical fold (precision.cpp:31-37
// `fold` with FpFormat::Binary32): acc = w_0 * o_0, acc = acc + w_j * o_j for j ascending, every
// product and sum rounded to fp32 (no FMA contraction), then one RNE to bf16:
// y = round_to_bf16(accumulate(plan, Binary32)) bit for bit; backward dx the same fold with unit
// weights (dx = bf16(dX_0 + dX_1 + ...)). The fold of one token is a warp job: the token's k
// replica rows are one contiguous block [t*k, t*k+k) x H, each lane keeps KT x U 16-byte loads in
// flight (KT >= k replicas x U column chunks, 16 per lane), so the HBM-bound fold is not
// latency-bound.
template <int KT>
__device__ __forceinline__ void fold_token(const MkArgs& a, int ph, long long t) {
  constexpr int U = 16 / KT;
  const Dims& d = a.d;
  const int k = d.topk, vecs = d.H / 8;
  const SymPtrs& me = a.peers.p[d.rank];
  const int lane = threadIdx.x & 31;
  const int4* rep = reinterpret_cast<const int4*>(ph == 0 ? me.rep : me.rep_dx);
  int4* out = reinterpret_cast<int4*>(ph == 0 ? a.y : a.dx);
  float w[KT];
#pragma unroll
  for (int j = 0; j < KT; ++j) w[j] = (j < k && ph == 0) ? a.p.gate_w[t * k + j] : 1.0f;
  const int4* base = rep + (size_t)t * k * vecs;
  for (int c = lane; c < vecs; c += 32 * U) {
    int4 v[KT][U];
#pragma unroll
    for (int j = 0; j < KT; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j < k && c + 32 * u < vecs) v[j][u] = base[(size_t)j * vecs + c + 32 * u];
    float acc[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[u][q] = 0.f;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      if (j >= k) break;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&v[j][u]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(hv[q]);
          // fp32 product and sum rounded separately (__fmul_rn / __fadd_rn are never contracted);
          // j = 0 starts the fold with the product itself (keeps the sign of a -0 term)
          const float px = ph == 0 ? __fmul_rn(w[j], f.x) : f.x;
          const float py = ph == 0 ? __fmul_rn(w[j], f.y) : f.y;
          acc[u][2 * q] = j == 0 ? px : __fadd_rn(acc[u][2 * q], px);
          acc[u][2 * q + 1] = j == 0 ? py : __fadd_rn(acc[u][2 * q + 1], py);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c + 32 * u >= vecs) continue;
      int4 o;
      o.x = (int)pack_bf16(acc[u][0], acc[u][1]);
      o.y = (int)pack_bf16(acc[u][2], acc[u][3]);
      o.z = (int)pack_bf16(acc[u][4], acc[u][5]);
      o.w = (int)pack_bf16(acc[u][6], acc[u][7]);
      out[(size_t)t * vecs + c + 32 * u] = o;
    }
  }
  if (ph == 1 && lane < k) {  // the token's gate gradients: its k entries' partials, tiles in order
    const int ncb = d.F / BN;
    const float* g = me.dgp + ((size_t)t * k + lane) * ncb;
    float s = g[0];
    for (int c = 1; c < ncb; ++c) s = __fadd_rn(s, g[c]);
    a.dgate[t * k + lane] = s;
  }
}

// Reduce workers: warps claim RCHUNK-token chunks from one atomic counter (the post-task CTAs
// after their GEMM tiles and, in the backward combine, the GEMM CTAs' spare warps from the start:
// there dX tokens complete during the up-dgrad tiles and fold under the up-wgrad tiles that
// follow). A warp polls its chunk's arrival counters (lane i <-> token i) and folds the tokens in
// the order they complete; who folds a token and when never changes its value. (In the forward
// combine no tiles follow the down GEMM and, with random routing, tokens complete with its last
// tiles: spare warps would only hold chunks they fold slowly, so they stay out.)
constexpr int RCHUNK = 8;
template <int KT>
__device__ void reduce_chunks_t(const MkArgs& a, int ph, bool backoff, const SpareStop* stop) {
  const Dims& d = a.d;
  const SymPtrs& me = a.peers.p[d.rank];
  const int lane = threadIdx.x & 31;
  const uint32_t need = (uint32_t)(d.topk * (d.H / BN));
  const int n_chunks = (a.p.n_tok + RCHUNK - 1) / RCHUNK;
  for (;;) {
    // spare workers hand the rest to the post-task CTAs once the GEMM phase ends: a spare warp
    // folds ~5x slower than a whole post-task CTA, and its CTA cannot move on to the post-tasks
    // while it holds chunks (k <= 4, 32K tokens: bwd combine 1.04 -> 0.62 ms)
    if (stop && stop->tiles_claimed()) break;
    int c = 0;
    if (lane == 0) c = (int)atomicAdd(a.red_cursor, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= n_chunks) break;
    const long long t = (long long)c * RCHUNK + lane;
    unsigned todo = __ballot_sync(0xffffffffu, lane < RCHUNK && t < a.p.n_tok);
    const unsigned long long t0 = globaltimer();
    while (todo) {
      bool ready = false;
      if ((todo >> lane) & 1u) ready = ld_acquire_sys(tok_counter(me, d, ph, PAR(a), (int)t)) >= need;
      unsigned r = __ballot_sync(0xffffffffu, ready);
      if (!r) {
        if (aborted(a.err)) return;
        if (globaltimer() - t0 > a.timeout_ns) {
          if (lane == 0) report_timeout(a.err, 20 + ph, need, 0, (int)(c * RCHUNK + __ffs(todo) - 1));
          return;
        }
        if (backoff) __nanosleep(500);  // (post-task pollers must not sleep: 100 ns costs 0.1-0.4 ms)
        continue;
      }
      todo &= ~r;
      while (r) {
        const int i = __ffs(r) - 1;
        r &= r - 1;
        fold_token<KT>(a, ph, (long long)c * RCHUNK + i);
      }
    }
  }
}

__device__ void reduce_chunks(const MkArgs& a, int ph, bool backoff, const SpareStop* stop = nullptr) {
  if (a.dbg & 64) return;  // experiment: no reduce (wrong y / dx; measures the reduce's share)
  if (a.d.topk <= 8)
    reduce_chunks_t<8>(a, ph, backoff, stop);
  else
    reduce_chunks_t<16>(a, ph, backoff, stop);
}

__device__ void reduce_task(const MkArgs& a, int, int ph) { reduce_chunks(a, ph, false); }

// spare warps of the backward combine MegaKernel's GEMM CTAs join the reduce pool from the start
__device__ __forceinline__ void spare_reduce(const MkArgs& a, const Timeline& tl, int ph, const SpareStop& stop) {
  if (!(a.spare_warps & 2)) return;
  const unsigned long long t0 = globaltimer();
  reduce_chunks(a, ph, true, &stop);
  if ((threadIdx.x & 31) == 0) timeline_push(tl, t0, globaltimer(), ROLE_REDUCE, -1 - (int)(threadIdx.x >> 5));
}

// ------------------------------------------------------------------ GEMM modes
// tensor maps: m[0]/m[1] = A/B of the first tile type, m[2]/m[3] = A/B of the second.

// Forward up projection: A = recv_x (K-major over H), B = W_up gate rows [f0,f0+128) and up
// rows [F+f0, ..) (K-major). Epilogue: GU (bf16) and h = bf16(silu(g) * u) from the bf16 g, u.
// Spare warps of the dispatch MegaKernels' GEMM CTAs drain the comm pool too (warp split);
// their activity goes into the device timeline as one comm interval per warp.
__device__ __forceinline__ void spare_comm(const MkArgs& a, const Timeline& tl, int ph) {
  if (!(a.spare_warps & 1) || a.comm_bulk) return;
  unsigned long long t0 = globaltimer();
  const int n = comm_rounds(a, ph);
  if (n > 0 && (threadIdx.x & 31) == 0) timeline_push(tl, t0, globaltimer(), ROLE_COMM, -1 - (int)(threadIdx.x >> 5));
  if (a.n_relay > 0) {  // then the relay pool (it waits on rows; the comm pool never waits)
    t0 = globaltimer();
    const int nr = relay_rowgroups(a, ph);
    if (nr > 0 && (threadIdx.x & 31) == 0)
      timeline_push(tl, t0, globaltimer(), ROLE_RELAY, -1 - (int)(threadIdx.x >> 5));
  }
}

struct ModeUp {
  using Args = MkArgs;
  static constexpr bool HAS_TILE_DONE = false;
  static constexpr bool SPARE = true;
  __device__ static void spare(const Args& a, const Timeline& tl, const SpareStop&) { spare_comm(a, tl, 0); }
  __device__ static int a_mn(const TileDesc&) { return 0; }
  __device__ static int b_mn(const TileDesc&) { return 0; }
  __device__ static TileDesc tile(const Args& a, int t) {
    return nt_tile(a.d, a.p, t, a.d.F / 128, 128, a.d.H / BK);
  }
  __device__ static void before_loads(const Args& a, const TileDesc& td) {
    if (a.unfused) return;
    const SymPtrs& me = a.peers.p[a.d.rank];
    wait_geq_sys(rg_counter(me, a.d, 0, PAR(a), td.m0 >> 7), (uint32_t)td.rows, a.timeout_ns, a.err,
                 30, td.m0 >> 7);
  }
  __device__ static void epilogue_prefetch(const Args&, const TileDesc&, int) {}
  // ---- CTA pair: rank 0 stages the gate rows, rank 1 the up rows of the same f-block
  __device__ static TileDesc tile_pair(const Args& a, int t) {
    return nt_tile_pair(a.d, a.p, t, a.d.F / 128, 128, a.d.H / BK, a.rgp);
  }
  __device__ static void before_loads_pair(const Args& a, const TileDesc& td) { wait_pair_rows(a, 0, td, 30); }
  __device__ static void load_a_pair(const Args&, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    tma_load_2d_pair(&tm.m[0], bar, s, kb * BK, td.m0 + BM * rank);
  }
  __device__ static void load_b_pair(const Args& a, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    tma_load_2d_pair(&tm.m[1], bar, s, kb * BK, td.e * 2 * a.d.F + td.n0 + rank * a.d.F);
  }
  __device__ static TileDesc half_of(const TileDesc& td, uint32_t rank) { return half_tile(td, rank); }
  __device__ static bool half_has_work(const TileDesc& h) { return h.rows > 0; }
  __device__ static void load_a(const Args&, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    tma_load_2d(&tm.m[0], bar, s, kb * BK, td.m0);
  }
  __device__ static void load_b(const Args& a, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    const int row = td.e * 2 * a.d.F + td.n0;
    tma_load_2d(&tm.m[1], bar, s, kb * BK, row);
    tma_load_2d(&tm.m[1], bar, s + 128 * 128, kb * BK, row + a.d.F);
  }
  __device__ static void epilogue(const Args& a, const TmaSet& tm, const TileDesc& td,
                                  uint32_t taddr, int r, uint8_t* stg) {
    const uint32_t lane = r & 31;
    const bool live = r < td.rows;  // tcgen05.ld is warp-collective: every lane loads
    const int row0 = td.m0 + (r & ~31);
    const int F = a.d.F;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      float g[32], u[32], h[32];
      acc_chunk(taddr, c, g);
      acc_chunk(taddr, 4 + c, u);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float gb = __bfloat162float(__float2bfloat16_rn(g[i]));
        const float ub = __bfloat162float(__float2bfloat16_rn(u[i]));
        h[i] = silu_f(gb) * ub;
      }
      stage_acquire(lane);
      if (live) {
        stage_row(stg, lane, g);
        stage_row(stg + EPI_TILE_BYTES, lane, u);
        stage_row(stg + 2 * EPI_TILE_BYTES, lane, h);
      } else {
        stage_zero_row(stg, lane);
        stage_zero_row(stg + EPI_TILE_BYTES, lane);
        stage_zero_row(stg + 2 * EPI_TILE_BYTES, lane);
      }
      stage_release();
      if (lane == 0) {
        const int col = td.n0 + c * 32;
        tma_store_2d(&tm.m[4], stg, col, row0);                       // GU gate half
        tma_store_2d(&tm.m[4], stg + EPI_TILE_BYTES, F + col, row0);  // GU up half
        tma_store_2d(&tm.m[5], stg + 2 * EPI_TILE_BYTES, col, row0);  // h
        tma_store_commit();
      }
    }
  }
  template <class A>
  __device__ static void tile_done(const A&, const TileDesc&) {}
};

// Push the 128x256 output tile row by row into the source's replica slots (over NVLink when
// the source is a peer) and count the column tile on the source token (combine scoreboard).
// The warp's 32 rows x 64 columns (two accumulator chunks) go through its staging area
// (32 rows x 128 B, 16-byte granules XOR-swizzled by row) so that every store instruction writes
// four whole 128-byte row segments -- full lines to the (possibly remote, over NVLink) replica
// slots instead of 32 scattered 16-byte pieces.
__device__ __forceinline__ void push_rows(const MkArgs& a, const TileDesc& td, uint32_t taddr,
                                          int r, int ph, uint8_t* stg) {
  const int lane = r & 31;
  const bool live = r < td.rows;
  SlotMeta mt{0, 0, 0.f, 0};
  if (live) mt = a.peers.p[a.d.rank].meta[td.m0 + r];
  const SymPtrs& S = a.peers.p[live ? mt.src : 0];
  __nv_bfloat16* dst = a.unfused ? a.ret + (size_t)(live ? a.ret_pos[td.m0 + r] : 0) * a.d.H + td.n0
                                 : (ph == 0 ? S.rep : S.rep_dx) + (size_t)mt.rep * a.d.H + td.n0;
  const unsigned live_mask = __ballot_sync(0xffffffffu, live);
#pragma unroll 1
  for (int c = 0; c < BN / 32; c += 2) {
    float v0[32], v1[32];
    acc_chunk(taddr, c, v0);
    acc_chunk(taddr, c + 1, v1);
    __syncwarp();  // the previous pair's reads of the staging area are done
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float* v = g < 4 ? v0 : v1;
      const int o = (g & 3) * 8;
      const int4 w = make_int4((int)pack_bf16(v[o], v[o + 1]), (int)pack_bf16(v[o + 2], v[o + 3]),
                               (int)pack_bf16(v[o + 4], v[o + 5]), (int)pack_bf16(v[o + 6], v[o + 7]));
      *reinterpret_cast<int4*>(stg + lane * 128 + ((g ^ (lane & 7)) << 4)) = w;
    }
    __syncwarp();
    // 4 rows per instruction, 8 lanes x 16 B per row
    const int sub = lane >> 3, gran = lane & 7;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = i * 4 + sub;
      const unsigned long long dp =
          __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), row);
      if ((live_mask >> row) & 1u) {
        const int4 w = *reinterpret_cast<const int4*>(stg + row * 128 + ((gran ^ (row & 7)) << 4));
        reinterpret_cast<int4*>(reinterpret_cast<__nv_bfloat16*>(dp) + c * 32)[gran] = w;
      }
    }
  }
  __syncwarp();  // staging free for the next tile; every row's stores precede its owner's release
}

// The combine push's scoreboard update (RELEASE_AFTER hook, after the accumulator went back to
// the MMA issuer): this thread's replica row of the tile is counted on its source token.
__device__ __forceinline__ void push_release(const MkArgs& a, const TileDesc& td, int r, int ph) {
  if (a.unfused) return;  // the return all-to-all runs after the kernel
  const bool live = r < td.rows;
  if (a.d.world == 1)
    fence_acq_rel_gpu();  // one GPU: the reducer is on this device
  else
    fence_acq_rel_sys();
  if (!live) return;
  const SlotMeta mt = a.peers.p[a.d.rank].meta[td.m0 + r];
  red_relaxed_sys_add(tok_counter(a.peers.p[mt.src], a.d, ph, PAR(a), mt.rep / a.d.topk), 1u);
}

// The same publication for a whole (half) tile, by the CTA's release warp (CTA-pair engine): the
// four epilogue warps' row stores happen-before this warp through the release queue's mbarrier
// (release / acquire at CTA scope), so ONE cumulative fence of this warp orders all 128 rows before
// the counter updates; the epilogue warps go straight on to the next accumulator.
__device__ __forceinline__ void push_release_tile(const MkArgs& a, const TileDesc& td, int lane, int ph) {
  if (a.unfused) return;
  if (a.d.world == 1)
    fence_acq_rel_gpu();  // one GPU: the reducer is on this device
  else
    fence_acq_rel_sys();
  const SymPtrs& me = a.peers.p[a.d.rank];
  for (int r = lane; r < td.rows; r += 32) {
    const SlotMeta mt = me.meta[td.m0 + r];
    red_relaxed_sys_add(tok_counter(a.peers.p[mt.src], a.d, ph, PAR(a), mt.rep / a.d.topk), 1u);
  }
}

// Pull this row's slot metadata (return address / gate weight) into L1 before the accumulator
// is ready, so the epilogue's first dependent load does not wait on L2.
__device__ __forceinline__ void prefetch_meta_l1(const MkArgs& a, const TileDesc& td, int r) {
  if (td.pad1 || r >= td.rows) return;
  asm volatile("prefetch.global.L1 [%0];" ::"l"(a.peers.p[a.d.rank].meta + td.m0 + r));
}

// Forward down projection + combine push: A = hact (K-major over F), B = W_down (K-major).
struct ModeDown {
  using Args = MkArgs;
  static constexpr bool HAS_TILE_DONE = false;
  static constexpr bool RELEASE_AFTER = true;   // single-CTA engine: per-row release by the epilogue
  static constexpr bool RELEASE_WARP = true;    // CTA-pair engine: per-tile release by warp 2
  __device__ static void epilogue_release(const Args& a, const TileDesc& td, int r) { push_release(a, td, r, 0); }
  __device__ static bool wants_release(const Args& a, const TileDesc&) { return !a.unfused; }
  __device__ static void release_tile(const Args& a, const TileDesc& td, int lane) { push_release_tile(a, td, lane, 0); }
  __device__ static void epilogue_prefetch(const Args& a, const TileDesc& td, int r) { prefetch_meta_l1(a, td, r); }
  __device__ static TileDesc tile_pair(const Args& a, int t) {
    return nt_tile_pair(a.d, a.p, t, a.d.H / BN, BN, a.d.F / BK, a.rgp);
  }
  __device__ static void before_loads_pair(const Args&, const TileDesc&) {}
  __device__ static void load_a_pair(const Args&, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    tma_load_2d_pair(&tm.m[0], bar, s, kb * BK, td.m0 + BM * rank);
  }
  __device__ static void load_b_pair(const Args& a, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    tma_load_2d_pair(&tm.m[2], bar, s, kb * BK, td.e * a.d.H + td.n0 + BM * rank);
  }
  __device__ static TileDesc half_of(const TileDesc& td, uint32_t rank) { return half_tile(td, rank); }
  __device__ static bool half_has_work(const TileDesc& h) { return h.rows > 0; }
  __device__ static int a_mn(const TileDesc&) { return 0; }
  __device__ static int b_mn(const TileDesc&) { return 0; }
  __device__ static TileDesc tile(const Args& a, int t) {
    return nt_tile(a.d, a.p, t, a.d.H / BN, BN, a.d.F / BK);
  }
  __device__ static void before_loads(const Args&, const TileDesc&) {}
  __device__ static void load_a(const Args&, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    tma_load_2d(&tm.m[0], bar, s, kb * BK, td.m0);
  }
  __device__ static void load_b(const Args& a, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    tma_load_2d(&tm.m[1], bar, s, kb * BK, td.e * a.d.H + td.n0);
  }
  __device__ static void epilogue(const Args& a, const TmaSet&, const TileDesc& td, uint32_t taddr,
                                  int r, uint8_t* stg) {
    push_rows(a, td, taddr, r, 0, stg);
  }
  template <class A>
  __device__ static void tile_done(const A&, const TileDesc&) {}
};

// Weight-gradient tile (128 x 256 fp32 in TMEM) -> bf16 through the warp's three staging tiles
// (round robin, two store groups in flight) and TMA stores into dW viewed as [epr*NO][KO].
__device__ __forceinline__ void wgrad_store(const CUtensorMap* map, const TileDesc& td, int NO,
                                            uint32_t taddr, int r, uint8_t* stg) {
  const uint32_t lane = r & 31;
  const int row0 = td.e * NO + td.m0 + (r & ~31);
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    float v[32];
    if (td.nkb > 0) {
      acc_chunk(taddr, c, v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    uint8_t* buf = stg + (c % 3) * EPI_TILE_BYTES;
    if (lane == 0) tma_store_wait_read<2>();
    __syncwarp();
    stage_row(buf, lane, v);
    stage_release();
    if (lane == 0) {
      tma_store_2d(map, buf, td.n0 + c * 32, row0);
      tma_store_commit();
    }
  }
}

// Backward: down-dgrad tiles then down-wgrad tiles.
//   dgrad : A = recv_dy (K-major over H), B = W_down[e] as [H rows = K][F cols] (MN-major).
//           Epilogue: dh = w * acc; SwiGLU backward from the saved bf16 g, u; writes dGU and
//           HW = bf16(w * h) (zeros on padding rows), then counts the (expert, f-block).
//   wgrad : dW_down[e] = recv_dy_e^T . HW_e, A and B MN-major over the expert's rows, which
//           are walked in ascending 64-row K-blocks (deterministic, no split-K).
struct ModeDgradDown {
  using Args = MkArgs;
  static constexpr bool HAS_TILE_DONE = true;
  static constexpr bool SPARE = true;
  __device__ static void spare(const Args& a, const Timeline& tl, const SpareStop&) { spare_comm(a, tl, 1); }
  __device__ static int n_dgrad_pair(const Args& a) { return a.p.mpair_pre[a.d.epr] * (a.d.F / BN); }
  __device__ static TileDesc tile_pair(const Args& a, int t) {
    const int nd = n_dgrad_pair(a);
    if (t < nd) return nt_tile_pair(a.d, a.p, t, a.d.F / BN, BN, a.d.H / BK, a.rgp);
    return tn_tile_pair(a.d, a.p, t - nd, a.d.H, a.d.F, a.tngp_d);
  }
  __device__ static void before_loads_pair(const Args& a, const TileDesc& td) {
    if (!td.pad1)
      wait_pair_rows(a, 1, td, 31);
    else
      wait_geq_sys(a.wg_cnt + td.e * (a.d.F / BN) + td.pad0, (uint32_t)a.p.mblocks[td.e],
                   a.timeout_ns, a.err, 32, td.e * 1000 + td.pad0);
  }
  __device__ static void load_a_pair(const Args&, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    if (!td.pad1) {
      tma_load_2d_pair(&tm.m[0], bar, s, kb * BK, td.m0 + BM * rank);
    } else {
#pragma unroll
      for (int i = 0; i < 2; ++i)
        tma_load_2d_pair(&tm.m[2], bar, s + i * 8192, td.m0 + BM * rank + 64 * i, td.kb0 + kb * BK);
    }
  }
  __device__ static void load_b_pair(const Args& a, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    const CUtensorMap* map = td.pad1 ? &tm.m[3] : &tm.m[1];
    const int row = td.pad1 ? td.kb0 + kb * BK : td.e * a.d.H + kb * BK;
#pragma unroll
    for (int i = 0; i < 2; ++i) tma_load_2d_pair(map, bar, s + i * 8192, td.n0 + BM * rank + 64 * i, row);
  }
  __device__ static TileDesc half_of(const TileDesc& td, uint32_t rank) { return half_tile(td, rank); }
  __device__ static bool half_has_work(const TileDesc& h) { return h.pad1 || h.rows > 0; }
  __device__ static int n_dgrad(const Args& a) { return a.p.mblock_pre[a.d.epr] * (a.d.F / BN); }
  __device__ static int a_mn(const TileDesc& td) { return td.pad1; }
  __device__ static int b_mn(const TileDesc&) { return 1; }
  __device__ static TileDesc tile(const Args& a, int t) {
    const int nd = n_dgrad(a);
    if (t < nd) return nt_tile(a.d, a.p, t, a.d.F / BN, BN, a.d.H / BK);
    return tn_tile(a.d, a.p, t - nd, a.d.H, a.d.F);
  }
  __device__ static void before_loads(const Args& a, const TileDesc& td) {
    if (!td.pad1) {
      if (a.unfused) return;
      const SymPtrs& me = a.peers.p[a.d.rank];
      wait_geq_sys(rg_counter(me, a.d, 1, PAR(a), td.m0 >> 7), (uint32_t)td.rows, a.timeout_ns,
                   a.err, 31, td.m0 >> 7);
    } else {
      wait_geq_sys(a.wg_cnt + td.e * (a.d.F / BN) + td.pad0, (uint32_t)a.p.mblocks[td.e],
                   a.timeout_ns, a.err, 32, td.e * 1000 + td.pad0);
    }
  }
  // dgrad tiles: pull this row's saved g, u (the SwiGLU backward inputs) toward L2 before the
  // accumulator is ready
  __device__ static void epilogue_prefetch(const Args& a, const TileDesc& td, int r) {
    if (td.pad1 || r >= td.rows) return;
    prefetch_meta_l1(a, td, r);
    const char* g = reinterpret_cast<const char*>(a.gu + ((size_t)td.m0 + r) * 2 * a.d.F + td.n0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(g + i * 128));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(g + (size_t)a.d.F * 2 + i * 128));
    }
  }
  __device__ static void load_a(const Args&, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    if (!td.pad1) {
      tma_load_2d(&tm.m[0], bar, s, kb * BK, td.m0);
    } else {
#pragma unroll
      for (int i = 0; i < BM / 64; ++i)
        tma_load_2d(&tm.m[2], bar, s + i * 8192, td.m0 + 64 * i, td.kb0 + kb * BK);
    }
  }
  __device__ static void load_b(const Args& a, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    if (!td.pad1) {
#pragma unroll
      for (int i = 0; i < BN / 64; ++i)
        tma_load_2d(&tm.m[1], bar, s + i * 8192, td.n0 + 64 * i, td.e * a.d.H + kb * BK);
    } else {
#pragma unroll
      for (int i = 0; i < BN / 64; ++i)
        tma_load_2d(&tm.m[3], bar, s + i * 8192, td.n0 + 64 * i, td.kb0 + kb * BK);
    }
  }
  // CTA pair: 5 operand stages; the freed 32 KB hold each epilogue warp's saved-g/u input ring. The
  // SwiGLU backward reads the forward's g, u of its 32 rows x 32 columns per chunk: with per-lane
  // global loads (one row per lane, 16 B pieces, one chunk ahead in registers) the math waited for
  // them (removing the loads cut the epilogue's cycles by 40 %, profiles/r02_epilogue_gather_probes.md);
  // TMA loads them into the ring two chunks ahead, the first two before the accumulator wait.
  static constexpr int PAIR_STAGES = 5;
  static constexpr bool GU_RING = true;
  __device__ static void gu_load(const Args& a, const TmaSet& tm, const TileDesc& td, int row0, int c,
                                 const EpiRing& ring) {
    uint8_t* b = ring.buf + (c & 1) * 4096;
    mbar_arrive_expect_tx(&ring.bar[c & 1], 4096);
    tma_load_2d(&tm.m[7], &ring.bar[c & 1], b, td.n0 + c * 32, row0);               // g
    tma_load_2d(&tm.m[7], &ring.bar[c & 1], b + 2048, a.d.F + td.n0 + c * 32, row0);  // u
  }
  __device__ static void epilogue_issue(const Args& a, const TmaSet& tm, const TileDesc& td, int lane,
                                        int q, const EpiRing& ring) {
    if (td.pad1 || lane != 0) return;
    gu_load(a, tm, td, td.m0 + q * 32, 0, ring);
    gu_load(a, tm, td, td.m0 + q * 32, 1, ring);
  }
  __device__ static void epilogue(const Args& a, const TmaSet& tm, const TileDesc& td,
                                  uint32_t taddr, int r, uint8_t* stg) {
    epi<false>(a, tm, td, taddr, r, stg, EpiRing{nullptr, nullptr});
  }
  __device__ static void epilogue_ring(const Args& a, const TmaSet& tm, const TileDesc& td,
                                       uint32_t taddr, int r, uint8_t* stg, const EpiRing& ring) {
    epi<true>(a, tm, td, taddr, r, stg, ring);
  }
  template <bool RING>
  __device__ static void epi(const Args& a, const TmaSet& tm, const TileDesc& td, uint32_t taddr, int r,
                             uint8_t* stg, const EpiRing& ring) {
    const int F = a.d.F;
    if (td.pad1) {  // weight-gradient tile
      wgrad_store(&tm.m[6], td, a.d.H, taddr, r, stg);
      return;  // (pair: td is this CTA's 128-row half of the 256-row dW tile)
    }
    const uint32_t lane = r & 31;
    const size_t m = (size_t)td.m0 + r;
    const int row0 = td.m0 + (r & ~31);
    const bool live = r < td.rows;
    SlotMeta mt{0, 0, 0.f, 0};
    if (live) mt = a.peers.p[a.d.rank].meta[m];
    const float w = mt.w;
    // gate gradient: dgate_{t,j} = <dY_t, o_{t,j}> = <dY_t W_down, h_{t,j}> -- the accumulator
    // before the gate weight, dotted with the (recomputed bf16) h, fp32 fmaf in column order; one
    // partial per (row, column tile), summed over the tiles in order by the source's reduce
    float gpart = 0.f;
    const int4* gsrc = reinterpret_cast<const int4*>(a.gu + m * 2 * F + td.n0);
    const int4* usrc = reinterpret_cast<const int4*>(a.gu + m * 2 * F + F + td.n0);
    // saved g, u of chunk c+1 are in flight while chunk c is computed (software pipelining)
    int4 gq[4] = {}, uq[4] = {};
    const bool ld_gu = live && !(a.dbg & 16);  // experiment: dbg 16 skips the saved g, u loads
    if (!RING && ld_gu) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        gq[i] = gsrc[i];
        uq[i] = usrc[i];
      }
    }
    // experiment (dbg 1024 + timeline): cycles per epilogue section of warp 0, one record per tile
    const bool sect = (a.dbg & 1024) && a.tl.rec && r == 0;
    long long cs[5] = {0, 0, 0, 0, 0}, ct = sect ? clock64() : 0;
    const unsigned long long gt0 = sect ? globaltimer() : 0;
    auto mark = [&](int i) {
      if (sect) {
        const long long n = clock64();
        cs[i] += n - ct;
        ct = n;
      }
    };
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      int4 gn[4], un[4];  // issued before this chunk's TMEM load so they also overlap its wait
      if constexpr (RING) {  // this chunk's g, u from the ring, then the refill two chunks ahead
        mbar_wait(&ring.bar[c & 1], (c >> 1) & 1);
        const uint8_t* b = ring.buf + (c & 1) * 4096 + lane * 64;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t off = (uint32_t)((i ^ ((lane >> 1) & 3)) << 4);
          gq[i] = ld_gu ? *reinterpret_cast<const int4*>(b + off) : make_int4(0, 0, 0, 0);
          uq[i] = ld_gu ? *reinterpret_cast<const int4*>(b + 2048 + off) : make_int4(0, 0, 0, 0);
        }
        __syncwarp();
        if (lane == 0 && c + 2 < BN / 32) {
          fence_proxy_async();  // the warp's reads of the buffer before the TMA refill
          gu_load(a, tm, td, row0, c + 2, ring);
        }
      } else if (ld_gu && c + 1 < BN / 32) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          gn[i] = gsrc[(c + 1) * 4 + i];
          un[i] = usrc[(c + 1) * 4 + i];
        }
      }
      mark(0);
      float v[32];
      acc_chunk(taddr, c, v);
      mark(1);
      uint32_t pdg[16], pdu[16], phw[16];
      if (live) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float2 g2 = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(gq)[q]);
          const float2 u2 = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(uq)[q]);
          float dg[2], du[2], hv[2];
          const float gg[2] = {g2.x, g2.y}, uu[2] = {u2.x, u2.y};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float dh = w * v[2 * q + h];
            const float sg = __fdividef(1.0f, 1.0f + __expf(-gg[h]));
            const float si = gg[h] * sg;
            const float ds = sg * (1.0f + gg[h] * (1.0f - sg));
            const float hh = __bfloat162float(__float2bfloat16_rn(si * uu[h]));
            dg[h] = dh * uu[h] * ds;
            du[h] = dh * si;
            hv[h] = w * hh;
            gpart = fmaf(v[2 * q + h], hh, gpart);
          }
          pdg[q] = pack_bf16(dg[0], dg[1]);
          pdu[q] = pack_bf16(du[0], du[1]);
          phw[q] = pack_bf16(hv[0], hv[1]);
        }
      }
      const int f0 = td.n0 + c * 32;
      if (sect) {  // the compute section ends when its results exist (not at the issue of the math)
        uint32_t z = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) z ^= pdg[q] ^ pdu[q] ^ phw[q];
        asm volatile("" ::"r"(z));
      }
      mark(2);
      if (a.dbg & 4) continue;  // experiment: no staging / stores at all
      stage_acquire(lane);
      mark(3);
      if (live) {
        stage_row_packed(stg, lane, pdg);
        stage_row_packed(stg + EPI_TILE_BYTES, lane, pdu);
        stage_row_packed(stg + 2 * EPI_TILE_BYTES, lane, phw);
      } else {  // zero padding rows: the K padding of the transposed weight-gradient GEMM
        stage_zero_row(stg, lane);
        stage_zero_row(stg + EPI_TILE_BYTES, lane);
        stage_zero_row(stg + 2 * EPI_TILE_BYTES, lane);
      }
      stage_release();
      if (lane == 0 && !(a.dbg & 2)) {
        tma_store_2d(&tm.m[4], stg, f0, row0);                       // dGU gate half
        tma_store_2d(&tm.m[4], stg + EPI_TILE_BYTES, F + f0, row0);  // dGU up half
        tma_store_2d(&tm.m[5], stg + 2 * EPI_TILE_BYTES, f0, row0);  // HW
        tma_store_commit();
      }
      mark(4);
      if (!RING && ld_gu && c + 1 < BN / 32) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          gq[i] = gn[i];
          uq[i] = un[i];
        }
      }
    }
    if (sect)
      for (int i = 0; i < 5; ++i) timeline_push(a.tl, gt0, gt0 + (unsigned long long)cs[i], ROLE_COMP, -9011 - i);
    if (live) {  // this tile's gate-gradient partial, to the source (peer memory at EP > 1)
      const int ncb = F / BN;
      float* dst = a.unfused ? a.ret_dgp + (size_t)a.ret_pos[m] * ncb
                             : a.peers.p[mt.src].dgp + (size_t)mt.rep * ncb;
      dst[td.pad0] = gpart;
    }
    // the weight-gradient tiles of this (expert, f-block) read HW / dGU through TMA: complete
    // the stores before tile_done publishes the count
    if (lane == 0) {
      tma_store_wait<0>();
      fence_proxy_async_global();
    }
    __syncwarp();
  }
  __device__ static void tile_done(const Args& a, const TileDesc& td) {
    if (td.pad1) return;
    __threadfence();
    red_release_gpu_add(a.wg_cnt + td.e * (a.d.F / BN) + td.pad0, 1u);
  }
};

// Backward: up-dgrad tiles (push dX replicas to the source) then up-wgrad tiles.
//   dgrad : A = dGU (K-major over 2F), B = W_up[e] as [2F rows = K][H cols] (MN-major).
//   wgrad : dW_up[e] = dGU_e^T . recv_x_e (both MN-major over the expert's rows).
struct ModeDgradUp {
  using Args = MkArgs;
  static constexpr bool HAS_TILE_DONE = false;
  static constexpr bool RELEASE_AFTER = true;
  __device__ static void epilogue_release(const Args& a, const TileDesc& td, int r) {
    if (!td.pad1) push_release(a, td, r, 1);  // dgrad tiles push dX replicas; wgrad tiles do not
  }
  static constexpr bool RELEASE_WARP = true;  // CTA pair: warp 2 publishes; the non-leader's warps
                                              // 1 and 3 remain the spare reduce workers
  __device__ static bool wants_release(const Args& a, const TileDesc& td) { return !a.unfused && !td.pad1; }
  __device__ static void release_tile(const Args& a, const TileDesc& td, int lane) { push_release_tile(a, td, lane, 1); }
  static constexpr bool SPARE = true;
  __device__ static void spare(const Args& a, const Timeline& tl, const SpareStop& stop) {
    spare_reduce(a, tl, 1, stop);
  }
  __device__ static void epilogue_prefetch(const Args& a, const TileDesc& td, int r) { prefetch_meta_l1(a, td, r); }
  __device__ static int n_dgrad_pair(const Args& a) { return a.p.mpair_pre[a.d.epr] * (a.d.H / BN); }
  __device__ static TileDesc tile_pair(const Args& a, int t) {
    const int nd = n_dgrad_pair(a);
    if (t < nd) return nt_tile_pair(a.d, a.p, t, a.d.H / BN, BN, 2 * a.d.F / BK, a.rgp);
    return tn_tile_pair(a.d, a.p, t - nd, 2 * a.d.F, a.d.H, a.tngp);
  }
  __device__ static void before_loads_pair(const Args&, const TileDesc&) {}
  __device__ static void load_a_pair(const Args&, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    if (!td.pad1) {
      tma_load_2d_pair(&tm.m[0], bar, s, kb * BK, td.m0 + BM * rank);
    } else {
#pragma unroll
      for (int i = 0; i < 2; ++i)
        tma_load_2d_pair(&tm.m[2], bar, s + i * 8192, td.m0 + BM * rank + 64 * i, td.kb0 + kb * BK);
    }
  }
  __device__ static void load_b_pair(const Args& a, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    const CUtensorMap* map = td.pad1 ? &tm.m[3] : &tm.m[1];
    const int row = td.pad1 ? td.kb0 + kb * BK : td.e * 2 * a.d.F + kb * BK;
#pragma unroll
    for (int i = 0; i < 2; ++i) tma_load_2d_pair(map, bar, s + i * 8192, td.n0 + BM * rank + 64 * i, row);
  }
  __device__ static TileDesc half_of(const TileDesc& td, uint32_t rank) { return half_tile(td, rank); }
  __device__ static bool half_has_work(const TileDesc& h) { return h.pad1 || h.rows > 0; }
  __device__ static int n_dgrad(const Args& a) { return a.p.mblock_pre[a.d.epr] * (a.d.H / BN); }
  __device__ static int a_mn(const TileDesc& td) { return td.pad1; }
  __device__ static int b_mn(const TileDesc&) { return 1; }
  __device__ static TileDesc tile(const Args& a, int t) {
    const int nd = n_dgrad(a);
    if (t < nd) return nt_tile(a.d, a.p, t, a.d.H / BN, BN, 2 * a.d.F / BK);
    return tn_tile(a.d, a.p, t - nd, 2 * a.d.F, a.d.H);
  }
  __device__ static void before_loads(const Args&, const TileDesc&) {}
  __device__ static void load_a(const Args&, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    if (!td.pad1) {
      tma_load_2d(&tm.m[0], bar, s, kb * BK, td.m0);
    } else {
#pragma unroll
      for (int i = 0; i < BM / 64; ++i)
        tma_load_2d(&tm.m[2], bar, s + i * 8192, td.m0 + 64 * i, td.kb0 + kb * BK);
    }
  }
  __device__ static void load_b(const Args& a, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    if (!td.pad1) {
#pragma unroll
      for (int i = 0; i < BN / 64; ++i)
        tma_load_2d(&tm.m[1], bar, s + i * 8192, td.n0 + 64 * i, td.e * 2 * a.d.F + kb * BK);
    } else {
#pragma unroll
      for (int i = 0; i < BN / 64; ++i)
        tma_load_2d(&tm.m[3], bar, s + i * 8192, td.n0 + 64 * i, td.kb0 + kb * BK);
    }
  }
  __device__ static void epilogue(const Args& a, const TmaSet& tm, const TileDesc& td,
                                  uint32_t taddr, int r, uint8_t* stg) {
    if (!td.pad1) {
      push_rows(a, td, taddr, r, 1, stg);
      return;
    }
    wgrad_store(&tm.m[6], td, 2 * a.d.F, taddr, r, stg);
  }
  template <class A>
  __device__ static void tile_done(const A&, const TileDesc&) {}
};

// Exit of every (non-aborted) CTA: the last one to leave returns the kernel's work counters -- the
// task cursor, comm-round / reduce-chunk / relay-rowgroup counters (cursor[0..5]) and, after the
// backward dispatch, the weight-gradient tile counts -- to zero for the next launch, so no memset
// launches separate the MegaKernels (cursor[6] counts the CTAs out). Every CTA has finished with
// the counters when it arrives; an aborted iteration touches none of them.
__device__ __forceinline__ void finish_kernel(const MkArgs& a, int kind) {
  __shared__ int sh_last;
  __syncthreads();
  unsigned* done = reinterpret_cast<unsigned*>(a.cursor + 6);
  if (threadIdx.x == 0) {
    __threadfence();
    sh_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!sh_last) return;
  __threadfence();
  // The scoreboard counters this kernel waited on (this phase, this parity) are complete -- every
  // increment, local or from a peer, was awaited by a CTA of this grid -- so they are zeroed here
  // too, not only one iteration later by the other parity's kernel: a restored iteration
  // (eplab_stash_restore) may run this phase twice in a row with the same parity.
  const SymPtrs& me = a.peers.p[a.d.rank];
  const int ph = kind >= 2 ? 1 : 0;
  if (kind == 0 || kind == 2)
    for (int g = threadIdx.x; g < a.d.RG_cap; g += blockDim.x) *rg_counter(me, a.d, ph, PAR(a), g) = 0;
  else
    for (int t = threadIdx.x; t < a.p.n_tok; t += blockDim.x) *tok_counter(me, a.d, ph, PAR(a), t) = 0;
  if (kind == 2)
    for (int i = threadIdx.x; i < a.d.epr * (a.d.F / BN); i += blockDim.x) a.wg_cnt[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) a.cursor[i] = 0;
    *done = 0;
  }
  __threadfence();
}

// ------------------------------------------------------------------ the MegaKernel
// KIND 0: fwd dispatch+GEMM, 1: fwd GEMM+combine, 2: bwd dispatch+GEMM, 3: bwd GEMM+combine.
template <int KIND, class Mode>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    megakernel(const __grid_constant__ TmaSet tm, const __grid_constant__ MkArgs a) {
  extern __shared__ uint8_t raw_smem[];
  uint8_t* base = smem_aligned(raw_smem);
  GemmSmem* S = reinterpret_cast<GemmSmem*>(base + TILES_BYTES + EPI_BYTES);
  const int ph = (KIND >= 2) ? 1 : 0;
  const bool has_pre = (KIND == 0 || KIND == 2);
  const bool has_post = (KIND == 1 || KIND == 3);

  load_epoch(a);
  // Reset the other parity of this phase's counters (used one iteration ago, all their
  // increments have landed) -- see DESIGN.md §Scoreboard.
  if (blockIdx.x == 0) {
    const SymPtrs& me = a.peers.p[a.d.rank];
    if (has_pre)
      for (int g = threadIdx.x; g < a.d.RG_cap; g += blockDim.x)
        *rg_counter(me, a.d, ph, (PAR(a) ^ 1), g) = 0;
    if (has_post)
      for (int t = threadIdx.x; t < a.d.T_max; t += blockDim.x)
        *tok_counter(me, a.d, ph, (PAR(a) ^ 1), t) = 0;
  }
  if (iteration_aborted(a)) return;  // after the reset: the next iteration's parity stays clean
  gemm_setup(S);

  const int n_pre = has_pre ? a.n_disp + a.n_relay : 0;
  int n_tiles = 0;
  if (KIND == 0) n_tiles = a.p.mblock_pre[a.d.epr] * (a.d.F / 128);
  if (KIND == 1) n_tiles = a.p.mblock_pre[a.d.epr] * (a.d.H / BN);
  if (KIND == 2)
    n_tiles = a.p.mblock_pre[a.d.epr] * (a.d.F / BN) + a.d.epr * (a.d.H / BM) * (a.d.F / BN);
  if (KIND == 3)
    n_tiles = a.p.mblock_pre[a.d.epr] * (a.d.H / BN) + a.d.epr * (2 * a.d.F / BM) * (a.d.H / BN);
  const int n_post = has_post ? a.n_red : 0;
  const int total = n_pre + n_tiles + n_post;

  if (threadIdx.x == 0) S->bcast = atomicAdd(a.cursor, 1);
  __syncthreads();
  int id = S->bcast;
  __syncthreads();
  // pre-tasks (comm / relay): the whole CTA
  while (id < n_pre) {
    const unsigned long long t0 = globaltimer();
    if (id < a.n_disp)
      comm_task(a, id, ph, S, base);
    else
      relay_task(a, id - a.n_disp, ph);
    __syncthreads();
    if (threadIdx.x == 0) {
      timeline_push(a.tl, t0, globaltimer(), id < a.n_disp ? ROLE_COMM : ROLE_RELAY, id);
      S->bcast = atomicAdd(a.cursor, 1);
    }
    __syncthreads();
    id = S->bcast;
    __syncthreads();
  }
  // compute tiles: warp-specialised engine
  if (id < n_pre + n_tiles)
    id = gemm_roles<Mode>(a, tm, base, S, id, n_pre, n_pre + n_tiles, a.cursor, a.tl);
  // post-tasks (reduce): the whole CTA
  while (id < total) {
    const unsigned long long t0 = globaltimer();
    reduce_task(a, id - n_pre - n_tiles, ph);
    __syncthreads();
    if (threadIdx.x == 0) {
      timeline_push(a.tl, t0, globaltimer(), ROLE_REDUCE, id);
      S->bcast = atomicAdd(a.cursor, 1);
    }
    __syncthreads();
    id = S->bcast;
    __syncthreads();
  }
  gemm_teardown(S);
  finish_kernel(a, KIND);
}


// CTA-pair MegaKernel: the same task space with 256-row (pair) tiles. Each CTA resolves
// pre-tasks (comm / relay) on its own; the pair then enters the GEMM phase together (the
// leader schedules tiles for both) and afterwards each CTA resolves post-tasks (reduce).
template <int KIND, class Mode>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    megakernel_pair(const __grid_constant__ TmaSet tm, const __grid_constant__ MkArgs a) {
  extern __shared__ uint8_t raw_smem[];
  uint8_t* base = smem_aligned(raw_smem);
  GemmSmem* S = reinterpret_cast<GemmSmem*>(base + TILES_BYTES + EPI_BYTES);
  const uint32_t rank = cluster_ctarank();
  const int ph = (KIND >= 2) ? 1 : 0;
  const bool has_pre = (KIND == 0 || KIND == 2);
  const bool has_post = (KIND == 1 || KIND == 3);
  // Programmatic dependent launch: let the next MegaKernel's CTAs take the SMs ours leave (it can only
  // launch once every CTA of this grid has started), build this CTA's barriers and TMEM allocation
  // while the previous kernel drains, and touch no global state before it has completed.
  if (a.pdl) griddep_launch_dependents();
  gemm_setup_pair(S, rank);
  if (a.pdl) griddep_wait();
  load_epoch(a);
  if (blockIdx.x == 0) {
    const SymPtrs& me = a.peers.p[a.d.rank];
    if (has_pre)
      for (int g = threadIdx.x; g < a.d.RG_cap; g += blockDim.x) *rg_counter(me, a.d, ph, (PAR(a) ^ 1), g) = 0;
    if (has_post)
      for (int t = threadIdx.x; t < a.d.T_max; t += blockDim.x) *tok_counter(me, a.d, ph, (PAR(a) ^ 1), t) = 0;
  }
  if (iteration_aborted(a)) {  // both CTAs of the pair read the same words and leave together
    gemm_teardown_pair(S);
    return;
  }
  const int n_pre = has_pre ? a.n_disp + a.n_relay : 0;
  const int pairs = a.p.mpair_pre[a.d.epr];
  int n_tiles = 0;
  if (KIND == 0) n_tiles = pairs * (a.d.F / 128);
  if (KIND == 1) n_tiles = pairs * (a.d.H / BN);
  if (KIND == 2) n_tiles = pairs * (a.d.F / BN) + a.d.epr * (a.d.H / (2 * BM)) * (a.d.F / BN);
  if (KIND == 3) n_tiles = pairs * (a.d.H / BN) + a.d.epr * (2 * a.d.F / (2 * BM)) * (a.d.H / BN);
  const int n_post = has_post ? a.n_red : 0;
  const int total = n_pre + n_tiles + n_post;

  auto claim = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) S->bcast = atomicAdd(a.cursor, 1);
    __syncthreads();
    return S->bcast;
  };
  int id = claim();
  while (id < n_pre) {
    const unsigned long long t0 = globaltimer();
    if (id < a.n_disp)
      comm_task(a, id, ph, S, base);
    else
      relay_task(a, id - a.n_disp, ph);
    __syncthreads();
    if (threadIdx.x == 0) timeline_push(a.tl, t0, globaltimer(), id < a.n_disp ? ROLE_COMM : ROLE_RELAY, id);
    id = claim();
  }
  // pair up: the leader learns both CTAs' first non-pre ids
  if (threadIdx.x == 0) st_cluster_u32(mapa_shared(smem_u32(&S->pend[rank]), 0), (uint32_t)id);
  cluster_sync_all();
#if EPLAB_ENGINE_WD
  // engine mbarrier waits report error 3 (sites 40-47); a debug build (make EXTRA=-DEPLAB_ENGINE_WD=1):
  // the timed waits in the MMA / producer / epilogue loops cost 6 % (Qwen3, Mixtral), profiles/r02_dgrad_ring_ab.txt
  const Watchdog wd{a.err, a.timeout_ns};
#else
  const Watchdog wd{};
#endif
  gemm_roles_pair<Mode>(a, tm, base, S, n_pre, n_pre + n_tiles, a.cursor, a.tl, rank, wd);
  cluster_sync_all();
  if (threadIdx.x == 0) {
    const int pn = (int)ld_cluster_u32(mapa_shared(smem_u32(&S->post_n), 0));
    S->bcast = (int)rank < pn ? (int)ld_cluster_u32(mapa_shared(smem_u32(&S->post_ids[rank]), 0))
                              : atomicAdd(a.cursor, 1);
  }
  __syncthreads();
  id = S->bcast;
  while (id < total) {
    const unsigned long long t0 = globaltimer();
    reduce_task(a, id - n_pre - n_tiles, ph);
    __syncthreads();
    if (threadIdx.x == 0) timeline_push(a.tl, t0, globaltimer(), ROLE_REDUCE, id);
    id = claim();
  }
  gemm_teardown_pair(S);
  finish_kernel(a, KIND);
}

}  // namespace eplab_dev

// ------------------------------------------------------------------ host launchers
namespace eplab_launch {
using namespace eplab_dev;

// Loads every MegaKernel into the current device's context and sets its shared-memory size --
// called by eplab_init on each context's device. With CUDA's lazy module loading the first
// launch of a function can wait for the device to idle, which never happens while another
// virtual rank's kernel spins on a scoreboard fed by a kernel this host thread has yet to launch.
int preload_megakernels() {
  auto set = [](auto fn) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM_BYTES) ==
           cudaSuccess;
  };
  const bool ok = set(megakernel<0, ModeUp>) && set(megakernel<1, ModeDown>) &&
                  set(megakernel<2, ModeDgradDown>) && set(megakernel<3, ModeDgradUp>) &&
                  set(megakernel_pair<0, ModeUp>) && set(megakernel_pair<1, ModeDown>) &&
                  set(megakernel_pair<2, ModeDgradDown>) && set(megakernel_pair<3, ModeDgradUp>);
  return ok ? 0 : 1;
}

template <int KIND, class Mode>
static int launch_mk(const TmaSet& tm, const MkArgs& a, int grid, cudaStream_t st) {
  // (the work counters are zero: eplab_init clears them and every MegaKernel's last CTA resets them)
  if (!a.pair) {
    auto fn = megakernel<KIND, Mode>;
    fn<<<grid, GEMM_THREADS, GEMM_SMEM_BYTES, st>>>(tm, a);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
  }
  auto fn = megakernel_pair<KIND, Mode>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((grid / 2) * 2);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = GEMM_SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cudaLaunchAttribute at2[2] = {at[0], {}};
  at2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at2[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a.pdl ? at2 : at;
  cfg.numAttrs = a.pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, fn, tm, a);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_fwd_dispatch(const TmaSet& tm, const MkArgs& a, int grid, cudaStream_t st) {
  return launch_mk<0, ModeUp>(tm, a, grid, st);
}
int launch_fwd_combine(const TmaSet& tm, const MkArgs& a, int grid, cudaStream_t st) {
  return launch_mk<1, ModeDown>(tm, a, grid, st);
}
int launch_bwd_dispatch(const TmaSet& tm, const MkArgs& a, int grid, cudaStream_t st) {
  return launch_mk<2, ModeDgradDown>(tm, a, grid, st);
}
int launch_bwd_combine(const TmaSet& tm, const MkArgs& a, int grid, cudaStream_t st) {
  return launch_mk<3, ModeDgradUp>(tm, a, grid, st);
}

}  // namespace eplab_launch
