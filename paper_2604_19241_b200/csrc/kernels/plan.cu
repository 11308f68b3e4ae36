// Device token map (Alg. 1; token_map.cpp:10-126) with the count
// AllGather done as P2P stores into every peer's symmetric count table -- no host sync.
//
//   plan_hist     : per-chunk BinCount of the routing entries            (Alg. 1 l.1)
//   plan_global   : chunk bases (CumSum), count exchange (l.3), global offsets (l.4,
//                   token_map.cpp:30-53), receive geometry (:71-82), schedule bucket bases
//                   (:108-126); one CTA
//   plan_entries  : stable within-expert rank of every (t, j) -> Alg. 1 final_idx, the
//                   destination slot and the priority-ordered send schedule
//   (plan_entries' extra CTAs) zero the alignment rows between expert segments (they are the zero
//                   K-padding of the transposed weight-gradient GroupGEMM)
#include "moe_common.cuh"
#include "ptx.cuh"

#include <climits>

namespace eplab_dev {

// BinCount of one chunk, and the routing checks of validate_routing (types.cpp:74-94) on device:
// expert id in [0, E), no duplicate expert within a token, finite gate weight. A violation is
// recorded as a bit set in p.scalars[4] (1 range, 2 duplicate, 4 non-finite; the offending entry
// in p.scalars[5]) and the entry is not counted; plan_global turns it into an iteration abort.
__global__ void plan_hist_kernel(const int* __restrict__ ids, const float* __restrict__ gw, int n, int k,
                                 int E, int* __restrict__ hist, int* __restrict__ scalars) {
  __shared__ int h[MAX_EXPERTS];
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = 0;
  __syncthreads();
  const int base = blockIdx.x * PLAN_CHUNK;
  const int end = min(n, base + PLAN_CHUNK);
  for (int i = base + threadIdx.x; i < end; i += blockDim.x) {
    const int e = ids[i];
    int bad = (e < 0 || e >= E) ? 1 : 0;
    const int t0 = i - i % k;
    for (int q = t0; q < i; ++q)
      if (ids[q] == e) bad |= 2;
    if (!isfinite(gw[i])) bad |= 4;
    if (bad) {
      atomicOr(scalars + 4, bad);
      atomicMin(scalars + 5, i);
    } else {
      atomicAdd(&h[e], 1);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[(size_t)blockIdx.x * E + e] = h[e];
}

// Advances the device iteration counter (every MegaKernel of the iteration reads it, so a captured
// graph of plan + MegaKernels replays with fresh flags and counter parities). Returns the epoch.
__device__ uint32_t plan_advance_epoch(uint32_t* epoch_dev) {
  __shared__ uint32_t epoch_s;
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch_s = *epoch_dev + 1;
    *epoch_dev = epoch_s;
  }
  __syncthreads();
  return epoch_s;
}

// A restored iteration (eplab_stash_restore) runs its backward under a fresh epoch: slot flags and
// counter parities of the MegaKernels never see an epoch twice.
__global__ void epoch_advance_kernel(uint32_t* epoch_dev) { plan_advance_epoch(epoch_dev); }

// (a) CumSum over chunks (chunk bases, in place in p.hist) and C_exp -> p.counts and cnt_s.
// Two passes over (expert, chunk-range) segments -- every thread of the CTA, S = blockDim / E
// segments per expert -- so the chunk scan is not one thread walking all chunks of an expert with a
// dependent load per chunk (Qwen3, 64 chunks: ~40 us of the planner).
__device__ void plan_scan_chunks(const Dims& d, const PlanDev& p, int nchunks, int* cnt_s) {
  __shared__ int part[1024];  // [segment][expert] partial sums, S * E <= blockDim <= 1024
  const int E = d.E;
  const int S = max(1, (int)blockDim.x / E);
  const int per = (nchunks + S - 1) / S;
  const int e = threadIdx.x % E, sg = threadIdx.x / E;
  const bool active = sg < S && (int)threadIdx.x < S * E;
  const int c0 = sg * per, c1 = min(nchunks, c0 + per);
  int sum = 0;
  if (active)
    for (int c = c0; c < c1; ++c) sum += p.hist[(size_t)c * E + e];
  if (active) part[sg * E + e] = sum;
  __syncthreads();
  if (active) {
    int s = 0;  // chunks before this segment
    for (int q = 0; q < sg; ++q) s += part[q * E + e];
    for (int c = c0; c < c1; ++c) {
      const int v = p.hist[(size_t)c * E + e];
      p.hist[(size_t)c * E + e] = s;
      s += v;
    }
    if (sg == S - 1) {
      p.counts[e] = s;
      cnt_s[e] = s;
    }
  }
  __syncthreads();
}

// (d)... the layout from every rank's counts call[src * stride + e]: receive totals, segment bases
// (reference and 128-aligned), the capacity check of every destination, the abort decision, the
// schedule bucket bases, the local receive geometry and the global offsets (Eq. 1) of my copies.
// bad_bits / bad_rank: the routing checks of all ranks (plus 16 = a count-exchange timeout).
__device__ void plan_layout(const Dims& d, const PlanDev& p, const int* call, int stride, const int* cnt_s,
                            int bad_bits, int bad_rank, int* err) {
  const int E = d.E, W = d.world, epr = d.epr, me = d.rank;
  __shared__ int rt[MAX_EXPERTS];  // recv totals per (dst, e_loc) = global expert
  // receive totals of every (rank, local expert)  (token_map.cpp:71-74)
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int s = 0;
    for (int src = 0; src < W; ++src) s += call[src * stride + e];
    rt[e] = s;
    p.rt_all[e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // segment bases, reference (unaligned) and the 128-aligned layout used here. The receive
    // capacity of EVERY destination is checked: all ranks see the same counts, so they all reach
    // the same abort decision and no sender writes past a peer's M_cap.
    int over_rank = -1;
    long long over_rows = 0;
    for (int dst = 0; dst < W; ++dst) {
      long long a = 0, b = 0;
      for (int el = 0; el < epr; ++el) {
        const int e = dst * epr + el;
        p.sb_all_ref[e] = (int)min(a, (long long)INT_MAX);
        p.sb_all[e] = (int)min(b, (long long)INT_MAX);
        a += rt[e];
        b += (rt[e] + 127) & ~127;
      }
      if (b > d.M_cap && over_rank < 0) {
        over_rank = dst;
        over_rows = b;
      }
      if (dst == me) {
        p.scalars[0] = (int)min(b, (long long)d.M_cap);
        p.scalars[1] = (int)(min(b, (long long)d.M_cap) >> 7);
        p.scalars[2] = (int)min(a, (long long)INT_MAX);
      }
    }
    int abort_bits = bad_bits;
    if (over_rank >= 0) abort_bits |= 8;
    // iteration abort: every kernel of this iteration (entries, padding, the four MegaKernels)
    // sees scalars[3] != 0 and skips its work; eplab_check reports error 2 (3 for a timeout)
    p.scalars[3] = abort_bits;
    if (abort_bits & ~16) {
      if (atomicCAS(err, 0, 2) == 0) {
        err[1] = abort_bits;
        err[2] = (abort_bits & 8) ? over_rank : bad_rank;
        err[3] = (abort_bits & 8) ? (int)min(over_rows, (long long)INT_MAX) : d.M_cap;
        err[4] = (abort_bits & 7) ? p.scalars[5] : -1;
      }
    }
    p.scalars[5] = INT_MAX;
    // priority schedule bucket bases: buckets ordered (e_loc, dst)  (token_map.cpp:117-124)
    int acc = 0;
    for (int el = 0; el < epr; ++el)
      for (int dst = 0; dst < W; ++dst) {
        const int e = dst * epr + el;
        p.bucket_base[e] = acc;
        acc += cnt_s[e];
      }
    // local receive geometry: 128-row blocks per local expert and their prefix
    int mp = 0, pp = 0;
    for (int el = 0; el < epr; ++el) {
      const int mb = (rt[me * epr + el] + 127) >> 7;
      p.mblocks[el] = mb;
      p.mblock_pre[el] = mp;
      p.mpair_pre[el] = pp;
      mp += mb;
      pp += (mb + 1) >> 1;
    }
    p.mblock_pre[epr] = mp;
    p.mpair_pre[epr] = pp;
  }
  __syncthreads();
  // global offsets of my copies: O_all[dst][e_loc][me] = sum_{s<me} C_all[s][e]  (Eq. 1)
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int o = 0;
    for (int src = 0; src < me; ++src) o += call[src * stride + e];
    p.o_all[e] = o;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) p.send_base[e] = p.sb_all[e] + p.o_all[e];
}

// Fused path: (a), then the count AllGather as P2P stores into every peer's symmetric table and a
// release flag that also carries this rank's routing-check result, then the layout. One CTA.
__global__ void plan_global_kernel(Dims d, Peers peers, PlanDev p, int nchunks, uint32_t* epoch_dev,
                                   uint64_t timeout_ns, int* err) {
  const int E = d.E, W = d.world, me = d.rank;
  const uint32_t epoch = plan_advance_epoch(epoch_dev);
  __shared__ int cnt_s[MAX_EXPERTS];
  plan_scan_chunks(d, p, nchunks, cnt_s);
  // (b) AllGather of C_exp: P2P store of my row into every peer's table, then release flag
  for (int i = threadIdx.x; i < W * E; i += blockDim.x) {
    const int dst = i / E, e = i % E;
    peers.p[dst].cnt_all[me * E + e] = cnt_s[e];
  }
  // this rank's routing-check result travels in bit 0 of its count flag: (epoch << 1) | bad
  __shared__ int bad_s, bad_rank_s;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int bad = p.scalars[4];
    bad_s = bad ? bad : 0;
    bad_rank_s = bad ? me : -1;
    p.scalars[4] = 0;  // consumed (the next iteration's checks start clean)
    __threadfence_system();
    const uint32_t flag = ((epoch & 0x7fffffffu) << 1) | (bad ? 1u : 0u);
    for (int dst = 0; dst < W; ++dst) st_release_sys(peers.p[dst].cnt_flag + me, flag);
  }
  // (c) wait for every source's row; a source that failed its routing checks aborts everyone
  __syncthreads();
  if (threadIdx.x < W) {
    const uint64_t t0 = globaltimer();
    uint32_t v;
    while (((v = ld_acquire_sys(peers.p[me].cnt_flag + threadIdx.x)) >> 1) != (epoch & 0x7fffffffu)) {
      if (globaltimer() - t0 > timeout_ns) {
        if (atomicCAS(err, 0, 3) == 0) {
          err[1] = 1;  // site 1: the count AllGather
          err[2] = (int)epoch;
          err[3] = (int)(v >> 1);
          err[4] = threadIdx.x;
        }
        atomicOr(&bad_s, 16);
        v = 0;
        break;
      }
    }
    if ((v & 1u) && threadIdx.x != me) {
      atomicOr(&bad_s, 32);
      atomicCAS(&bad_rank_s, -1, threadIdx.x);
    }
  }
  __syncthreads();
  plan_layout(d, p, peers.p[me].cnt_all, E, cnt_s, bad_s, bad_rank_s, err);
}

// Unfused path (the NCCL baseline), step 1: (a) and this rank's count row for the
// host's ncclAllGather: out[0..E) = C_exp, out[E] = its routing-check bits.
__global__ void plan_counts_kernel(Dims d, PlanDev p, int nchunks, uint32_t* epoch_dev, int* out) {
  plan_advance_epoch(epoch_dev);
  __shared__ int cnt_s[MAX_EXPERTS];
  plan_scan_chunks(d, p, nchunks, cnt_s);
  for (int e = threadIdx.x; e < d.E; e += blockDim.x) out[e] = cnt_s[e];
  if (threadIdx.x == 0) {
    out[d.E] = p.scalars[4];
    p.scalars[4] = 0;
  }
}

// Unfused path, step 2: the layout from the all-gathered rows call [W][E + 1].
__global__ void plan_layout_ext_kernel(Dims d, PlanDev p, const int* call, int* err) {
  __shared__ int cnt_s[MAX_EXPERTS];
  __shared__ int bad_s, bad_rank_s;
  if (threadIdx.x == 0) {
    bad_s = 0;
    bad_rank_s = -1;
    for (int r = 0; r < d.world; ++r) {
      const int b = call[r * (d.E + 1) + d.E];
      if (b) {
        bad_s |= r == d.rank ? b : 32;
        if (bad_rank_s < 0) bad_rank_s = r;
      }
    }
  }
  for (int e = threadIdx.x; e < d.E; e += blockDim.x) cnt_s[e] = call[d.rank * (d.E + 1) + e];
  __syncthreads();
  plan_layout(d, p, call, d.E + 1, cnt_s, bad_s, bad_rank_s, err);
}

// 256 threads = 8 warps; warp w owns entries [w*256, w*256+256) of the chunk in 8 rounds of 32.
// The PAD_BLOCKS extra CTAs (blockIdx.x >= nchunks) zero the alignment rows between this rank's
// expert segments in both receive buffers (rows [sb + rt, sb + align128(rt))): they are the zero
// K-padding of the transposed weight-gradient GroupGEMMs. (One launch instead of three.)
constexpr int PAD_BLOCKS = 148;  // the padding is up to 127 rows per expert and buffer (Qwen3: ~64 MB)
__device__ void zero_padding(const Dims& d, const PlanDev& p, __nv_bfloat16* recv_x, __nv_bfloat16* recv_dy,
                             int b) {
  // work item = (local expert, padding row < 128): one warp per item, items dealt round-robin over
  // all the padding warps (a serial loop over the experts with dependent segment loads cost ~0.1 ms)
  const int vec_per_row = d.H / 8;
  const int lane = threadIdx.x & 31, nw = blockDim.x / 32;
  for (int it = b * nw + (int)(threadIdx.x >> 5); it < d.epr * 128; it += PAD_BLOCKS * nw) {
    const int el = it >> 7, r = it & 127;
    const int e = d.rank * d.epr + el;
    const int rows = p.rt_all[e];
    if (r >= (((rows + 127) & ~127) - rows)) continue;
    int4* xrow = reinterpret_cast<int4*>(recv_x) + ((size_t)p.sb_all[e] + rows + r) * vec_per_row;
    int4* dyrow = reinterpret_cast<int4*>(recv_dy) + ((size_t)p.sb_all[e] + rows + r) * vec_per_row;
    for (int c = lane; c < vec_per_row; c += 32) {
      xrow[c] = make_int4(0, 0, 0, 0);
      dyrow[c] = make_int4(0, 0, 0, 0);
    }
  }
}

__global__ void __launch_bounds__(256) plan_entries_kernel(Dims d, PlanDev p, int n, int nchunks,
                                                           __nv_bfloat16* recv_x, __nv_bfloat16* recv_dy) {
  if (p.scalars[3]) return;  // aborted iteration (bad routing / capacity / timeout)
  if ((int)blockIdx.x >= nchunks) {
    zero_padding(d, p, recv_x, recv_dy, blockIdx.x - nchunks);
    return;
  }
  __shared__ int wcnt[8][MAX_EXPERTS];
  const int E = d.E;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * E; i += blockDim.x) wcnt[i / E][i % E] = 0;
  __syncthreads();
  const int base = blockIdx.x * PLAN_CHUNK + warp * 256;
  int ev[8], pos[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = base + r * 32 + lane;
    const bool valid = i < n;
    const int e = valid ? p.topk_ids[i] : -1 - lane;  // invalid lanes never match
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int before = valid ? wcnt[warp][e] : 0;
    const int rk = __popc(peers & ((1u << lane) - 1));
    __syncwarp();
    if (valid && rk == 0) wcnt[warp][e] = before + __popc(peers);
    __syncwarp();
    ev[r] = e;
    pos[r] = before + rk;
  }
  __syncthreads();
  // exclusive prefix over warps, per expert
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int v = wcnt[w][e];
      wcnt[w][e] = s;
      s += v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = base + r * 32 + lane;
    if (i >= n) continue;
    const int e = ev[r];
    const int local = p.hist[(size_t)blockIdx.x * E + e] + wcnt[warp][e] + pos[r];
    p.offset[i] = p.o_all[e] + local;
    p.dst_slot[i] = p.send_base[e] + local;
    p.sched[p.bucket_base[e] + local] = i;
  }
}

}  // namespace eplab_dev

namespace eplab_launch {
using namespace eplab_dev;

int plan_counts_launch(const Dims& d, const PlanDev& p, uint32_t* epoch, int* out, cudaStream_t st) {
  const int n = p.n_tok * d.topk;
  const int nchunks = n > 0 ? (n + PLAN_CHUNK - 1) / PLAN_CHUNK : 0;
  if (nchunks > 0)
    plan_hist_kernel<<<nchunks, 256, 0, st>>>(p.topk_ids, p.gate_w, n, d.topk, d.E, p.hist, p.scalars);
  plan_counts_kernel<<<1, 1024, 0, st>>>(d, p, nchunks, epoch, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int plan_layout_ext_launch(const Dims& d, const PlanDev& p, const int* call, int* err, __nv_bfloat16* recv_x,
                           __nv_bfloat16* recv_dy, cudaStream_t st) {
  const int n = p.n_tok * d.topk;
  const int nchunks = n > 0 ? (n + PLAN_CHUNK - 1) / PLAN_CHUNK : 0;
  plan_layout_ext_kernel<<<1, 1024, 0, st>>>(d, p, call, err);
  plan_entries_kernel<<<nchunks + PAD_BLOCKS, 256, 0, st>>>(d, p, n, nchunks, recv_x, recv_dy);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int plan_launch(const Dims& d, const Peers& peers, const PlanDev& p, uint32_t* epoch,
                uint64_t timeout_ns, int* err, __nv_bfloat16* recv_x, __nv_bfloat16* recv_dy, cudaStream_t st) {
  const int n = p.n_tok * d.topk;
  const int nchunks = n > 0 ? (n + PLAN_CHUNK - 1) / PLAN_CHUNK : 0;
  if (nchunks > 0)
    plan_hist_kernel<<<nchunks, 256, 0, st>>>(p.topk_ids, p.gate_w, n, d.topk, d.E, p.hist, p.scalars);
  plan_global_kernel<<<1, 1024, 0, st>>>(d, peers, p, nchunks, epoch, timeout_ns, err);
  plan_entries_kernel<<<nchunks + PAD_BLOCKS, 256, 0, st>>>(d, p, n, nchunks, recv_x, recv_dy);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int epoch_advance_launch(uint32_t* epoch, cudaStream_t st) {
  epoch_advance_kernel<<<1, 32, 0, st>>>(epoch);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// Loads the planning kernels into the current context up front (see preload_megakernels): the
// count exchange of plan_global_kernel spins until every virtual rank's planner has run.
int preload_plan() {
  cudaFuncAttributes fa;
  const bool ok = cudaFuncGetAttributes(&fa, plan_hist_kernel) == cudaSuccess &&
                  cudaFuncGetAttributes(&fa, plan_global_kernel) == cudaSuccess &&
                  cudaFuncGetAttributes(&fa, plan_entries_kernel) == cudaSuccess &&
                  cudaFuncGetAttributes(&fa, plan_counts_kernel) == cudaSuccess &&
                  cudaFuncGetAttributes(&fa, plan_layout_ext_kernel) == cudaSuccess &&
                  cudaFuncGetAttributes(&fa, epoch_advance_kernel) == cudaSuccess;
  return ok ? 0 : 1;
}

}  // namespace eplab_launch
