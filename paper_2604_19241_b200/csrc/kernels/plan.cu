// Device token map (Alg. 1; token_map.cpp:10-126) with the count
// AllGather done as P2P stores into every peer's symmetric count table -- no host sync.
//
//   plan_hist     : per-chunk BinCount of the routing entries            (Alg. 1 l.1)
//   plan_global   : chunk bases (CumSum), count exchange (l.3), global offsets (l.4,
//                   token_map.cpp:30-53), receive geometry (:71-82), schedule bucket bases
//                   (:108-126); one CTA
//   plan_entries  : stable within-expert rank of every (t, j) -> Alg. 1 final_idx, the
//                   destination slot and the priority-ordered send schedule
//   zero_padding  : zero the alignment rows between expert segments (they are the zero
//                   K-padding of the transposed weight-gradient GroupGEMM)
#include "moe_common.cuh"
#include "ptx.cuh"

namespace eplab_dev {

__global__ void plan_hist_kernel(const int* __restrict__ ids, int n, int E, int* __restrict__ hist) {
  __shared__ int h[MAX_EXPERTS];
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = 0;
  __syncthreads();
  const int base = blockIdx.x * PLAN_CHUNK;
  const int end = min(n, base + PLAN_CHUNK);
  for (int i = base + threadIdx.x; i < end; i += blockDim.x) atomicAdd(&h[ids[i]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[(size_t)blockIdx.x * E + e] = h[e];
}

__global__ void plan_global_kernel(Dims d, Peers peers, PlanDev p, int nchunks, uint32_t* epoch_dev,
                                   uint64_t timeout_ns, int* err) {
  const int E = d.E, W = d.world, epr = d.epr, me = d.rank;
  // a new iteration: advance the device epoch (every MegaKernel of the iteration reads it, so a
  // captured graph of plan + MegaKernels replays with fresh flags and counter parities)
  __shared__ uint32_t epoch_s;
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch_s = *epoch_dev + 1;
    *epoch_dev = epoch_s;
  }
  __syncthreads();
  const uint32_t epoch = epoch_s;
  __shared__ int rt[MAX_EXPERTS];   // recv totals per (dst, e_loc) = global expert
  __shared__ int cnt_s[MAX_EXPERTS];
  // (a) CumSum over chunks (chunk bases) and C_exp
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int s = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int v = p.hist[(size_t)c * E + e];
      p.hist[(size_t)c * E + e] = s;
      s += v;
    }
    p.counts[e] = s;
    cnt_s[e] = s;
  }
  __syncthreads();
  // (b) AllGather of C_exp: P2P store of my row into every peer's table, then release flag
  for (int i = threadIdx.x; i < W * E; i += blockDim.x) {
    const int dst = i / E, e = i % E;
    peers.p[dst].cnt_all[me * E + e] = cnt_s[e];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int dst = 0; dst < W; ++dst) st_release_sys(peers.p[dst].cnt_flag + me, epoch);
  }
  // (c) wait for every source's row
  if (threadIdx.x < W) {
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(peers.p[me].cnt_flag + threadIdx.x) != epoch) {
      if (globaltimer() - t0 > timeout_ns) {
        if (atomicCAS(err, 0, 3) == 0) {
          err[1] = 1;
          err[4] = threadIdx.x;
        }
        break;
      }
    }
  }
  __syncthreads();
  const int* call = peers.p[me].cnt_all;
  // (d) receive totals of every (rank, local expert)  (token_map.cpp:71-74)
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int s = 0;
    for (int src = 0; src < W; ++src) s += call[src * E + e];
    rt[e] = s;
    p.rt_all[e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // segment bases, reference (unaligned) and the 128-aligned layout used here
    for (int dst = 0; dst < W; ++dst) {
      int a = 0, b = 0;
      for (int el = 0; el < epr; ++el) {
        const int e = dst * epr + el;
        p.sb_all_ref[e] = a;
        p.sb_all[e] = b;
        a += rt[e];
        b += (rt[e] + 127) & ~127;
      }
      if (dst == me) {
        p.scalars[0] = b;
        p.scalars[1] = b >> 7;
        p.scalars[2] = a;
        if (b > d.M_cap) atomicExch(err, 2);
      }
    }
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
    for (int src = 0; src < me; ++src) o += call[src * E + e];
    p.o_all[e] = o;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) p.send_base[e] = p.sb_all[e] + p.o_all[e];
}

// 256 threads = 8 warps; warp w owns entries [w*256, w*256+256) of the chunk in 8 rounds of 32.
__global__ void __launch_bounds__(256) plan_entries_kernel(Dims d, PlanDev p, int n) {
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

// Zero the alignment rows of my receive buffer (rows [sb + rt, sb + align128(rt))).
__global__ void zero_padding_kernel(Dims d, PlanDev p, __nv_bfloat16* recv) {
  const int el = blockIdx.y;
  const int e = d.rank * d.epr + el;
  const int rows = p.rt_all[e];
  const int pad = ((rows + 127) & ~127) - rows;
  const int row0 = p.sb_all[e] + rows;
  const int vec_per_row = d.H / 8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pad * vec_per_row;
       i += gridDim.x * blockDim.x) {
    const int r = i / vec_per_row, c = i % vec_per_row;
    reinterpret_cast<int4*>(recv + (size_t)(row0 + r) * d.H)[c] = make_int4(0, 0, 0, 0);
  }
}

}  // namespace eplab_dev

namespace eplab_launch {
using namespace eplab_dev;

int plan_launch(const Dims& d, const Peers& peers, const PlanDev& p, uint32_t* epoch,
                uint64_t timeout_ns, int* err, cudaStream_t st) {
  const int n = p.n_tok * d.topk;
  const int nchunks = n > 0 ? (n + PLAN_CHUNK - 1) / PLAN_CHUNK : 0;
  if (nchunks > 0) plan_hist_kernel<<<nchunks, 256, 0, st>>>(p.topk_ids, n, d.E, p.hist);
  plan_global_kernel<<<1, 1024, 0, st>>>(d, peers, p, nchunks, epoch, timeout_ns, err);
  if (nchunks > 0) plan_entries_kernel<<<nchunks, 256, 0, st>>>(d, p, n);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// Loads the planning kernels into the current context up front (see preload_megakernels): the
// count exchange of plan_global_kernel spins until every virtual rank's planner has run.
int preload_plan() {
  cudaFuncAttributes fa;
  const bool ok = cudaFuncGetAttributes(&fa, plan_hist_kernel) == cudaSuccess &&
                  cudaFuncGetAttributes(&fa, plan_global_kernel) == cudaSuccess &&
                  cudaFuncGetAttributes(&fa, plan_entries_kernel) == cudaSuccess &&
                  cudaFuncGetAttributes(&fa, zero_padding_kernel) == cudaSuccess;
  return ok ? 0 : 1;
}

int zero_padding_launch(const Dims& d, const PlanDev& p, __nv_bfloat16* recv, cudaStream_t st) {
  dim3 grid(4, d.epr);
  zero_padding_kernel<<<grid, 256, 0, st>>>(d, p, recv);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace eplab_launch
