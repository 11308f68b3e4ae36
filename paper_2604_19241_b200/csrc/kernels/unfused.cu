// The unfused EP-MoE baseline of SURVEY.md §8(d): NCCL all-to-all -> grouped GEMM -> NCCL all-to-all
// back -> k-order reduce, as separate kernels with the collectives (issued by the host through
// NCCL) in between -- no overlap of communication with the GEMMs, host synchronisation for the
// split sizes. Its GroupGEMM tiles are the MegaKernels' (same engine, same epilogues, same K order)
// with every collective removed (MkArgs::unfused), and the reduce below is the MegaKernels' fold, so
// the unfused step is the bitwise reference of the fused one (precision.cpp:54-96
// fused_vs_sequential: "fused combine == sequential combine").
//
//   pack     : x (or dY) rows -> the all-to-all send buffer, ordered by destination rank, then by
//              (local expert, t, j) -- the local stable-sort position m_loc of Alg. 1 l.1-2 -- plus
//              each row's (gate weight, t*k+j) for the receiver
//   scatter  : received rows (source-major, as the all-to-all delivers them) -> the receive layout
//              of the fused path (128-aligned expert segments in global (src, t, j) order, Alg. 1
//              final_idx) + slot metadata + the slot's position in the return all-to-all
//   fold     : the k-ascending reference fold over the returned rows (precision.cpp:31-37)
//   dgate    : the sum of the returned gate-gradient partials, in the fused reduce's order
#include <algorithm>

#include "moe_common.cuh"
#include "ptx.cuh"

namespace eplab_dev {

// Exclusive prefix of this rank's per-expert counts (expert order = (dst, e_loc) order) in smem.
__device__ __forceinline__ void count_prefix(const Dims& d, const PlanDev& p, int* pre) {
  if (threadIdx.x == 0) {
    int s = 0;
    for (int e = 0; e < d.E; ++e) {
      pre[e] = s;
      s += p.counts[e];
    }
  }
  __syncthreads();
}

// One warp per routing entry i = t*k + j.
__global__ void __launch_bounds__(256) unfused_pack_kernel(Dims d, PlanDev p, const __nv_bfloat16* src,
                                                           __nv_bfloat16* send, int2* send_meta, int* spos) {
  if (p.scalars[3]) return;
  __shared__ int pre[MAX_EXPERTS];
  count_prefix(d, p, pre);
  const int lane = threadIdx.x & 31, vecs = d.H / 8;
  const long long n = (long long)p.n_tok * d.topk;
  for (long long i = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); i < n; i += (long long)gridDim.x * 8) {
    const int e = p.topk_ids[i];
    const int pos = pre[e] + (p.dst_slot[i] - p.send_base[e]);  // m_loc of Alg. 1
    const int4* s = reinterpret_cast<const int4*>(src + (size_t)(i / d.topk) * d.H);
    int4* o = reinterpret_cast<int4*>(send + (size_t)pos * d.H);
    for (int c = lane; c < vecs; c += 32) o[c] = ld_nc_v4(s + c);
    if (lane == 0) {
      spos[i] = pos;
      if (send_meta) send_meta[pos] = make_int2(__float_as_int(p.gate_w[i]), (int)i);
    }
  }
}

// One warp per received row r. call = the all-gathered counts [W][E + 1].
__global__ void __launch_bounds__(256) unfused_scatter_kernel(Dims d, PlanDev p, const int* call,
                                                              const __nv_bfloat16* recv, const int2* recv_meta,
                                                              int n_recv, __nv_bfloat16* dst, SlotMeta* meta,
                                                              int* ret_pos) {
  if (p.scalars[3]) return;
  const int W = d.world, epr = d.epr, me = d.rank, stride = d.E + 1;
  __shared__ int rb[MAX_EXPERTS + 1];  // received-row base of (src, e_loc), src-major
  __shared__ int ob[MAX_EXPERTS];      // slot base of (src, e_loc): segment base + O_all (Eq. 1)
  if (threadIdx.x == 0) {
    int r = 0;
    for (int s = 0; s < W; ++s)
      for (int el = 0; el < epr; ++el) {
        const int q = s * epr + el;
        rb[q] = r;
        r += call[s * stride + me * epr + el];
        int o = 0;
        for (int s2 = 0; s2 < s; ++s2) o += call[s2 * stride + me * epr + el];
        ob[q] = p.sb_all[me * epr + el] + o;
      }
    rb[W * epr] = r;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, vecs = d.H / 8;
  for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < n_recv; r += gridDim.x * 8) {
    int lo = 0, hi = W * epr - 1;  // last q with rb[q] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rb[mid] <= r)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int slot = ob[lo] + (r - rb[lo]);
    const int4* s = reinterpret_cast<const int4*>(recv + (size_t)r * d.H);
    int4* o = reinterpret_cast<int4*>(dst + (size_t)slot * d.H);
    for (int c = lane; c < vecs; c += 32) o[c] = ld_nc_v4(s + c);
    if (lane == 0) {
      ret_pos[slot] = r;
      if (recv_meta) {
        const int2 m = recv_meta[r];
        meta[slot] = SlotMeta{lo / epr, m.y, __int_as_float(m.x), -1};
      }
    }
  }
}

// One warp per token: the reference fold of its k returned rows (the same arithmetic as the
// MegaKernels' reduce role: products and sums rounded to fp32, no contraction, one RNE).
__global__ void __launch_bounds__(256) unfused_fold_kernel(Dims d, PlanDev p, const __nv_bfloat16* rows,
                                                           const int* spos, __nv_bfloat16* out, int ph) {
  if (p.scalars[3]) return;
  const int lane = threadIdx.x & 31, vecs = d.H / 8, k = d.topk;
  for (long long t = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); t < p.n_tok; t += (long long)gridDim.x * 8) {
    for (int c = lane; c < vecs; c += 32) {
      float acc[8];
      for (int j = 0; j < k; ++j) {
        const int4 v = ld_nc_v4(reinterpret_cast<const int4*>(rows + (size_t)spos[t * k + j] * d.H) + c);
        const float w = ph == 0 ? p.gate_w[t * k + j] : 1.0f;
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(hv[q]);
          const float px = ph == 0 ? __fmul_rn(w, f.x) : f.x;
          const float py = ph == 0 ? __fmul_rn(w, f.y) : f.y;
          acc[2 * q] = j == 0 ? px : __fadd_rn(acc[2 * q], px);
          acc[2 * q + 1] = j == 0 ? py : __fadd_rn(acc[2 * q + 1], py);
        }
      }
      int4 o;
      o.x = (int)pack_bf16(acc[0], acc[1]);
      o.y = (int)pack_bf16(acc[2], acc[3]);
      o.z = (int)pack_bf16(acc[4], acc[5]);
      o.w = (int)pack_bf16(acc[6], acc[7]);
      reinterpret_cast<int4*>(out + (size_t)t * d.H)[c] = o;
    }
  }
}

// One thread per routing entry: dgate_{t,j} = the sum of the entry's gate-gradient partials
// <dY W_down, h> over the down-dgrad column tiles (returned by the all-to-all), in tile order -- the
// fused reduce role's sum.
__global__ void __launch_bounds__(256) unfused_dgate_kernel(Dims d, PlanDev p, const float* parts,
                                                            const int* spos, float* dgate) {
  if (p.scalars[3]) return;
  const int ncb = d.F / 256;
  const long long n = (long long)p.n_tok * d.topk;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float* g = parts + (size_t)spos[i] * ncb;
    float s = g[0];
    for (int c = 1; c < ncb; ++c) s = __fadd_rn(s, g[c]);
    dgate[i] = s;
  }
}

}  // namespace eplab_dev

namespace eplab_launch {
using namespace eplab_dev;

static int grid_for(long long items, int sms) {
  const long long g = (items + 7) / 8;
  return (int)std::max(1LL, std::min(g, (long long)sms * 8));
}

int unfused_pack_launch(const Dims& d, const PlanDev& p, const __nv_bfloat16* src, __nv_bfloat16* send,
                        int2* send_meta, int* spos, int sms, cudaStream_t st) {
  unfused_pack_kernel<<<grid_for((long long)p.n_tok * d.topk, sms), 256, 0, st>>>(d, p, src, send, send_meta, spos);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
int unfused_scatter_launch(const Dims& d, const PlanDev& p, const int* call, const __nv_bfloat16* recv,
                           const int2* recv_meta, int n_recv, __nv_bfloat16* dst, SlotMeta* meta, int* ret_pos,
                           int sms, cudaStream_t st) {
  unfused_scatter_kernel<<<grid_for(n_recv, sms), 256, 0, st>>>(d, p, call, recv, recv_meta, n_recv, dst, meta,
                                                                 ret_pos);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
int unfused_fold_launch(const Dims& d, const PlanDev& p, const __nv_bfloat16* rows, const int* spos,
                        __nv_bfloat16* out, int ph, int sms, cudaStream_t st) {
  unfused_fold_kernel<<<grid_for(p.n_tok, sms), 256, 0, st>>>(d, p, rows, spos, out, ph);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
int unfused_dgate_launch(const Dims& d, const PlanDev& p, const float* parts, const int* spos, float* dgate,
                         int sms, cudaStream_t st) {
  const long long n = (long long)p.n_tok * d.topk;
  const int grid = (int)std::max(1LL, std::min((n + 255) / 256, (long long)sms * 8));
  unfused_dgate_kernel<<<grid, 256, 0, st>>>(d, p, parts, spos, dgate);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace eplab_launch
