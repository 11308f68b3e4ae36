// Router / gating step in front of the dispatch path: router
// logits [T][E] fp32 -> top-k expert ids [T][k] int32 + gate weights [T][k] fp32, and its
// backward dgate [T][k] -> dlogits [T][E]. The reference treats routing as an input
// (routing.cpp sample_routing); this produces the same a1/a3 tensors on device so
// eplab_plan can consume them directly.
//
// Semantics (oracle/eplab_oracle.c orc_router_topk restates them):
//   selection: the k largest logits, descending; equal logits -> lower expert index first;
//              ordering on the IEEE total order of the bit pattern (+NaN above +inf).
//   renorm=1 : w_j = exp(l_j - l_max) / sum_{i<k} exp(l_i - l_max)   (softmax over the selected)
//   renorm=0 : w_j = exp(l_j - l_max) / Z, Z = sum over all E experts (full-softmax probability)
//   backward : S = sum_j g_j w_j (fmaf, j ascending);
//              renorm=1: dl_{s_j} = w_j (g_j - S), other experts 0
//              renorm=0: dl_i = p_i ([i selected] g_i - S) with p_i recomputed as in the forward
// Every floating-point operation is spelled out (fmaf, IEEE divide, a fixed-order warp
// butterfly for Z, a portable exp) so the CPU oracle reproduces the outputs bit for bit.
//
// Layout: one warp per token; lane l holds experts l, l+32, ... (coalesced 128 B loads), 8 warps
// per CTA. HBM-bound: 4E bytes read + 8k written per token (bwd: 4E + 12k read, 4E written).
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "eplab_b200.h"
#include "../host/errors.hpp"

namespace eplab_dev {

// exp(x) for x <= 0 from fmaf/multiply only (Cody-Waite reduction + degree-7 Taylor); 0 below
// -87 (the result would be subnormal). Identical operation sequence in the oracle.
__device__ __forceinline__ float exp_portable(float x) {
  if (!(x >= -87.0f)) return 0.0f;  // also -inf and NaN
  const float n = rintf(__fmul_rn(x, 1.44269504088896341f));
  float r = fmaf(-n, 0.693145751953125f, x);
  r = fmaf(-n, 1.42860682030941723212e-6f, r);
  float p = 1.98412698412698413e-4f;  // 1/5040
  p = fmaf(p, r, 1.38888888888888889e-3f);
  p = fmaf(p, r, 8.33333333333333333e-3f);
  p = fmaf(p, r, 4.16666666666666667e-2f);
  p = fmaf(p, r, 1.66666666666666667e-1f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  const int e = (int)n;
  // 2^e for e in [-126, 0] (normal), product rounded once
  return __fmul_rn(p, __int_as_float((e + 127) << 23));
}

__device__ __forceinline__ uint32_t order_key(float v) {
  const uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// fixed-order warp sum: butterfly over xor offsets 16, 8, 4, 2, 1 (commutative adds: every lane
// ends with the same bits)
__device__ __forceinline__ float warp_sum_fixed(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

template <int NPL>
__device__ __forceinline__ void load_row(const float* __restrict__ row, int E, int lane, float (&l)[NPL]) {
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int i = lane + 32 * j;
    l[j] = i < E ? __ldg(row + i) : 0.0f;
  }
}

template <int NPL>
__device__ __forceinline__ float full_partition(const float (&l)[NPL], int E, int lane, float m) {
  float s = 0.0f;
#pragma unroll
  for (int q = 0; q < NPL; ++q)
    if (lane + 32 * q < E) s = __fadd_rn(s, exp_portable(__fsub_rn(l[q], m)));
  return warp_sum_fixed(s);
}

template <int NPL>
__global__ void __launch_bounds__(256) router_topk_kernel(const float* __restrict__ logits, int T, int E,
                                                          int k, int renorm, int32_t* __restrict__ ids,
                                                          float* __restrict__ gw) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  float l[NPL];
  load_row<NPL>(logits + (size_t)t * E, E, lane, l);
  // k rounds of a warp arg-max on (order key, lowest index); lane j keeps the j-th winner
  uint32_t taken = 0;
  int my_id = 0;
  float my_val = 0.0f, m = 0.0f, den = 0.0f;
  for (int j = 0; j < k; ++j) {
    uint32_t bk = 0, bi = 0;  // best key / (0xFFFFFFFF - idx) of this lane, bi == 0: none
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
      const int i = lane + 32 * q;
      if (i < E && !((taken >> q) & 1u)) {
        const uint32_t key = order_key(l[q]);
        if (bi == 0 || key > bk) {  // ascending i within the lane: the first max is the lowest index
          bk = key;
          bi = 0xFFFFFFFFu - (uint32_t)i;
        }
      }
    }
    const uint32_t kmax = __reduce_max_sync(0xFFFFFFFFu, bi ? bk : 0u);
    const uint32_t cmax = __reduce_max_sync(0xFFFFFFFFu, (bi && bk == kmax) ? bi : 0u);
    const int win = (int)(0xFFFFFFFFu - cmax);
    float v = 0.0f;  // the owner's register, compile-time indices only
#pragma unroll
    for (int q = 0; q < NPL; ++q)
      if ((win >> 5) == q) v = l[q];
    v = __shfl_sync(0xFFFFFFFFu, v, win & 31);
    if ((win & 31) == lane) taken |= 1u << (win >> 5);
    if (j == 0) m = v;
    if (renorm) den = __fadd_rn(den, exp_portable(__fsub_rn(v, m)));
    if (lane == j) {
      my_id = win;
      my_val = v;
    }
  }
  if (!renorm) den = full_partition<NPL>(l, E, lane, m);
  if (lane < k) {
    ids[(size_t)t * k + lane] = my_id;
    gw[(size_t)t * k + lane] = __fdiv_rn(exp_portable(__fsub_rn(my_val, m)), den);
  }
}

template <int NPL>
__global__ void __launch_bounds__(256) router_topk_bwd_kernel(const float* __restrict__ logits,
                                                              const int32_t* __restrict__ ids,
                                                              const float* __restrict__ gw,
                                                              const float* __restrict__ dgate, int T, int E,
                                                              int k, int renorm, float* __restrict__ dlogits) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const int my_id = lane < k ? __ldg(ids + (size_t)t * k + lane) : -1;
  const float my_w = lane < k ? __ldg(gw + (size_t)t * k + lane) : 0.0f;
  const float my_g = lane < k ? __ldg(dgate + (size_t)t * k + lane) : 0.0f;
  float S = 0.0f;  // sum_j g_j w_j, j ascending (every lane the same)
  for (int j = 0; j < k; ++j)
    S = fmaf(__shfl_sync(0xFFFFFFFFu, my_g, j), __shfl_sync(0xFFFFFFFFu, my_w, j), S);
  // per owned expert: selected? and its (g, w)
  uint32_t sel = 0;
  float gq[NPL], wq[NPL];
#pragma unroll
  for (int q = 0; q < NPL; ++q) gq[q] = wq[q] = 0.0f;
  for (int j = 0; j < k; ++j) {
    const int idj = __shfl_sync(0xFFFFFFFFu, my_id, j);
    const float gj = __shfl_sync(0xFFFFFFFFu, my_g, j), wj = __shfl_sync(0xFFFFFFFFu, my_w, j);
    if ((idj & 31) == lane) {
#pragma unroll
      for (int q = 0; q < NPL; ++q)
        if ((idj >> 5) == q) {
          gq[q] = gj;
          wq[q] = wj;
        }
      sel |= 1u << (idj >> 5);
    }
  }
  float* out = dlogits + (size_t)t * E;
  if (renorm) {
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
      const int i = lane + 32 * q;
      if (i < E) out[i] = ((sel >> q) & 1u) ? __fmul_rn(wq[q], __fsub_rn(gq[q], S)) : 0.0f;
    }
  } else {
    float l[NPL];
    load_row<NPL>(logits + (size_t)t * E, E, lane, l);
    uint32_t kmax = 0;  // max logit on the key order (== the forward's top-1 value)
#pragma unroll
    for (int q = 0; q < NPL; ++q)
      if (lane + 32 * q < E) kmax = max(kmax, order_key(l[q]));
    kmax = __reduce_max_sync(0xFFFFFFFFu, kmax);
    const float m = __uint_as_float((kmax & 0x80000000u) ? (kmax & 0x7FFFFFFFu) : ~kmax);
    const float Z = full_partition<NPL>(l, E, lane, m);
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
      const int i = lane + 32 * q;
      if (i >= E) continue;
      const float p = __fdiv_rn(exp_portable(__fsub_rn(l[q], m)), Z);
      out[i] = __fmul_rn(p, ((sel >> q) & 1u) ? __fsub_rn(gq[q], S) : -S);
    }
  }
}

template <int NPL>
static void launch_fwd(const float* lg, int T, int E, int k, int renorm, int32_t* ids, float* gw,
                       cudaStream_t st) {
  router_topk_kernel<NPL><<<(T + 7) / 8, 256, 0, st>>>(lg, T, E, k, renorm, ids, gw);
}

template <int NPL>
static void launch_bwd(const float* lg, const int32_t* ids, const float* gw, const float* dg, int T, int E,
                       int k, int renorm, float* dl, cudaStream_t st) {
  router_topk_bwd_kernel<NPL><<<(T + 7) / 8, 256, 0, st>>>(lg, ids, gw, dg, T, E, k, renorm, dl);
}

static int npl_of(int E) {
  int n = 1;
  while (n * 32 < E) n <<= 1;
  return n;
}

static int check_args(int T, int E, int k) {
  if (T < 0 || E < 1 || E > 1024 || k < 1 || k > 32 || k > E) {
    eplab_host::set_last_error("router: need T >= 0, 1 <= n_experts <= 1024, 1 <= topk <= min(32, n_experts)");
    return EPLAB_ERR_VALIDATION;
  }
  return EPLAB_OK;
}

static int finish() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    eplab_host::set_last_error(std::string("router launch: ") + cudaGetErrorString(e));
    return EPLAB_ERR_INTERNAL;
  }
  return EPLAB_OK;
}

}  // namespace eplab_dev

using namespace eplab_dev;

extern "C" {

int eplab_router_topk(const float* logits, int n_tok, int n_experts, int topk, int renorm, int32_t* topk_ids,
                      float* gate_w, void* stream) {
  if (int rc = check_args(n_tok, n_experts, topk)) return rc;
  if (n_tok == 0) return EPLAB_OK;
  const cudaStream_t st = (cudaStream_t)stream;
  switch (npl_of(n_experts)) {
    case 1: launch_fwd<1>(logits, n_tok, n_experts, topk, renorm, topk_ids, gate_w, st); break;
    case 2: launch_fwd<2>(logits, n_tok, n_experts, topk, renorm, topk_ids, gate_w, st); break;
    case 4: launch_fwd<4>(logits, n_tok, n_experts, topk, renorm, topk_ids, gate_w, st); break;
    case 8: launch_fwd<8>(logits, n_tok, n_experts, topk, renorm, topk_ids, gate_w, st); break;
    case 16: launch_fwd<16>(logits, n_tok, n_experts, topk, renorm, topk_ids, gate_w, st); break;
    default: launch_fwd<32>(logits, n_tok, n_experts, topk, renorm, topk_ids, gate_w, st); break;
  }
  return finish();
}

int eplab_router_topk_bwd(const float* logits, const int32_t* topk_ids, const float* gate_w, const float* dgate,
                          int n_tok, int n_experts, int topk, int renorm, float* dlogits, void* stream) {
  if (int rc = check_args(n_tok, n_experts, topk)) return rc;
  if (n_tok == 0) return EPLAB_OK;
  const cudaStream_t st = (cudaStream_t)stream;
  switch (npl_of(n_experts)) {
    case 1: launch_bwd<1>(logits, topk_ids, gate_w, dgate, n_tok, n_experts, topk, renorm, dlogits, st); break;
    case 2: launch_bwd<2>(logits, topk_ids, gate_w, dgate, n_tok, n_experts, topk, renorm, dlogits, st); break;
    case 4: launch_bwd<4>(logits, topk_ids, gate_w, dgate, n_tok, n_experts, topk, renorm, dlogits, st); break;
    case 8: launch_bwd<8>(logits, topk_ids, gate_w, dgate, n_tok, n_experts, topk, renorm, dlogits, st); break;
    case 16: launch_bwd<16>(logits, topk_ids, gate_w, dgate, n_tok, n_experts, topk, renorm, dlogits, st); break;
    default: launch_bwd<32>(logits, topk_ids, gate_w, dgate, n_tok, n_experts, topk, renorm, dlogits, st); break;
  }
  return finish();
}

}  // extern "C"
