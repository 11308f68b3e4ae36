/*
 * eplab_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference `eplab` algorithms on the EP-MoE hot
 * path (/root/reference/proj/src/eplab) plus the MoE-layer numerics the
 * reference leaves undefined (GEMM / SwiGLU / backward).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it -- and only as the checker / CPU baseline, never as the product path.
 *
 * Pinning: the addressing / traffic / perf-model / tuner / fold functions are
 * checked against the reference's own golden vectors (proj/tests/*.cpp) and
 * against the reference compiled from its sources into oracle/_ref
 * (oracle/Makefile). The layer numerics (a22) have no reference implementation:
 * "parity unpinned" for GEMM/SwiGLU/backward values.
 */
#ifndef EPLAB_ORACLE_H_
#define EPLAB_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------- routing (a2) */
/* routing.cpp:32-73. sel[r][t*topk+j] (int32), gw same layout (float); arrays are
 * world * n_tok * topk long, rank-major. Returns 0, or 2 if topk > n_exp. */
int orc_sample_routing(int n_exp, int topk, long long n_tok, int world, uint64_t seed,
                       int32_t* sel, float* gw);

/* -------------------------------------------------------- token map (a3-a6) */
/* token_map.cpp:10-28: counts/offsets [n_exp], m_loc [n]. */
void orc_local_stable_sort(const int32_t* sel, long long n, int n_exp, int64_t* m_loc,
                           int64_t* counts, int64_t* offsets);
/* token_map.cpp:30-53: counts_all [world][n_exp] -> o_all [world(dst)][epr][world(src)]. */
int orc_global_offsets(const int64_t* counts_all, int world, int n_exp, int64_t* o_all);
/* token_map.cpp:55-106 for all ranks at once. sel is rank-major [world][n_tok*topk].
 * Outputs (rank-major [world][n_tok*topk]): target_rank, local_expert, offset;
 * recv_totals/seg_base [world*epr]. Returns 0 or 2 (validation). */
int orc_token_map(const int32_t* sel, int world, int n_exp, long long n_tok, int topk,
                  int32_t* target_rank, int32_t* local_expert, int64_t* offset,
                  int64_t* recv_totals, int64_t* seg_base);
/* token_map.cpp:108-126 for one source rank; item arrays [n_tok*topk]. */
void orc_send_schedule(const int32_t* target_rank, const int32_t* local_expert,
                       const int64_t* offset, long long n_tok, int topk, int world, int epr,
                       int64_t* item_token, int32_t* item_slot, int32_t* item_dst_rank,
                       int32_t* item_dst_expert, int64_t* item_dst_offset);
/* sim.cpp:384-390: primary[i] = first (token, dst_rank) in schedule order (world > 1). */
void orc_primary_flags(const int64_t* item_token, const int32_t* item_dst_rank, long long n,
                       int world, int8_t* primary);

/* ------------------------------------------------------------ traffic (a21) */
/* traffic.cpp:11-22 / :49-78. numerators as (hi, lo) 64-bit halves of an unsigned
 * 128-bit integer, index x-1. Returns 0 or 2. */
int orc_stirling2(int n, int k, uint64_t* hi, uint64_t* lo);
int orc_distinct_rank_distribution(int world, int topk, uint64_t* num_hi, uint64_t* num_lo,
                                   double* probs, double* expectation, double* saving);
typedef struct {
  double v_allgather, v_alltoall, v_megakernel_nvl, v_megakernel_hbm;
} orc_traffic;
/* traffic.cpp:103-112 (remote_only = SelfRankAccounting::RemoteOnly). */
int orc_volume_expected(long long n_tok, int topk, long long s_tok, int world, int remote_only,
                        orc_traffic* out);
/* traffic.cpp:114-140 over a routing instance (rank-major sel). */
int orc_volume_exact(const int32_t* sel, int world, int n_exp, long long n_tok, int topk,
                     long long s_tok, int remote_only, orc_traffic* out);

/* --------------------------------------------------------- perf model (a18) */
typedef struct {
  int n_sm;
  double p_peak, bw_hbm, bw_nvl, w_sat, tau_sync;
  int world_size;
} orc_hw;
typedef struct {
  int h_dim, h_inter, n_exp, topk;
  long long n_tok, s_tok;
  int b_m, b_n;
  int mu_n; /* entries in mu_w / mu_v */
  int mu_w[8];
  double mu_v[8];
} orc_shape;
typedef struct {
  int n_disp, n_relay, n_comb, n_red, w;
} orc_cfg;
typedef struct {
  double t_up, t_down, l_swiglu, l_disp, l_up, l_comb, l_down, t_red, l_s1, l_s2, l_total;
  long long n_tiles_up, n_tiles_down;
  double w_gap, w_red, w_rem;
} orc_breakdown;

double orc_effective_bandwidth(int n_sm_active, int w, double beta, double w_sat);
int orc_gemm_block_time(const orc_hw* hw, const orc_shape* s, long long k_dim, int w,
                        double* out);
double orc_swiglu(const orc_shape* s, const orc_hw* hw, long long expanded);
long long orc_tiles_up(const orc_shape* s, int world);
long long orc_tiles_down(const orc_shape* s, int world);
/* perf_model.cpp:94-135; redistributed = ResidualScaling::Redistributed. Returns 0 or 2. */
int orc_predict_latency(const orc_shape* s, const orc_hw* hw, const orc_cfg* cfg,
                        const orc_traffic* t, int redistributed, orc_breakdown* out);

/* -------------------------------------------------------------- tuner (a19) */
/* tuner.cpp:15-45: raw / enumerated / feasible grid sizes. */
int orc_space_sizes(int n_sm, long long* raw, long long* enumerated, long long* feasible);
/* tuner.cpp:90-148 (single thread; the tie-break makes the result worker-count
 * independent). Returns 0 or 2. */
int orc_search(const orc_shape* s, const orc_hw* hw, const orc_traffic* t, int redistributed,
               orc_cfg* best, double* l_min, long long* evaluated);

/* ------------------------------------------------------------ numerics (a15) */
float orc_round_to_bf16(float x);                /* softfloat.cpp:27-33 */
/* precision.cpp:31-37 left fold of w*v terms; bf16 = per-op rounding. */
float orc_fold(const float* w, const float* v, int n, int bf16);

/* ----------------------------------------------- MoE layer numerics (a11-a17, a22) */
/* The product's numeric contract, restated on the CPU.
 * Simulated EP=world over rank-major inputs. bf16 tensors are uint16 payloads.
 *   x, dy  : [world][n_tok][H]          sel/gw : [world][n_tok*topk]
 *   w_up   : [E][2F][H] (gate rows [0,F), up rows [F,2F))   w_down : [E][H][F]
 * Outputs: y, dx [world][n_tok][H] bf16; dgate [world][n_tok*topk] fp32;
 *          dw_up [E][2F][H] bf16; dw_down [E][H][F] bf16. Any output may be NULL.
 * threads <= 0 uses all OpenMP threads. Returns 0 or 2. */
typedef struct {
  int world, n_exp, topk, H, F;
  long long n_tok;
} orc_layer_dims;
int orc_moe_layer(const orc_layer_dims* d, const int32_t* sel, const float* gw,
                  const uint16_t* x, const uint16_t* w_up, const uint16_t* w_down,
                  const uint16_t* dy, uint16_t* y, uint16_t* dx, float* dgate, uint16_t* dw_up,
                  uint16_t* dw_down, int threads);

/* ------------------------------------------------------------- router (§8 f1) */
/* No reference implementation exists (the reference takes routing as input, routing.cpp:32-73;
 * gating is described at PAPER.md:54-55). These define the product's router semantics, spelled
 * operation by operation so the CUDA kernel (csrc/kernels/router.cu) is bit-exact with them:
 * top-k by the IEEE total order of the logits (descending, ties -> lower index); renorm=1 softmax
 * over the selected, renorm=0 full-softmax probabilities with Z summed in the warp's order
 * (lane-strided partials, xor butterfly 16..1); exp from a fixed fmaf polynomial. Pinned by
 * tests/test_oracle.py against an independent float64 softmax/top-k (numpy). */
float orc_exp_portable(float x);
int orc_router_topk(const float* logits, long long n_tok, int n_exp, int topk, int renorm, int32_t* ids,
                    float* gw);
int orc_router_topk_bwd(const float* logits, const int32_t* ids, const float* gw, const float* dgate,
                        long long n_tok, int n_exp, int topk, int renorm, float* dlogits);

/* Deterministic synthetic bf16 data: N(0,1)*scale via splitmix64 + Box-Muller. */
void orc_fill_normal_bf16(uint16_t* out, long long n, uint64_t seed, float scale);

#ifdef __cplusplus
}
#endif
#endif
