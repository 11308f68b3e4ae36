/*
 * eplab_b200.h -- C-ABI of libeplab_b200.so, the B200-native (sm_100a) data path
 * for the expert-parallel MoE layer of arXiv 2604.19241 (Dispatch+GroupGEMM and
 * GroupGEMM+Combine MegaKernels, forward and backward).
 *
 * The reference (`/root/reference/proj`, namespace `eplab`) is a CPU lab whose
 * data-path entry points are addressing / control-flow / numerics models:
 *   dispatch   ~ build_global_token_map / build_send_schedule  (token_map.hpp:68, :88)
 *                + run_dispatch_gemm_sim                        (sim.hpp:87)
 *   group_gemm ~ the simulators' compute tasks, tile time/count (perf_model.hpp:40, :57-58)
 *   combine    ~ run_gemm_combine_sim (sim.hpp:88) + k-ordered fold `accumulate`
 *                (precision.hpp:30)
 * Each export below names the reference interface it replaces. Conventions:
 *   - plain pointers and sizes only; device pointers are marked `d_`;
 *   - return 0 ok, 1 internal/CUDA error, 2 validation error, 3 deadlock/timeout
 *     (the reference CLI's exit codes, tools/main.cpp:503-511); the message of the
 *     last failure is available from eplab_last_error();
 *   - every device call is ordered on the caller's stream (`stream` is a
 *     cudaStream_t) and performs no host synchronisation unless stated.
 */
#ifndef EPLAB_B200_H_
#define EPLAB_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define EPLAB_API __attribute__((visibility("default")))
#else
#define EPLAB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum { EPLAB_OK = 0, EPLAB_ERR_INTERNAL = 1, EPLAB_ERR_VALIDATION = 2, EPLAB_ERR_DEADLOCK = 3 };

/* ------------------------------------------------------------------ misc */

/* Library version string (reference: version.hpp:7 kVersion). */
EPLAB_API const char* eplab_version(void);

/* Copies the thread's last error message into buf (NUL-terminated). Returns its length. */
EPLAB_API size_t eplab_last_error(char* buf, size_t len);

/* ------------------------------------------------------- grouped GEMMs (unfused) */

/* C[m, n] = sum_k A[m, k] * B[e][n, k] for each expert segment e: rows
 * [seg_start[e], seg_start[e] + seg_rows[e]) of A (seg_start multiples of 128, host arrays).
 * bf16 in, fp32 accumulate, bf16 out. The GroupGEMM compute task of the reference
 * (perf_model.cpp:16-23 tile time, :74-92 tile count) as a stand-alone op; also the
 * GEMM of the unfused NCCL baseline. d_workspace >= 32 * tiles + 4 bytes. */
EPLAB_API int eplab_grouped_gemm_nt(const void* d_A, const void* d_B, void* d_C, int M_total,
                                    int N, int K, int n_experts, const int* seg_start,
                                    const int* seg_rows, void* d_workspace, void* stream);

/* Transposed GroupGEMM (weight-gradient shape):
 * C[e][i, j] = sum_{m in seg e} A[m, i] * B[m, j]; padded segment rows must be zero. */
EPLAB_API int eplab_grouped_gemm_tn(const void* d_A, const void* d_B, void* d_C, int M_total,
                                    int NA, int NB, int n_experts, const int* seg_start,
                                    const int* seg_rows_padded, void* d_workspace, void* stream);

/* The same two GEMMs on CTA pairs (cta_group::2, 256x256 tiles, B fetched once per pair). */
EPLAB_API int eplab_grouped_gemm_nt_pair(const void* d_A, const void* d_B, void* d_C, int M_total,
                                         int N, int K, int n_experts, const int* seg_start,
                                         const int* seg_rows, void* d_workspace, void* stream);
EPLAB_API int eplab_grouped_gemm_tn_pair(const void* d_A, const void* d_B, void* d_C, int M_total,
                                         int NA, int NB, int n_experts, const int* seg_start,
                                         const int* seg_rows_padded, void* d_workspace,
                                         void* stream);

/* ------------------------------------------------------- router
 * The gating step in front of dispatch. The reference takes routing as input
 * (routing.cpp sample_routing: k distinct experts per token + weights summing to 1); these
 * produce the same topk_ids [T][k] int32 / gate_w [T][k] fp32 on device from router logits
 * [T][E] fp32, ready for eplab_plan. Top-k descending, ties -> lower expert index.
 * renorm = 1: softmax over the k selected logits (weights sum to 1, like sample_routing);
 * renorm = 0: full softmax probabilities of the selected experts.
 * Backward: dgate [T][k] (eplab_moe_bwd's d_dgate) -> dlogits [T][E].
 * 1 <= topk <= min(32, E), E <= 1024. Bit-exact with oracle/eplab_oracle.c orc_router_topk. */
EPLAB_API int eplab_router_topk(const float* d_logits, int n_tok, int n_experts, int topk, int renorm,
                                int32_t* d_topk_ids, float* d_gate_w, void* stream);
EPLAB_API int eplab_router_topk_bwd(const float* d_logits, const int32_t* d_topk_ids, const float* d_gate_w,
                                    const float* d_dgate, int n_tok, int n_experts, int topk, int renorm,
                                    float* d_dlogits, void* stream);


/* ------------------------------------------- NB split-batch backward
 * d_acc[i] = bf16_rne(float(d_acc[i]) + float(d_add[i])) for n bf16 elements (16-byte aligned):
 * sums the per-sub-batch weight gradients of the opt-in non-bitwise split-batch backward
 * (PAPER.md:647-651), the two-way split of precision.cpp:98-134 on real gradients. */
EPLAB_API int eplab_bf16_accumulate(void* d_acc, const void* d_add, size_t n, void* stream);

/* ------------------------------------------------------- EP-MoE context (per rank) */

typedef struct eplab_ctx eplab_ctx;

/* Launch parameters chosen by the performance model (reference TuneConfig, types.hpp:45-53).
 * n_disp: comm tasks; n_relay: relay tasks (0 = AllToAll-style, every replica sent directly;
 * >0 = AllGather-style dedup + intra-rank multicast); n_red: reduce tasks. n_comb must be 0 or 1
 * (the combine push is the GEMM epilogue: there are no combine CTAs) and w must be 8 (one
 * 256-thread CTA per SM; comm workers are single warps, the warp split is
 * eplab_set_comm_options); other values return 2. The tile is fixed at 256 x 256 (CTA pairs). */
typedef struct {
  int n_disp, n_relay, n_comb, n_red, w;
} eplab_tune_config;

typedef struct {
  int rank, world, device;
  int max_tokens;         /* tokens per rank per call (T_max) */
  int hidden, ffn;        /* H, F (F = moe_ffn; W_up is [E_loc][2F][H]) */
  int n_experts, topk;    /* global expert count E (sharded contiguously, e // (E/W)) */
  long long max_recv_rows;/* 0 = worst case */
  double timeout_s;       /* scoreboard watchdog (0 = 10 s) */
} eplab_init_args;

/* Allocates the symmetric region (receive buffers, scoreboard, replica slots, count table)
 * and local activations for one rank on `device`. Reference analogue: the simulator state
 * built by DispatchSim::build / CombineSim::build (sim.cpp:355-442, :767-864). */
EPLAB_API int eplab_init(const eplab_init_args* args, eplab_ctx** out);
EPLAB_API int eplab_destroy(eplab_ctx* ctx);

/* Peer wiring. Multi-process: export my region's record (EPLAB_IPC_HANDLE_BYTES: the CUDA IPC
 * handle, then a layout signature -- hidden, ffn, experts, topk, world, max_tokens, receive
 * capacity, device SM count, region size), all-gather the records (NCCL / torch.distributed
 * bootstrap) and import them (world records, rank order). eplab_connect_ipc returns 2 when any
 * peer's layout differs (its peer pointers and the senders' slot writes would be wrong).
 * Single process (several contexts on one or more devices): link them directly (same check). */
#define EPLAB_IPC_HANDLE_BYTES 128
EPLAB_API int eplab_ipc_handle(eplab_ctx* ctx, void* handle);
EPLAB_API int eplab_connect_ipc(eplab_ctx* ctx, const void* handles);
EPLAB_API int eplab_connect_local(eplab_ctx* const* ctxs, int n);

EPLAB_API int eplab_set_tune_config(eplab_ctx* ctx, const eplab_tune_config* cfg);
EPLAB_API int eplab_get_tune_config(const eplab_ctx* ctx, eplab_tune_config* cfg);
/* Auto-tune (the default until eplab_set_tune_config is called): every eplab_plan picks the launch
 * parameters for its n_tok from the B200 performance model (search_layer), cached per 4096-token
 * bucket as the reference TuneCache does (tuner.hpp:60). on = 1 re-enables it (clears the cache). */
EPLAB_API int eplab_set_auto_tune(eplab_ctx* ctx, int on);
/* Work for the GEMM CTAs' idle warps (the unified primitive's warp split), a bit set:
 * bit 0 (comm): they drain the dispatch MegaKernels' priority-ordered round pool together with
 * the n_disp comm CTAs, so n_disp may be 0; bit 1 (reduce): they fold completed dX tokens in the
 * backward combine MegaKernel while its weight-gradient tiles run. Default 3. bulk_mover = 1 moves
 * rows through the TMA bulk-copy engine (comm CTAs only) instead of warp copies. Results are
 * bitwise identical for every setting. */
EPLAB_API int eplab_set_comm_options(eplab_ctx* ctx, int spare_warps, int bulk_mover);
/* Experiment knobs (A/B measurements; never read from the environment): "engine_pair" (1: CTA-pair
 * engine, 0: single-CTA), "spare" / "comm_bulk" (as eplab_set_comm_options), "rgp" / "tngp" /
 * "tngp_d" (raster groups of the NT / up-TN / down-TN pair tiles), "bwd_disp_scale" (comm CTAs of
 * the backward dispatch relative to the forward's), "pdl" (1, default: the CTA-pair MegaKernels use
 * programmatic dependent launch when the rank owns the whole device), "dbg" (debug bits that SKIP work: results
 * wrong, for measuring a role's share only). Unknown names return 2. */
EPLAB_API int eplab_set_option(eplab_ctx* ctx, const char* name, int value);
/* Persistent grid size (default: all SMs). Several ranks sharing one GPU (the single-device
 * multi-rank test mode) each get a disjoint budget so their MegaKernels are co-resident. */
EPLAB_API int eplab_set_sm_budget(eplab_ctx* ctx, int n_sm);

/* Device token map (Alg. 1 + count AllGather + priority schedule), token_map.hpp:68 and :88.
 * d_topk_ids int32 [n_tok][topk], d_gate_w fp32 [n_tok][topk]; both must stay valid until
 * the backward calls of this iteration. Starts a new iteration (epoch).
 * On the device the planner applies validate_routing's checks (types.cpp:74-94: expert id in
 * [0, E), distinct experts per token, finite gate weights) and checks the receive capacity of
 * EVERY rank (max_recv_rows). A failure on any rank aborts the iteration on all ranks -- every
 * kernel of it returns without reading or writing rows -- and eplab_check reports 2 with the
 * reason (the host cannot see device routing without a synchronisation). */
EPLAB_API int eplab_plan(eplab_ctx* ctx, const int32_t* d_topk_ids, const float* d_gate_w,
                         int n_tok, void* stream);

/* Dispatch+GroupGEMM MegaKernel, forward (run_dispatch_gemm_sim, sim.hpp:87): pushes x rows to
 * the expert ranks and runs the up GroupGEMM + SwiGLU as rowgroups land. */
EPLAB_API int eplab_dispatch_group_gemm(eplab_ctx* ctx, const void* d_x, const void* d_w_up,
                                        void* stream);
/* GroupGEMM+Combine MegaKernel, forward (run_gemm_combine_sim, sim.hpp:88 + accumulate,
 * precision.hpp:30): down GroupGEMM whose epilogue pushes each replica to its source, then
 * the top-k barrier and the k-ordered reduction into d_y [n_tok][H] bf16. */
EPLAB_API int eplab_group_gemm_combine(eplab_ctx* ctx, const void* d_w_down, void* d_y,
                                       void* stream);
/* Backward Dispatch+GroupGEMM: dY dispatch, down dgrad + SwiGLU backward (whose epilogue also
 * forms the gate-gradient partials <dY W_down, h> per column tile), down weight gradient
 * (deterministic transposed GroupGEMM). d_dgate [n_tok][k] is completed by the following
 * eplab_group_gemm_combine_bwd (its reduce sums the partials in tile order). */
EPLAB_API int eplab_dispatch_group_gemm_bwd(eplab_ctx* ctx, const void* d_dy,
                                            const void* d_w_down, void* d_dw_down,
                                            float* d_dgate, void* stream);
/* Backward GroupGEMM+Combine: up dgrad pushed back and k-reduced into d_dx, up weight grad. */
EPLAB_API int eplab_group_gemm_combine_bwd(eplab_ctx* ctx, const void* d_w_up, void* d_dx,
                                           void* d_dw_up, void* stream);

/* Several forwards in flight on one context (pipelined micro-batches, layers sharing a context,
 * activation recomputation). A context holds ONE iteration's state -- the plan tables, the
 * received rows and slot metadata (symmetric region) and the saved g/u and h activations --
 * which the next eplab_plan overwrites. A stash is a copy of that state in caller-owned device
 * memory, sized to the iteration's actual receive rows (not the worst-case capacity):
 *   eplab_stash_bytes    bytes the current iteration's stash needs (synchronises `stream`: the
 *                        receive row count is on the device)
 *   eplab_stash_save     copies the state into d_dst (>= that many bytes) and fills *info
 *   eplab_stash_restore  copies a stash back; the context's current iteration becomes the stashed
 *                        one and its backward (eplab_moe_bwd / the two backward MegaKernels) may run.
 * The restored backward runs under a fresh epoch (every rank must restore in the same order: the
 * MegaKernels' flags and counter parities follow the epoch). Copies are enqueued on `stream`;
 * the routing / gate-weight tensors of the stashed plan must stay alive until its backward. */
typedef struct {
  uint32_t magic;     /* EPLAB_STASH_MAGIC */
  uint32_t epoch;     /* epoch of the stashed plan */
  int n_tok;
  int rows;           /* receive rows (128-aligned segments) */
  const int32_t* topk_ids;
  const float* gate_w;
  size_t bytes;       /* bytes used in the stash buffer */
} eplab_stash_info;
#define EPLAB_STASH_MAGIC 0x5354a5a5u
EPLAB_API int eplab_stash_bytes(eplab_ctx* ctx, size_t* bytes, void* stream);
EPLAB_API int eplab_stash_save(eplab_ctx* ctx, void* d_dst, size_t dst_bytes, eplab_stash_info* info,
                               void* stream);
EPLAB_API int eplab_stash_restore(eplab_ctx* ctx, const void* d_src, const eplab_stash_info* info,
                                  void* stream);

/* Whole layer. fwd = plan + the two forward MegaKernels; bwd = the two backward ones. */
EPLAB_API int eplab_moe_fwd(eplab_ctx* ctx, const int32_t* d_topk_ids, const float* d_gate_w,
                            int n_tok, const void* d_x, const void* d_w_up, const void* d_w_down,
                            void* d_y, void* stream);
EPLAB_API int eplab_moe_bwd(eplab_ctx* ctx, const void* d_dy, const void* d_w_up,
                            const void* d_w_down, void* d_dx, void* d_dw_up, void* d_dw_down,
                            float* d_dgate, void* stream);
/* fwd+bwd with HOST routing/activations (pinned for asynchronous copies): H2D copies, the
 * four MegaKernels on `stream`, D2H of y, dx and dgate. dY's upload runs under the forward
 * MegaKernels and y's download under the backward ones (two copy streams). Synchronises before
 * returning. */
EPLAB_API int eplab_moe_step_host(eplab_ctx* ctx, const int32_t* h_topk_ids,
                                  const float* h_gate_w, int n_tok, const void* h_x,
                                  const void* h_dy, const void* d_w_up, const void* d_w_down,
                                  void* h_y, void* h_dx, float* h_dgate, void* d_dw_up,
                                  void* d_dw_down, void* stream);
/* The same step enqueued without blocking the host. Consecutive steps alternate between two
 * device staging sets, so step i+1's uploads overlap step i's MegaKernels and step i's
 * downloads overlap step i+1's. Host inputs must stay unchanged and host outputs are valid only
 * after eplab_host_join(ctx, s) + a synchronisation of s (or a later blocking step). */
EPLAB_API int eplab_moe_step_host_async(eplab_ctx* ctx, const int32_t* h_topk_ids,
                                        const float* h_gate_w, int n_tok, const void* h_x,
                                        const void* h_dy, const void* d_w_up, const void* d_w_down,
                                        void* h_y, void* h_dx, float* h_dgate, void* d_dw_up,
                                        void* d_dw_down, void* stream);
/* Makes `stream` wait (on the device) for every enqueued host-step copy. */
EPLAB_API int eplab_host_join(eplab_ctx* ctx, void* stream);

/* Synchronises `stream` and reports the device error word: 0 ok, 2 the iteration was aborted by
 * the planner's checks (bad routing on some rank, or a rank's receive capacity exceeded), 3 a
 * scoreboard watchdog fired (DeadlockError analogue, error.hpp:19-22; the message names the wait
 * site). Clears it. Until it is cleared every later kernel of the context skips its work. */
EPLAB_API int eplab_check(eplab_ctx* ctx, void* stream);

/* Bit-exact exports of the device token map (synchronising). Arrays of n_tok*topk entries;
 * recv_totals / seg_base have world*epr entries (GlobalTokenMap, token_map.hpp:52-66). */
EPLAB_API int eplab_export_token_map(eplab_ctx* ctx, int32_t* target_rank, int32_t* local_expert,
                                     int64_t* offset, int64_t* recv_totals, int64_t* seg_base);
/* Priority send schedule (SendSchedule, token_map.hpp:70-88): token and k-slot per item. */
EPLAB_API int eplab_export_schedule(eplab_ctx* ctx, int64_t* item_token, int32_t* item_slot);
/* Receive-side geometry actually used: 128-aligned segment base and rows per local expert. */
EPLAB_API int eplab_export_layout(eplab_ctx* ctx, int32_t* seg_base_aligned, int32_t* rows);
/* Device pointer of a named internal buffer (tests / profiling): "recv_x", "recv_dy", "gu",
 * "hact", "dgu", "hw", "rep", "rep_dx". */
EPLAB_API void* eplab_buffer(eplab_ctx* ctx, const char* name);

/* Device timeline (per-task %globaltimer intervals, role, SM) for overlap analysis, exported in
 * the reference's Chrome-trace format (trace.cpp:13-34). cap = 0 disables. */
EPLAB_API int eplab_timeline_enable(eplab_ctx* ctx, int cap);
EPLAB_API int eplab_timeline_export(eplab_ctx* ctx, const char* path, double* overlap_frac);

/* ------------------------------------------ unfused baseline
 * NCCL all-to-all -> grouped GEMM (+SwiGLU) -> NCCL all-to-all back -> k-order reduce, as separate
 * kernels with the caller's collectives in between (host-synchronised split sizes, no overlap).
 * The GEMM tiles are the MegaKernels' own (same engine, epilogues, K order) with the collectives
 * removed and the fold is the MegaKernels' fold, so a step through these entry points is BITWISE
 * equal to the fused step: the reference's fused_vs_sequential contract (precision.cpp:54-96).
 * Per step and rank (A2A = the caller's all-to-all, rows as the first dimension):
 *   plan_counts(row[E+1]) ; AllGather rows -> rows_all[W][E+1] ; plan_finish(rows_all)
 *   pack(x, send, send_meta[n][2]) ; A2A(send, send_meta) ; scatter(recv, recv_meta, n_recv, 0)
 *   up(w_up) ; down(w_down, o_ret[n_recv]) ; A2A back -> o_src[n_send] ; combine(o_src, y, 0)
 *   pack(dy, send, NULL) ; A2A ; scatter(recv, NULL, n_recv, 1)
 *   bwd_down(w_down, dw_down, dgp_ret[n_recv][F/256] f32) ; A2A back -> dgp_src ; dgate(dgp_src, dgate)
 *   bwd_up(w_up, dx_ret, dw_up) ; A2A back -> dx_src ; combine(dx_src, dx, 1)
 * Send split to rank d = sum of rows_all[me][d*epr .. d*epr+epr); receive split from rank s = sum of
 * rows_all[s][me*epr .. me*epr+epr). Paper_2604_19241_b200/unfused.py drives it over NCCL. */
EPLAB_API int eplab_unfused_plan_counts(eplab_ctx* ctx, const int32_t* d_topk_ids, const float* d_gate_w,
                                        int n_tok, int32_t* d_row, void* stream);
EPLAB_API int eplab_unfused_plan_finish(eplab_ctx* ctx, const int32_t* d_rows_all, void* stream);
EPLAB_API int eplab_unfused_pack(eplab_ctx* ctx, const void* d_src, void* d_send, int32_t* d_send_meta,
                                 void* stream);
EPLAB_API int eplab_unfused_scatter(eplab_ctx* ctx, const void* d_recv, const int32_t* d_recv_meta, int n_recv,
                                    int phase, void* stream);
EPLAB_API int eplab_unfused_up(eplab_ctx* ctx, const void* d_w_up, void* stream);
EPLAB_API int eplab_unfused_down(eplab_ctx* ctx, const void* d_w_down, void* d_o_ret, void* stream);
EPLAB_API int eplab_unfused_combine(eplab_ctx* ctx, const void* d_rows, void* d_out, int phase, void* stream);
EPLAB_API int eplab_unfused_dgate(eplab_ctx* ctx, const float* d_dgp_src, float* d_dgate, void* stream);
EPLAB_API int eplab_unfused_bwd_down(eplab_ctx* ctx, const void* d_w_down, void* d_dw_down, float* d_dgp_ret,
                                     void* stream);
EPLAB_API int eplab_unfused_bwd_up(eplab_ctx* ctx, const void* d_w_up, void* d_dx_ret, void* d_dw_up,
                                   void* stream);

/* ------------------------------------------------ host model API (C view of eplab::, eplab.hpp) */

typedef struct {
  int n_sm;
  double p_peak, bw_hbm, bw_nvl, w_sat, tau_sync;
  int world_size;
} eplab_hw;                          /* HardwareSpec, types.hpp:16-25 */
typedef struct {
  int h_dim, h_inter, n_exp, topk;
  long long n_tok, s_tok;
  int b_m, b_n;
  int mu_n;
  int mu_w[8];
  double mu_v[8];
} eplab_shape;                       /* MoEShape, types.hpp:28-42 */
typedef struct {
  double v_allgather, v_alltoall, v_megakernel_nvl, v_megakernel_hbm;
} eplab_traffic;                     /* TrafficReport, traffic.hpp:39-44 */
typedef struct {
  double t_up, t_down, l_swiglu, l_disp, l_up, l_comb, l_down, t_red, l_s1, l_s2, l_total;
  long long n_tiles_up, n_tiles_down;
  double w_gap, w_red, w_rem;
} eplab_breakdown;                   /* LatencyBreakdown, perf_model.hpp:17-35 */
typedef struct {
  double mu, tile_overhead, comm_bw_per_sm, relay_bw_per_sm, reduce_bw, launch, epi_bw_per_sm,
      spare_sm_equiv, hbm_overlap, startup;
} eplab_b200_calib;                  /* B200 calibration of this build's MegaKernels (eplab::B200Calib) */
typedef struct {
  double fwd_dispatch, fwd_combine, bwd_dispatch, bwd_combine, total, t_gemm_bound, t_nvl_bound;
} eplab_layer_prediction;

/* sample_routing (routing.hpp:15): sel int32 / gw fp32, rank-major [world][n_tok*topk]. */
EPLAB_API int eplab_sample_routing(int n_exp, int topk, long long n_tok, int world, uint64_t seed,
                                   int32_t* sel, float* gw);
/* build_global_token_map (token_map.hpp:68) on the host, all ranks; outputs rank-major. */
EPLAB_API int eplab_host_token_map(const int32_t* sel, int world, int n_exp, long long n_tok,
                                   int topk, int32_t* target_rank, int32_t* local_expert,
                                   int64_t* offset, int64_t* recv_totals, int64_t* seg_base);
/* One rank's part of build_global_token_map, as each rank computes it in an EP run: its own
 * routing sel [n_tok*topk] (local stable sort, Alg. 1 l.1-2) and the all-gathered per-expert
 * counts of every rank counts_all [world][n_exp] (l.3) give its map entries (l.4-16). */
EPLAB_API int eplab_host_rank_token_map(const int32_t* sel, const int64_t* counts_all, int rank, int world,
                                        int n_exp, long long n_tok, int topk, int32_t* target_rank,
                                        int32_t* local_expert, int64_t* offset);
/* build_send_schedule (token_map.hpp:88) for one rank. */
EPLAB_API int eplab_host_send_schedule(const int32_t* sel, int world, int n_exp, long long n_tok,
                                       int topk, int rank, int64_t* item_token, int32_t* item_slot,
                                       int32_t* item_dst_rank, int32_t* item_dst_expert,
                                       int64_t* item_dst_offset);
/* build_task_list (sim.hpp:84): one rank's dispatch-kernel task layout -- comm_slices [n_disp][2] (send
 * schedule ranges balanced by NVLink transmissions), relay_ranges [n_relay][2] (up-GEMM tile ranges),
 * n_comp (up-GEMM tiles). Routing sel [world][n_tok*topk] with the shape's n_exp, n_tok, topk. */
EPLAB_API int eplab_host_build_task_list(const int32_t* sel, int world, const eplab_shape* s,
                                         const eplab_tune_config* c, int rank, int64_t* comm_slices,
                                         int64_t* relay_ranges, int64_t* n_comp);
/* volume_expected (traffic.hpp:46); remote_only = SelfRankAccounting::RemoteOnly. */
EPLAB_API int eplab_volume_expected(const eplab_shape* s, const eplab_hw* h, int remote_only,
                                    eplab_traffic* out);
/* predict_latency (perf_model.hpp:60), reference-compatible forward model. */
EPLAB_API int eplab_predict_latency(const eplab_shape* s, const eplab_hw* h,
                                    const eplab_tune_config* c, const eplab_traffic* t,
                                    int redistributed, eplab_breakdown* out);
/* search (tuner.hpp:49): exhaustive, deterministic for any worker count. */
EPLAB_API int eplab_search(const eplab_shape* s, const eplab_hw* h, const eplab_traffic* t,
                           int n_workers, int redistributed, eplab_tune_config* best,
                           double* l_min, long long* evaluated);
/* B200 fwd+bwd model of this build's MegaKernels (calib NULL = built-in constants). */
EPLAB_API int eplab_predict_layer(const eplab_shape* s, const eplab_hw* h,
                                  const eplab_tune_config* c, const eplab_b200_calib* calib,
                                  eplab_layer_prediction* out);
/* Minimises eplab_predict_layer over (n_disp, n_relay incl. 0 = AllToAll mode). */
EPLAB_API int eplab_search_layer(const eplab_shape* s, const eplab_hw* h,
                                 const eplab_b200_calib* calib, eplab_tune_config* best,
                                 double* l_min, long long* evaluated);

#ifdef __cplusplus
}
#endif
#endif /* EPLAB_B200_H_ */
