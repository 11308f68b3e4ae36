// Device data path for reference-style C++ callers: the reference's simulated operators -- the
// token map (build_global_token_map, token_map.hpp:68), run_dispatch_gemm_sim and
// run_gemm_combine_sim (sim.hpp:87-88) -- as device-executing calls on a per-rank context, in
// namespace eplab, over the C-ABI of libeplab_b200.so (include/eplab_b200.h). Header-only: C++
// host code calls CUDA only through that thin C layer. Errors come back as the reference's
// exception types (ValidationError for rc 2, DeadlockError for rc 3, error.hpp:12-22).
//
//   g++ -std=c++20 -I<repo>/include app.cpp -L<repo>/paper_2604_19241_b200 -leplab_b200 -lcudart
#pragma once
#include <stdexcept>
#include <string>

#include "eplab/eplab.hpp"
#include "eplab_b200.h"

namespace eplab {

inline void check_rc(int rc) {
  if (rc == EPLAB_OK) return;
  char buf[1024] = {0};
  eplab_last_error(buf, sizeof buf);
  if (rc == EPLAB_ERR_VALIDATION) throw ValidationError(buf);
  if (rc == EPLAB_ERR_DEADLOCK) throw DeadlockError(buf);
  throw std::runtime_error(std::string("eplab internal error: ") + buf);
}

// One rank's MegaKernel context (symmetric buffers, scoreboard, plan arrays). `stream` arguments
// are cudaStream_t values passed as void* so this header needs no CUDA include.
class Context {
 public:
  struct Options {
    int rank = 0, world = 1, device = 0;
    int max_tokens = 0;             // tokens per rank per call
    int hidden = 0, ffn = 0;        // H, F
    int n_experts = 0, topk = 0;    // global expert count, top-k
    long long max_recv_rows = 0;    // 0: worst case
    double timeout_s = 10.0;        // scoreboard watchdog
  };
  explicit Context(const Options& o) {
    eplab_init_args a{o.rank, o.world, o.device, o.max_tokens, o.hidden, o.ffn, o.n_experts, o.topk,
                      o.max_recv_rows, o.timeout_s};
    check_rc(eplab_init(&a, &c_));
  }
  ~Context() { eplab_destroy(c_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  eplab_ctx* get() const { return c_; }

  // TuneConfig (types.hpp:45-53); until set, every plan auto-tunes per 4096-token bucket
  void set_tune_config(const TuneConfig& t) {
    eplab_tune_config c{t.n_disp, t.n_relay, t.n_comb, t.n_red, t.w};
    check_rc(eplab_set_tune_config(c_, &c));
  }
  TuneConfig tune_config() const {
    eplab_tune_config c{};
    check_rc(eplab_get_tune_config(c_, &c));
    return TuneConfig{c.n_disp, c.n_relay, c.n_comb, c.n_red, c.w};
  }
  // synchronises `stream`; throws DeadlockError if a scoreboard watchdog fired
  void check(void* stream = nullptr) { check_rc(eplab_check(c_, stream)); }

 private:
  eplab_ctx* c_ = nullptr;
};

// Device token map + priority send schedule of this iteration (Alg. 1 with the count AllGather
// done on device): d_topk_ids int32 [n_tok][topk], d_gate_w fp32 [n_tok][topk].
inline void build_global_token_map(Context& ctx, const int32_t* d_topk_ids, const float* d_gate_w,
                                   int n_tok, void* stream = nullptr) {
  check_rc(eplab_plan(ctx.get(), d_topk_ids, d_gate_w, n_tok, stream));
}
// Dispatch+GroupGEMM MegaKernel (run_dispatch_gemm_sim): x rows to the expert ranks, up
// GroupGEMM + SwiGLU as rowgroups land. d_x bf16 [n_tok][H], d_w_up bf16 [E_loc][2F][H].
inline void dispatch_group_gemm(Context& ctx, const void* d_x, const void* d_w_up, void* stream = nullptr) {
  check_rc(eplab_dispatch_group_gemm(ctx.get(), d_x, d_w_up, stream));
}
// GroupGEMM+Combine MegaKernel (run_gemm_combine_sim + accumulate): down GroupGEMM, replica
// pushes to the source, top-k barrier, k-ordered fold into d_y bf16 [n_tok][H].
inline void group_gemm_combine(Context& ctx, const void* d_w_down, void* d_y, void* stream = nullptr) {
  check_rc(eplab_group_gemm_combine(ctx.get(), d_w_down, d_y, stream));
}
// Backward twins: dY dispatch + gate gradient + down dgrad/wgrad; up dgrad pushed back and
// k-reduced into dX + up wgrad.
inline void dispatch_group_gemm_bwd(Context& ctx, const void* d_dy, const void* d_w_down, void* d_dw_down,
                                    float* d_dgate, void* stream = nullptr) {
  check_rc(eplab_dispatch_group_gemm_bwd(ctx.get(), d_dy, d_w_down, d_dw_down, d_dgate, stream));
}
inline void group_gemm_combine_bwd(Context& ctx, const void* d_w_up, void* d_dx, void* d_dw_up,
                                   void* stream = nullptr) {
  check_rc(eplab_group_gemm_combine_bwd(ctx.get(), d_w_up, d_dx, d_dw_up, stream));
}

}  // namespace eplab
