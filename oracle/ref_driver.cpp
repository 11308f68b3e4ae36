// C wrappers over the UNMODIFIED reference eplab library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libeplab_ref.so).
// Test infrastructure only: used to pin the C oracle and the product host code
// against the reference itself, and as the "reference" CPU baseline.
#include <chrono>
#include <cstring>
#include <exception>

#include "eplab/perf_model.hpp"
#include "eplab/precision.hpp"
#include "eplab/routing.hpp"
#include "eplab/sim.hpp"
#include "eplab/token_map.hpp"
#include "eplab/traffic.hpp"
#include "eplab/tuner.hpp"
#include "eplab_oracle.h"

using namespace eplab;

namespace {
MoEShape to_shape(const orc_shape* s) {
  MoEShape m;
  m.name = "ref";
  m.h_dim = s->h_dim;
  m.h_inter = s->h_inter;
  m.n_exp = s->n_exp;
  m.topk = s->topk;
  m.n_tok = s->n_tok;
  m.s_tok = s->s_tok;
  m.b_m = s->b_m;
  m.b_n = s->b_n;
  m.mu_table.clear();
  for (int i = 0; i < s->mu_n; ++i) m.mu_table[s->mu_w[i]] = s->mu_v[i];
  return m;
}
HardwareSpec to_hw(const orc_hw* h) {
  HardwareSpec s;
  s.name = "ref";
  s.n_sm = h->n_sm;
  s.p_peak = h->p_peak;
  s.bw_hbm = h->bw_hbm;
  s.bw_nvl = h->bw_nvl;
  s.w_sat = h->w_sat;
  s.tau_sync = h->tau_sync;
  s.world_size = h->world_size;
  return s;
}
RoutingInstance to_routing(const int32_t* sel, const float* gw, int world, int n_exp,
                           long long n_tok, int topk) {
  RoutingInstance r;
  r.world = world;
  r.n_exp = n_exp;
  r.topk = topk;
  r.n_tok = n_tok;
  r.selected_experts.resize(world);
  r.gate_weights.resize(world);
  const size_t n = (size_t)n_tok * topk;
  for (int w = 0; w < world; ++w) {
    r.selected_experts[w].assign(sel + w * n, sel + (w + 1) * n);
    if (gw)
      r.gate_weights[w].assign(gw + w * n, gw + (w + 1) * n);
    else
      r.gate_weights[w].assign(n, 1.0f / topk);
  }
  return r;
}
TrafficReport to_traffic(const orc_traffic* t) {
  TrafficReport r;
  r.v_allgather = t->v_allgather;
  r.v_alltoall = t->v_alltoall;
  r.v_megakernel_nvl = t->v_megakernel_nvl;
  r.v_megakernel_hbm = t->v_megakernel_hbm;
  return r;
}
void from_traffic(const TrafficReport& r, orc_traffic* t) {
  t->v_allgather = r.v_allgather;
  t->v_alltoall = r.v_alltoall;
  t->v_megakernel_nvl = r.v_megakernel_nvl;
  t->v_megakernel_hbm = r.v_megakernel_hbm;
}
void from_breakdown(const LatencyBreakdown& b, orc_breakdown* o) {
  o->t_up = b.t_up;
  o->t_down = b.t_down;
  o->l_swiglu = b.l_swiglu;
  o->l_disp = b.l_disp;
  o->l_up = b.l_up;
  o->l_comb = b.l_comb;
  o->l_down = b.l_down;
  o->t_red = b.t_red;
  o->l_s1 = b.l_s1;
  o->l_s2 = b.l_s2;
  o->l_total = b.l_total;
  o->n_tiles_up = b.n_tiles_up;
  o->n_tiles_down = b.n_tiles_down;
  o->w_gap = b.w_gap;
  o->w_red = b.w_red;
  o->w_rem = b.w_rem;
}
}  // namespace

#define REF_TRY(...)                     \
  try {                                  \
    __VA_ARGS__;                         \
    return 0;                            \
  } catch (const ValidationError&) {     \
    return 2;                            \
  } catch (const DeadlockError&) {       \
    return 3;                            \
  } catch (const std::exception&) {      \
    return 1;                            \
  }

extern "C" {

int ref_sample_routing(int n_exp, int topk, long long n_tok, int world, uint64_t seed,
                       int32_t* sel, float* gw) {
  REF_TRY({
    MoEShape s;
    s.h_dim = s.h_inter = 8;
    s.n_exp = n_exp;
    s.topk = topk;
    s.n_tok = n_tok;
    RoutingInstance r = sample_routing(s, world, seed);
    const size_t n = (size_t)n_tok * topk;
    for (int w = 0; w < world; ++w) {
      std::memcpy(sel + w * n, r.selected_experts[w].data(), n * sizeof(int32_t));
      std::memcpy(gw + w * n, r.gate_weights[w].data(), n * sizeof(float));
    }
  })
}

int ref_token_map(const int32_t* sel, int world, int n_exp, long long n_tok, int topk,
                  int32_t* target_rank, int32_t* local_expert, int64_t* offset,
                  int64_t* recv_totals, int64_t* seg_base) {
  REF_TRY({
    auto maps = build_global_token_map(to_routing(sel, nullptr, world, n_exp, n_tok, topk));
    const size_t n = (size_t)n_tok * topk;
    for (int w = 0; w < world; ++w)
      for (size_t i = 0; i < n; ++i) {
        target_rank[w * n + i] = maps[w].entries[i].target_rank;
        local_expert[w * n + i] = maps[w].entries[i].local_expert;
        offset[w * n + i] = maps[w].entries[i].offset;
      }
    if (recv_totals)
      std::memcpy(recv_totals, maps[0].recv_totals.data(), maps[0].recv_totals.size() * 8);
    if (seg_base)
      std::memcpy(seg_base, maps[0].recv_segment_base.data(),
                  maps[0].recv_segment_base.size() * 8);
  })
}

int ref_send_schedule(const int32_t* sel, int world, int n_exp, long long n_tok, int topk,
                      int rank, int64_t* item_token, int32_t* item_slot, int32_t* item_dst_rank,
                      int32_t* item_dst_expert, int64_t* item_dst_offset) {
  REF_TRY({
    auto maps = build_global_token_map(to_routing(sel, nullptr, world, n_exp, n_tok, topk));
    SendSchedule s = build_send_schedule(maps[rank]);
    for (size_t i = 0; i < s.items.size(); ++i) {
      item_token[i] = s.items[i].token;
      item_slot[i] = s.items[i].slot;
      item_dst_rank[i] = s.items[i].dst_rank;
      item_dst_expert[i] = s.items[i].dst_expert;
      item_dst_offset[i] = s.items[i].dst_offset;
    }
  })
}

int ref_distinct_rank_distribution(int world, int topk, uint64_t* num_lo, double* probs,
                                   double* expectation, double* saving) {
  REF_TRY({
    auto d = distinct_rank_distribution(world, topk);
    for (size_t i = 0; i < d.numerators.size(); ++i) {
      num_lo[i] = d.numerators[i].convert_to<uint64_t>();
      probs[i] = d.probs[i];
    }
    *expectation = d.expectation;
    *saving = d.expected_saving_fraction;
  })
}

int ref_volume_expected(const orc_shape* s, const orc_hw* h, int remote_only, orc_traffic* out) {
  REF_TRY({
    from_traffic(volume_expected(to_shape(s), to_hw(h),
                                 remote_only ? SelfRankAccounting::RemoteOnly
                                             : SelfRankAccounting::IncludeSelf),
                 out);
  })
}

int ref_volume_exact(const int32_t* sel, const orc_shape* s, const orc_hw* h, int world,
                     int remote_only, orc_traffic* out) {
  REF_TRY({
    auto r = to_routing(sel, nullptr, world, s->n_exp, s->n_tok, s->topk);
    from_traffic(volume_exact(r, to_shape(s), to_hw(h),
                              remote_only ? SelfRankAccounting::RemoteOnly
                                          : SelfRankAccounting::IncludeSelf),
                 out);
  })
}

int ref_predict_latency(const orc_shape* s, const orc_hw* h, const orc_cfg* c,
                        const orc_traffic* t, int redistributed, orc_breakdown* out) {
  REF_TRY({
    TuneConfig cfg{c->n_disp, c->n_relay, c->n_comb, c->n_red, c->w};
    from_breakdown(predict_latency(to_shape(s), to_hw(h), cfg, to_traffic(t),
                                   redistributed ? ResidualScaling::Redistributed
                                                 : ResidualScaling::AsPrinted),
                   out);
  })
}

int ref_search(const orc_shape* s, const orc_hw* h, const orc_traffic* t, int n_workers,
               orc_cfg* best, double* l_min, long long* evaluated, double* wall_s) {
  REF_TRY({
    TuneResult r = search(to_hw(h), to_shape(s), to_traffic(t), n_workers);
    *best = orc_cfg{r.best.n_disp, r.best.n_relay, r.best.n_comb, r.best.n_red, r.best.w};
    *l_min = r.l_min;
    *evaluated = r.evaluated;
    if (wall_s) *wall_s = r.wall_seconds;
  })
}

int ref_space_sizes(int n_sm, long long* raw, long long* enumerated, long long* feasible) {
  REF_TRY({
    HardwareSpec h;
    h.name = "x";
    h.n_sm = n_sm;
    h.p_peak = 1;
    h.bw_hbm = 1;
    h.bw_nvl = 1;
    MoEShape s;
    SearchSpace sp = enumerate_space(h, s);
    *raw = sp.raw_grid_size;
    *enumerated = sp.enumerated_count;
    long long f = 0;
    for_each_candidate(sp, true, [&](const TuneConfig&) { ++f; });
    *feasible = f;
  })
}

float ref_round_to_bf16(float x) { return round_to_bf16(x); }

float ref_fold(const float* w, const float* v, int n, int bf16) {
  ReductionPlan plan;
  plan.tokens.emplace_back();
  for (int i = 0; i < n; ++i) plan.tokens[0].push_back(ReductionTerm{i, w[i], v[i]});
  return accumulate(plan, bf16 ? FpFormat::Bfloat16 : FpFormat::Binary32)[0];
}

// Task layout of the dispatch MegaKernel (sim.cpp:226-250): comm slices then relay ranges.
int ref_build_task_list(const int32_t* sel, int world, const orc_shape* s, const orc_cfg* c,
                        int rank, int64_t* comm_slices, int64_t* relay_ranges, int64_t* n_comp) {
  REF_TRY({
    auto r = to_routing(sel, nullptr, world, s->n_exp, s->n_tok, s->topk);
    TaskQueueInfo tq =
        build_task_list(to_shape(s), TuneConfig{c->n_disp, c->n_relay, c->n_comb, c->n_red, c->w},
                        r, rank);
    for (size_t i = 0; i < tq.comm_slices.size(); ++i) {
      comm_slices[2 * i] = tq.comm_slices[i].first;
      comm_slices[2 * i + 1] = tq.comm_slices[i].second;
    }
    for (size_t i = 0; i < tq.relay_ranges.size(); ++i) {
      relay_ranges[2 * i] = tq.relay_ranges[i].first;
      relay_ranges[2 * i + 1] = tq.relay_ranges[i].second;
    }
    *n_comp = tq.n_comp;
  })
}

// Wall time of the reference's CPU addressing path (a2, a5, a6) on one routing instance.
int ref_time_addressing(int n_exp, int topk, long long n_tok, int world, uint64_t seed,
                        double* t_routing, double* t_map, double* t_sched) {
  REF_TRY({
    MoEShape s;
    s.h_dim = s.h_inter = 8;
    s.n_exp = n_exp;
    s.topk = topk;
    s.n_tok = n_tok;
    auto t0 = std::chrono::steady_clock::now();
    RoutingInstance r = sample_routing(s, world, seed);
    auto t1 = std::chrono::steady_clock::now();
    auto maps = build_global_token_map(r);
    auto t2 = std::chrono::steady_clock::now();
    size_t total = 0;
    for (const auto& m : maps) total += build_send_schedule(m).items.size();
    auto t3 = std::chrono::steady_clock::now();
    (void)total;
    *t_routing = std::chrono::duration<double>(t1 - t0).count();
    *t_map = std::chrono::duration<double>(t2 - t1).count();
    *t_sched = std::chrono::duration<double>(t3 - t2).count();
  })
}

}  // extern "C"
