// C-ABI over the host eplab:: API (routing, token map, traffic, perf model, tuner).
#include <cstring>

#include "eplab/eplab.hpp"
#include "eplab_b200.h"
#include "host/errors.hpp"

namespace {
using namespace eplab;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return EPLAB_OK;
  } catch (const ValidationError& e) {
    eplab_host::set_last_error(e.what());
    return EPLAB_ERR_VALIDATION;
  } catch (const DeadlockError& e) {
    eplab_host::set_last_error(e.what());
    return EPLAB_ERR_DEADLOCK;
  } catch (const std::exception& e) {
    eplab_host::set_last_error(e.what());
    return EPLAB_ERR_INTERNAL;
  }
}

MoEShape to_shape(const eplab_shape* s) {
  MoEShape m;
  m.name = "c-abi";
  m.h_dim = s->h_dim;
  m.h_inter = s->h_inter;
  m.n_exp = s->n_exp;
  m.topk = s->topk;
  m.n_tok = s->n_tok;
  m.s_tok = s->s_tok;
  m.b_m = s->b_m;
  m.b_n = s->b_n;
  if (s->mu_n > 0) {
    m.mu_table.clear();
    for (int i = 0; i < s->mu_n && i < 8; ++i) m.mu_table[s->mu_w[i]] = s->mu_v[i];
  }
  return m;
}
HardwareSpec to_hw(const eplab_hw* h) {
  HardwareSpec s;
  s.name = "c-abi";
  s.n_sm = h->n_sm;
  s.p_peak = h->p_peak;
  s.bw_hbm = h->bw_hbm;
  s.bw_nvl = h->bw_nvl;
  s.w_sat = h->w_sat;
  s.tau_sync = h->tau_sync;
  s.world_size = h->world_size;
  return s;
}
TrafficReport to_traffic(const eplab_traffic* t) {
  return TrafficReport{t->v_allgather, t->v_alltoall, t->v_megakernel_nvl, t->v_megakernel_hbm};
}
B200Calib to_calib(const eplab_b200_calib* c) {
  B200Calib k;
  if (c)
    k = B200Calib{c->mu,        c->tile_overhead, c->comm_bw_per_sm, c->relay_bw_per_sm,
                  c->reduce_bw, c->launch,        c->epi_bw_per_sm,  c->spare_sm_equiv, c->hbm_overlap,
                  c->startup};
  return k;
}
RoutingInstance to_routing(const int32_t* sel, int world, int n_exp, long long n_tok, int topk) {
  RoutingInstance r;
  r.world = world;
  r.n_exp = n_exp;
  r.topk = topk;
  r.n_tok = n_tok;
  const size_t n = (size_t)n_tok * topk;
  for (int w = 0; w < world; ++w) {
    r.selected_experts.emplace_back(sel + w * n, sel + (w + 1) * n);
    r.gate_weights.emplace_back(n, 1.0f / topk);
  }
  return r;
}
}  // namespace

extern "C" {

int eplab_sample_routing(int n_exp, int topk, long long n_tok, int world, uint64_t seed,
                         int32_t* sel, float* gw) {
  return guarded([&] {
    MoEShape s;
    s.h_dim = s.h_inter = 8;
    s.n_exp = n_exp;
    s.topk = topk;
    s.n_tok = n_tok;
    RoutingInstance r = sample_routing(s, world, seed);
    const size_t n = (size_t)n_tok * topk;
    for (int w = 0; w < world; ++w) {
      std::memcpy(sel + w * n, r.selected_experts[w].data(), n * 4);
      std::memcpy(gw + w * n, r.gate_weights[w].data(), n * 4);
    }
  });
}

int eplab_host_token_map(const int32_t* sel, int world, int n_exp, long long n_tok, int topk,
                         int32_t* target_rank, int32_t* local_expert, int64_t* offset,
                         int64_t* recv_totals, int64_t* seg_base) {
  return guarded([&] {
    if (world < 1 || n_exp % world) throw ValidationError("n_exp not divisible by world");
    auto maps = build_global_token_map(to_routing(sel, world, n_exp, n_tok, topk));
    const size_t n = (size_t)n_tok * topk;
    for (int w = 0; w < world; ++w)
      for (size_t i = 0; i < n; ++i) {
        target_rank[w * n + i] = maps[w].entries[i].target_rank;
        local_expert[w * n + i] = maps[w].entries[i].local_expert;
        offset[w * n + i] = maps[w].entries[i].offset;
      }
    for (size_t i = 0; i < maps[0].recv_totals.size(); ++i) {
      if (recv_totals) recv_totals[i] = maps[0].recv_totals[i];
      if (seg_base) seg_base[i] = maps[0].recv_segment_base[i];
    }
  });
}

int eplab_host_rank_token_map(const int32_t* sel, const int64_t* counts_all, int rank, int world,
                              int n_exp, long long n_tok, int topk, int32_t* target_rank,
                              int32_t* local_expert, int64_t* offset) {
  return guarded([&] {
    if (world < 1 || n_exp % world) throw ValidationError("n_exp not divisible by world");
    if (rank < 0 || rank >= world) throw ValidationError("rank out of range");
    // this rank's routing alone (Alg. 1 l.1-2) + every rank's counts (l.3) -> its map (l.4-16)
    RoutingInstance one;
    one.world = 1;
    one.n_exp = n_exp;
    one.topk = topk;
    one.n_tok = n_tok;
    one.selected_experts.assign(1, std::vector<int>(sel, sel + (size_t)n_tok * topk));
    one.gate_weights.assign(1, std::vector<float>((size_t)n_tok * topk, 1.0f));
    validate_routing(one);
    const LocalSortResult loc = local_stable_sort(one.selected_experts[0], n_tok, topk, n_exp);
    std::vector<std::vector<long long>> counts(world, std::vector<long long>(n_exp));
    for (int r = 0; r < world; ++r)
      for (int e = 0; e < n_exp; ++e) counts[r][e] = counts_all[(size_t)r * n_exp + e];
    if (counts[rank] != loc.expert_counts)
      throw ValidationError("all_expert_counts row of this rank differs from its own routing");
    const GlobalOffsets oall = compute_global_offsets(counts, world, n_exp);
    const int epr = n_exp / world;
    for (size_t i = 0; i < loc.m_loc.size(); ++i) {
      const int e = one.selected_experts[0][i];
      target_rank[i] = e / epr;
      local_expert[i] = e % epr;
      offset[i] = loc.m_loc[i] - loc.expert_offsets[e] + oall.at(e / epr, e % epr, rank);
    }
  });
}

int eplab_host_send_schedule(const int32_t* sel, int world, int n_exp, long long n_tok, int topk,
                             int rank, int64_t* item_token, int32_t* item_slot,
                             int32_t* item_dst_rank, int32_t* item_dst_expert,
                             int64_t* item_dst_offset) {
  return guarded([&] {
    if (world < 1 || n_exp % world) throw ValidationError("n_exp not divisible by world");
    if (rank < 0 || rank >= world) throw ValidationError("rank out of range");
    auto maps = build_global_token_map(to_routing(sel, world, n_exp, n_tok, topk));
    SendSchedule s = build_send_schedule(maps[rank]);
    for (size_t i = 0; i < s.items.size(); ++i) {
      item_token[i] = s.items[i].token;
      item_slot[i] = s.items[i].slot;
      item_dst_rank[i] = s.items[i].dst_rank;
      item_dst_expert[i] = s.items[i].dst_expert;
      item_dst_offset[i] = s.items[i].dst_offset;
    }
  });
}

int eplab_host_build_task_list(const int32_t* sel, int world, const eplab_shape* s, const eplab_tune_config* c,
                               int rank, int64_t* comm_slices, int64_t* relay_ranges, int64_t* n_comp) {
  return guarded([&] {
    if (world < 1 || s->n_exp % world) throw ValidationError("n_exp not divisible by world");
    if (rank < 0 || rank >= world) throw ValidationError("rank out of range");
    TaskQueueInfo tq = build_task_list(to_shape(s), TuneConfig{c->n_disp, c->n_relay, c->n_comb, c->n_red, c->w},
                                       to_routing(sel, world, s->n_exp, s->n_tok, s->topk), rank);
    for (size_t i = 0; i < tq.comm_slices.size(); ++i) {
      comm_slices[2 * i] = tq.comm_slices[i].first;
      comm_slices[2 * i + 1] = tq.comm_slices[i].second;
    }
    for (size_t i = 0; i < tq.relay_ranges.size(); ++i) {
      relay_ranges[2 * i] = tq.relay_ranges[i].first;
      relay_ranges[2 * i + 1] = tq.relay_ranges[i].second;
    }
    *n_comp = tq.n_comp;
  });
}

int eplab_volume_expected(const eplab_shape* s, const eplab_hw* h, int remote_only,
                          eplab_traffic* out) {
  return guarded([&] {
    TrafficReport t = volume_expected(to_shape(s), to_hw(h),
                                      remote_only ? SelfRankAccounting::RemoteOnly
                                                  : SelfRankAccounting::IncludeSelf);
    *out = eplab_traffic{t.v_allgather, t.v_alltoall, t.v_megakernel_nvl, t.v_megakernel_hbm};
  });
}

int eplab_predict_latency(const eplab_shape* s, const eplab_hw* h, const eplab_tune_config* c,
                          const eplab_traffic* t, int redistributed, eplab_breakdown* out) {
  return guarded([&] {
    LatencyBreakdown b = predict_latency(
        to_shape(s), to_hw(h), TuneConfig{c->n_disp, c->n_relay, c->n_comb, c->n_red, c->w},
        to_traffic(t), redistributed ? ResidualScaling::Redistributed : ResidualScaling::AsPrinted);
    *out = eplab_breakdown{b.t_up,   b.t_down, b.l_swiglu,    b.l_disp,       b.l_up,
                           b.l_comb, b.l_down, b.t_red,       b.l_s1,         b.l_s2,
                           b.l_total, b.n_tiles_up, b.n_tiles_down, b.w_gap, b.w_red, b.w_rem};
  });
}

int eplab_search(const eplab_shape* s, const eplab_hw* h, const eplab_traffic* t, int n_workers,
                 int redistributed, eplab_tune_config* best, double* l_min, long long* evaluated) {
  return guarded([&] {
    TuneResult r = search(to_hw(h), to_shape(s), to_traffic(t), n_workers,
                          redistributed ? ResidualScaling::Redistributed : ResidualScaling::AsPrinted);
    *best = eplab_tune_config{r.best.n_disp, r.best.n_relay, r.best.n_comb, r.best.n_red, r.best.w};
    *l_min = r.l_min;
    *evaluated = r.evaluated;
  });
}

int eplab_predict_layer(const eplab_shape* s, const eplab_hw* h, const eplab_tune_config* c,
                        const eplab_b200_calib* calib, eplab_layer_prediction* out) {
  return guarded([&] {
    LayerPrediction p = predict_layer(to_shape(s), to_hw(h),
                                      TuneConfig{c->n_disp, c->n_relay, c->n_comb, c->n_red, c->w},
                                      to_calib(calib));
    *out = eplab_layer_prediction{p.fwd_dispatch, p.fwd_combine, p.bwd_dispatch, p.bwd_combine,
                                  p.total,        p.t_gemm_bound, p.t_nvl_bound};
  });
}

int eplab_search_layer(const eplab_shape* s, const eplab_hw* h, const eplab_b200_calib* calib,
                       eplab_tune_config* best, double* l_min, long long* evaluated) {
  return guarded([&] {
    TuneResult r = search_layer(to_hw(h), to_shape(s), 0, to_calib(calib));
    *best = eplab_tune_config{r.best.n_disp, r.best.n_relay, r.best.n_comb, r.best.n_red, r.best.w};
    *l_min = r.l_min;
    *evaluated = r.evaluated;
  });
}

}  // extern "C"
