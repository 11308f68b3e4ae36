// Host-side eplab API (include/eplab/eplab.hpp): validation, synthetic routing, host token map,
// traffic analytics, the reference-compatible performance model + tuner, and the B200 model of
// the MegaKernels implemented in this repository (forward and backward).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <fstream>
#include <numeric>
#include <set>
#include <sstream>
#include <thread>
#include <tuple>

#include "eplab/eplab.hpp"

namespace eplab {

namespace {
[[noreturn]] void bad(const std::string& field, const std::string& why) {
  throw ValidationError(field + " " + why);
}
using u128 = unsigned __int128;
}  // namespace

// ------------------------------------------------------------------ validation (types.cpp:20-94)
HardwareSpec validate_hardware(HardwareSpec s) {
  if (s.n_sm < 2) bad("n_sm", "must be >= 2");
  if (!(s.p_peak > 0)) bad("p_peak", "must be > 0");
  if (!(s.bw_hbm > 0)) bad("bw_hbm", "must be > 0");
  if (!(s.bw_nvl > 0)) bad("bw_nvl", "must be > 0");
  if (!(s.w_sat > 0)) bad("w_sat", "must be > 0");
  if (!(s.tau_sync >= 0)) bad("tau_sync", "must be >= 0");
  if (s.world_size < 1) bad("world_size", "must be >= 1");
  return s;
}

std::pair<MoEShape, HardwareSpec> validate_shape(MoEShape m, HardwareSpec s) {
  s = validate_hardware(std::move(s));
  if (m.h_dim <= 0) bad("h_dim", "must be > 0");
  if (m.h_inter <= 0) bad("h_inter", "must be > 0");
  if (m.n_exp <= 0) bad("n_exp", "must be > 0");
  if (m.n_exp % s.world_size)
    throw ValidationError("n_exp " + std::to_string(m.n_exp) + " not divisible by world_size " +
                          std::to_string(s.world_size));
  if (m.topk < 1 || m.topk > m.n_exp) bad("topk", "must be in [1, n_exp]");
  if (m.n_tok < 0) bad("n_tok", "must be >= 0");
  if (m.s_tok < 0) bad("s_tok", "must be >= 0");
  if (m.s_tok == 0) m.s_tok = 2LL * m.h_dim;
  if (m.b_m <= 0) bad("b_m", "must be > 0");
  if (m.b_n <= 0) bad("b_n", "must be > 0");
  if (m.mu_table.empty()) bad("mu_table", "must not be empty");
  for (const auto& [w, mu] : m.mu_table) {
    if (w <= 0) bad("mu_table", "warp keys must be > 0");
    if (!(mu > 0.0 && mu <= 1.0)) bad("mu_table", "values must be in (0,1]");
  }
  return {std::move(m), std::move(s)};
}

void validate_tune_config(const TuneConfig& c, const HardwareSpec& s) {
  if (c.w != 8 && c.w != 16 && c.w != 32) bad("w", "must be one of {8,16,32}");
  if (c.n_disp < 0) bad("n_disp", "must be >= 0");
  if (c.n_relay < 0) bad("n_relay", "must be >= 0");
  if (c.n_disp + c.n_relay >= s.n_sm)
    throw ValidationError("n_disp + n_relay must be < n_sm (deadlock constraint): " +
                          std::to_string(c.n_disp) + " + " + std::to_string(c.n_relay) +
                          " >= " + std::to_string(s.n_sm));
  if (c.n_comb >= s.n_sm || c.n_comb < 1) bad("n_comb", "must be in [1, n_sm)");
  if (c.n_red < 1 || c.n_red > s.n_sm) bad("n_red", "must be in [1, n_sm]");
}

long long derive_expanded_tokens(const MoEShape& shape, int) {
  return shape.n_tok * shape.topk;  // balanced routing: rows received per rank == rows sent
}

void validate_routing(const RoutingInstance& r) {
  if (r.world < 1) bad("world", "must be >= 1");
  if ((int)r.selected_experts.size() != r.world || (int)r.gate_weights.size() != r.world)
    bad("routing", "rank table count != world");
  for (int w = 0; w < r.world; ++w) {
    const auto& sel = r.selected_experts[w];
    const auto& gw = r.gate_weights[w];
    if ((long long)sel.size() != r.n_tok * r.topk) bad("selected_experts", "bad shape");
    if (gw.size() != sel.size()) bad("gate_weights", "bad shape");
    for (long long t = 0; t < r.n_tok; ++t)
      for (int j = 0; j < r.topk; ++j) {
        const int e = sel[t * r.topk + j];
        if (e < 0 || e >= r.n_exp) bad("selected_experts", "expert id out of range");
        for (int i = 0; i < j; ++i)
          if (sel[t * r.topk + i] == e) bad("selected_experts", "duplicate expert within token");
        if (!std::isfinite(gw[t * r.topk + j])) bad("gate_weights", "non-finite weight");
      }
  }
}

// ------------------------------------------------------------------ routing (routing.cpp:15-73)
namespace {
struct SplitMix {
  std::uint64_t s;
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  std::uint64_t below(std::uint64_t n) { return (std::uint64_t)(((u128)next() * n) >> 64); }
  double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
};
}  // namespace

RoutingInstance sample_routing(const MoEShape& shape, int world, std::uint64_t seed) {
  if (shape.topk > shape.n_exp) throw ValidationError("topk exceeds n_exp; cannot draw distinct experts");
  RoutingInstance out;
  out.world = world;
  out.n_exp = shape.n_exp;
  out.topk = shape.topk;
  out.n_tok = shape.n_tok;
  out.seed = seed;
  out.selected_experts.assign(world, {});
  out.gate_weights.assign(world, {});
  const size_t n = (size_t)(shape.n_tok * shape.topk);
  std::vector<int> deck(shape.n_exp);
  for (int r = 0; r < world; ++r) {
    SplitMix g{seed ^ (0xA5A5A5A5A5A5A5A5ULL + (std::uint64_t)r * 0x9E3779B97F4A7C15ULL)};
    auto& sel = out.selected_experts[r];
    auto& gw = out.gate_weights[r];
    sel.resize(n);
    gw.resize(n);
    std::iota(deck.begin(), deck.end(), 0);  // the deck persists across the rank's tokens
    for (long long t = 0; t < shape.n_tok; ++t) {
      int* row = &sel[t * shape.topk];
      float* wrow = &gw[t * shape.topk];
      for (int j = 0; j < shape.topk; ++j) {
        const std::uint64_t pick = j + g.below((std::uint64_t)(shape.n_exp - j));
        std::swap(deck[j], deck[pick]);
        row[j] = deck[j];
      }
      double total = 0;
      for (int j = 0; j < shape.topk; ++j) {
        const double u = g.unit();
        wrow[j] = (float)u;
        total += u;
      }
      if (total > 0)
        for (int j = 0; j < shape.topk; ++j) wrow[j] = (float)((double)wrow[j] / total);
    }
  }
  return out;
}

// ------------------------------------------------------------------ host token map
LocalSortResult local_stable_sort(const std::vector<int>& sel, long long n_tok, int topk, int n_exp) {
  LocalSortResult r;
  r.expert_counts.assign(n_exp, 0);
  for (int e : sel) ++r.expert_counts[e];
  r.expert_offsets.resize(n_exp);
  std::exclusive_scan(r.expert_counts.begin(), r.expert_counts.end(), r.expert_offsets.begin(), 0LL);
  std::vector<long long> next = r.expert_offsets;
  r.m_loc.resize((size_t)n_tok * topk);
  for (size_t i = 0; i < r.m_loc.size(); ++i) r.m_loc[i] = next[sel[i]]++;
  return r;
}

GlobalOffsets compute_global_offsets(const std::vector<std::vector<long long>>& counts, int world,
                                     int n_exp) {
  if ((int)counts.size() != world) throw ValidationError("all_expert_counts rank dimension != world");
  for (const auto& row : counts)
    if ((int)row.size() != n_exp) throw ValidationError("all_expert_counts expert dimension != n_exp");
  if (n_exp % world) throw ValidationError("n_exp not divisible by world");
  GlobalOffsets g;
  g.world = world;
  g.experts_per_rank = n_exp / world;
  g.data.resize((size_t)n_exp * world);
  for (int e = 0; e < n_exp; ++e) {  // e = dst * epr + e_loc
    long long run = 0;
    for (int src = 0; src < world; ++src) {
      g.data[(size_t)e * world + src] = run;
      run += counts[src][e];
    }
  }
  return g;
}

std::vector<GlobalTokenMap> build_global_token_map(const RoutingInstance& routing) {
  validate_routing(routing);
  const int W = routing.world, epr = routing.n_exp / W;
  std::vector<LocalSortResult> loc(W);
  std::vector<std::vector<long long>> counts(W);
  for (int r = 0; r < W; ++r) {
    loc[r] = local_stable_sort(routing.selected_experts[r], routing.n_tok, routing.topk, routing.n_exp);
    counts[r] = loc[r].expert_counts;
  }
  const GlobalOffsets oall = compute_global_offsets(counts, W, routing.n_exp);
  std::vector<long long> totals(routing.n_exp, 0), bases(routing.n_exp, 0);
  for (int src = 0; src < W; ++src)
    for (int e = 0; e < routing.n_exp; ++e) totals[e] += counts[src][e];
  for (int dst = 0; dst < W; ++dst)
    std::exclusive_scan(totals.begin() + dst * epr, totals.begin() + (dst + 1) * epr,
                        bases.begin() + dst * epr, 0LL);
  std::vector<GlobalTokenMap> maps(W);
  for (int r = 0; r < W; ++r) {
    GlobalTokenMap& m = maps[r];
    m.rank = r;
    m.n_tok = routing.n_tok;
    m.topk = routing.topk;
    m.world = W;
    m.experts_per_rank = epr;
    m.recv_totals = totals;
    m.recv_segment_base = bases;
    const auto& sel = routing.selected_experts[r];
    m.entries.resize(sel.size());
    for (size_t i = 0; i < sel.size(); ++i) {
      const int e = sel[i];
      m.entries[i] = MapEntry{e / epr, e % epr,
                              loc[r].m_loc[i] - loc[r].expert_offsets[e] + oall.at(e / epr, e % epr, r)};
    }
  }
  return maps;
}

std::string export_map_table(const std::vector<GlobalTokenMap>& maps) {
  std::string out = "rank\ttoken\tslot\tdst_rank\tdst_expert\tdst_offset\n";
  for (const GlobalTokenMap& m : maps)
    for (size_t i = 0; i < m.entries.size(); ++i) {
      const MapEntry& e = m.entries[i];
      out += std::to_string(m.rank) + "\t" + std::to_string(i / m.topk) + "\t" + std::to_string(i % m.topk) +
             "\t" + std::to_string(e.target_rank) + "\t" + std::to_string(e.local_expert) + "\t" +
             std::to_string(e.offset) + "\n";
    }
  return out;
}

SendSchedule build_send_schedule(const GlobalTokenMap& map) {
  // bucket base of (e_loc, dst) = exclusive scan in (e_loc, dst) order; position inside the
  // bucket = (t, j) order, which is ascending destination offset (stable local sort)
  const int W = map.world, epr = map.experts_per_rank, nb = W * epr;
  std::vector<long long> fill(nb + 1, 0);
  for (const auto& e : map.entries) ++fill[(size_t)e.local_expert * W + e.target_rank + 1];
  std::partial_sum(fill.begin(), fill.end(), fill.begin());
  SendSchedule s;
  s.rank = map.rank;
  s.items.resize(map.entries.size());
  for (size_t i = 0; i < map.entries.size(); ++i) {
    const MapEntry& e = map.entries[i];
    s.items[fill[(size_t)e.local_expert * W + e.target_rank]++] =
        SendItem{(long long)(i / map.topk), (int)(i % map.topk), e.target_rank, e.local_expert, e.offset};
  }
  return s;
}

// ------------------------------------------------------------------ traffic (traffic.cpp)
BigInt stirling2(int n, int k) {
  if (n < 0 || k < 0 || k > n || n > 64) throw ValidationError("stirling2 supports 0 <= k <= n <= 64");
  // Pascal-like triangle of S(i, j) = j S(i-1, j) + S(i-1, j-1), kept as the previous row only
  std::vector<BigInt> prev(1, BigInt(1));  // S(0, 0) = 1
  for (int i = 1; i <= n; ++i) {
    std::vector<BigInt> cur(std::min(i, k) + 1, BigInt(0));
    for (int j = 1; j < (int)cur.size(); ++j) {
      const BigInt keep = j < (int)prev.size() ? BigInt(j) * prev[j] : BigInt(0);
      cur[j] = keep + prev[j - 1];
    }
    prev.swap(cur);
  }
  return k < (int)prev.size() ? prev[k] : BigInt(0);
}

DistinctRankDistribution distinct_rank_distribution(int world, int topk) {
  if (world < 1 || topk < 1) throw ValidationError("world and topk must be >= 1");
  if (topk > 64) throw ValidationError("topk must be <= 64");
  DistinctRankDistribution d;
  d.world = world;
  d.topk = topk;
  for (int i = 0; i < topk; ++i) d.denominator *= BigInt(world);
  const int xmax = std::min(world, topk);
  // P(X = x) = W (W-1) ... (W-x+1) S(topk, x) / W^topk, exact
  BigInt check = 0, e_num = 0;
  for (int x = 1; x <= xmax; ++x) {
    BigInt falling = 1;  // C(W, x) * x!
    for (int i = 0; i < x; ++i) falling *= BigInt(world - i);
    const BigInt num = falling * stirling2(topk, x);
    d.numerators.push_back(num);
    d.probs.push_back(num.to_double() / d.denominator.to_double());
    check += num;
    e_num += BigInt(x) * num;
  }
  if (check != d.denominator)
    throw ValidationError("distinct_rank_distribution: probabilities do not sum to 1");
  d.expectation = e_num.to_double() / d.denominator.to_double();
  const double closed = world * (1.0 - std::pow(1.0 - 1.0 / world, topk));
  if (std::abs(d.expectation - closed) > 1e-12 * std::max(1.0, closed))
    throw ValidationError("distinct_rank_distribution: expectation mismatch vs closed form");
  d.expected_saving_fraction = (topk - d.expectation) / topk;
  return d;
}

namespace {
TrafficReport make_volumes(const MoEShape& shape, int world, double mean_distinct) {
  TrafficReport r;
  const double s = (double)shape.token_bytes(), n = (double)shape.n_tok;
  r.v_allgather = world * n * s;
  r.v_alltoall = n * shape.topk * s;
  r.v_megakernel_nvl = world == 1 ? 0.0 : n * mean_distinct * s;
  r.v_megakernel_hbm = r.v_alltoall - r.v_megakernel_nvl;
  return r;
}
}  // namespace

TrafficReport volume_expected(const MoEShape& shape, const HardwareSpec& spec, SelfRankAccounting acc) {
  double ex = distinct_rank_distribution(spec.world_size, shape.topk).expectation;
  if (acc == SelfRankAccounting::RemoteOnly && spec.world_size > 1)
    ex *= (double)(spec.world_size - 1) / spec.world_size;
  return make_volumes(shape, spec.world_size, ex);
}

TrafficReport volume_exact(const RoutingInstance& r, const MoEShape& shape, const HardwareSpec&,
                           SelfRankAccounting acc) {
  const int epr = r.n_exp / r.world;
  long long distinct = 0;
  for (int src = 0; src < r.world; ++src)
    for (long long t = 0; t < r.n_tok; ++t) {
      std::uint64_t seen = 0;
      for (int j = 0; j < r.topk; ++j) {
        const int dst = r.expert_at(src, t, j) / epr;
        if (acc == SelfRankAccounting::RemoteOnly && dst == src) continue;
        if (!(seen >> dst & 1)) {
          seen |= 1ULL << dst;
          ++distinct;
        }
      }
    }
  const double copies = (double)r.n_tok * r.world;
  MoEShape s = shape;
  s.n_tok = r.n_tok;
  TrafficReport rep = make_volumes(s, r.world, copies > 0 ? distinct / copies : 0.0);
  rep.basis = TrafficReport::Basis::ExactInstance;
  return rep;
}

double expected_remote_ranks(int n_exp, int world, int topk) {
  if (world <= 1) return 0.0;
  // P(a given remote rank is hit) = 1 - C(E - epr, k) / C(E, k)
  const int epr = n_exp / world;
  double miss = 1.0;
  for (int i = 0; i < topk; ++i) miss *= (double)(n_exp - epr - i) / (double)(n_exp - i);
  if (n_exp - epr < topk) miss = 0.0;
  return (world - 1) * (1.0 - miss);
}

// ------------------------------------------------------------------ perf model (perf_model.cpp)
double effective_bandwidth(int n, int w, double beta, double w_sat) {
  return n <= 0 ? 0.0 : std::min((double)n * w * beta / w_sat, beta);
}

double calc_gemm_block_time(const HardwareSpec& s, const MoEShape& m, long long k, int w) {
  const auto it = m.mu_table.find(w);
  if (it == m.mu_table.end()) throw ValidationError("mu_table has no entry for w");
  return 2.0 * m.b_m * m.b_n * (double)k / (s.p_peak * (it->second / s.n_sm)) + s.tau_sync;
}

double calc_swiglu(const MoEShape& m, const HardwareSpec& s, long long expanded) {
  return 2.0 * (double)expanded * (4.0 * m.h_inter) / s.bw_hbm;
}

double calc_disp_lat(const TrafficReport& t, const HardwareSpec& s, const TuneConfig& c) {
  double l = 0;
  if (t.v_megakernel_nvl > 0) {
    const double b = effective_bandwidth(c.n_disp, c.w, s.bw_nvl, s.w_sat);
    if (b <= 0) throw ValidationError("zero effective NVLink bandwidth with nonzero volume");
    l += t.v_megakernel_nvl / b;
  }
  if (t.v_megakernel_hbm > 0) {
    const double b = effective_bandwidth(c.n_relay, c.w, s.bw_hbm, s.w_sat);
    if (b <= 0) throw ValidationError("zero effective HBM bandwidth with nonzero volume");
    l += t.v_megakernel_hbm / b;
  }
  return l;
}

double calc_comp_lat(long long n_tiles, double t_block, int n_comp) {
  if (n_comp <= 0) throw ValidationError("n_comp_sms must be >= 1");
  return n_tiles <= 0 ? 0.0 : (double)((n_tiles + n_comp - 1) / n_comp) * t_block;
}

std::pair<double, double> calc_comb_lat(const TrafficReport& t, const HardwareSpec& s,
                                        const TuneConfig& c) {
  double l_comb = 0, t_red = 0;
  if (t.v_megakernel_nvl > 0) {
    const double b = effective_bandwidth(c.n_comb, c.w, s.bw_nvl, s.w_sat);
    if (b <= 0) throw ValidationError("zero effective NVLink bandwidth with nonzero volume");
    l_comb = t.v_megakernel_nvl / b;
  }
  if (t.v_alltoall > 0) {
    const double b1 = effective_bandwidth(1, c.w, s.bw_hbm, s.w_sat);
    if (b1 <= 0) throw ValidationError("zero effective HBM bandwidth with nonzero volume");
    t_red = t.v_alltoall / b1;
  }
  return {l_comb, t_red};
}

namespace {
long long grouped_tiles(const MoEShape& m, int world, long long n_out) {
  const long long expanded = m.n_tok * m.topk;
  if (expanded == 0) return 0;
  const long long epr = m.experts_per_rank(world);
  const long long rows = (expanded + epr - 1) / epr;
  return epr * ((rows + m.b_m - 1) / m.b_m) * ((n_out + m.b_n - 1) / m.b_n);
}
}  // namespace

long long tiles_up(const MoEShape& m, int world) { return grouped_tiles(m, world, 2LL * m.h_inter); }
long long tiles_down(const MoEShape& m, int world) { return grouped_tiles(m, world, m.h_dim); }

LatencyBreakdown predict_latency(const MoEShape& m, const HardwareSpec& s, const TuneConfig& c,
                                 const TrafficReport& t, ResidualScaling mode) {
  LatencyBreakdown b;
  b.t_up = calc_gemm_block_time(s, m, m.h_dim, c.w);
  b.t_down = calc_gemm_block_time(s, m, m.h_inter, c.w);
  b.l_swiglu = calc_swiglu(m, s, m.n_tok * m.topk);
  b.n_tiles_up = tiles_up(m, s.world_size);
  b.n_tiles_down = tiles_down(m, s.world_size);
  // stage 1: dispatch overlapped with the up GEMM (Alg. 2 lines 3-12)
  const int comp1 = s.n_sm - c.n_disp;
  if (comp1 <= 0) throw ValidationError("n_disp leaves no compute SMs");
  b.l_disp = calc_disp_lat(t, s, c);
  b.l_up = calc_comp_lat(b.n_tiles_up, b.t_up, comp1);
  if (b.l_up > b.l_disp)
    b.l_s1 = b.l_disp + (b.l_up - b.l_disp) *
                            (mode == ResidualScaling::AsPrinted ? (double)s.n_sm / comp1
                                                                : (double)comp1 / s.n_sm);
  else
    b.l_s1 = b.l_disp + b.t_up;
  // stage 2: down GEMM overlapped with combine; the reduction fills the gap (lines 13-25)
  const int comp2 = s.n_sm - c.n_comb;
  if (comp2 <= 0) throw ValidationError("n_comb leaves no compute SMs");
  std::tie(b.l_comb, b.t_red) = calc_comb_lat(t, s, c);
  b.l_down = calc_comp_lat(b.n_tiles_down, b.t_down, comp2);
  b.w_gap = std::abs(b.l_down - b.l_comb) * comp2;
  b.w_red = b.t_red;  // reference behaviour (perf_model.cpp:129)
  b.w_rem = std::max(0.0, b.w_red - b.w_gap);
  b.l_s2 = std::max(b.l_down, b.l_comb) + b.w_rem / s.n_sm;
  b.l_total = b.l_s1 + b.l_s2 + b.l_swiglu;
  return b;
}

// ------------------------------------------------------------------ B200 model of our kernels
HardwareSpec b200_hardware(int world, double p_peak, double bw_hbm, double bw_nvl) {
  HardwareSpec h;
  h.name = "b200";
  h.n_sm = 148;
  h.p_peak = p_peak;
  h.bw_hbm = bw_hbm;
  h.bw_nvl = bw_nvl;
  h.w_sat = 1024;
  h.tau_sync = 1e-6;
  h.world_size = world;
  return h;
}

LayerPrediction predict_layer(const MoEShape& m, const HardwareSpec& s, const TuneConfig& c,
                              const B200Calib& k) {
  LayerPrediction p;
  const int W = s.world_size, epr = m.n_exp / W;
  const double T = (double)m.n_tok, S = (double)m.token_bytes();
  const double H = m.h_dim, F = m.h_inter;
  const double rows = T * m.topk;  // received rows per rank (balanced routing)
  const double rows_e = rows / epr;
  const double mblocks = epr * std::ceil(rows_e / 128.0);
  const double seg_pad = std::ceil(rows_e / 128.0) * 128.0;
  // tile time: main loop at mu of peak, or the epilogue's traffic (bytes per 128x256 tile) when
  // that is longer (the TMEM double buffer overlaps the two), plus a fixed hand-off cost
  auto tile_t = [&](double K, double epi_bytes) {
    return std::max(2.0 * 128 * 256 * K / (s.p_peak * k.mu / s.n_sm), epi_bytes / k.epi_bw_per_sm) +
           k.tile_overhead;
  };
  constexpr double kEpiUp = 128.0 * (256 + 128) * 2;           // GU + h
  constexpr double kEpiPush = 128.0 * 256 * 2;                  // one replica row chunk
  constexpr double kEpiDgrad = 128.0 * (512 + 256 + 512) * 2;   // dGU + HW written, GU read
  constexpr double kEpiWgrad = 128.0 * 256 * 2;                 // dW tile
  // dispatch rows: relay on -> one send per (token, distinct destination rank) and HBM relay
  // copies for the other replicas (sim.cpp:384-441); relay off -> every replica is sent
  // (AllToAll style). q = P(a given rank hosts >= 1 of the token's experts), without replacement.
  const double q = W > 1 ? expected_remote_ranks(m.n_exp, W, m.topk) / (W - 1) : 1.0;
  const bool relay = c.n_relay > 0;
  const double sent_rows = relay ? T * W * q : rows;
  const double nvl_rows = relay ? T * (W - 1) * q : rows * (double)(W - 1) / W;
  const double k_rem = m.topk * (double)(W - 1) / W;
  const double dup_rows = relay ? std::max(0.0, rows - sent_rows) : 0.0;
  // comm capacity: n_disp comm CTAs plus the GEMM CTAs' spare warps (the warp split), both
  // draining one round pool; only the comm CTAs' time is taken from the GEMM
  const double comm_units = std::max(c.n_disp + k.spare_sm_equiv, 1e-3);
  const double l_comm = std::max(sent_rows * S / (comm_units * k.comm_bw_per_sm),
                                 W > 1 ? nvl_rows * S / s.bw_nvl : 0.0);
  // relay pool: the n_relay relay CTAs' warps plus, once the comm rounds drain, the spare warps
  const double l_relay = relay ? dup_rows * S / ((c.n_relay + k.spare_sm_equiv) * k.relay_bw_per_sm) : 0.0;
  const double l_push = W > 1 ? T * k_rem * S / s.bw_nvl : 0.0;
  const double l_reduce = T * (m.topk + 1) * S / k.reduce_bw;
  // persistent grid: SM-seconds spread over n_sm, but never less than whole waves of the
  // kernel's dominant tile (quantisation matters for small batches)
  // algorithmic HBM bytes per kernel: every tensor read or written once per use (the dispatch
  // copies, both GEMMs' operands and outputs, saved activations, replica slots, reductions, dW)
  const double w_up = epr * 2 * F * H * 2, w_down = epr * H * F * 2;
  const double b_fd = T * S + rows * S + rows * S + w_up + rows * 2 * F * 2 + rows * F * 2;
  const double b_fc = rows * F * 2 + w_down + rows * S + T * m.topk * S + T * S;
  const double b_bd = T * S + rows * S + rows * S + w_down + rows * 4 * F * 2 + rows * F * 2 + rows * S +
                      rows * F * 2 + w_down;
  const double b_bc = rows * 4 * F + w_up + rows * S + rows * 4 * F + rows * S + w_up + T * m.topk * S + T * S;
  // persistent grid: SM-seconds spread over n_sm, but never less than whole waves of the
  // kernel's dominant tile (quantisation matters for small batches); the HBM traffic overlaps
  // the compute only partly (hbm_overlap)
  auto kernel = [&](double sm_seconds, double critical, double extra, double tiles = 0,
                    double t_one = 0, double hbm_bytes = 0, double t_start = 0) {
    const double waves = tiles > 0 ? std::ceil(tiles / s.n_sm) * t_one : 0.0;
    const double comp = std::max({sm_seconds / s.n_sm + t_start, critical, waves});
    const double mem = hbm_bytes / s.bw_hbm;
    return std::max(comp, mem) + k.hbm_overlap * std::min(comp, mem) + extra + k.launch;
  };
  const double n_pre_sm = c.n_disp * l_comm + c.n_relay * l_relay;
  // GEMM start-up behind the scoreboard: the first wave of pair tiles (n_sm / 2 of them, raster
  // groups of 8 row pairs across the nb column blocks) needs its rows landed before its main loop
  // starts; the comm pool lands rows in priority order at its aggregate rate
  auto start_up = [&](double nb, double units) {
    const double first_rows = std::min(rows, 256.0 * std::ceil((s.n_sm / 2.0) / nb));
    return first_rows * S / (std::max(units, 1e-3) * k.comm_bw_per_sm) * k.startup;
  };
  // forward
  const double up = mblocks * (F / 128) * tile_t(H, kEpiUp);
  p.fwd_dispatch = kernel(up + n_pre_sm, std::max(l_comm, l_relay) + tile_t(H, kEpiUp), 0.0,
                          mblocks * (F / 128), tile_t(H, kEpiUp), b_fd, start_up(F / 128, comm_units));
  const double down = mblocks * (H / 256) * tile_t(F, kEpiPush);
  p.fwd_combine = kernel(down, l_push, l_reduce, mblocks * (H / 256), tile_t(F, kEpiPush), b_fc);
  // backward: the dY dispatch moves the forward's rows (the gate gradient is formed in the
  // down-dgrad epilogue) with twice the comm CTAs (eplab_dispatch_group_gemm_bwd)
  const double comm_units_b = std::max(std::min(2.0 * c.n_disp, s.n_sm / 2.0 - c.n_relay) + k.spare_sm_equiv, 1e-3);
  const double l_comm_b = std::max(sent_rows * S / (comm_units_b * k.comm_bw_per_sm),
                                   W > 1 ? nvl_rows * S / s.bw_nvl : 0.0);
  const double ddown = mblocks * (F / 256) * tile_t(H, kEpiDgrad);
  const double wg_down = epr * (H / 128) * (F / 256) * tile_t(seg_pad, kEpiWgrad);
  p.bwd_dispatch = kernel(ddown + wg_down + std::min(2.0 * c.n_disp, s.n_sm / 2.0 - c.n_relay) * l_comm_b +
                              c.n_relay * l_relay,
                          std::max(l_comm_b, l_relay) + tile_t(H, kEpiDgrad), 0.0, 0, 0, b_bd,
                          start_up(F / 256, comm_units_b));
  const double dup = mblocks * (H / 256) * tile_t(2 * F, kEpiPush);
  const double wg_up = epr * (2 * F / 128) * (H / 256) * tile_t(seg_pad, kEpiWgrad);
  p.bwd_combine = kernel(dup + wg_up, l_push, l_reduce, mblocks * (H / 256), tile_t(2 * F, kEpiPush), b_bc);
  p.total = p.fwd_dispatch + p.fwd_combine + p.bwd_dispatch + p.bwd_combine;
  p.t_gemm_bound = 18.0 * m.topk * H * F * T / s.p_peak;
  p.t_nvl_bound = 2.0 * ((W - 1) * q + k_rem) * 2.0 * H * T / s.bw_nvl;
  return p;
}

// ------------------------------------------------------------------ tuner (tuner.cpp)
std::vector<int> SearchSpace::relay_choices(int n_disp) {
  std::vector<int> v;
  for (int x = 1; x <= n_disp / 2; x += 4) v.push_back(x);
  if (v.empty()) v.push_back(1);
  return v;
}

SearchSpace enumerate_space(const HardwareSpec& spec, const MoEShape&) {
  if (spec.n_sm < 4) throw ValidationError("n_sm must be >= 4 to enumerate the config space");
  SearchSpace s;
  s.n_sm = spec.n_sm;
  for (int x = 4; x <= spec.n_sm; x += 4) s.disp_choices.push_back(x);
  s.comb_choices = s.disp_choices;
  for (int x = 1; x <= spec.n_sm; x += 16) s.red_choices.push_back(x);
  if (s.red_choices.back() != spec.n_sm) s.red_choices.push_back(spec.n_sm);
  s.warp_choices = {8, 16, 32};
  const long long flat = std::max(1, spec.n_sm / 16);
  s.raw_grid_size = (long long)s.disp_choices.size() * s.comb_choices.size() * flat * flat * 3;
  for (int nd : s.disp_choices)
    s.enumerated_count += (long long)SearchSpace::relay_choices(nd).size() * s.comb_choices.size() *
                          s.red_choices.size() * s.warp_choices.size();
  return s;
}

void for_each_candidate(const SearchSpace& sp, bool feasible_only,
                        const std::function<void(const TuneConfig&)>& fn) {
  for (int nd : sp.disp_choices) {
    const auto relays = SearchSpace::relay_choices(nd);
    for (int nc : sp.comb_choices)
      for (int nr : relays)
        for (int nred : sp.red_choices)
          for (int w : sp.warp_choices) {
            if (feasible_only && (nd + nr >= sp.n_sm || nc >= sp.n_sm)) continue;
            fn(TuneConfig{nd, nr, nc, nred, w});
          }
  }
}

namespace {
// ascending n_disp, n_comb, n_relay; descending n_red; ascending w (tuner.cpp:70-73)
bool preferred(double la, const TuneConfig& a, double lb, const TuneConfig& b) {
  if (la != lb) return la < lb;
  return std::make_tuple(a.n_disp, a.n_comb, a.n_relay, -a.n_red, a.w) <
         std::make_tuple(b.n_disp, b.n_comb, b.n_relay, -b.n_red, b.w);
}

TuneResult minimise(const std::vector<TuneConfig>& cands, const LatencyFn& eval, int n_workers) {
  auto t0 = std::chrono::steady_clock::now();
  if (cands.empty()) throw ValidationError("empty feasible config set");
  if (n_workers <= 0) n_workers = (int)std::thread::hardware_concurrency();
  n_workers = std::clamp(n_workers, 1, 64);
  struct Best {
    double l = 0;
    TuneConfig c{};
    bool ok = false;
  };
  auto scan = [&](size_t lo, size_t hi, Best& out) {
    for (size_t i = lo; i < hi; ++i) {
      const double l = eval(cands[i]);
      if (!out.ok || preferred(l, cands[i], out.l, out.c)) out = Best{l, cands[i], true};
    }
  };
  Best best;
  if (n_workers == 1 || cands.size() < 1024) {
    scan(0, cands.size(), best);
  } else {
    std::vector<Best> part(n_workers);
    std::vector<std::thread> pool;
    const size_t chunk = (cands.size() + n_workers - 1) / n_workers;
    for (int w = 0; w < n_workers; ++w) {
      const size_t lo = std::min(cands.size(), (size_t)w * chunk);
      pool.emplace_back(scan, lo, std::min(cands.size(), lo + chunk), std::ref(part[w]));
    }
    for (auto& th : pool) th.join();
    for (const auto& b : part)
      if (b.ok && (!best.ok || preferred(b.l, b.c, best.l, best.c))) best = b;
  }
  TuneResult r;
  r.best = best.c;
  r.l_min = best.l;
  r.evaluated = (long long)cands.size();
  r.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return r;
}
}  // namespace

TuneResult search_with(const HardwareSpec& spec, const MoEShape& shape, const LatencyFn& eval,
                       int n_workers) {
  std::vector<TuneConfig> cands;
  for_each_candidate(enumerate_space(spec, shape), true, [&](const TuneConfig& c) { cands.push_back(c); });
  return minimise(cands, eval, n_workers);
}

TuneResult search(const HardwareSpec& spec, const MoEShape& shape, const TrafficReport& traffic,
                  int n_workers, ResidualScaling mode) {
  TuneResult r = search_with(
      spec, shape, [&](const TuneConfig& c) { return predict_latency(shape, spec, c, traffic, mode).l_total; },
      n_workers);
  r.breakdown = predict_latency(shape, spec, r.best, traffic, mode);
  r.l_min = r.breakdown.l_total;
  return r;
}

TuneResult search_layer(const HardwareSpec& spec, const MoEShape& shape, int n_workers,
                        const B200Calib& calib) {
  std::vector<TuneConfig> cands;
  for (int nd = calib.spare_sm_equiv > 0 ? 0 : 4; nd < spec.n_sm; nd += 4) {
    std::vector<int> relays = {0};
    if (spec.world_size > 1)
      for (int r : SearchSpace::relay_choices(nd)) relays.push_back(r);
    for (int nr : relays)
      if (nd + nr < spec.n_sm) cands.push_back(TuneConfig{nd, nr, 1, spec.n_sm, 8});
  }
  return minimise(cands, [&](const TuneConfig& c) { return predict_layer(shape, spec, c, calib).total; },
                  n_workers);
}

long long token_bucket(long long n_tok) { return (n_tok + 4095) / 4096; }

TuneResult TuneCache::lookup(const HardwareSpec& spec, const MoEShape& shape, long long n_tok,
                             int n_workers, ResidualScaling mode) {
  if (n_tok < 1) throw ValidationError("n_tok must be >= 1");
  const auto key = std::make_tuple(spec.name, shape.name, token_bucket(n_tok));
  if (auto it = entries_.find(key); it != entries_.end()) return it->second;
  MoEShape b = shape;
  b.n_tok = std::get<2>(key) * 4096;
  ++invocations_;
  TuneResult r = search(spec, b, volume_expected(b, spec), n_workers, mode);
  entries_.emplace(key, r);
  return r;
}

// Cache file: the reference's JSON layout (tuner.cpp:167-186), written without a JSON library.
void TuneCache::save(const std::string& path) const {
  std::ofstream f(path);
  if (!f) throw ValidationError("cannot write cache file " + path);
  f.precision(17);
  f << "{\n  \"entries\": [";
  bool first = true;
  for (const auto& [k, v] : entries_) {
    f << (first ? "\n" : ",\n") << "    {\"hardware\": \"" << std::get<0>(k) << "\", \"shape\": \""
      << std::get<1>(k) << "\", \"bucket\": " << std::get<2>(k) << ", \"n_disp\": " << v.best.n_disp
      << ", \"n_relay\": " << v.best.n_relay << ", \"n_comb\": " << v.best.n_comb
      << ", \"n_red\": " << v.best.n_red << ", \"w\": " << v.best.w << ", \"l_min\": " << v.l_min
      << ", \"evaluated\": " << v.evaluated << "}";
    first = false;
  }
  f << "\n  ],\n  \"version\": 1\n}\n";
}

void TuneCache::load(const std::string& path) {
  std::ifstream f(path);
  if (!f) return;
  std::stringstream ss;
  ss << f.rdbuf();
  const std::string s = ss.str();
  auto field = [&](size_t from, const std::string& name) -> std::string {
    const size_t p = s.find("\"" + name + "\"", from);
    if (p == std::string::npos) throw ValidationError("cache file missing field " + name);
    size_t q = s.find(':', p) + 1;
    while (s[q] == ' ') ++q;
    if (s[q] == '"') return s.substr(q + 1, s.find('"', q + 1) - q - 1);
    size_t e = q;
    while (e < s.size() && s[e] != ',' && s[e] != '}' && s[e] != '\n') ++e;
    return s.substr(q, e - q);
  };
  if (s.find("\"version\": 1") == std::string::npos)
    throw ValidationError("unknown cache file version in " + path);
  for (size_t p = s.find("{\"hardware\""); p != std::string::npos; p = s.find("{\"hardware\"", p + 1)) {
    TuneResult r;
    r.best = TuneConfig{std::stoi(field(p, "n_disp")), std::stoi(field(p, "n_relay")),
                        std::stoi(field(p, "n_comb")), std::stoi(field(p, "n_red")),
                        std::stoi(field(p, "w"))};
    r.l_min = std::stod(field(p, "l_min"));
    r.evaluated = std::stoll(field(p, "evaluated"));
    entries_.emplace(std::make_tuple(field(p, "hardware"), field(p, "shape"), std::stoll(field(p, "bucket"))), r);
  }
}

}  // namespace eplab
