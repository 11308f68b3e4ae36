// eplab C++ host API of the B200 build (namespace eplab), re-implemented from scratch so that
// callers written against the reference's headers (/root/reference/proj/src/eplab/*.hpp) find
// the same types and entry points. Device data-path entry points live in eplab_b200.h.
//
//   types.hpp:16-82      HardwareSpec, MoEShape, TuneConfig, RoutingInstance, validate_*
//   routing.hpp:15       sample_routing
//   token_map.hpp:22-93  local_stable_sort, compute_global_offsets, build_global_token_map,
//                        build_send_schedule
//   traffic.hpp:14-51    BigInt, stirling2, distinct_rank_distribution, volume_expected, volume_exact
//   precision.hpp:16-52  OrderPolicy, ReductionTerm, ReductionPlan, accumulate, PrecisionReport,
//                        fused_vs_sequential, split_batch_experiment
//   softfloat.hpp:10-28  FpFormat, round_to_bf16, fp_round, fp_add, fp_mul, bit_equal
//   perf_model.hpp:38-62 effective_bandwidth ... predict_latency (reference-compatible)
//   tuner.hpp:16-82      enumerate_space, search, TuneCache
//   sim.hpp:16-85        Role, role_name, TaskQueueInfo, build_task_list (the task layout, not the simulator)
// B200 additions: b200_hardware(), predict_layer() (fwd+bwd model of the MegaKernels built
// here, incl. the relay-off AllToAll mode), search_layer().
#pragma once
#include <algorithm>
#include <cstdint>
#include <functional>
#include <map>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

// The eplab:: API is exported from libeplab_b200.so (built with -fvisibility=hidden) so that
// reference-style C++ callers link against it directly.
#pragma GCC visibility push(default)
namespace eplab {

class ValidationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeadlockError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct HardwareSpec {
  std::string name;
  int n_sm = 0;
  double p_peak = 0;       // bf16 FLOP/s
  double bw_hbm = 0;       // B/s
  double bw_nvl = 0;       // B/s per direction
  double w_sat = 1024;     // warps to saturate a link
  double tau_sync = 2e-6;  // per-tile synchronisation, s
  int world_size = 1;
};

struct MoEShape {
  std::string name;
  int h_dim = 0, h_inter = 0, n_exp = 0, topk = 0;
  long long n_tok = 0;  // tokens per rank
  long long s_tok = 0;  // bytes per token row (0: 2*h_dim)
  int b_m = 128, b_n = 256;
  std::map<int, double> mu_table = {{8, 0.7}, {16, 0.65}, {32, 0.6}};
  long long token_bytes() const { return s_tok > 0 ? s_tok : 2LL * h_dim; }
  int experts_per_rank(int world) const { return n_exp / world; }
};

struct TuneConfig {
  int n_disp = 0, n_relay = 0, n_comb = 0, n_red = 0, w = 0;
  bool operator==(const TuneConfig&) const = default;
};

struct RoutingInstance {
  int world = 0, n_exp = 0, topk = 0;
  long long n_tok = 0;
  std::uint64_t seed = 0;
  std::vector<std::vector<int>> selected_experts;  // [rank][t*topk+j]
  std::vector<std::vector<float>> gate_weights;
  int expert_at(int r, long long t, int j) const { return selected_experts[r][t * topk + j]; }
  float weight_at(int r, long long t, int j) const { return gate_weights[r][t * topk + j]; }
};

HardwareSpec validate_hardware(HardwareSpec spec);
std::pair<MoEShape, HardwareSpec> validate_shape(MoEShape shape, HardwareSpec spec);
void validate_tune_config(const TuneConfig& cfg, const HardwareSpec& spec);
// Post-dispatch token count per rank under balanced routing (types.hpp:79).
long long derive_expanded_tokens(const MoEShape& shape, int world);
void validate_routing(const RoutingInstance& routing);

RoutingInstance sample_routing(const MoEShape& shape, int world, std::uint64_t seed);

// --------------------------------------------------------------- token map (host mirror)
struct LocalSortResult {
  std::vector<long long> m_loc, expert_counts, expert_offsets;
};
LocalSortResult local_stable_sort(const std::vector<int>& selected, long long n_tok, int topk,
                                  int n_exp);
struct GlobalOffsets {
  int world = 0, experts_per_rank = 0;
  std::vector<long long> data;  // [dst][e_loc][src]
  long long at(int dst, int e_loc, int src) const {
    return data[((size_t)dst * experts_per_rank + e_loc) * world + src];
  }
};
GlobalOffsets compute_global_offsets(const std::vector<std::vector<long long>>& counts, int world,
                                     int n_exp);
struct MapEntry {
  int target_rank = 0, local_expert = 0;
  long long offset = 0;
  bool operator==(const MapEntry&) const = default;
};
struct GlobalTokenMap {
  int rank = 0, topk = 0, world = 0, experts_per_rank = 0;
  long long n_tok = 0;
  std::vector<MapEntry> entries;
  std::vector<long long> recv_totals, recv_segment_base;
  const MapEntry& at(long long t, int j) const { return entries[t * topk + j]; }
  long long recv_total(int rank_, int e_loc) const { return recv_totals[(size_t)rank_ * experts_per_rank + e_loc]; }
  long long segment_base(int rank_, int e_loc) const {
    return recv_segment_base[(size_t)rank_ * experts_per_rank + e_loc];
  }
};
std::vector<GlobalTokenMap> build_global_token_map(const RoutingInstance& routing);
struct SendItem {
  long long token = 0;
  int slot = 0, dst_rank = 0, dst_expert = 0;
  long long dst_offset = 0;
  bool operator==(const SendItem&) const = default;
};
struct SendSchedule {
  int rank = 0;
  std::vector<SendItem> items;
};
SendSchedule build_send_schedule(const GlobalTokenMap& map);
// One row per (rank, t, j) plus a header, for diffing against oracles (token_map.hpp:91).
std::string export_map_table(const std::vector<GlobalTokenMap>& maps);

// --------------------------------------------------------------- traffic
// Exact non-negative integers of any size (the role of boost::multiprecision::cpp_int in
// traffic.hpp:6-10): base-2^32 limbs, the operations the exact traffic arithmetic needs.
class BigInt {
 public:
  BigInt(unsigned long long v = 0) { set(v); }  // NOLINT: implicit, like cpp_int
  BigInt(long long v) { set(v < 0 ? 0ULL : (unsigned long long)v); }
  BigInt(int v) { set(v < 0 ? 0ULL : (unsigned long long)v); }
  BigInt(unsigned __int128 v) {
    while (v) {
      l_.push_back((uint32_t)v);
      v >>= 32;
    }
  }
  explicit BigInt(const char* dec) {
    for (const char* c = dec; *c; ++c) {
      if (*c < '0' || *c > '9') throw std::invalid_argument("BigInt: not a decimal number");
      *this = *this * BigInt(10) + BigInt(*c - '0');
    }
  }
  BigInt& operator+=(const BigInt& o) {
    uint64_t carry = 0;
    if (l_.size() < o.l_.size()) l_.resize(o.l_.size(), 0);
    for (size_t i = 0; i < l_.size(); ++i) {
      const uint64_t s = (uint64_t)l_[i] + (i < o.l_.size() ? o.l_[i] : 0) + carry;
      l_[i] = (uint32_t)s;
      carry = s >> 32;
    }
    if (carry) l_.push_back((uint32_t)carry);
    return *this;
  }
  friend BigInt operator+(BigInt a, const BigInt& b) { return a += b; }
  friend BigInt operator*(const BigInt& a, const BigInt& b) {
    BigInt r;
    if (a.l_.empty() || b.l_.empty()) return r;
    std::vector<uint64_t> acc(a.l_.size() + b.l_.size() + 1, 0);
    for (size_t i = 0; i < a.l_.size(); ++i) {
      uint64_t carry = 0;
      for (size_t j = 0; j < b.l_.size(); ++j) {
        const uint64_t cur = acc[i + j] + (uint64_t)a.l_[i] * b.l_[j] + carry;
        acc[i + j] = cur & 0xFFFFFFFFull;
        carry = cur >> 32;
      }
      for (size_t k = i + b.l_.size(); carry; ++k) {
        const uint64_t cur = acc[k] + carry;
        acc[k] = cur & 0xFFFFFFFFull;
        carry = cur >> 32;
      }
    }
    r.l_.assign(acc.begin(), acc.end());
    r.trim();
    return r;
  }
  BigInt& operator*=(const BigInt& o) { return *this = *this * o; }
  friend bool operator==(const BigInt& a, const BigInt& b) { return a.l_ == b.l_; }
  friend bool operator!=(const BigInt& a, const BigInt& b) { return !(a == b); }
  friend bool operator<(const BigInt& a, const BigInt& b) {
    if (a.l_.size() != b.l_.size()) return a.l_.size() < b.l_.size();
    for (size_t i = a.l_.size(); i-- > 0;)
      if (a.l_[i] != b.l_[i]) return a.l_[i] < b.l_[i];
    return false;
  }
  friend bool operator>(const BigInt& a, const BigInt& b) { return b < a; }
  friend bool operator<=(const BigInt& a, const BigInt& b) { return !(b < a); }
  friend bool operator>=(const BigInt& a, const BigInt& b) { return !(a < b); }
  double to_double() const {
    double r = 0;
    for (size_t i = l_.size(); i-- > 0;) r = r * 4294967296.0 + l_[i];
    return r;
  }
  template <class T>
  T convert_to() const {
    return (T)to_double();
  }
  std::string str() const {
    if (l_.empty()) return "0";
    std::vector<uint32_t> v = l_;
    std::string out;
    while (!v.empty()) {  // repeated division by 10^9
      uint64_t rem = 0;
      for (size_t i = v.size(); i-- > 0;) {
        const uint64_t cur = (rem << 32) | v[i];
        v[i] = (uint32_t)(cur / 1000000000u);
        rem = cur % 1000000000u;
      }
      while (!v.empty() && v.back() == 0) v.pop_back();
      char buf[16];
      std::snprintf(buf, sizeof buf, v.empty() ? "%llu" : "%09llu", (unsigned long long)rem);
      out.insert(0, buf);
    }
    return out;
  }

 private:
  void set(unsigned long long v) {
    l_.clear();
    while (v) {
      l_.push_back((uint32_t)v);
      v >>= 32;
    }
  }
  void trim() {
    while (!l_.empty() && l_.back() == 0) l_.pop_back();
  }
  std::vector<uint32_t> l_;  // little-endian base-2^32 limbs, no leading zeros
};

// Stirling numbers of the second kind, exact, 0 <= k <= n <= 64 (traffic.hpp:16).
BigInt stirling2(int n, int k);
struct DistinctRankDistribution {
  int world = 0, topk = 0;
  std::vector<BigInt> numerators;  // index x-1, x in [1, min(topk, world)]
  BigInt denominator = 1;          // world^topk
  std::vector<double> probs;
  double expectation = 0, expected_saving_fraction = 0;
  double prob(int x) const { return probs[x - 1]; }
};
DistinctRankDistribution distinct_rank_distribution(int world, int topk);
enum class SelfRankAccounting { IncludeSelf, RemoteOnly };
struct TrafficReport {
  double v_allgather = 0, v_alltoall = 0, v_megakernel_nvl = 0, v_megakernel_hbm = 0;
  enum class Basis { Expected, ExactInstance } basis = Basis::Expected;  // traffic.hpp:44
};
TrafficReport volume_expected(const MoEShape& shape, const HardwareSpec& spec,
                              SelfRankAccounting acc = SelfRankAccounting::IncludeSelf);
TrafficReport volume_exact(const RoutingInstance& routing, const MoEShape& shape,
                           const HardwareSpec& spec,
                           SelfRankAccounting acc = SelfRankAccounting::IncludeSelf);
// Exact E[#distinct remote ranks] for top-k drawn WITHOUT replacement from n_exp experts
// spread evenly over `world` ranks.
double expected_remote_ranks(int n_exp, int world, int topk);

// --------------------------------------------------------------- softfloat / precision
// softfloat.hpp:10-28: round-to-nearest-even to bfloat16 carried in binary32; fp_add / fp_mul round
// their binary32 result to the format (an accumulate-then-round pipeline).
enum class FpFormat { Binary32, Bfloat16 };
float round_to_bf16(float x);
float fp_round(float x, FpFormat fmt);
float fp_add(float a, float b, FpFormat fmt);
float fp_mul(float a, float b, FpFormat fmt);
bool bit_equal(float a, float b);

// precision.hpp:16-52. The k-ordered combine: a token's replicas folded in plan order, every
// intermediate rounded to the format. With FpFormat::Binary32 this is, bit for bit, the fold of
// the MegaKernels' reduce role (y = round_to_bf16(accumulate(plan, Binary32)), tests/test_parity_gpu.py).
enum class OrderPolicy { Canonical, Permuted, SplitBatch };
struct ReductionTerm {
  int k = 0;
  float weight = 0;
  float value = 0;
};
struct ReductionPlan {
  std::vector<std::vector<ReductionTerm>> tokens;
};
std::vector<float> accumulate(const ReductionPlan& plan, FpFormat fmt);
struct PrecisionReport {
  double max_diff = 0;
  double frac_non_bitwise = 0;
  long long elements = 0;
  long long non_bitwise = 0;
};
// Path A: the sequential k-ascending fold; path B: the fused combine of this build -- a token is
// reduced only after all top-k replicas landed (the reduce role's top-k barrier) and folded in
// canonical slot order whatever order they arrived in (here: a seeded random arrival order per
// token, as replicas from different expert tiles and ranks land). control = Permuted folds path B
// in a seeded per-token permutation instead (the broken-reducer control). The reference derives
// arrival times from its combine simulator (precision.cpp:54-96); the fold order, the contract, is
// the same.
PrecisionReport fused_vs_sequential(const RoutingInstance& routing, const MoEShape& shape,
                                    const HardwareSpec& spec, const TuneConfig& cfg, std::uint64_t seed,
                                    FpFormat fmt, OrderPolicy control = OrderPolicy::Canonical);
// Weight-gradient style column sums: full left-fold over the token axis vs (first half) + (second
// half) (precision.cpp:98-134). split_at < 0 means n_tok / 2.
PrecisionReport split_batch_experiment(const MoEShape& shape, std::uint64_t seed, FpFormat fmt,
                                       long long split_at = -1);

// --------------------------------------------------------------- perf model (reference Alg. 2)
enum class ResidualScaling { AsPrinted, Redistributed };
struct LatencyBreakdown {
  double t_up = 0, t_down = 0, l_swiglu = 0, l_disp = 0, l_up = 0, l_comb = 0, l_down = 0,
         t_red = 0, l_s1 = 0, l_s2 = 0, l_total = 0;
  long long n_tiles_up = 0, n_tiles_down = 0;
  double w_gap = 0, w_red = 0, w_rem = 0;
};
double effective_bandwidth(int n_sm_active, int w, double beta, double w_sat);
double calc_gemm_block_time(const HardwareSpec& spec, const MoEShape& shape, long long k_dim, int w);
double calc_swiglu(const MoEShape& shape, const HardwareSpec& spec, long long expanded_tokens);
double calc_disp_lat(const TrafficReport& traffic, const HardwareSpec& spec, const TuneConfig& cfg);
double calc_comp_lat(long long n_tiles, double t_block, int n_comp_sms);
std::pair<double, double> calc_comb_lat(const TrafficReport& traffic, const HardwareSpec& spec,
                                        const TuneConfig& cfg);
long long tiles_up(const MoEShape& shape, int world);
long long tiles_down(const MoEShape& shape, int world);
LatencyBreakdown predict_latency(const MoEShape& shape, const HardwareSpec& spec,
                                 const TuneConfig& cfg, const TrafficReport& traffic,
                                 ResidualScaling mode = ResidualScaling::AsPrinted);

// --------------------------------------------------------------- B200 model of the MegaKernels
// Calibrated constants of this implementation on B200 (DESIGN.md §Performance model).
struct B200Calib {
  // fitted over 94 measured cases, EP=1 and EP=2/4/8 on virtual ranks (tools/model_sweep.py
  // --ep + tools/fit_model.py, profiles/r02_perf_model_validation.md: 6.6 % mean step error)
  double mu = 0.935;              // tensor-pipe efficiency of the tile main loop vs p_peak (sustained)
  double tile_overhead = 0.2e-6;  // per-tile hand-off cost not hidden behind the loop, s
  double comm_bw_per_sm = 28.94e9; // B/s one comm CTA sustains (8 warps of warp copies)
  double relay_bw_per_sm = 8.88e9;   // B/s one relay worker unit sustains on HBM copies (polling
                                     // the primaries' flags, then copying)
  double reduce_bw = 6.5e12;      // B/s of the reduce role when all SMs join
  double launch = 31.45e-6;       // per MegaKernel fixed cost: launch, prologue, pipeline fill
  double epi_bw_per_sm = 199.1e9; // B/s of epilogue traffic per SM (TMA stores, saved-input reads)
  double spare_sm_equiv = 29.04;  // comm capacity of the GEMM CTAs' spare warps, in comm-CTA units
                                  // (0: spare warps off / not modelled); also drains the relay pool
  double hbm_overlap = 0.528;     // kernel time = max(compute, HBM) + hbm_overlap * min(compute, HBM)
                                  // (HBM = the kernel's algorithmic bytes at bw_hbm)
  double startup = 2.0;           // weight of the GEMM start-up term: landing the first wave's rows
                                  // at the comm pool's rate before its main loops run
};
struct LayerPrediction {
  double fwd_dispatch = 0, fwd_combine = 0, bwd_dispatch = 0, bwd_combine = 0, total = 0;
  double t_gemm_bound = 0, t_nvl_bound = 0;  // roofline terms
};
HardwareSpec b200_hardware(int world, double p_peak = 1408.1e12, double bw_hbm = 6468.9e9,
                           double bw_nvl = 770e9);
// cfg.n_relay == 0 selects the AllToAll-style primitive (every replica crosses NVLink).
LayerPrediction predict_layer(const MoEShape& shape, const HardwareSpec& spec,
                              const TuneConfig& cfg, const B200Calib& calib = {});

// --------------------------------------------------------------- tuner
struct SearchSpace {
  int n_sm = 0;
  std::vector<int> disp_choices, comb_choices, red_choices, warp_choices;
  long long raw_grid_size = 0, enumerated_count = 0;
  static std::vector<int> relay_choices(int n_disp);
};
SearchSpace enumerate_space(const HardwareSpec& spec, const MoEShape& shape);
void for_each_candidate(const SearchSpace& space, bool feasible_only,
                        const std::function<void(const TuneConfig&)>& fn);
struct TuneResult {
  TuneConfig best;
  double l_min = 0;
  long long evaluated = 0;
  double wall_seconds = 0;
  LatencyBreakdown breakdown;
};
using LatencyFn = std::function<double(const TuneConfig&)>;
TuneResult search_with(const HardwareSpec& spec, const MoEShape& shape, const LatencyFn& eval,
                       int n_workers = 0);
TuneResult search(const HardwareSpec& spec, const MoEShape& shape, const TrafficReport& traffic,
                  int n_workers = 0, ResidualScaling mode = ResidualScaling::AsPrinted);
// B200: minimise predict_layer().total over (n_disp, n_relay in {0} U relay_choices, n_red) at
// the w this build implements (8).
TuneResult search_layer(const HardwareSpec& spec, const MoEShape& shape, int n_workers = 0,
                        const B200Calib& calib = {});
long long token_bucket(long long n_tok);
class TuneCache {
 public:
  TuneResult lookup(const HardwareSpec& spec, const MoEShape& shape, long long n_tok,
                    int n_workers = 0, ResidualScaling mode = ResidualScaling::AsPrinted);
  long long search_invocations() const { return invocations_; }
  size_t size() const { return entries_.size(); }
  void save(const std::string& path) const;
  void load(const std::string& path);

 private:
  std::map<std::tuple<std::string, std::string, long long>, TuneResult> entries_;
  long long invocations_ = 0;
};

// --------------------------------------------------------------- task list (sim.hpp:16-85, a9)
// The MegaKernel's linearised task space of one rank: [comm | relay | comp] for Dispatch+GroupGEMM
// (the reference's claim order; the device kernels claim the same order from one cursor). comm_slices
// are contiguous ranges of the rank's send schedule, balanced by NVLink transmissions (the first
// (token, dst rank) item of the priority order; a replica whose row a relay copy covers is free);
// relay_ranges are even ranges of the up-GEMM tiles (rowgroups of b_m rows x ceil(2F / b_n) columns).
// The discrete-event simulator of sim.hpp (run_*_sim) is not part of this build: the kernels are.
enum class Role { Comm, Relay, Comp, Reduce };
const char* role_name(Role r);
struct TaskQueueInfo {
  long long n_comm = 0, n_relay = 0, n_comp = 0, n_reduce = 0;
  std::vector<std::pair<long long, long long>> comm_slices;    // send item ranges
  std::vector<std::pair<long long, long long>> relay_ranges;   // tile ranges
  std::vector<std::pair<long long, long long>> reduce_ranges;  // token ranges
  long long total() const { return n_comm + n_relay + n_comp + n_reduce; }
};
TaskQueueInfo build_task_list(const MoEShape& shape, const TuneConfig& cfg, const RoutingInstance& routing,
                              int rank);

}  // namespace eplab
#pragma GCC visibility pop
