// Numerics contract of the combine (reference softfloat.cpp / precision.cpp, SURVEY.md §8(a)
// a15-a17), restated for the C++ API of this build. The device reduce role computes exactly
// round_to_bf16(accumulate(plan, FpFormat::Binary32)) per output element (tests/test_parity_gpu.py
// checks it bit for bit on the MegaKernels' own replica rows); these host functions let
// reference-style callers and the reference's own tests use the same contract.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "eplab/eplab.hpp"

namespace eplab {

namespace {

uint32_t bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return u;
}
float from_bits(uint32_t u) {
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

// splitmix64 stream (the generator every reference experiment uses, routing.cpp:15-28)
struct Stream {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double unit() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

// Synthetic replica values of the precision experiments: log-uniform magnitude in [2^-4, 2^8] with a
// random sign, rounded to the format -- wide enough that bf16 accumulation absorbs small terms.
float synth(Stream& g, FpFormat fmt) {
  const double mag = std::exp2(-4.0 + 12.0 * g.unit());
  const double sgn = (g.next() & 1) ? -1.0 : 1.0;
  return fp_round((float)(sgn * mag), fmt);
}

float fold_terms(const std::vector<ReductionTerm>& terms, FpFormat fmt) {
  if (terms.empty()) return 0.0f;
  float acc = fp_mul(terms[0].weight, terms[0].value, fmt);
  for (size_t i = 1; i < terms.size(); ++i) acc = fp_add(acc, fp_mul(terms[i].weight, terms[i].value, fmt), fmt);
  return acc;
}

void count(PrecisionReport& r, float a, float b) {
  ++r.elements;
  if (!bit_equal(a, b)) ++r.non_bitwise;
  r.max_diff = std::max(r.max_diff, std::fabs((double)a - (double)b));
}

void finish(PrecisionReport& r) { r.frac_non_bitwise = r.elements ? (double)r.non_bitwise / r.elements : 0.0; }

}  // namespace

float round_to_bf16(float x) {
  const uint32_t u = bits(x);
  if (std::isnan(x)) return from_bits((u | 0x00400000u) & 0xFFFF0000u);  // quiet NaN, payload cut
  return from_bits((u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u);      // nearest, ties to even
}
float fp_round(float x, FpFormat fmt) { return fmt == FpFormat::Bfloat16 ? round_to_bf16(x) : x; }
float fp_add(float a, float b, FpFormat fmt) { return fp_round(a + b, fmt); }
float fp_mul(float a, float b, FpFormat fmt) { return fp_round(a * b, fmt); }
bool bit_equal(float a, float b) { return bits(a) == bits(b); }

std::vector<float> accumulate(const ReductionPlan& plan, FpFormat fmt) {
  std::vector<float> out(plan.tokens.size());
  std::transform(plan.tokens.begin(), plan.tokens.end(), out.begin(),
                 [fmt](const std::vector<ReductionTerm>& t) { return fold_terms(t, fmt); });
  return out;
}

PrecisionReport fused_vs_sequential(const RoutingInstance& routing, const MoEShape& shape, const HardwareSpec& spec,
                                    const TuneConfig& cfg, std::uint64_t seed, FpFormat fmt, OrderPolicy control) {
  validate_routing(routing);
  validate_tune_config(cfg, spec);
  (void)shape;
  PrecisionReport rep;
  const int k = routing.topk;
  for (int r = 0; r < routing.world; ++r) {
    Stream values{seed ^ 0xC0FFEEULL ^ ((uint64_t)r << 17)};
    Stream arrival{(seed * 0x9E3779B97F4A7C15ULL) ^ (uint64_t)r};
    for (long long t = 0; t < routing.n_tok; ++t) {
      std::vector<ReductionTerm> canonical(k);
      for (int j = 0; j < k; ++j)
        canonical[j] = ReductionTerm{j, fp_round(routing.weight_at(r, t, j), fmt), synth(values, fmt)};
      const float a = fold_terms(canonical, fmt);  // path A: sequential, k ascending
      // path B: the replicas land in some order (expert tiles and ranks finish independently)...
      std::vector<ReductionTerm> landed = canonical;
      for (int j = k - 1; j > 0; --j) std::swap(landed[j], landed[(int)(arrival.next() % (uint64_t)(j + 1))]);
      // ...the reducer waits for all k (top-k barrier) and, unless it is the broken control,
      // folds them by slot, not by arrival -- the device reads rep[t*k + j] for j = 0..k-1
      if (control != OrderPolicy::Permuted)
        std::sort(landed.begin(), landed.end(),
                  [](const ReductionTerm& x, const ReductionTerm& y) { return x.k < y.k; });
      count(rep, a, fold_terms(landed, fmt));
    }
  }
  finish(rep);
  return rep;
}

PrecisionReport split_batch_experiment(const MoEShape& shape, std::uint64_t seed, FpFormat fmt, long long split_at) {
  const long long n = shape.n_tok;
  constexpr int kCols = 16;
  if (split_at < 0) split_at = n / 2;
  split_at = std::min(split_at, n);
  Stream g{seed ^ 0xBADC0DEULL};
  std::vector<float> v((size_t)n * kCols);
  for (auto& x : v) x = synth(g, fmt);
  auto fold_rows = [&](int c, long long lo, long long hi, float& acc) {  // left fold of rows [lo, hi)
    for (long long t = lo; t < hi; ++t) acc = t == lo ? v[(size_t)t * kCols + c] : fp_add(acc, v[(size_t)t * kCols + c], fmt);
    return hi > lo;
  };
  PrecisionReport rep;
  for (int c = 0; c < kCols; ++c) {
    float full = 0.0f, h1 = 0.0f, h2 = 0.0f;
    fold_rows(c, 0, n, full);
    const bool has1 = fold_rows(c, 0, split_at, h1), has2 = fold_rows(c, split_at, n, h2);
    count(rep, full, has1 && has2 ? fp_add(h1, h2, fmt) : (has1 ? h1 : h2));
  }
  finish(rep);
  return rep;
}

}  // namespace eplab
