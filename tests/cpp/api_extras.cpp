// Reference API surface not covered by the five reference test files compiled in
// tests/test_reference_suite.py (test_core.cpp needs the reference's config loader): the calls a
// reference-style caller makes, against this library, with the reference's documented results.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
#include "eplab/precision.hpp"
#include "eplab/routing.hpp"
#include "eplab/token_map.hpp"
#include "eplab/traffic.hpp"
#include "eplab/types.hpp"

using namespace eplab;

TEST_CASE("derive_expanded_tokens: balanced routing, n_tok * topk (types.hpp:79)") {
  MoEShape s;
  s.n_tok = 4096;
  s.topk = 8;
  CHECK(derive_expanded_tokens(s, 8) == 32768);
  s.n_tok = 3072;
  s.topk = 2;
  CHECK(derive_expanded_tokens(s, 8) == 6144);
}

TEST_CASE("TrafficReport::basis tells expected from exact volumes (traffic.hpp:44)") {
  MoEShape s;
  s.name = "m";
  s.h_dim = 1024;
  s.h_inter = 1024;
  s.n_exp = 16;
  s.topk = 4;
  s.n_tok = 64;
  HardwareSpec h;
  h.world_size = 4;
  CHECK(volume_expected(s, h).basis == TrafficReport::Basis::Expected);
  const RoutingInstance r = sample_routing(s, 4, 7);
  CHECK(volume_exact(r, s, h).basis == TrafficReport::Basis::ExactInstance);
}

TEST_CASE("BigInt stirling2 beyond 128 bits: S(64, 32) decimal digits") {
  const BigInt v = stirling2(64, 32);
  CHECK(v > BigInt("340282366920938463463374607431768211455"));  // > 2^128 - 1
  CHECK(stirling2(10, 3) == 9330);
  CHECK(stirling2(10, 3).str() == "9330");
}

TEST_CASE("accumulate(Binary32) is the device fold: w0*v0 then + wj*vj, each rounded to fp32") {
  ReductionPlan p;
  p.tokens.push_back({{0, 0.3f, 1.5f}, {1, 0.7f, -2.25f}, {2, 0.1f, 1e-3f}});
  float acc = 0.3f * 1.5f;
  acc = acc + 0.7f * -2.25f;
  acc = acc + 0.1f * 1e-3f;
  CHECK(bit_equal(accumulate(p, FpFormat::Binary32)[0], acc));
  CHECK(bit_equal(round_to_bf16(1.00390625f), 1.0f));  // tie -> even
}
