// A reference-style C++ caller: compiles against include/eplab/eplab.hpp -- the
// same names as the reference's headers (types.hpp, routing.hpp, token_map.hpp, perf_model.hpp,
// tuner.hpp) -- and links libeplab_b200.so. Prints one JSON line the CPU test checks against the
// C-ABI and the oracle. Host-only calls: runs without a GPU.
#include <cstdio>

#include "eplab/eplab.hpp"

int main() {
  eplab::MoEShape shape;
  shape.name = "qwen3";
  shape.h_dim = 2048;
  shape.h_inter = 768;
  shape.n_exp = 128;
  shape.topk = 8;
  shape.n_tok = 1024;
  const int world = 8;
  const eplab::RoutingInstance r = eplab::sample_routing(shape, world, 7);
  const std::vector<eplab::GlobalTokenMap> maps = eplab::build_global_token_map(r);
  const eplab::SendSchedule sched = eplab::build_send_schedule(maps[3]);
  long long off_sum = 0;
  for (const auto& m : maps)
    for (const auto& e : m.entries) off_sum += e.offset;
  const eplab::HardwareSpec hw = eplab::b200_hardware(world);
  eplab::MoEShape big = shape;
  big.n_tok = 16384;
  const eplab::TuneResult t = eplab::search_layer(hw, big);
  bool threw = false;
  try {
    eplab::validate_tune_config(eplab::TuneConfig{140, 10, 1, 148, 8}, hw);
  } catch (const eplab::ValidationError&) {
    threw = true;
  }
  std::printf("{\"sel0\": %d, \"gw0\": %.9g, \"off_sum\": %lld, \"sched3_first_token\": %lld, "
              "\"n_disp\": %d, \"n_relay\": %d, \"validation_error\": %s}\n",
              r.selected_experts[0][0], (double)r.gate_weights[0][0], off_sum,
              (long long)sched.items.at(0).token, t.best.n_disp, t.best.n_relay, threw ? "true" : "false");
  return 0;
}
