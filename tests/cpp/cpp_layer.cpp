// GPU half of the C++ boundary test: a reference-style caller runs one EP=1 layer step through
// include/eplab/device.hpp (build_global_token_map, dispatch_group_gemm, group_gemm_combine and
// the _bwd twins) twice, checks the two runs are bitwise identical, and writes inputs + outputs
// to argv[1] for the pytest to compare against the oracle.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "eplab/device.hpp"

static uint16_t bf16(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}
static std::vector<uint16_t> fill(size_t n, uint64_t seed, float scale) {
  std::vector<uint16_t> v(n);
  for (size_t i = 0; i < n; ++i) {
    seed = seed * 6364136223846793005ULL + 1442695040888963407ULL;
    const float u = (float)((seed >> 40) & 0xFFFFFF) / 16777216.0f - 0.5f;
    v[i] = bf16(u * 3.4641f * scale);  // uniform, unit variance before scaling
  }
  return v;
}
template <class T>
static T* to_dev(const std::vector<T>& h) {
  T* d = nullptr;
  cudaMalloc(&d, h.size() * sizeof(T));
  cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return d;
}
template <class T>
static std::vector<T> to_host(const T* d, size_t n) {
  std::vector<T> h(n);
  cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost);
  return h;
}

int main(int argc, char** argv) {
  const int E = 8, k = 2, H = 256, F = 256, T = 192;
  eplab::MoEShape shape;
  shape.h_dim = H;
  shape.h_inter = F;
  shape.n_exp = E;
  shape.topk = k;
  shape.n_tok = T;
  const eplab::RoutingInstance r = eplab::sample_routing(shape, 1, 3);
  const std::vector<int32_t> sel(r.selected_experts[0].begin(), r.selected_experts[0].end());
  const std::vector<float> gw = r.gate_weights[0];
  const auto x = fill((size_t)T * H, 1, 1.0f), dy = fill((size_t)T * H, 2, 0.5f);
  const auto w_up = fill((size_t)E * 2 * F * H, 3, 1.0f / 16), w_down = fill((size_t)E * H * F, 4, 1.0f / 16);
  int32_t* d_sel = to_dev(sel);
  float* d_gw = to_dev(gw);
  uint16_t *d_x = to_dev(x), *d_dy = to_dev(dy), *d_wu = to_dev(w_up), *d_wd = to_dev(w_down);
  uint16_t *d_y, *d_dx, *d_dwu, *d_dwd;
  float* d_dg;
  cudaMalloc(&d_y, (size_t)T * H * 2);
  cudaMalloc(&d_dx, (size_t)T * H * 2);
  cudaMalloc(&d_dwu, w_up.size() * 2);
  cudaMalloc(&d_dwd, w_down.size() * 2);
  cudaMalloc(&d_dg, (size_t)T * k * 4);

  eplab::Context::Options o;
  o.max_tokens = T;
  o.hidden = H;
  o.ffn = F;
  o.n_experts = E;
  o.topk = k;
  eplab::Context ctx(o);
  std::vector<std::vector<uint16_t>> runs;
  for (int rep = 0; rep < 2; ++rep) {
    eplab::build_global_token_map(ctx, d_sel, d_gw, T);
    eplab::dispatch_group_gemm(ctx, d_x, d_wu);
    eplab::group_gemm_combine(ctx, d_wd, d_y);
    eplab::dispatch_group_gemm_bwd(ctx, d_dy, d_wd, d_dwd, d_dg);
    eplab::group_gemm_combine_bwd(ctx, d_wu, d_dx, d_dwu);
    ctx.check();
    std::vector<uint16_t> all = to_host(d_y, (size_t)T * H);
    for (auto* p : {d_dx, d_dwu, d_dwd}) {
      const size_t n = p == d_dx ? (size_t)T * H : (p == d_dwu ? w_up.size() : w_down.size());
      const auto h = to_host(p, n);
      all.insert(all.end(), h.begin(), h.end());
    }
    runs.push_back(all);
  }
  const bool same = runs[0] == runs[1];
  bool threw = false;
  try {
    eplab::build_global_token_map(ctx, d_sel, d_gw, T + 1);  // more tokens than max_tokens
  } catch (const eplab::ValidationError&) {
    threw = true;
  }
  FILE* f = std::fopen(argv[1], "wb");
  std::fwrite(sel.data(), 4, sel.size(), f);
  std::fwrite(gw.data(), 4, gw.size(), f);
  for (const auto* v : {&x, &dy, &w_up, &w_down}) std::fwrite(v->data(), 2, v->size(), f);
  const auto y = to_host(d_y, (size_t)T * H), dx = to_host(d_dx, (size_t)T * H);
  const auto dg = to_host(d_dg, (size_t)T * k);
  const auto dwu = to_host(d_dwu, w_up.size()), dwd = to_host(d_dwd, w_down.size());
  std::fwrite(y.data(), 2, y.size(), f);
  std::fwrite(dx.data(), 2, dx.size(), f);
  std::fwrite(dg.data(), 4, dg.size(), f);
  std::fwrite(dwu.data(), 2, dwu.size(), f);
  std::fwrite(dwd.data(), 2, dwd.size(), f);
  std::fclose(f);
  std::printf("{\"bitwise_repeat\": %s, \"validation_error\": %s}\n", same ? "true" : "false",
              threw ? "true" : "false");
  return 0;
}
