// Plain grouped GEMMs on the tcgen05 engine (no fused collective):
//   eplab_grouped_gemm_nt : C[m, n] = sum_k A[m, k] * B[e][n, k]   (both K-major; forward shape)
//   eplab_grouped_gemm_tn : C[e][i, j] = sum_m A[m, i] * B[m, j]   (both MN-major; the transposed
//                           GroupGEMM of the weight gradient)
// These are the building blocks of the unfused baseline and the engine's
// own numerics tests; the MegaKernels reuse the same engine with fused roles.
#include <cuda_runtime.h>

#include <vector>

#include "gemm_engine.cuh"
#include "gemm_pair.cuh"
#include "tma_host.hpp"
#include "eplab_b200.h"

namespace eplab_dev {

struct ModeNT {
  static constexpr bool HAS_TILE_DONE = false;
  __device__ static int a_mn(const TileDesc&) { return 0; }
  __device__ static int b_mn(const TileDesc&) { return 0; }
  template <class A> __device__ static void tile_done(const A&, const TileDesc&) {}
  struct Args {
    const TileDesc* tiles;
    __nv_bfloat16* C;
    int ldc;
    int n_per_expert;  // rows of B per expert
  };
  __device__ static TileDesc tile(const Args& a, int t) { return a.tiles[t]; }
  __device__ static void before_loads(const Args&, const TileDesc&) {}
  __device__ static void epilogue_prefetch(const Args&, const TileDesc&, int) {}
  __device__ static void load_a(const Args&, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    tma_load_2d(&tm.m[0], bar, s, kb * BK, td.m0);
  }
  __device__ static void load_b(const Args& a, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
    tma_load_2d(&tm.m[1], bar, s, kb * BK, td.e * a.n_per_expert + td.n0);
  }
  __device__ static void epilogue(const Args& a, const TmaSet&, const TileDesc& td, uint32_t taddr, int r,
                                  uint8_t*) {
    __nv_bfloat16* row = a.C + (size_t)(td.m0 + r) * a.ldc + td.n0;
    const bool live = r < td.rows;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float v[32];
      acc_chunk(taddr, c, v);
      if (live) store_row_bf16_32(row + c * 32, v);
    }
  }
};

struct ModeTN {
  static constexpr bool HAS_TILE_DONE = false;
  __device__ static int a_mn(const TileDesc&) { return 1; }
  __device__ static int b_mn(const TileDesc&) { return 1; }
  template <class A> __device__ static void tile_done(const A&, const TileDesc&) {}
  struct Args {
    const TileDesc* tiles;
    __nv_bfloat16* C;  // [E][rows_out][ldc]
    int ldc;
    long long expert_stride;
  };
  __device__ static TileDesc tile(const Args& a, int t) { return a.tiles[t]; }
  __device__ static void before_loads(const Args&, const TileDesc&) {}
  __device__ static void epilogue_prefetch(const Args&, const TileDesc&, int) {}
  __device__ static void load_a(const Args&, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
#pragma unroll
    for (int i = 0; i < BM / 64; ++i)
      tma_load_2d(&tm.m[0], bar, s + i * 8192, td.m0 + 64 * i, td.kb0 + kb * BK);
  }
  __device__ static void load_b(const Args&, const TmaSet& tm, uint64_t* bar, uint8_t* s,
                                const TileDesc& td, int kb) {
#pragma unroll
    for (int i = 0; i < BN / 64; ++i)
      tma_load_2d(&tm.m[1], bar, s + i * 8192, td.n0 + 64 * i, td.kb0 + kb * BK);
  }
  __device__ static void epilogue(const Args& a, const TmaSet&, const TileDesc& td, uint32_t taddr, int r,
                                  uint8_t*) {
    __nv_bfloat16* row = a.C + td.e * a.expert_stride + (size_t)(td.m0 + r) * a.ldc + td.n0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float v[32];
      if (td.nkb > 0) {
        acc_chunk(taddr, c, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      store_row_bf16_32(row + c * 32, v);
    }
  }
};

template <class Mode>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    plain_gemm_kernel(const __grid_constant__ TmaSet tm, const typename Mode::Args args,
                      int ntiles, int* cursor) {
  extern __shared__ uint8_t raw_smem[];
  uint8_t* base = smem_aligned(raw_smem);
  GemmSmem* S = reinterpret_cast<GemmSmem*>(base + TILES_BYTES + EPI_BYTES);
  gemm_setup(S);
  if (threadIdx.x == 0) S->bcast = atomicAdd(cursor, 1);
  __syncthreads();
  const int first = S->bcast;
  __syncthreads();
  gemm_roles<Mode>(args, tm, base, S, first, 0, ntiles, cursor, Timeline{nullptr, nullptr, 0});
  gemm_teardown(S);
}


// CTA-pair versions: tiles are 256 rows (two 128-row halves) x 256 columns.
struct ModeNTPair : ModeNT {
  __device__ static TileDesc tile_pair(const Args& a, int t) { return a.tiles[t]; }
  __device__ static void before_loads_pair(const Args&, const TileDesc&) {}
  __device__ static void load_a_pair(const Args&, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    tma_load_2d_pair(&tm.m[0], bar, s, kb * BK, td.m0 + 128 * rank);
  }
  __device__ static void load_b_pair(const Args& a, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
    tma_load_2d_pair(&tm.m[2], bar, s, kb * BK, td.e * a.n_per_expert + td.n0 + 128 * rank);
  }
  __device__ static TileDesc half_of(const TileDesc& td, uint32_t rank) {
    TileDesc h = td;
    h.m0 = td.m0 + 128 * rank;
    h.rows = max(0, min(128, td.rows - 128 * (int)rank));
    return h;
  }
  __device__ static bool half_has_work(const TileDesc& h) { return h.rows > 0; }
};

struct ModeTNPair : ModeTN {
  __device__ static TileDesc tile_pair(const Args& a, int t) { return a.tiles[t]; }
  __device__ static void before_loads_pair(const Args&, const TileDesc&) {}
  __device__ static void load_a_pair(const Args&, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      tma_load_2d_pair(&tm.m[0], bar, s + i * 8192, td.m0 + 128 * rank + 64 * i, td.kb0 + kb * BK);
  }
  __device__ static void load_b_pair(const Args&, const TmaSet& tm, uint32_t bar, uint8_t* s,
                                     const TileDesc& td, int kb, uint32_t rank) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      tma_load_2d_pair(&tm.m[1], bar, s + i * 8192, td.n0 + 128 * rank + 64 * i, td.kb0 + kb * BK);
  }
  __device__ static TileDesc half_of(const TileDesc& td, uint32_t rank) {
    TileDesc h = td;
    h.m0 = td.m0 + 128 * rank;
    return h;
  }
  __device__ static bool half_has_work(const TileDesc&) { return true; }
};

template <class Mode>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    plain_gemm_pair_kernel(const __grid_constant__ TmaSet tm, const typename Mode::Args args,
                           int ntiles, int* cursor) {
  extern __shared__ uint8_t raw_smem[];
  uint8_t* base = smem_aligned(raw_smem);
  GemmSmem* S = reinterpret_cast<GemmSmem*>(base + TILES_BYTES + EPI_BYTES);
  const uint32_t rank = cluster_ctarank();
  gemm_setup_pair(S, rank);
  if (threadIdx.x == 0) {
    const int id = atomicAdd(cursor, 1);
    st_cluster_u32(mapa_shared(smem_u32(&S->pend[rank]), 0), (uint32_t)id);
  }
  cluster_sync_all();
  gemm_roles_pair<Mode>(args, tm, base, S, 0, ntiles, cursor, Timeline{nullptr, nullptr, 0}, rank);
  gemm_teardown_pair(S);
}

}  // namespace eplab_dev

using namespace eplab_dev;

namespace {
int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

template <class Mode>
int launch_plain(const TmaSet& tm, const typename Mode::Args& args, const TileDesc* d_tiles,
                 int ntiles, int* d_cursor, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(plain_gemm_kernel<Mode>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)GEMM_SMEM_BYTES);
    attr = true;
  }
  (void)d_tiles;
  cudaMemsetAsync(d_cursor, 0, sizeof(int), st);
  int grid = num_sms();
  if (grid > ntiles) grid = ntiles > 0 ? ntiles : 1;
  plain_gemm_kernel<Mode><<<grid, GEMM_THREADS, GEMM_SMEM_BYTES, st>>>(tm, args, ntiles, d_cursor);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
template <class Mode>
int launch_plain_pair(const TmaSet& tm, const typename Mode::Args& args, int ntiles, int* d_cursor,
                      cudaStream_t st) {
  static bool attr = false;
  auto fn = plain_gemm_pair_kernel<Mode>;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM_BYTES);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaMemsetAsync(d_cursor, 0, sizeof(int), st);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((num_sms() / 2) * 2);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = GEMM_SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, fn, tm, args, ntiles, d_cursor);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
}  // namespace

extern "C" {

// Grouped NT GEMM over expert segments. seg_rows[e] rows of A starting at
// seg_start[e] (multiples of 128) multiply B[e] ([N][K], K-major).
// workspace: >= 32 B * tiles + 4 B (device). Host arrays describe the groups.
int eplab_grouped_gemm_nt(const void* A, const void* B, void* C, int M_total, int N, int K,
                          int n_experts, const int* seg_start, const int* seg_rows,
                          void* d_workspace, void* stream) {
  try {
    std::vector<TileDesc> tiles;
    for (int e = 0; e < n_experts; ++e)
      for (int m = 0; m < seg_rows[e]; m += BM)
        for (int n = 0; n < N; n += BN) {
          TileDesc t{};
          t.e = e;
          t.m0 = seg_start[e] + m;
          t.n0 = n;
          t.rows = seg_rows[e] - m < BM ? seg_rows[e] - m : BM;
          t.nkb = K / BK;
          tiles.push_back(t);
        }
    cudaStream_t st = (cudaStream_t)stream;
    TileDesc* d_tiles = (TileDesc*)d_workspace;
    int* d_cursor = (int*)((char*)d_workspace + sizeof(TileDesc) * tiles.size());
    cudaMemcpyAsync(d_tiles, tiles.data(), sizeof(TileDesc) * tiles.size(),
                    cudaMemcpyHostToDevice, st);
    TmaSet tm;
    tm.m[0] = eplab_host::make_bf16_map(A, M_total, K, K, 64, BM);
    tm.m[1] = tm.m[2] = tm.m[3] = tm.m[4] = tm.m[5] = tm.m[6] = tm.m[7] = eplab_host::make_bf16_map(B, (uint64_t)n_experts * N, K, K, 64, BN);
    ModeNT::Args args{d_tiles, (__nv_bfloat16*)C, N, N};
    return launch_plain<ModeNT>(tm, args, d_tiles, (int)tiles.size(), d_cursor, st);
  } catch (...) {
    return 1;
  }
}

// Grouped TN GEMM (weight-gradient shape): C[e] ([NA][NB]) = A_seg^T * B_seg where
// A is [M_total][NA], B is [M_total][NB] and expert e owns rows
// [seg_start[e], seg_start[e] + seg_rows_padded[e]) (padded rows must be zero).
int eplab_grouped_gemm_tn(const void* A, const void* B, void* C, int M_total, int NA, int NB,
                          int n_experts, const int* seg_start, const int* seg_rows_padded,
                          void* d_workspace, void* stream) {
  try {
    std::vector<TileDesc> tiles;
    for (int e = 0; e < n_experts; ++e)
      for (int m = 0; m < NA; m += BM)
        for (int n = 0; n < NB; n += BN) {
          TileDesc t{};
          t.e = e;
          t.m0 = m;
          t.n0 = n;
          t.rows = BM;
          t.kb0 = seg_start[e];
          t.nkb = seg_rows_padded[e] / BK;
          tiles.push_back(t);
        }
    cudaStream_t st = (cudaStream_t)stream;
    TileDesc* d_tiles = (TileDesc*)d_workspace;
    int* d_cursor = (int*)((char*)d_workspace + sizeof(TileDesc) * tiles.size());
    cudaMemcpyAsync(d_tiles, tiles.data(), sizeof(TileDesc) * tiles.size(),
                    cudaMemcpyHostToDevice, st);
    TmaSet tm;
    tm.m[0] = eplab_host::make_bf16_map(A, M_total, NA, NA, 64, 64);
    tm.m[1] = tm.m[2] = tm.m[3] = tm.m[4] = tm.m[5] = tm.m[6] = tm.m[7] = eplab_host::make_bf16_map(B, M_total, NB, NB, 64, 64);
    ModeTN::Args args{d_tiles, (__nv_bfloat16*)C, NB, (long long)NA * NB};
    return launch_plain<ModeTN>(tm, args, d_tiles, (int)tiles.size(), d_cursor, st);
  } catch (...) {
    return 1;
  }
}

// CTA-pair (cta_group::2) versions of the two grouped GEMMs (same arguments).
int eplab_grouped_gemm_nt_pair(const void* A, const void* B, void* C, int M_total, int N, int K,
                               int n_experts, const int* seg_start, const int* seg_rows,
                               void* d_workspace, void* stream) {
  try {
    std::vector<TileDesc> tiles;
    for (int e = 0; e < n_experts; ++e)
      for (int m = 0; m < seg_rows[e]; m += 2 * BM)
        for (int n = 0; n < N; n += BN) {
          TileDesc t{};
          t.e = e;
          t.m0 = seg_start[e] + m;
          t.n0 = n;
          t.rows = seg_rows[e] - m < 2 * BM ? seg_rows[e] - m : 2 * BM;
          t.nkb = K / BK;
          tiles.push_back(t);
        }
    cudaStream_t st = (cudaStream_t)stream;
    TileDesc* d_tiles = (TileDesc*)d_workspace;
    int* d_cursor = (int*)((char*)d_workspace + sizeof(TileDesc) * tiles.size());
    cudaMemcpyAsync(d_tiles, tiles.data(), sizeof(TileDesc) * tiles.size(),
                    cudaMemcpyHostToDevice, st);
    TmaSet tm;
    tm.m[0] = eplab_host::make_bf16_map(A, M_total, K, K, 64, BM);
    tm.m[1] = tm.m[3] = tm.m[4] = tm.m[5] = tm.m[6] = tm.m[7] = tm.m[0];
    tm.m[2] = eplab_host::make_bf16_map(B, (uint64_t)n_experts * N, K, K, 64, 128);
    ModeNT::Args args{d_tiles, (__nv_bfloat16*)C, N, N};
    return launch_plain_pair<ModeNTPair>(tm, args, (int)tiles.size(), d_cursor, st);
  } catch (...) {
    return 1;
  }
}

int eplab_grouped_gemm_tn_pair(const void* A, const void* B, void* C, int M_total, int NA, int NB,
                               int n_experts, const int* seg_start, const int* seg_rows_padded,
                               void* d_workspace, void* stream) {
  try {
    std::vector<TileDesc> tiles;
    for (int e = 0; e < n_experts; ++e)
      for (int m = 0; m < NA; m += 2 * BM)
        for (int n = 0; n < NB; n += BN) {
          TileDesc t{};
          t.e = e;
          t.m0 = m;
          t.n0 = n;
          t.rows = 2 * BM;
          t.kb0 = seg_start[e];
          t.nkb = seg_rows_padded[e] / BK;
          tiles.push_back(t);
        }
    cudaStream_t st = (cudaStream_t)stream;
    TileDesc* d_tiles = (TileDesc*)d_workspace;
    int* d_cursor = (int*)((char*)d_workspace + sizeof(TileDesc) * tiles.size());
    cudaMemcpyAsync(d_tiles, tiles.data(), sizeof(TileDesc) * tiles.size(),
                    cudaMemcpyHostToDevice, st);
    TmaSet tm;
    tm.m[0] = eplab_host::make_bf16_map(A, M_total, NA, NA, 64, 64);
    tm.m[1] = eplab_host::make_bf16_map(B, M_total, NB, NB, 64, 64);
    tm.m[2] = tm.m[3] = tm.m[4] = tm.m[5] = tm.m[6] = tm.m[7] = tm.m[0];
    ModeTN::Args args{d_tiles, (__nv_bfloat16*)C, NB, (long long)NA * NB};
    return launch_plain_pair<ModeTNPair>(tm, args, (int)tiles.size(), d_cursor, st);
  } catch (...) {
    return 1;
  }
}

}  // extern "C"
