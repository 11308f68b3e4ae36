// Probe: does TMA tile::gather4 (4 rows x 128 B per instruction, 128B swizzle) land rows in shared
// memory in exactly the layout a tile-mode load of the same rows (in the same order) produces?
// Loads a 128-row x 64-col bf16 box both ways (tile mode from a pre-permuted copy; gather4 from
// the source with a row permutation) and compares the raw shared-memory bytes. Also times
// gather4 issue throughput (32 lanes issuing one gather4 each per stage).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_19241_b200/csrc tools/gather4_probe.cu -lcuda
#include <cstdio>
#include <vector>
#include "kernels/ptx.cuh"
#include "kernels/tma_host.hpp"

using namespace eplab_dev;

__device__ __forceinline__ void gather4(const CUtensorMap* m, uint64_t* bar, void* smem, int c0, int4 r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w)
      : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap src_g, const __grid_constant__ CUtensorMap perm_t,
                      const int* perm, int* mismatch, int col0) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  const int lane = threadIdx.x;
  if (lane == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  __syncwarp();
  if (lane == 0) {
    mbar_arrive_expect_tx(&bar[0], 16384);
    tma_load_2d(&perm_t, &bar[0], sm, col0, 0);
    mbar_arrive_expect_tx(&bar[1], 16384);
  }
  __syncwarp();
  const int4 r = reinterpret_cast<const int4*>(perm)[lane];
  gather4(&src_g, &bar[1], sm + 16384 + lane * 512, col0, r);
  mbar_wait(&bar[0], 0);
  mbar_wait(&bar[1], 0);
  int bad = 0;
  for (int i = lane; i < 16384 / 4; i += 32)
    bad += reinterpret_cast<const int*>(sm)[i] != reinterpret_cast<const int*>(sm + 16384)[i];
  atomicAdd(mismatch, bad);
}

// throughput: ITER stages of 128x64 gathered by the 32 lanes of warp 0 (one gather4 each),
// 4-stage ring, consumer = nobody (stage reused after its barrier completes)
template <int NST, int TILE, int WARPS = 1>
__global__ void thru(const __grid_constant__ CUtensorMap src_g, const __grid_constant__ CUtensorMap src_t,
                     const int* perm, int iters, int nrows) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[NST];
  const int lane = threadIdx.x;
  if (lane == 0) { for (int i = 0; i < NST; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    const int s = it % NST;
    if (it >= NST) mbar_wait(&bar[s], ((it / NST) - 1) & 1);
    if (lane == 0) mbar_arrive_expect_tx(&bar[s], 16384);
    if (WARPS > 1) __syncthreads(); else __syncwarp();
    const int base = ((blockIdx.x * 977 + it * 128) % (nrows / 128)) * 128;
    if (TILE) {
      if (lane == 0) tma_load_2d(&src_t, &bar[s], sm + s * 16384, (it % 32) * 64, base);
    } else {
      if (WARPS == 0) {  // one thread issues all 32
        if (lane == 0)
          for (int q = 0; q < 32; ++q)
            gather4(&src_g, &bar[s], sm + s * 16384 + q * 512, (it % 32) * 64,
                    reinterpret_cast<const int4*>(perm + base)[q]);
      } else {
        const int per = 32 / (WARPS > 1 ? WARPS : 1), w = lane >> 5, l = lane & 31;
        if (l < per) {
          const int q = w * per + l;
          const int4 r = reinterpret_cast<const int4*>(perm + base)[q];
          gather4(&src_g, &bar[s], sm + s * 16384 + q * 512, (it % 32) * 64, r);
        }
      }
    }
  }
  for (int i = iters - NST; i < iters; ++i) mbar_wait(&bar[i % NST], (i / NST) & 1);
}

int main() {
  const int rows = 65536, cols = 2048;
  std::vector<uint16_t> h((size_t)rows * cols);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
  std::vector<int> perm(rows);
  for (int i = 0; i < rows; ++i) perm[i] = (int)(((long long)i * 7919 + 13) % rows);
  std::vector<uint16_t> hp((size_t)128 * cols);
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < cols; ++c) hp[(size_t)r * cols + c] = h[(size_t)perm[r] * cols + c];
  uint16_t *d, *dp;
  int *dperm, *mis;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&dp, hp.size() * 2);
  cudaMalloc(&dperm, rows * 4);
  cudaMalloc(&mis, 4);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, hp.data(), hp.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dperm, perm.data(), rows * 4, cudaMemcpyHostToDevice);
  cudaMemset(mis, 0, 4);
  CUtensorMap g = eplab_host::make_bf16_map(d, rows, cols, cols, 64, 1);
  CUtensorMap t = eplab_host::make_bf16_map(dp, 128, cols, cols, 64, 128);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int c0 : {0, 64, 1984}) {
    cudaMemset(mis, 0, 4);
    probe<<<1, 32, 40000>>>(g, t, dperm, mis, c0);
    int m = -1;
    cudaMemcpy(&m, mis, 4, cudaMemcpyDeviceToHost);
    printf("gather4 vs tile layout, col0=%d: %d mismatching words of 4096 (%s)\n", c0, m,
           cudaGetErrorString(cudaGetLastError()));
  }
  CUtensorMap tt = eplab_host::make_bf16_map(d, rows, cols, cols, 64, 128);
  auto run = [&](auto kern, const char* name, int grid, int bs = 32) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    const int iters = 4096;
    kern<<<grid, bs, 200000>>>(g, tt, dperm, 64, rows);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, bs, 200000>>>(g, tt, dperm, iters, rows);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-16s grid %3d: %.1f ns per 16 KB stage per CTA, %.1f GB/s per CTA, %.0f GB/s total (%s)\n", name, grid,
           ms * 1e6 / iters, 16384.0 * iters / (ms * 1e6), 16384.0 * iters * grid / (ms * 1e6),
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int grid : {1, 148}) {
    run(thru<8, 0>, "gather4 8st", grid);
    run(thru<8, 0, 0>, "g4 1thread", grid);
    run(thru<8, 0, 4>, "g4 4warps", grid, 128);
    run(thru<8, 0, 8>, "g4 8warps", grid, 256);
    run(thru<4, 1>, "tile 4st", grid);
    run(thru<11, 1>, "tile 11st", grid);
  }
  return 0;
}
