// Micro-benchmark of row copies through the TMA bulk-copy engine (the comm role's data mover):
// global row -> smem slot (cp.async.bulk + mbarrier) -> global row (cp.async.bulk bulk_group).
//   variant 0: one issuing thread, wait_group<NSLOT-L-1> before every slot reuse (the kernel's way)
//   variant 1: one issuing thread, stores waited only at the end (no per-item wait_group)
//   variant 2: ISS issuing warps (lane 0 each), each owning NSLOT/ISS slots
//   variant 3: warp copies (8 warps, 8 x 16 B in flight per lane)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_19241_b200/csrc tools/bulk_copy_probe.cu
#include <cstdio>
#include <vector>

#include "kernels/ptx.cuh"

using namespace eplab_dev;

template <int NSLOT, int ISS>
__global__ void __launch_bounds__(256, 1) probe(const int4* src, int4* dst, const int* perm, int rows,
                                                int row_bytes, int variant) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[NSLOT];
  const int per = (rows + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * per, hi = min(rows, lo + per);
  const int SLOT = 196608 / NSLOT;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSLOT; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (variant == 3) {
    const int vecs = row_bytes / 16;
    for (int r = lo + warp; r < hi; r += 8) {
      const int4* s = src + (size_t)perm[r] * vecs;
      int4* d = dst + (size_t)r * vecs;
      for (int c = lane; c < vecs; c += 256) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c + u * 32 < vecs) v[u] = ld_nc_v4(s + c + u * 32);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c + u * 32 < vecs) d[c + u * 32] = v[u];
      }
    }
    return;
  }
  if (variant == 4) {  // warp copies, two rows per warp in flight (16 x 16 B per lane)
    const int vecs = row_bytes / 16;
    for (int r = lo + warp * 2; r < hi; r += 16) {
      const bool two = r + 1 < hi;
      const int4* s0 = src + (size_t)perm[r] * vecs;
      const int4* s1 = src + (size_t)perm[two ? r + 1 : r] * vecs;
      int4* d0 = dst + (size_t)r * vecs;
      int4* d1 = dst + (size_t)(two ? r + 1 : r) * vecs;
      for (int c = lane; c < vecs; c += 256) {
        int4 v[8], w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c + u * 32 < vecs) { v[u] = ld_nc_v4(s0 + c + u * 32); w[u] = ld_nc_v4(s1 + c + u * 32); }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c + u * 32 < vecs) { d0[c + u * 32] = v[u]; if (two) d1[c + u * 32] = w[u]; }
      }
    }
    return;
  }
  const int iss = variant == 2 ? ISS : 1;
  if (warp >= iss || lane != 0) return;
  constexpr int NS = NSLOT;  // slots owned by this issuer
  const int ns = NS / iss, base_slot = warp * ns, L = ns / 2;
  uint64_t par = 0;
  int nl = 0, nst = 0;
  for (int r = lo + warp; r <= hi + iss; r += iss) {
    if (r < hi) {
      const int q = nl, slot = base_slot + q % ns;
      if (q >= ns && variant != 1) {
        // completion of the store that used this slot (ns - L - 1 newer groups may be pending)
        if (ns - L - 1 >= 8) tma_store_wait<8>(); else if (ns - L - 1 >= 4) tma_store_wait<4>();
        else if (ns - L - 1 >= 2) tma_store_wait<2>(); else tma_store_wait<0>();
      }
      mbar_arrive_expect_tx(&bar[slot], row_bytes);
      bulk_load(sm + slot * SLOT, reinterpret_cast<const char*>(src) + (size_t)perm[r] * row_bytes,
                row_bytes, &bar[slot]);
      ++nl;
    }
    while (nst < nl && (nl - nst > L || r >= hi)) {
      const int slot = base_slot + nst % ns;
      const int rr = lo + warp + nst * iss;
      mbar_wait(&bar[slot], (par >> (slot - base_slot)) & 1u);
      par ^= 1ull << (slot - base_slot);
      bulk_store(reinterpret_cast<char*>(dst) + (size_t)rr * row_bytes, sm + slot * SLOT, row_bytes);
      tma_store_commit();
      ++nst;
    }
  }
  tma_store_wait<0>();
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int rows = 131072;
  for (int row_bytes : {4096, 8192, 14336}) {
    const size_t n = (size_t)rows * row_bytes;
    char *src, *dst;
    int* perm;
    cudaMalloc(&src, n);
    cudaMalloc(&dst, n);
    cudaMalloc(&perm, rows * 4);
    std::vector<int> hp(rows);
    for (int i = 0; i < rows; ++i) hp[i] = (int)(((long long)i * 7919) % (rows / 8));  // k=8 reuse
    cudaMemcpy(perm, hp.data(), rows * 4, cudaMemcpyHostToDevice);
    auto run = [&](auto kern, int grid, int variant) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      kern<<<grid, 256, 196608 + 1024>>>((int4*)src, (int4*)dst, perm, rows, row_bytes, variant);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      for (int i = 0; i < 5; ++i)
        kern<<<grid, 256, 196608 + 1024>>>((int4*)src, (int4*)dst, perm, rows, row_bytes, variant);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("row %5d B grid %3d variant %d: %7.3f ms  %6.1f GB/s total  %5.1f GB/s per CTA  (%s)\n",
             row_bytes, grid, variant, ms, n / ms / 1e6, n / ms / 1e6 / grid,
             cudaGetErrorString(cudaGetLastError()));
    };
    for (int grid : {32, 64, 148}) {
      if (row_bytes <= 4096) {
        run(probe<48, 4>, grid, 0);
        run(probe<48, 4>, grid, 1);
        run(probe<48, 4>, grid, 2);
      } else if (row_bytes <= 8192) {
        run(probe<24, 4>, grid, 0);
        run(probe<24, 4>, grid, 1);
        run(probe<24, 4>, grid, 2);
      } else {
        run(probe<12, 4>, grid, 0);
        run(probe<12, 4>, grid, 1);
        run(probe<12, 4>, grid, 2);
      }
      run(probe<12, 4>, grid, 3);
      run(probe<12, 4>, grid, 4);
    }
    cudaFree(src);
    cudaFree(dst);
    cudaFree(perm);
  }
  return 0;
}
