/*
 * eplab_b200.h -- C-ABI of libeplab_b200.so, the B200-native (sm_100a) data path
 * for the expert-parallel MoE layer of arXiv 2604.19241 (Dispatch+GroupGEMM and
 * GroupGEMM+Combine MegaKernels, forward and backward).
 *
 * The reference (`/root/reference/proj`, namespace `eplab`) is a CPU lab whose
 * data-path entry points are addressing / control-flow / numerics models:
 *   dispatch   ~ build_global_token_map / build_send_schedule  (token_map.hpp:68, :88)
 *                + run_dispatch_gemm_sim                        (sim.hpp:87)
 *   group_gemm ~ the simulators' compute tasks, tile time/count (perf_model.hpp:40, :57-58)
 *   combine    ~ run_gemm_combine_sim (sim.hpp:88) + k-ordered fold `accumulate`
 *                (precision.hpp:30)
 * Each export below names the reference interface it replaces. Conventions:
 *   - plain pointers and sizes only; device pointers are marked `d_`;
 *   - return 0 ok, 1 internal/CUDA error, 2 validation error, 3 deadlock/timeout
 *     (the reference CLI's exit codes, tools/main.cpp:503-511); the message of the
 *     last failure is available from eplab_last_error();
 *   - every device call is ordered on the caller's stream (`stream` is a
 *     cudaStream_t) and performs no host synchronisation unless stated.
 */
#ifndef EPLAB_B200_H_
#define EPLAB_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define EPLAB_API __attribute__((visibility("default")))
#else
#define EPLAB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum { EPLAB_OK = 0, EPLAB_ERR_INTERNAL = 1, EPLAB_ERR_VALIDATION = 2, EPLAB_ERR_DEADLOCK = 3 };

/* ------------------------------------------------------------------ misc */

/* Library version string (reference: version.hpp:7 kVersion). */
EPLAB_API const char* eplab_version(void);

/* Copies the thread's last error message into buf (NUL-terminated). Returns its length. */
EPLAB_API size_t eplab_last_error(char* buf, size_t len);

/* ------------------------------------------------------- grouped GEMMs (unfused) */

/* C[m, n] = sum_k A[m, k] * B[e][n, k] for each expert segment e: rows
 * [seg_start[e], seg_start[e] + seg_rows[e]) of A (seg_start multiples of 128, host arrays).
 * bf16 in, fp32 accumulate, bf16 out. The GroupGEMM compute task of the reference
 * (perf_model.cpp:16-23 tile time, :74-92 tile count) as a stand-alone op; also the
 * GEMM of the unfused NCCL baseline. d_workspace >= 32 * tiles + 4 bytes. */
EPLAB_API int eplab_grouped_gemm_nt(const void* d_A, const void* d_B, void* d_C, int M_total,
                                    int N, int K, int n_experts, const int* seg_start,
                                    const int* seg_rows, void* d_workspace, void* stream);

/* Transposed GroupGEMM (weight-gradient shape):
 * C[e][i, j] = sum_{m in seg e} A[m, i] * B[m, j]; padded segment rows must be zero. */
EPLAB_API int eplab_grouped_gemm_tn(const void* d_A, const void* d_B, void* d_C, int M_total,
                                    int NA, int NB, int n_experts, const int* seg_start,
                                    const int* seg_rows_padded, void* d_workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EPLAB_B200_H_ */
