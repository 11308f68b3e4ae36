// Declarations of the device launchers (implemented in kernels/*.cu).
#pragma once
#include <cuda_runtime.h>

#include "kernels/moe_common.cuh"

namespace eplab_launch {
int preload_megakernels();
int preload_plan();
int plan_launch(const eplab_dev::Dims& d, const eplab_dev::Peers& peers,
                const eplab_dev::PlanDev& p, uint32_t* epoch, uint64_t timeout_ns, int* err,
                __nv_bfloat16* recv_x, __nv_bfloat16* recv_dy, cudaStream_t st);
int epoch_advance_launch(uint32_t* epoch, cudaStream_t st);
int plan_counts_launch(const eplab_dev::Dims& d, const eplab_dev::PlanDev& p, uint32_t* epoch, int* out,
                       cudaStream_t st);
int plan_layout_ext_launch(const eplab_dev::Dims& d, const eplab_dev::PlanDev& p, const int* call, int* err,
                           __nv_bfloat16* recv_x, __nv_bfloat16* recv_dy, cudaStream_t st);
int unfused_pack_launch(const eplab_dev::Dims& d, const eplab_dev::PlanDev& p, const __nv_bfloat16* src,
                        __nv_bfloat16* send, int2* send_meta, int* spos, int sms, cudaStream_t st);
int unfused_scatter_launch(const eplab_dev::Dims& d, const eplab_dev::PlanDev& p, const int* call,
                           const __nv_bfloat16* recv, const int2* recv_meta, int n_recv, __nv_bfloat16* dst,
                           eplab_dev::SlotMeta* meta, int* ret_pos, int sms, cudaStream_t st);
int unfused_fold_launch(const eplab_dev::Dims& d, const eplab_dev::PlanDev& p, const __nv_bfloat16* rows,
                        const int* spos, __nv_bfloat16* out, int ph, int sms, cudaStream_t st);
int unfused_dgate_launch(const eplab_dev::Dims& d, const eplab_dev::PlanDev& p, const float* parts,
                         const int* spos, float* dgate, int sms, cudaStream_t st);
int launch_fwd_dispatch(const eplab_dev::TmaSet& tm, const eplab_dev::MkArgs& a, int grid,
                        cudaStream_t st);
int launch_fwd_combine(const eplab_dev::TmaSet& tm, const eplab_dev::MkArgs& a, int grid,
                       cudaStream_t st);
int launch_bwd_dispatch(const eplab_dev::TmaSet& tm, const eplab_dev::MkArgs& a, int grid,
                        cudaStream_t st);
int launch_bwd_combine(const eplab_dev::TmaSet& tm, const eplab_dev::MkArgs& a, int grid,
                       cudaStream_t st);
}  // namespace eplab_launch
