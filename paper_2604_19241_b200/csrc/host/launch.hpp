// Declarations of the device launchers (implemented in kernels/*.cu).
#pragma once
#include <cuda_runtime.h>

#include "kernels/moe_common.cuh"

namespace eplab_launch {
int preload_megakernels();
int preload_plan();
int plan_launch(const eplab_dev::Dims& d, const eplab_dev::Peers& peers,
                const eplab_dev::PlanDev& p, uint32_t* epoch, uint64_t timeout_ns, int* err,
                cudaStream_t st);
int zero_padding_launch(const eplab_dev::Dims& d, const eplab_dev::PlanDev& p,
                        __nv_bfloat16* recv, cudaStream_t st);
int launch_fwd_dispatch(const eplab_dev::TmaSet& tm, const eplab_dev::MkArgs& a, int grid,
                        cudaStream_t st);
int launch_fwd_combine(const eplab_dev::TmaSet& tm, const eplab_dev::MkArgs& a, int grid,
                       cudaStream_t st);
int launch_bwd_dispatch(const eplab_dev::TmaSet& tm, const eplab_dev::MkArgs& a, int grid,
                        cudaStream_t st);
int launch_bwd_combine(const eplab_dev::TmaSet& tm, const eplab_dev::MkArgs& a, int grid,
                       cudaStream_t st);
}  // namespace eplab_launch
