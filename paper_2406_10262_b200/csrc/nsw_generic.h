// Host launchers of the streaming fused step (nsw_step_generic.cuh), for the
// shapes no compiled on-chip tile holds.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "nsw_step_kernel.cuh"

namespace nsw {
constexpr int GEN_NT = 256;   // threads per CTA of the streaming step
// scratch elements (of the scalar type) per CTA
size_t gen_scratch_elems(int n, int m);
// CTAs of one launch for U users (persistent over users)
int gen_ctas(int dtype, int U);
cudaError_t gen_launch(const StepArgs<float>& a, float* scratch, int ctas, cudaStream_t st);
cudaError_t gen_launch(const StepArgs<double>& a, double* scratch, int ctas, cudaStream_t st);
}  // namespace nsw
