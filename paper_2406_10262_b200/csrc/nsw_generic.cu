// Streaming fused step (any n, m): instantiations and launchers.
#include "nsw_generic.h"
#include "nsw_step_generic.cuh"

#include <algorithm>

namespace nsw {

size_t gen_scratch_elems(int n, int m) { return GenScratch<float>::elems(n, m); }

int gen_ctas(int dtype, int U) {
  int per_sm = 1;
  const void* fn = dtype == 1 ? (const void*)&step_kernel_gen<double> : (const void*)&step_kernel_gen<float>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, GEN_NT, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  per_sm = std::min(per_sm, 4);
  return std::max(1, std::min(U, sm_count() * per_sm));
}

cudaError_t gen_launch(const StepArgs<float>& a, float* scratch, int ctas, cudaStream_t st) {
  step_kernel_gen<float><<<ctas, GEN_NT, 0, st>>>(a, GenScratch<float>{scratch, a.n, a.m});
  return cudaGetLastError();
}

cudaError_t gen_launch(const StepArgs<double>& a, double* scratch, int ctas, cudaStream_t st) {
  step_kernel_gen<double><<<ctas, GEN_NT, 0, st>>>(a, GenScratch<double>{scratch, a.n, a.m});
  return cudaGetLastError();
}

}  // namespace nsw
