// Cross-user pieces of one outer step: the impact reduction (solver.py:206)
// and the scalar epilogue (objective, gradient norm, best iterate, stopping
// rule; solver.py:207-223).  Both are latency kernels; they are ordered on
// the solver's stream right after the fused per-user step kernel.
#include "nsw_step.cuh"

namespace nsw {

__global__ void __launch_bounds__(128) impact_reduce_kernel(const double* __restrict__ partial, int U, int n,
                                                            int chunks, double* __restrict__ split,
                                                            double* __restrict__ imp_local,
                                                            unsigned int* counter,
                                                            const int* __restrict__ state) {
  const int phase = state[ST_PHASE];
  if (phase != PHASE_INIT && phase != PHASE_RUNNING && phase != PHASE_RESUME) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int u0 = int((long long)y * U / chunks), u1 = int((long long)(y + 1) * U / chunks);
  if (i < n) {
    double acc = 0.0;
    for (int u = u0; u < u1; ++u) acc += partial[size_t(u) * n + i];
    split[size_t(y) * n + i] = acc;
  }
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < chunks; ++c) acc += __ldcg(split + size_t(c) * n + j);
    imp_local[j] = acc;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

__global__ void __launch_bounds__(512) finalize_kernel(FinalizeArgs f) {
  constexpr int NT = 512;
  __shared__ double sF[NT];
  __shared__ double sG[NT];
  __shared__ int sBad;
  const int tid = threadIdx.x;
  const int phase = f.state[ST_PHASE];
  if (phase == PHASE_FINISHED) return;
  if (phase == PHASE_DONE_PENDING) {
    if (tid == 0) f.state[ST_PHASE] = PHASE_FINISHED;
    return;
  }
  if (tid == 0) sBad = 0;
  __syncthreads();
  double accF = 0.0, accG = 0.0;
  int bad = 0;
  for (int i = tid; i < f.n; i += NT) {
    double imp = 0.0;
    for (int g = 0; g < f.world; ++g) imp += f.imp_all[size_t(g) * f.n + i];
    f.imp_cur[i] = imp;
    if (!(imp > 0.0) || !isfinite(imp)) bad = 1;
    accF += log(imp);
    accG += f.rel_sq[i] * f.exp_sq / (imp * imp);
  }
  if (bad) atomicOr(&sBad, 1);
  sF[tid] = accF;
  sG[tid] = accG;
  __syncthreads();
  for (int w = NT / 2; w > 0; w >>= 1) {
    if (tid < w) {
      sF[tid] += sF[tid + w];
      sG[tid] += sG[tid + w];
    }
    __syncthreads();
  }
  if (tid != 0) return;
  const int k = f.state[ST_STEP];
  if (sBad) {  // DomainError (solver.py:207-208): stop before recording the step
    f.state[ST_ERR] |= ERR_IMPACT;
    f.state[ST_PHASE] = PHASE_FINISHED;
    return;
  }
  const double F = sF[0];
  const double gn = sqrt(sG[0]);
  f.objective[k] = F;
  f.grad_norm[k] = gn;
  f.stamp[k + 1] = globaltimer_ns();
  const int improved = F >= *f.best;  // ties go to the later step (solver.py:217)
  if (improved) *f.best = F;
  const int k1 = k + 1;
  f.state[ST_STEP] = k1;
  f.state[ST_IMPROVED] = improved;
  f.state[ST_PHASE] = (gn <= f.grad_threshold || k1 >= f.outer_max) ? PHASE_DONE_PENDING : PHASE_RUNNING;
}

__global__ void stamp_kernel(unsigned long long* stamp) { stamp[0] = globaltimer_ns(); }

__global__ void flush_kernel(float* buf, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    buf[i] = buf[i] * 0.5f + 1.0f;
}

}  // namespace nsw
