// Cross-user pieces of one outer step: the impact reduction (solver.py:206)
// and the scalar epilogue (objective, gradient norm, best iterate, stopping
// rule; solver.py:207-223).  Both are latency kernels; they are ordered on
// the solver's stream right after the fused per-user step kernel.
#include "nsw_step_kernel.cuh"

namespace nsw {

// One CTA per IMP_ITEMS consecutive items; its 256 threads stride over the
// users (thread t: item t % IMP_ITEMS, user lane t / IMP_ITEMS), then a fixed
// shared-memory tree combines the lanes: one pass, deterministic order.
__global__ void __launch_bounds__(IMP_THREADS) impact_reduce_kernel(const double* __restrict__ partial, int U,
                                                                    int n, double* __restrict__ imp_local,
                                                                    const int* __restrict__ state) {
  const int phase = state[ST_PHASE];
  if (phase != PHASE_INIT && phase != PHASE_RUNNING && phase != PHASE_RESUME) return;
  constexpr int LANES = IMP_THREADS / IMP_ITEMS;
  __shared__ double red[IMP_THREADS];
  const int j = threadIdx.x % IMP_ITEMS;
  const int l = threadIdx.x / IMP_ITEMS;
  const int i = blockIdx.x * IMP_ITEMS + j;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (i < n) {
    int u = l;
    for (; u + 3 * LANES < U; u += 4 * LANES) {
      a0 += partial[size_t(u) * n + i];
      a1 += partial[size_t(u + LANES) * n + i];
      a2 += partial[size_t(u + 2 * LANES) * n + i];
      a3 += partial[size_t(u + 3 * LANES) * n + i];
    }
    for (; u < U; u += LANES) a0 += partial[size_t(u) * n + i];
  }
  red[threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  for (int w = LANES / 2; w > 0; w >>= 1) {
    if (l < w) red[threadIdx.x] += red[threadIdx.x + w * IMP_ITEMS];
    __syncthreads();
  }
  if (l == 0 && i < n) imp_local[i] = red[threadIdx.x];
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
