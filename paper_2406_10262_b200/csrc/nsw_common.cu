// Cross-user pieces of one outer step: the impact reduction (solver.py:206),
// the tolerance-mode stopping test (sinkhorn.py:244) and the scalar epilogue
// (objective, gradient norm, best iterate, stopping rule; solver.py:200-223).
// All are latency kernels ordered on the solver's stream after the fused
// per-user step kernel.
#include "nsw_step_kernel.cuh"

namespace nsw {

// The forward whose impact terms are ready: the fused launch in the fixed
// schedule, the finish launch (PHASE_FWD_FIN) in tolerance mode.
__device__ __forceinline__ bool forward_ready(int phase, int tol_mode) {
  return tol_mode ? phase == PHASE_FWD_FIN
                  : (phase == PHASE_INIT || phase == PHASE_RUNNING || phase == PHASE_RESUME);
}

template <int NTH>
__device__ void finalize_body(const FinalizeArgs& f, double* sF, double* sG, int& sBad, int& sConv);

// Two-level, fixed-order reduction.  Level 1: CTA (x, y) sums items
// [8x, 8x+8) over user chunk y (thread t: item t % IMP_ITEMS, user lane
// t / IMP_ITEMS, then a fixed shared-memory tree) into split[y][i].  Level
// 2: the last CTA to finish sums the chunks in chunk order.
__global__ void __launch_bounds__(IMP_THREADS) impact_reduce_kernel(const double* __restrict__ partial, int U,
                                                                    int n, int chunks, double* __restrict__ split,
                                                                    unsigned int* counter,
                                                                    double* __restrict__ imp_local,
                                                                    const int* __restrict__ state, int tol_mode,
                                                                    const double* __restrict__ res, int T,
                                                                    double tol, int fuse_finalize, FinalizeArgs fin) {
  const int phase0 = state[ST_PHASE];
  if (!forward_ready(phase0, tol_mode)) {
    // single shard: the step's finalize is fused here, including the
    // DONE_PENDING -> FINISHED transition of a launch with no forward
    if (fuse_finalize && phase0 == PHASE_DONE_PENDING && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
      fin.state[ST_PHASE] = PHASE_FINISHED;
    return;
  }
  constexpr int LANES = IMP_THREADS / IMP_ITEMS;
  __shared__ double red[IMP_THREADS];
  __shared__ bool last;
  const int j = threadIdx.x % IMP_ITEMS;
  const int l = threadIdx.x / IMP_ITEMS;
  const int i = blockIdx.x * IMP_ITEMS + j;
  const int y = blockIdx.y;
  const int ub = int((long long)y * U / chunks), ue = int((long long)(y + 1) * U / chunks);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (i < n) {
    int u = ub + l;
    for (; u + 3 * LANES < ue; u += 4 * LANES) {
      a0 += partial[size_t(u) * n + i];
      a1 += partial[size_t(u + LANES) * n + i];
      a2 += partial[size_t(u + 2 * LANES) * n + i];
      a3 += partial[size_t(u + 3 * LANES) * n + i];
    }
    for (; u < ue; u += LANES) a0 += partial[size_t(u) * n + i];
  }
  red[threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  for (int w = LANES / 2; w > 0; w >>= 1) {
    if (l < w) red[threadIdx.x] += red[threadIdx.x + w * IMP_ITEMS];
    __syncthreads();
  }
  if (l == 0 && i < n) split[size_t(y) * n + i] = red[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int ii = threadIdx.x; ii < n; ii += IMP_THREADS) {
    double acc = 0.0;
    for (int c = 0; c < chunks; ++c) acc += __ldcg(split + size_t(c) * n + ii);
    imp_local[ii] = acc;
  }
  // converged = residual <= tol at the final iteration t* (sinkhorn.py:253)
  int cnt = 0;
  if (tol_mode) {
    const int tstar = state[ST_TSTAR];
    for (int u = threadIdx.x; u < U; u += IMP_THREADS) cnt += res[size_t(u) * (T + 1) + tstar] <= tol;
  }
  __shared__ int sc;
  if (threadIdx.x == 0) sc = 0;
  __syncthreads();
  if (cnt) atomicAdd(&sc, cnt);
  __syncthreads();
  if (threadIdx.x == 0) {
    imp_local[n] = double(sc);
    *counter = 0u;
  }
  if (fuse_finalize) {
    __shared__ double sF[512];
    __shared__ double sG[512];
    __shared__ int sBad, sConv;
    __threadfence_block();
    __syncthreads();
    finalize_body<IMP_THREADS>(fin, sF, sG, sBad, sConv);
  }
}

__global__ void __launch_bounds__(256) tol_chunk_max_kernel(const double* __restrict__ res, int U, int T,
                                                            int chunk, const int* state, double* __restrict__ cmax) {
  const int phase = state[ST_PHASE];
  if (!(phase == PHASE_INIT || phase == PHASE_RUNNING || phase == PHASE_RESUME || phase == PHASE_FWD_CONT)) return;
  __shared__ double red[256];
  const int t0 = state[ST_T0];
  const int t1 = min(t0 + chunk, T);
  for (int j = 0; j < chunk; ++j) {
    const int t = t0 + 1 + j;
    double mx = 0.0;
    if (t <= t1)
      for (int u = threadIdx.x; u < U; u += blockDim.x) mx = fmax(mx, res[size_t(u) * (T + 1) + t]);
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) cmax[j] = red[0];
    __syncthreads();
  }
}

// cond (nonzero): the while-conditional of the single-shard tolerance graph,
// set to "another forward chunk follows" in every path
__global__ void tol_decide_kernel(const double* __restrict__ cmax, int T, int chunk, double tol, int* state,
                                  unsigned long long cond) {
  if (threadIdx.x != 0) return;
  const int phase = state[ST_PHASE];
  if (!(phase == PHASE_INIT || phase == PHASE_RUNNING || phase == PHASE_RESUME || phase == PHASE_FWD_CONT)) {
    if (cond) cudaGraphSetConditional(cond, 0u);
    return;
  }
  const int t0 = state[ST_T0];
  const int t1 = min(t0 + chunk, T);
  int tstar = 0;
  for (int t = t0 + 1; t <= t1; ++t)
    if (cmax[t - t0 - 1] <= tol) {   // residual.max() <= tol (sinkhorn.py:244)
      tstar = t;
      break;
    }
  if (tstar > 0 || t1 == T) {
    state[ST_TSTAR] = tstar > 0 ? tstar : T;
    state[ST_PHASE] = PHASE_FWD_FIN;
  } else {
    state[ST_T0] = t1;
    state[ST_PHASE] = PHASE_FWD_CONT;
  }
  if (cond) cudaGraphSetConditional(cond, state[ST_PHASE] == PHASE_FWD_CONT ? 1u : 0u);
}

// Objective, gradient norm, trace, best iterate, stop and error decisions
// from the (gathered) impacts.  The sums run over 512 virtual lanes in a fixed
// tree whatever the block size (NTH threads take 512 / NTH lanes each), so
// the standalone kernel and the copy fused into the impact reduction give
// bitwise-identical results.
template <int NTH>
__device__ void finalize_body(const FinalizeArgs& f, double* sF, double* sG, int& sBad, int& sConv) {
  constexpr int NT = 512;
  static_assert(NT % NTH == 0, "virtual lanes");
  const int tid = threadIdx.x;
  if (tid == 0) {
    sBad = 0;
    sConv = 0;
  }
  __syncthreads();
  const int tstar = f.tol_mode ? f.state[ST_TSTAR] : f.T;
  if (f.tol_mode && tid == 0) {
    // converged users over all ranks (each rank's count rides in slot n of
    // its exchanged impact vector)
    double c = 0.0;
    for (int g = 0; g < f.world; ++g) c += f.imp_all[size_t(g) * (f.n + 1) + f.n];
    sConv = int(c);
  }
  int bad = 0;
  for (int v = tid; v < NT; v += NTH) {
    double accF = 0.0, accG = 0.0;
    for (int i = v; i < f.n; i += NT) {
      double imp = 0.0;
      for (int g = 0; g < f.world; ++g) imp += f.imp_all[size_t(g) * (f.n + 1) + i];
      f.imp_cur[i] = imp;
      if (!(imp > 0.0) || !isfinite(imp)) bad = 1;
      accF += log(imp);
      accG += f.rel_sq[i] * f.exp_sq / (imp * imp);
    }
    sF[v] = accF;
    sG[v] = accG;
  }
  if (bad) atomicOr(&sBad, 1);
  __syncthreads();
  for (int w = NT / 2; w > 0; w >>= 1) {
    for (int v = tid; v < w; v += NTH) {
      sF[v] += sF[v + w];
      sG[v] += sG[v + w];
    }
    __syncthreads();
  }
  if (tid != 0) return;
  const int k = f.state[ST_STEP];
  if (f.tol_mode) {
    f.state[ST_CONV] = sConv;
    f.state[ST_T0] = 0;
    // SolverError if more than half the users missed the tolerance
    // (solver.py:200-205), checked before the impact (solver.py:206-208)
    if (1.0 - double(sConv) / double(f.U_total) > 0.5) {
      f.state[ST_ERR] |= ERR_SOLVER;
      f.state[ST_PHASE] = PHASE_FINISHED;
      return;
    }
  }
  if (sBad) {  // DomainError (solver.py:207-208): stop before recording the step
    f.state[ST_ERR] |= ERR_IMPACT;
    f.state[ST_PHASE] = PHASE_FINISHED;
    return;
  }
  const double F = sF[0];
  const double gn = sqrt(sG[0]);
  f.objective[k] = F;
  f.grad_norm[k] = gn;
  f.iters[k] = tstar;
  f.stamp[k + 1] = globaltimer_ns();
  const int improved = F >= *f.best;  // ties go to the later step (solver.py:217)
  if (improved) *f.best = F;
  const int k1 = k + 1;
  f.state[ST_STEP] = k1;
  f.state[ST_IMPROVED] = improved;
  f.state[ST_PHASE] = (gn <= f.grad_threshold || k1 >= f.outer_max) ? PHASE_DONE_PENDING : PHASE_RUNNING;
}


__global__ void __launch_bounds__(512) finalize_kernel(FinalizeArgs f) {
  __shared__ double sF[512];
  __shared__ double sG[512];
  __shared__ int sBad, sConv;
  const int phase = f.state[ST_PHASE];
  if (phase == PHASE_FINISHED) return;
  if (phase == PHASE_DONE_PENDING) {
    if (threadIdx.x == 0) f.state[ST_PHASE] = PHASE_FINISHED;
    return;
  }
  if (!forward_ready(phase, f.tol_mode)) return;
  finalize_body<512>(f, sF, sG, sBad, sConv);
}

__global__ void stamp_kernel(unsigned long long* stamp) { stamp[0] = globaltimer_ns(); }

__global__ void flush_kernel(float* buf, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    buf[i] = buf[i] * 0.5f + 1.0f;
}

// float64 -> float32 (round to nearest, as the host's float(x))
__global__ void narrow_kernel(const double* __restrict__ src, float* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = __double2float_rn(src[i]);
}

// bit 0: a non-finite relevance; bit 1: a value outside (0, 1]  (core.py:90-93)
__global__ void rel_check_kernel(const double* __restrict__ rel, size_t count, unsigned* __restrict__ flags) {
  unsigned f = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
    const double v = rel[i];
    if (!isfinite(v)) f |= 1u;
    else if (v <= 0.0 || v > 1.0) f |= 2u;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (f != 0 && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

// rsq_i = sum_u r_ui^2 in user order with separate multiply / add roundings
// (the closed-form gradient norm's item weights, solver.py:211)
__global__ void rel_sq_kernel(const double* __restrict__ rel, int U, int n, double* __restrict__ rsq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
#pragma unroll 8
  for (int u = 0; u < U; ++u) {
    const double r = rel[size_t(u) * n + i];
    acc = __dadd_rn(acc, __dmul_rn(r, r));
  }
  rsq[i] = acc;
}

__global__ void widen_kernel(const float* __restrict__ src, double* __restrict__ dst, size_t n, unsigned* bad) {
  bool ok = true;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float x = src[i];
    ok &= isfinite(x);
    dst[i] = double(x);
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

__global__ void discard_kernel(float* buf, size_t n) {
  // one discard per 128-byte line (n floats, 128-byte aligned buffer)
  for (size_t l = blockIdx.x * size_t(blockDim.x) + threadIdx.x; l < n / 32; l += size_t(gridDim.x) * blockDim.x)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(buf + l * 32) : "memory");
}

}  // namespace nsw
