// Policy evaluation metrics on the device (reference metrics.py:16-69):
//   user_utility     = sum_{u,i,k<m-1} r_ui e_k x_uik / |U|
//   mean_max_envy    = mean_i ( max_j cross_ij - cross_ii ),
//                      cross = R^T A, A_uj = sum_{k<m-1} x_ujk e_k
//   items_better_off = mean_i [ Imp_i > (1 + th) Imp^unif_i ]
//   items_worse_off  = mean_i [ Imp_i < (1 - th) Imp^unif_i ]
// Everything is accumulated in float64 in a fixed order (deterministic).
// The one dense product (cross = R' A, n x n x |U|, reference metrics.py:38)
// never materialises: envy_gemm_kernel runs it on the FP64 tensor cores
// (mma.sync m8n8k4 f64, DMMA) with the row maximum and the diagonal fused
// into the epilogue, so only [n / 64][n] partial maxima reach HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "../../include/nswrank_b200.h"
#include "nsw_device.cuh"
#include "nsw_pool.h"

namespace nsw {
namespace {

// A_uj = sum_{k<m-1} x_ujk e_k  (float64), one thread per (u, j)
template <typename S>
__global__ void alloc_kernel(const S* __restrict__ X, const double* __restrict__ e, int U, int n, int m,
                             double* __restrict__ A) {
  const size_t cells = size_t(U) * n;
  for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < cells; q += size_t(gridDim.x) * blockDim.x) {
    const S* x = X + q * m;
    double acc = 0.0;
    for (int k = 0; k < m - 1; ++k) acc += double(x[k]) * e[k];
    A[q] = acc;
  }
}

// Imp_j = sum_u r_uj A_uj and Imp^unif_j = (sum_k e_k / n) sum_u r_uj in two
// fixed-order levels: chunk c of the users (grid.y) sums its users in index
// order per item (coalesced over items), then chunk partials add in chunk order
template <typename S>
__global__ void impact_partial_kernel(const S* __restrict__ rel, const double* __restrict__ A, int U, int n,
                                      int chunks, double* __restrict__ pa, double* __restrict__ pb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int c = blockIdx.y;
  const int ub = int((long long)c * U / chunks), ue = int((long long)(c + 1) * U / chunks);
  double a = 0.0, b = 0.0;
  for (int u = ub; u < ue; ++u) {
    const double r = double(rel[size_t(u) * n + j]);
    a += r * A[size_t(u) * n + j];
    b += r;
  }
  pa[size_t(c) * n + j] = a;
  pb[size_t(c) * n + j] = b;
}

__global__ void impact_combine_kernel(const double* __restrict__ pa, const double* __restrict__ pb, int n,
                                      int chunks, double e_sum_over_n, double* __restrict__ imp,
                                      double* __restrict__ imp_unif) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double a = 0.0, b = 0.0;
  for (int c = 0; c < chunks; ++c) {
    a += pa[size_t(c) * n + j];
    b += pb[size_t(c) * n + j];
  }
  imp[j] = a;
  imp_unif[j] = b * e_sum_over_n;
}

// ---------------------------------------------------------------------------
// envy_i = max_j cross(i, j) - cross(i, i),  cross(i, j) = sum_u r_ui A_uj
// (reference metrics.py:38-41), as one fused FP64 tensor-core GEMM.
// CTA: 64 x 64 output tile (4 warps, 2 x 2 warp tiles of 32 x 32 = 4 x 4 DMMA
// m8n8k4 tiles), users staged 16 at a time through shared memory (both
// operands are [U][n] row-major: coalesced 64-item rows), the next stage
// prefetched into registers during the MMAs.  Epilogue: row maxima over the
// tile's 64 columns -> part[jt][i]; diagonal tiles also write cross(i, i).
// The user sum runs in index order (fixed): deterministic.
// ---------------------------------------------------------------------------
constexpr int EG_T = 64;       // output tile edge
constexpr int EG_KS = 16;      // users per shared-memory stage
constexpr int EG_P = 72;       // padded row pitch (doubles): conflict-free fragment loads

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Split-K (few output tiles, e.g. n = 500): blockIdx.z takes users
// [z U / S, (z + 1) U / S) and writes its partial 64 x 64 tile to
// pcross[z][i][j] (pcross != nullptr); envy_splitk_combine sums the splits in
// split order, then takes the row maxima and the diagonal.
template <typename S>
__global__ void __launch_bounds__(128) envy_gemm_kernel(const S* __restrict__ rel, const double* __restrict__ A,
                                                        int U, int n, double* __restrict__ part,
                                                        double* __restrict__ diag, double* __restrict__ pcross) {
  __shared__ __align__(16) double sR[EG_KS][EG_P];   // r_ui  (k = user, i = row item)
  __shared__ __align__(16) double sA[EG_KS][EG_P];   // A_uj  (k = user, j = column item)
  __shared__ double smax[2][EG_T];
  const int it = blockIdx.y, jt = blockIdx.x;
  const int i0 = it * EG_T, j0 = jt * EG_T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = warp >> 1, wj = warp & 1;   // warp tile (rows wi*32.., columns wj*32..)
  const int g = lane >> 2, q = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // each thread stages 8 elements of each operand per stage: rows k = tid/16 + 8e, 4 items at (tid%16)*4
  const int lk = tid >> 4, li = (tid & 15) * 4;
  double pr[2][4], pa[2][4];
  auto fetch = [&](int u0) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int u = u0 + lk + 8 * e;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = i0 + li + c, j = j0 + li + c;
        pr[e][c] = (u < U && i < n) ? double(rel[size_t(u) * n + i]) : 0.0;
        pa[e][c] = (u < U && j < n) ? A[size_t(u) * n + j] : 0.0;
      }
    }
  };
  const int ub = int((long long)U * blockIdx.z / gridDim.z), ue = int((long long)U * (blockIdx.z + 1) / gridDim.z);
  U = ue;   // fetch() masks users >= U
  fetch(ub);
  for (int u0 = ub; u0 < ue; u0 += EG_KS) {
    __syncthreads();   // the previous stage's fragments are consumed
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sR[lk + 8 * e][li + c] = pr[e][c];
        sA[lk + 8 * e][li + c] = pa[e][c];
      }
    __syncthreads();
    if (u0 + EG_KS < U) fetch(u0 + EG_KS);   // next stage in flight during the MMAs
#pragma unroll
    for (int k0 = 0; k0 < EG_KS; k0 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        af[t] = sR[k0 + q][wi * 32 + t * 8 + g];   // A fragment: row g, column (user) q
        bf[t] = sA[k0 + q][wj * 32 + t * 8 + g];   // B fragment: row (user) q, column g
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_m8n8k4(acc[a][b], af[a], bf[b]);
    }
  }
  // epilogue: accumulator (a, b, c) is cross(i0 + wi*32 + a*8 + g, j0 + wj*32 + b*8 + 2q + c)
  if (pcross != nullptr) {
    double* pc = pcross + size_t(blockIdx.z) * n * n;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int i = i0 + wi * 32 + a * 8 + g, j = j0 + wj * 32 + b * 8 + 2 * q + c;
          if (i < n && j < n) pc[size_t(i) * n + j] = acc[a][b][c];
        }
    return;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int il = wi * 32 + a * 8 + g;
    double mx = -INFINITY;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int jl = wj * 32 + b * 8 + 2 * q + c;
        if (j0 + jl < n) mx = fmax(mx, acc[a][b][c]);
        if (it == jt && il == jl && i0 + il < n) diag[i0 + il] = acc[a][b][c];
      }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    if (q == 0) smax[wj][il] = mx;
  }
  __syncthreads();
  if (tid < EG_T && i0 + tid < n) part[size_t(jt) * n + i0 + tid] = fmax(smax[0][tid], smax[1][tid]);
}

__global__ void envy_splitk_combine(const double* __restrict__ pcross, int n, int splits,
                                    double* __restrict__ envy) {
  const int i = blockIdx.x;
  __shared__ double smx[128];
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double c = 0.0;
    for (int z = 0; z < splits; ++z) c += pcross[(size_t(z) * n + i) * n + j];
    mx = fmax(mx, c);
  }
  smx[threadIdx.x] = mx;
  __syncthreads();
  for (int w = 64; w > 0; w >>= 1) {
    if (threadIdx.x < w) smx[threadIdx.x] = fmax(smx[threadIdx.x], smx[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double d = 0.0;
    for (int z = 0; z < splits; ++z) d += pcross[(size_t(z) * n + i) * n + i];
    envy[i] = smx[0] - d;
  }
}

__global__ void envy_combine_kernel(const double* __restrict__ part, const double* __restrict__ diag, int n,
                                    int tiles, double* __restrict__ envy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double mx = -INFINITY;
  for (int t = 0; t < tiles; ++t) mx = fmax(mx, part[size_t(t) * n + i]);
  envy[i] = mx - diag[i];
}

// one block: the four metrics from the per-item vectors, fixed-order sums
__global__ void metrics_finish_kernel(const double* __restrict__ imp, const double* __restrict__ imp_unif,
                                      const double* __restrict__ envy, int n, int U, double th,
                                      double* __restrict__ out) {
  __shared__ double s_imp[256], s_env[256];
  __shared__ int s_b[256], s_w[256];
  double a = 0.0, c = 0.0;
  int b = 0, w = 0;
  for (int i = threadIdx.x; i < n; i += 256) {
    a += imp[i];
    c += envy[i];
    b += imp[i] > (1.0 + th) * imp_unif[i];
    w += imp[i] < (1.0 - th) * imp_unif[i];
  }
  s_imp[threadIdx.x] = a;
  s_env[threadIdx.x] = c;
  s_b[threadIdx.x] = b;
  s_w[threadIdx.x] = w;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s_imp[threadIdx.x] += s_imp[threadIdx.x + s];
      s_env[threadIdx.x] += s_env[threadIdx.x + s];
      s_b[threadIdx.x] += s_b[threadIdx.x + s];
      s_w[threadIdx.x] += s_w[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s_imp[0] / double(U);
    out[1] = s_env[0] / double(n);
    out[2] = double(s_b[0]) / double(n);
    out[3] = double(s_w[0]) / double(n);
  }
}

template <typename S>
nsw_status policy_metrics(const void* X, const void* rel, const double* expo_host, int32_t U, int32_t n,
                          int32_t m, double threshold, double* out_host, void* stream) {
  if (!X || !rel || !expo_host || !out_host) return NSW_ERR_ARG;
  if (U <= 0 || n <= 0 || m < 2 || m > n) return NSW_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t cells = size_t(U) * n;
  // user chunks of the impact sums: ~4 CTAs of 128 items per SM
  const int chunks = std::max(1, std::min(U, (sm_count() * 4 * 128 + n - 1) / n));
  const int tiles = (n + EG_T - 1) / EG_T;
  // e[m] | A[U n] | part[tiles n] | diag[n] | imp[n] | unif[n] | envy[n] | out[4] | pa, pb [chunks n]
  double* buf = nullptr;
  const size_t words = size_t(m) + cells + size_t(tiles) * n + 4 * size_t(n) + 4 + 2 * size_t(chunks) * n;
  if (private_malloc((void**)&buf, words * sizeof(double), st) != cudaSuccess) return NSW_ERR_CUDA;
  double* e = buf;
  double* A = e + m;
  double* part = A + cells;
  double* diag = part + size_t(tiles) * n;
  double* imp = diag + n;
  double* unif = imp + n;
  double* envy = unif + n;
  double* out = envy + n;
  double* pa = out + 4;
  double* pb = pa + size_t(chunks) * n;
  double esum = 0.0;
  for (int k = 0; k < m - 1; ++k) esum += expo_host[k];
  nsw_status status = NSW_OK;
  if (cudaMemcpyAsync(e, expo_host, size_t(m - 1) * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess) {
    status = NSW_ERR_CUDA;
  } else {
    alloc_kernel<S><<<sm_count() * 8, 256, 0, st>>>(static_cast<const S*>(X), e, U, n, m, A);
    impact_partial_kernel<S><<<dim3((n + 127) / 128, chunks), 128, 0, st>>>(static_cast<const S*>(rel), A, U, n,
                                                                             chunks, pa, pb);
    impact_combine_kernel<<<(n + 127) / 128, 128, 0, st>>>(pa, pb, n, chunks, esum / n, imp, unif);
    // envy: the fused FP64 tensor-core product R' A with row maxima / diagonal
    // few output tiles: split the user sum so about two CTAs per SM run
    const int splits = std::max(1, std::min((2 * sm_count() + tiles * tiles - 1) / (tiles * tiles), (U + 63) / 64));
    double* pcross = nullptr;
    if (splits > 1 && private_malloc((void**)&pcross, size_t(splits) * n * n * sizeof(double), st) != cudaSuccess)
      status = NSW_ERR_CUDA;
    if (status == NSW_OK) {
      envy_gemm_kernel<S><<<dim3(tiles, tiles, splits), 128, 0, st>>>(static_cast<const S*>(rel), A, U, n, part,
                                                                        diag, pcross);
      if (splits > 1) envy_splitk_combine<<<n, 128, 0, st>>>(pcross, n, splits, envy);
      else envy_combine_kernel<<<(n + 127) / 128, 128, 0, st>>>(part, diag, n, tiles, envy);
    }
    if (pcross) cudaFreeAsync(pcross, st);
    metrics_finish_kernel<<<1, 256, 0, st>>>(imp, unif, envy, n, U, threshold, out);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(out_host, out, 4 * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      status = NSW_ERR_CUDA;
  }
  cudaFreeAsync(buf, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) status = NSW_ERR_CUDA;
  return status;
}

// Imp only (reference solver.py:46-53): allocation masses + two-level sums
template <typename S>
nsw_status policy_impact(const void* X, const void* rel, const double* expo_host, int32_t U, int32_t n, int32_t m,
                         double* imp_host, void* stream) {
  if (!X || !rel || !expo_host || !imp_host) return NSW_ERR_ARG;
  if (U <= 0 || n <= 0 || m < 2) return NSW_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t cells = size_t(U) * n;
  const int chunks = std::max(1, std::min(U, (sm_count() * 4 * 128 + n - 1) / n));
  double* buf = nullptr;   // e[m] | A[U n] | imp[n] | unif[n] | pa, pb [chunks n]
  const size_t words = size_t(m) + cells + 2 * size_t(n) + 2 * size_t(chunks) * n;
  if (private_malloc((void**)&buf, words * sizeof(double), st) != cudaSuccess) return NSW_ERR_CUDA;
  double* e = buf;
  double* A = e + m;
  double* imp = A + cells;
  double* unif = imp + n;
  double* pa = unif + n;
  double* pb = pa + size_t(chunks) * n;
  nsw_status status = NSW_OK;
  if (cudaMemcpyAsync(e, expo_host, size_t(m - 1) * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess) {
    status = NSW_ERR_CUDA;
  } else {
    alloc_kernel<S><<<sm_count() * 8, 256, 0, st>>>(static_cast<const S*>(X), e, U, n, m, A);
    impact_partial_kernel<S><<<dim3((n + 127) / 128, chunks), 128, 0, st>>>(static_cast<const S*>(rel), A, U, n,
                                                                             chunks, pa, pb);
    impact_combine_kernel<<<(n + 127) / 128, 128, 0, st>>>(pa, pb, n, chunks, 0.0, imp, unif);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(imp_host, imp, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      status = NSW_ERR_CUDA;
  }
  cudaFreeAsync(buf, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) status = NSW_ERR_CUDA;
  return status;
}

// grad[u][i][k] = r_ui e_k / Imp_i for k < m-1, 0 at the dummy (solver.py:68-90)
template <typename S>
__global__ void welfare_gradient_kernel(const S* __restrict__ rel, const double* __restrict__ e,
                                        const double* __restrict__ imp, int U, int n, int m, S* __restrict__ grad) {
  const size_t total = size_t(U) * n * m;
  for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < total; q += size_t(gridDim.x) * blockDim.x) {
    const int k = int(q % m);
    const size_t ui = q / m;
    const int i = int(ui % n);
    grad[q] = k < m - 1 ? S((double(rel[ui]) * e[k]) / imp[i]) : S(0);
  }
}

template <typename S>
nsw_status welfare_gradient(const void* rel, const double* expo_host, const double* imp_host, int32_t U, int32_t n,
                            int32_t m, void* grad, void* stream) {
  if (!rel || !expo_host || !imp_host || !grad) return NSW_ERR_ARG;
  if (U <= 0 || n <= 0 || m < 2) return NSW_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* buf = nullptr;
  if (private_malloc((void**)&buf, (size_t(m) + n) * sizeof(double), st) != cudaSuccess) return NSW_ERR_CUDA;
  nsw_status status = NSW_OK;
  if (cudaMemcpyAsync(buf, expo_host, size_t(m - 1) * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(buf + m, imp_host, size_t(n) * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess) {
    status = NSW_ERR_CUDA;
  } else {
    welfare_gradient_kernel<S><<<sm_count() * 8, 256, 0, st>>>(static_cast<const S*>(rel), buf, buf + m, U, n, m,
                                                        static_cast<S*>(grad));
    if (cudaGetLastError() != cudaSuccess) status = NSW_ERR_CUDA;
  }
  cudaFreeAsync(buf, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) status = NSW_ERR_CUDA;
  return status;
}

// One Adam ascent step in place (solver.py:105-122), the reference's
// operation order; bias corrections bc1 = 1 - b1^step, bc2 = 1 - b2^step
// come from the host exactly as Python computes them.
// IEEE round-to-nearest operations, never contracted into FMAs (numpy order)
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double rsqrt_(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float rsqrt_(float a) { return __fsqrt_rn(a); }

template <typename S>
__global__ void adam_kernel(S* __restrict__ p, const S* __restrict__ g, S* __restrict__ m1, S* __restrict__ v1,
                            size_t count, double lr, double b1, double b2, double eps, double bc1, double bc2) {
  for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < count; q += size_t(gridDim.x) * blockDim.x) {
    const S gg = g[q];
    const S mm = radd(rmul(S(b1), m1[q]), rmul(S(1.0 - b1), gg));
    const S vv = radd(rmul(S(b2), v1[q]), rmul(rmul(S(1.0 - b2), gg), gg));
    m1[q] = mm;
    v1[q] = vv;
    const S mh = rdiv(mm, S(bc1));
    const S vh = rdiv(vv, S(bc2));
    p[q] = radd(p[q], rdiv(rmul(S(lr), mh), radd(rsqrt_(vh), S(eps))));
  }
}

}  // namespace
}  // namespace nsw

extern "C" {

nsw_status nsw_policy_impact_f32(const float* X, const float* rel, const double* expo, int32_t U, int32_t n,
                                 int32_t m, double* imp, void* stream) {
  return nsw::policy_impact<float>(X, rel, expo, U, n, m, imp, stream);
}

nsw_status nsw_policy_impact_f64(const double* X, const double* rel, const double* expo, int32_t U, int32_t n,
                                 int32_t m, double* imp, void* stream) {
  return nsw::policy_impact<double>(X, rel, expo, U, n, m, imp, stream);
}

nsw_status nsw_welfare_gradient_f32(const float* rel, const double* expo, const double* imp, int32_t U, int32_t n,
                                    int32_t m, float* grad, void* stream) {
  return nsw::welfare_gradient<float>(rel, expo, imp, U, n, m, grad, stream);
}

nsw_status nsw_welfare_gradient_f64(const double* rel, const double* expo, const double* imp, int32_t U, int32_t n,
                                    int32_t m, double* grad, void* stream) {
  return nsw::welfare_gradient<double>(rel, expo, imp, U, n, m, grad, stream);
}

nsw_status nsw_adam_update_f32(float* params, const float* grads, float* adam_m, float* adam_v, size_t count,
                               double lr, double beta1, double beta2, double eps, double bias1, double bias2,
                               void* stream) {
  if (!params || !grads || !adam_m || !adam_v) return NSW_ERR_ARG;
  nsw::adam_kernel<float><<<nsw::sm_count() * 8, 256, 0, (cudaStream_t)stream>>>(params, grads, adam_m, adam_v, count, lr, beta1,
                                                                     beta2, eps, bias1, bias2);
  return cudaGetLastError() == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}

nsw_status nsw_adam_update_f64(double* params, const double* grads, double* adam_m, double* adam_v, size_t count,
                               double lr, double beta1, double beta2, double eps, double bias1, double bias2,
                               void* stream) {
  if (!params || !grads || !adam_m || !adam_v) return NSW_ERR_ARG;
  nsw::adam_kernel<double><<<nsw::sm_count() * 8, 256, 0, (cudaStream_t)stream>>>(params, grads, adam_m, adam_v, count, lr, beta1,
                                                                      beta2, eps, bias1, bias2);
  return cudaGetLastError() == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}


nsw_status nsw_policy_metrics_f32(const float* X, const float* rel, const double* expo, int32_t U, int32_t n,
                                  int32_t m, double threshold, double* out, void* stream) {
  return nsw::policy_metrics<float>(X, rel, expo, U, n, m, threshold, out, stream);
}

nsw_status nsw_policy_metrics_f64(const double* X, const double* rel, const double* expo, int32_t U, int32_t n,
                                  int32_t m, double threshold, double* out, void* stream) {
  return nsw::policy_metrics<double>(X, rel, expo, U, n, m, threshold, out, stream);
}

}  // extern "C"
