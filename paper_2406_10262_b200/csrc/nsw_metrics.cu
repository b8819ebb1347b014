// Policy evaluation metrics on the device (reference metrics.py:16-69):
//   user_utility     = sum_{u,i,k<m-1} r_ui e_k x_uik / |U|
//   mean_max_envy    = mean_i ( max_j cross_ij - cross_ii ),
//                      cross = R^T A, A_uj = sum_{k<m-1} x_ujk e_k
//   items_better_off = mean_i [ Imp_i > (1 + th) Imp^unif_i ]
//   items_worse_off  = mean_i [ Imp_i < (1 - th) Imp^unif_i ]
// Everything is accumulated in float64 in a fixed order (deterministic).
// The one dense product (cross, n x n x |U|) is a plain cuBLAS DGEMM; the
// allocation masses, impacts and row maxima are kernels here.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "../../include/nswrank_b200.h"
#include "nsw_device.cuh"

namespace nsw {
namespace {

__global__ void widen_to_f64(const float* __restrict__ src, double* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = double(src[i]);
}

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

// envy_i = max_j cross(i, j) - cross(i, i); cross column-major (n x n)
__global__ void envy_kernel(const double* __restrict__ cross, int n, double* __restrict__ envy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double mx = -INFINITY;
  for (int j = 0; j < n; ++j) mx = fmax(mx, cross[size_t(j) * n + i]);
  envy[i] = mx - cross[size_t(i) * n + i];
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

// cuBLAS is loaded on first use (dlopen), so the solver library does not pull
// it in at import time; only the envy product of the metrics needs it.
struct Cublas {
  using create_t = cublasStatus_t (*)(cublasHandle_t*);
  using stream_t = cublasStatus_t (*)(cublasHandle_t, cudaStream_t);
  using dgemm_t = cublasStatus_t (*)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                                     const double*, const double*, int, const double*, int, const double*, double*,
                                     int);
  create_t create = nullptr;
  stream_t set_stream = nullptr;
  dgemm_t dgemm = nullptr;
  bool ok = false;
  Cublas() {
    void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libcublas.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    create = reinterpret_cast<create_t>(dlsym(h, "cublasCreate_v2"));
    set_stream = reinterpret_cast<stream_t>(dlsym(h, "cublasSetStream_v2"));
    dgemm = reinterpret_cast<dgemm_t>(dlsym(h, "cublasDgemm_v2"));
    ok = create && set_stream && dgemm;
  }
};

const Cublas& cublas() {
  static const Cublas c;
  return c;
}

// one cuBLAS handle per host thread and device (creating one costs ms)
cublasHandle_t cublas_handle() {
  thread_local cublasHandle_t handles[64] = {};
  int dev = 0;
  if (!cublas().ok || cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!handles[dev] && cublas().create(&handles[dev]) != CUBLAS_STATUS_SUCCESS) handles[dev] = nullptr;
  return handles[dev];
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
  double* buf = nullptr;   // e[m] | A[U n] | cross[n n] | imp[n] | unif[n] | envy[n] | out[4] | pa, pb [chunks n]
  const size_t words = size_t(m) + cells + size_t(n) * n + 3 * size_t(n) + 4 + 2 * size_t(chunks) * n;
  {
    // keep the pool's memory between calls (large transient buffers)
    int dev = 0;
    cudaMemPool_t pool;
    uint64_t keep = ~uint64_t(0);
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (cudaMallocAsync((void**)&buf, words * sizeof(double), st) != cudaSuccess) return NSW_ERR_CUDA;
  double* e = buf;
  double* A = e + m;
  double* cross = A + cells;
  double* imp = cross + size_t(n) * n;
  double* unif = imp + n;
  double* envy = unif + n;
  double* out = envy + n;
  double* pa = out + 4;
  double* pb = pa + size_t(chunks) * n;
  double esum = 0.0;
  for (int k = 0; k < m - 1; ++k) esum += expo_host[k];
  nsw_status status = NSW_OK;
  cublasHandle_t h = nullptr;
  const double one = 1.0, zero = 0.0;
  if (cudaMemcpyAsync(e, expo_host, size_t(m - 1) * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess) {
    status = NSW_ERR_CUDA;
  } else {
    alloc_kernel<S><<<sm_count() * 8, 256, 0, st>>>(static_cast<const S*>(X), e, U, n, m, A);
    impact_partial_kernel<S><<<dim3((n + 127) / 128, chunks), 128, 0, st>>>(static_cast<const S*>(rel), A, U, n,
                                                                             chunks, pa, pb);
    impact_combine_kernel<<<(n + 127) / 128, 128, 0, st>>>(pa, pb, n, chunks, esum / n, imp, unif);
    // cross(i, j) = sum_u r_ui A_uj: column-major n x n = R' A with R, A
    // read as column-major n x U matrices (their row-major [U][n] layout)
    double* Rd = nullptr;
    if constexpr (sizeof(S) == 8) {
      Rd = const_cast<double*>(static_cast<const double*>(rel));
    } else {
      // widen R for DGEMM (float64 products, as the reference's numpy matmul)
      if (cudaMallocAsync((void**)&Rd, cells * sizeof(double), st) != cudaSuccess) status = NSW_ERR_CUDA;
      else widen_to_f64<<<sm_count() * 8, 256, 0, st>>>(static_cast<const float*>(rel), Rd, cells);
    }
    if (status == NSW_OK && (h = cublas_handle()) == nullptr) status = NSW_ERR_CUDA;
    if (status == NSW_OK && cublas().set_stream(h, st) != CUBLAS_STATUS_SUCCESS) status = NSW_ERR_CUDA;
    if (status == NSW_OK && cublas().dgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, n, n, U, &one, Rd, n, A, n, &zero, cross,
                                           n) != CUBLAS_STATUS_SUCCESS)
      status = NSW_ERR_CUDA;
    if (status == NSW_OK) {
      envy_kernel<<<(n + 127) / 128, 128, 0, st>>>(cross, n, envy);
      metrics_finish_kernel<<<1, 256, 0, st>>>(imp, unif, envy, n, U, threshold, out);
      if (cudaGetLastError() != cudaSuccess ||
          cudaMemcpyAsync(out_host, out, 4 * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
        status = NSW_ERR_CUDA;
    }
    if constexpr (sizeof(S) == 4) {
      if (Rd) cudaFreeAsync(Rd, st);
    }
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
  if (cudaMallocAsync((void**)&buf, words * sizeof(double), st) != cudaSuccess) return NSW_ERR_CUDA;
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
  if (cudaMallocAsync((void**)&buf, (size_t(m) + n) * sizeof(double), st) != cudaSuccess) return NSW_ERR_CUDA;
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
