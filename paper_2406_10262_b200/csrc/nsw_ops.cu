// Inner operator seam: the reference's private batch functions as device
// operators with its log-domain inputs and outputs (fixed schedule, ranking
// marginals of sinkhorn.py:55-60):
//   nsw_sinkhorn_batch_*          <- _sinkhorn_batch(..., tol<=0, record=True)   (sinkhorn.py:204-255)
//   nsw_sinkhorn_backward_batch_* <- _sinkhorn_backward_batch                    (sinkhorn.py:258-309)
// One CTA per batch element; the absorbed kernel K~ (and the adjoint G) live
// in shared memory.  These are the seam for callers that drive the Sinkhorn
// layer themselves; the solver's hot path is the fused step kernel.
#include <cuda_runtime.h>

#include <string>

#include "../../include/nswrank_b200.h"
#include "nsw_device.cuh"

namespace nsw {
namespace {

constexpr int OP_NT = 256;

template <typename S, int M>
__device__ __forceinline__ S dotrow(const S* row, const S (&y)[M]) {
  S s0 = S(0), s1 = S(0);
#pragma unroll
  for (int k = 0; k + 1 < M; k += 2) {
    s0 = fma(row[k], y[k], s0);
    s1 = fma(row[k + 1], y[k + 1], s1);
  }
  if constexpr (M % 2) s0 = fma(row[M - 1], y[M - 1], s0);
  return s0 + s1;
}

template <typename S>
__device__ __forceinline__ S colmass(int k, int n, int m) {
  return k == m - 1 ? S(n - m + 1) : S(1);
}

// Absorb beta = lvi, alpha_i = -max_k (K_ik + beta_k): K~ = exp(K + beta + alpha).
template <typename S, int M>
__device__ void absorb(const S* __restrict__ K, const S* __restrict__ lvi, int n, int m, S* Kt, S* alpha) {
  constexpr int P = Pitch<S, M>::value;
  for (int i = threadIdx.x; i < n; i += OP_NT) {
    S mx = Fp<S>::ninf();
    for (int k = 0; k < m; ++k) mx = fmax(mx, K[size_t(i) * m + k] + lvi[k]);
    alpha[i] = -mx;
    for (int k = 0; k < P; ++k) Kt[i * P + k] = k < m ? Fp<S>::exp_((K[size_t(i) * m + k] + lvi[k]) - mx) : S(0);
  }
}

template <typename S, int M>
__global__ void __launch_bounds__(OP_NT) sinkhorn_fwd_op(const S* __restrict__ log_kernel, const S* __restrict__ lvi_all,
                                                       int B, int n, int m, int T, S* __restrict__ plan,
                                                       S* __restrict__ log_u, S* __restrict__ log_v,
                                                       S* __restrict__ hist) {
  constexpr int P = Pitch<S, M>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* vv = reinterpret_cast<S*>(smem_raw);   // [P]   (16-byte aligned vectors first)
  S* red = vv + P;                          // [NW][P]
  S* Kt = red + (OP_NT / 32) * P;           // [n][P]
  S* alpha = Kt + size_t(n) * P;            // [n]
  S* ut = alpha + n;                        // [n]
  const int b = blockIdx.x;
  const S* K = log_kernel + size_t(b) * n * m;
  const S* lvi = lvi_all + size_t(b) * m;
  absorb<S, M>(K, lvi, n, m, Kt, alpha);
  if (threadIdx.x < P) vv[threadIdx.x] = threadIdx.x < m ? S(1) : S(0);
  __syncthreads();
  for (int t = 1; t <= T; ++t) {
    S v[M], c[M];
    lds_vec<S, M>(v, vv);
#pragma unroll
    for (int k = 0; k < M; ++k) c[k] = S(0);
    for (int i = threadIdx.x; i < n; i += OP_NT) {
      const S* row = Kt + size_t(i) * P;
      const S u = Fp<S>::rcp(dotrow<S, M>(row, v));
      ut[i] = u;
#pragma unroll
      for (int k = 0; k < M; ++k) c[k] = fma(row[k], u, c[k]);
    }
    cta_reduce_cols<S, M, OP_NT, OpSum>(c, red, m, [&](int k, S tot) {
      const S vn = Fp<S>::div(colmass<S>(k, n, m), tot);
      vv[k] = vn;
      hist[(size_t(t - 1) * B + b) * m + k] = lvi[k] + Fp<S>::log_(vn);   // v^t
    });
  }
  for (int i = threadIdx.x; i < n; i += OP_NT) {
    log_u[size_t(b) * n + i] = alpha[i] + Fp<S>::log_(ut[i]);
    for (int k = 0; k < m; ++k) plan[(size_t(b) * n + i) * m + k] = (Kt[i * P + k] * ut[i]) * vv[k];
  }
  if (threadIdx.x < m) log_v[size_t(b) * m + threadIdx.x] = lvi[threadIdx.x] + Fp<S>::log_(vv[threadIdx.x]);
}

template <typename S, int M>
__global__ void __launch_bounds__(OP_NT) sinkhorn_bwd_op(const S* __restrict__ log_kernel,
                                                       const S* __restrict__ hist_all,
                                                       const S* __restrict__ lvi_all,
                                                       const S* __restrict__ grad_plan,
                                                       const S* __restrict__ plan, const S* __restrict__ log_u_T,
                                                       int B, int n, int m, int T, S* __restrict__ grad_kernel) {
  constexpr int P = Pitch<S, M>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* cvs = reinterpret_cast<S*>(smem_raw);  // [P]   (16-byte aligned vectors first)
  S* red = cvs + P;                         // [NW][P]
  S* Kt = red + (OP_NT / 32) * P;           // [n][P]
  S* G = Kt + size_t(n) * P;                // [n][P]
  S* vh = G + size_t(n) * P;                // [T+1][P]  v~^t
  S* alpha = vh + size_t(T + 1) * P;        // [n]
  S* ut = alpha + n;                        // [n]
  S* gu = ut + n;                           // [n]
  const int b = blockIdx.x;
  const S* K = log_kernel + size_t(b) * n * m;
  const S* lvi = lvi_all + size_t(b) * m;
  const S* gp = grad_plan + size_t(b) * n * m;
  const S* X = plan + size_t(b) * n * m;
  absorb<S, M>(K, lvi, n, m, Kt, alpha);
  for (int idx = threadIdx.x; idx < (T + 1) * P; idx += OP_NT) {
    const int t = idx / P, k = idx - t * P;
    S v = S(0);
    if (k < m) v = t == 0 ? S(1) : Fp<S>::exp_(hist_all[(size_t(t - 1) * B + b) * m + k] - lvi[k]);
    vh[idx] = v;
  }
  __syncthreads();
  // seed W = grad_plan * plan (sinkhorn.py:272-275); u~^T from log_u_final
  S c[M];
#pragma unroll
  for (int k = 0; k < M; ++k) c[k] = S(0);
  for (int i = threadIdx.x; i < n; i += OP_NT) {
    ut[i] = Fp<S>::exp_(log_u_T[size_t(b) * n + i] - alpha[i]);
    S s = S(0);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      G[i * P + k] = S(0);
      if (k < m) {
        const S w = gp[size_t(i) * m + k] * X[size_t(i) * m + k];
        s += w;
        c[k] += w;
      }
    }
    gu[i] = s;
  }
  cta_reduce_cols<S, M, OP_NT, OpSum>(c, red, m, [&](int k, S tot) {
    cvs[k] = vh[size_t(T) * P + k] * tot / colmass<S>(k, n, m);
  });
  for (int t = T; t >= 1; --t) {
    S cv[M], vp[M], vpp[M];
    lds_vec<S, M>(cv, cvs);
    lds_vec<S, M>(vp, vh + size_t(t - 1) * P);
    lds_vec<S, M>(vpp, vh + size_t(t >= 2 ? t - 2 : 0) * P);
#pragma unroll
    for (int k = 0; k < M; ++k) c[k] = S(0);
    for (int i = threadIdx.x; i < n; i += OP_NT) {
      const S* row = Kt + size_t(i) * P;
      S* g = G + size_t(i) * P;
      const S u = ut[i];
      const S gg = (t == T ? gu[i] : S(0)) - u * dotrow<S, M>(row, cv);   // column VJP
      const S h = u * gg;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        g[k] = g[k] - u * cv[k] - h * vp[k];   // both softmax VJPs into gK
        c[k] = fma(row[k], h, c[k]);
      }
      if (t >= 2) ut[i] = Fp<S>::rcp(dotrow<S, M>(row, vpp));   // replay u~^{t-1}
    }
    if (t >= 2) {
      cta_reduce_cols<S, M, OP_NT, OpSum>(c, red, m, [&](int k, S tot) {
        const S vpk = vh[size_t(t - 1) * P + k];
        cvs[k] = vpk * (-(vpk * tot)) / colmass<S>(k, n, m);
      });
    }
  }
  for (int i = threadIdx.x; i < n; i += OP_NT)
    for (int k = 0; k < m; ++k) {
      const size_t o = size_t(i) * m + k;
      grad_kernel[size_t(b) * n * m + o] = fma(Kt[i * P + k], G[i * P + k], gp[o] * X[o]);
    }
}

thread_local std::string g_op_err;

template <typename S, int M>
nsw_status launch_fwd(const S* K, const S* lvi, int B, int n, int m, int T, S* plan, S* lu, S* lv, S* hist,
                      cudaStream_t st) {
  constexpr int P = Pitch<S, M>::value;
  const size_t smem = sizeof(S) * (size_t(n) * P + 2 * size_t(n) + (OP_NT / 32) * P + P);
  if (smem > 227 * 1024) return NSW_ERR_UNSUPPORTED;
  auto fn = sinkhorn_fwd_op<S, M>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return NSW_ERR_CUDA;
  fn<<<B, OP_NT, smem, st>>>(K, lvi, B, n, m, T, plan, lu, lv, hist);
  return cudaGetLastError() == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}

template <typename S, int M>
nsw_status launch_bwd(const S* K, const S* hist, const S* lvi, const S* gp, const S* X, const S* lu, int B, int n,
                      int m, int T, S* gk, cudaStream_t st) {
  constexpr int P = Pitch<S, M>::value;
  const size_t smem =
      sizeof(S) * (2 * size_t(n) * P + size_t(T + 1) * P + 3 * size_t(n) + (OP_NT / 32) * P + P);
  if (smem > 227 * 1024) return NSW_ERR_UNSUPPORTED;
  auto fn = sinkhorn_bwd_op<S, M>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return NSW_ERR_CUDA;
  fn<<<B, OP_NT, smem, st>>>(K, hist, lvi, gp, X, lu, B, n, m, T, gk);
  return cudaGetLastError() == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}

template <typename S>
nsw_status dispatch_fwd(const S* K, const S* lvi, int B, int n, int m, int T, S* plan, S* lu, S* lv, S* hist,
                        void* stream) {
  if (!K || !lvi || !plan || !lu || !lv || !hist || B <= 0 || T <= 0) return NSW_ERR_ARG;
  if (m < 2 || m > n) return NSW_ERR_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  if (m <= 4) return launch_fwd<S, 4>(K, lvi, B, n, m, T, plan, lu, lv, hist, st);
  if (m <= 8) return launch_fwd<S, 8>(K, lvi, B, n, m, T, plan, lu, lv, hist, st);
  if (m <= 11) return launch_fwd<S, 11>(K, lvi, B, n, m, T, plan, lu, lv, hist, st);
  if (m <= 16) return launch_fwd<S, 16>(K, lvi, B, n, m, T, plan, lu, lv, hist, st);
  if (m <= 21) return launch_fwd<S, 21>(K, lvi, B, n, m, T, plan, lu, lv, hist, st);
  if (m <= 32) return launch_fwd<S, 32>(K, lvi, B, n, m, T, plan, lu, lv, hist, st);
  return NSW_ERR_UNSUPPORTED;
}

template <typename S>
nsw_status dispatch_bwd(const S* K, const S* hist, const S* lvi, const S* gp, const S* X, const S* lu, int B, int n,
                        int m, int T, S* gk, void* stream) {
  if (!K || !hist || !lvi || !gp || !X || !lu || !gk || B <= 0 || T <= 0) return NSW_ERR_ARG;
  if (m < 2 || m > n) return NSW_ERR_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  if (m <= 4) return launch_bwd<S, 4>(K, hist, lvi, gp, X, lu, B, n, m, T, gk, st);
  if (m <= 8) return launch_bwd<S, 8>(K, hist, lvi, gp, X, lu, B, n, m, T, gk, st);
  if (m <= 11) return launch_bwd<S, 11>(K, hist, lvi, gp, X, lu, B, n, m, T, gk, st);
  if (m <= 16) return launch_bwd<S, 16>(K, hist, lvi, gp, X, lu, B, n, m, T, gk, st);
  if (m <= 21) return launch_bwd<S, 21>(K, hist, lvi, gp, X, lu, B, n, m, T, gk, st);
  if (m <= 32) return launch_bwd<S, 32>(K, hist, lvi, gp, X, lu, B, n, m, T, gk, st);
  return NSW_ERR_UNSUPPORTED;
}

}  // namespace
}  // namespace nsw

extern "C" {

nsw_status nsw_sinkhorn_batch_f64(const double* log_kernel, const double* log_v_init, int32_t B, int32_t n, int32_t m,
                                  int32_t iters, double* plan, double* log_u, double* log_v, double* log_v_hist,
                                  void* stream) {
  return nsw::dispatch_fwd<double>(log_kernel, log_v_init, B, n, m, iters, plan, log_u, log_v, log_v_hist, stream);
}

nsw_status nsw_sinkhorn_batch_f32(const float* log_kernel, const float* log_v_init, int32_t B, int32_t n, int32_t m,
                                  int32_t iters, float* plan, float* log_u, float* log_v, float* log_v_hist,
                                  void* stream) {
  return nsw::dispatch_fwd<float>(log_kernel, log_v_init, B, n, m, iters, plan, log_u, log_v, log_v_hist, stream);
}

nsw_status nsw_sinkhorn_backward_batch_f64(const double* log_kernel, const double* log_v_hist,
                                           const double* log_v_init, const double* grad_plan, const double* plan,
                                           const double* log_u_final, int32_t B, int32_t n, int32_t m, int32_t iters,
                                           double* grad_log_kernel, void* stream) {
  return nsw::dispatch_bwd<double>(log_kernel, log_v_hist, log_v_init, grad_plan, plan, log_u_final, B, n, m, iters,
                                   grad_log_kernel, stream);
}

nsw_status nsw_sinkhorn_backward_batch_f32(const float* log_kernel, const float* log_v_hist, const float* log_v_init,
                                           const float* grad_plan, const float* plan, const float* log_u_final,
                                           int32_t B, int32_t n, int32_t m, int32_t iters, float* grad_log_kernel,
                                           void* stream) {
  return nsw::dispatch_bwd<float>(log_kernel, log_v_hist, log_v_init, grad_plan, plan, log_u_final, B, n, m, iters,
                                  grad_log_kernel, stream);
}

}  // extern "C"
