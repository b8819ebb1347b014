// Inner operator seam: the reference's batch Sinkhorn functions as device
// operators with its log-domain inputs and outputs and arbitrary positive
// marginals (the ranking marginals of sinkhorn.py:55-60 when none are given):
//   nsw_sinkhorn_solve_batch_*    <- _sinkhorn_batch(log_kernel, log_row, log_col, row, col, tol,
//                                                    max_iters, log_v_init, record)  (sinkhorn.py:204-255)
//   nsw_sinkhorn_batch_*          <- the same with the ranking marginals and tol <= 0 (fixed schedule)
//   nsw_sinkhorn_backward_batch_* <- _sinkhorn_backward_batch                       (sinkhorn.py:258-309)
//   nsw_cost_from_policy_*        <- cost_from_policy (sinkhorn.py:176-188)
// One CTA per batch element; the absorbed kernel K~ (and the adjoint G) live
// in shared memory.  The tolerance stop is lock-step over the batch
// (sinkhorn.py:244): chunks of iterations record every element's residual,
// the host finds the first iteration whose maximum is <= tol, and a finish
// launch emits the plan of that iteration from the recorded duals.  These are
// the seam for callers that drive the Sinkhorn layer themselves; the
// solver's hot path is the fused step kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/nswrank_b200.h"
#include "nsw_device.cuh"
#include "nsw_pool.h"

namespace nsw {
namespace {

constexpr int OP_NT = 256;
constexpr int OP_NW = OP_NT / 32;
constexpr int OP_CHUNK = 16;   // tolerance mode: iterations per launch

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

template <typename T>
__device__ __forceinline__ double* align8(T* p) {
  return reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + 7) & ~uintptr_t(7));
}

// Marginal masses: caller-provided (row[n], col[m]) or, when null, the
// ranking marginals (rows 1; columns 1 and the dummy n - m + 1).
template <typename S>
struct Marg {
  const S* row;
  const S* col;
  int n, m;
  __device__ S r(int i) const { return row ? row[i] : S(1); }
  __device__ S c(int k) const { return col ? col[k] : (k == m - 1 ? S(n - m + 1) : S(1)); }
  // u~ = row_i / (K~ v~)_i ; the ranking form keeps the reciprocal
  __device__ S udiv(int i, S d) const { return row ? Fp<S>::div(row[i], d) : Fp<S>::rcp(d); }
};

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

__device__ __forceinline__ double warp_maxd(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Iterations t0+1 .. t1 of every batch element.  The multiplicative form
// (SURVEY Appendix A): u~ = row / (K~ v~), v~ = col / (K~' u~); v~^t is kept
// in vt [B][T+1][m] (exact, for the next chunk and the finish launch) and
// v^t = lvi + log v~^t goes to hist [T][B][m].  With res != nullptr the L-inf
// marginal residual of X^t = diag(u~^t) K~ diag(v~^t) is recorded in
// res [B][T+1] (rows: u~^t (K~ v~^t) - row, the next iteration's own dot;
// columns: v~^t (K~' u~^t) - col).
template <typename S, int M>
__global__ void __launch_bounds__(OP_NT) fwd_chunk_op(const S* __restrict__ log_kernel, const S* __restrict__ lvi_all,
                                                     Marg<S> mg, int B, int n, int m, int T, int t0, int t1,
                                                     S* __restrict__ hist, S* __restrict__ vt,
                                                     double* __restrict__ res) {
  constexpr int P = Pitch<S, M>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  nsw_poison_smem(smem_raw);
  S* vv = reinterpret_cast<S*>(smem_raw);   // [P]   (16-byte aligned vectors first)
  S* red = vv + P;                          // [NW][P]
  S* Kt = red + OP_NW * P;                  // [n][P]
  S* alpha = Kt + size_t(n) * P;            // [n]
  S* ut = alpha + n;                        // [n]
  double* colres = align8(ut + n);                                 // [2][P]
  double* rowmax = colres + 2 * P;                                 // [NW]
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const S* K = log_kernel + size_t(b) * n * m;
  const S* lvi = lvi_all + size_t(b) * m;
  S* vtb = vt + size_t(b) * (T + 1) * m;
  absorb<S, M>(K, lvi, n, m, Kt, alpha);
  if (threadIdx.x < P) {
    const S v0 = t0 == 0 ? S(1) : vtb[size_t(t0) * m + (threadIdx.x < m ? threadIdx.x : 0)];
    vv[threadIdx.x] = threadIdx.x < m ? v0 : S(0);
    if (t0 == 0 && threadIdx.x < m) vtb[threadIdx.x] = S(1);
  }
  __syncthreads();
  for (int t = t0 + 1; t <= t1; ++t) {
    S v[M], c[M];
    lds_vec<S, M>(v, vv);
#pragma unroll
    for (int k = 0; k < M; ++k) c[k] = S(0);
    double rmax = 0.0;
    for (int i = threadIdx.x; i < n; i += OP_NT) {
      const S* row = Kt + size_t(i) * P;
      const S d = dotrow<S, M>(row, v);
      if (res && t - 1 > t0) rmax = fmax(rmax, fabs(double(ut[i] * d) - double(mg.r(i))));
      const S u = mg.udiv(i, d);
      ut[i] = u;
#pragma unroll
      for (int k = 0; k < M; ++k) c[k] = fma(row[k], u, c[k]);
    }
    if (res) {
      rmax = warp_maxd(rmax);
      if (lane == 0) rowmax[warp] = rmax;
    }
    cta_reduce_cols<S, M, OP_NT, OpSum>(c, red, m, [&](int k, S tot) {
      const S vn = Fp<S>::div(mg.c(k), tot);
      vv[k] = vn;
      vtb[size_t(t) * m + k] = vn;
      hist[(size_t(t - 1) * B + b) * m + k] = lvi[k] + Fp<S>::log_(vn);   // v^t
      if (res) {
        colres[(t & 1) * P + k] = fabs(double(vn * tot) - double(mg.c(k)));
        if (k == 0 && t - 1 > t0) {
          double r = 0.0;
          for (int w = 0; w < OP_NW; ++w) r = fmax(r, rowmax[w]);
          for (int kk = 0; kk < m; ++kk) r = fmax(r, colres[((t - 1) & 1) * P + kk]);
          res[size_t(b) * (T + 1) + t - 1] = r;
        }
      }
    });
  }
  if (res) {
    // residual of the chunk's last iteration: one more row pass
    S v[M];
    lds_vec<S, M>(v, vv);
    double rmax = 0.0;
    for (int i = threadIdx.x; i < n; i += OP_NT)
      rmax = fmax(rmax, fabs(double(ut[i] * dotrow<S, M>(Kt + size_t(i) * P, v)) - double(mg.r(i))));
    rmax = warp_maxd(rmax);
    if (lane == 0) rowmax[warp] = rmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double r = 0.0;
      for (int w = 0; w < OP_NW; ++w) r = fmax(r, rowmax[w]);
      for (int kk = 0; kk < m; ++kk) r = fmax(r, colres[(t1 & 1) * P + kk]);
      res[size_t(b) * (T + 1) + t1] = r;
    }
  }
}

// Plan, duals and final residual of iteration ts from the recorded v~:
// u~ = row / (K~ v~^{ts-1}), X = diag(u~) K~ diag(v~^ts); residual as the
// reference measures it on X (row and column sums, sinkhorn.py:237-243).
template <typename S, int M>
__global__ void __launch_bounds__(OP_NT) finish_op(const S* __restrict__ log_kernel, const S* __restrict__ lvi_all,
                                                  Marg<S> mg, int B, int n, int m, int T, int ts,
                                                  const S* __restrict__ vt, S* __restrict__ plan,
                                                  S* __restrict__ log_u, S* __restrict__ log_v,
                                                  double* __restrict__ resid) {
  constexpr int P = Pitch<S, M>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  nsw_poison_smem(smem_raw);
  S* vp = reinterpret_cast<S*>(smem_raw);   // [P] v~^{ts-1}
  S* vs = vp + P;                           // [P] v~^{ts}
  S* red = vs + P;                          // [NW][P]
  S* Kt = red + OP_NW * P;                  // [n][P]
  S* alpha = Kt + size_t(n) * P;            // [n]
  double* rowmax = align8(alpha + n);                                 // [NW]
  double* cmax = rowmax + OP_NW;                                      // [1]
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const S* K = log_kernel + size_t(b) * n * m;
  const S* lvi = lvi_all + size_t(b) * m;
  const S* vtb = vt + size_t(b) * (T + 1) * m;
  absorb<S, M>(K, lvi, n, m, Kt, alpha);
  if (threadIdx.x < P) {
    const int k = threadIdx.x < m ? threadIdx.x : 0;
    vp[threadIdx.x] = threadIdx.x < m ? vtb[size_t(ts - 1) * m + k] : S(0);
    vs[threadIdx.x] = threadIdx.x < m ? vtb[size_t(ts) * m + k] : S(0);
  }
  __syncthreads();
  S v1[M], v2[M], c[M];
  lds_vec<S, M>(v1, vp);
  lds_vec<S, M>(v2, vs);
#pragma unroll
  for (int k = 0; k < M; ++k) c[k] = S(0);
  double rmax = 0.0;
  for (int i = threadIdx.x; i < n; i += OP_NT) {
    const S* row = Kt + size_t(i) * P;
    const S u = mg.udiv(i, dotrow<S, M>(row, v1));
    log_u[size_t(b) * n + i] = alpha[i] + Fp<S>::log_(u);
    S rs = S(0);
    for (int k = 0; k < m; ++k) {
      const S x = (row[k] * u) * v2[k];
      plan[(size_t(b) * n + i) * m + k] = x;
      rs += x;
    }
#pragma unroll
    for (int k = 0; k < M; ++k) c[k] += (row[k] * u) * v2[k];
    rmax = fmax(rmax, fabs(double(rs) - double(mg.r(i))));
  }
  rmax = warp_maxd(rmax);
  if (lane == 0) rowmax[warp] = rmax;
  if (threadIdx.x == 0) *cmax = 0.0;
  cta_reduce_cols<S, M, OP_NT, OpSum>(c, red, m, [&](int k, S tot) {
    atomicMax(reinterpret_cast<unsigned long long*>(cmax),
              __double_as_longlong(fabs(double(tot) - double(mg.c(k)))));   // nonnegative doubles order as ints
  });
  if (threadIdx.x < m) log_v[size_t(b) * m + threadIdx.x] = lvi[threadIdx.x] + Fp<S>::log_(vs[threadIdx.x]);
  if (threadIdx.x == 0) {
    double r = *cmax;
    for (int w = 0; w < OP_NW; ++w) r = fmax(r, rowmax[w]);
    resid[b] = r;
  }
}

template <typename S, int M>
__global__ void __launch_bounds__(OP_NT) sinkhorn_bwd_op(const S* __restrict__ log_kernel,
                                                       const S* __restrict__ hist_all,
                                                       const S* __restrict__ lvi_all, Marg<S> mg,
                                                       const S* __restrict__ grad_plan,
                                                       const S* __restrict__ plan, const S* __restrict__ log_u_T,
                                                       int B, int n, int m, int T, S* __restrict__ grad_kernel) {
  constexpr int P = Pitch<S, M>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  nsw_poison_smem(smem_raw);
  S* cvs = reinterpret_cast<S*>(smem_raw);  // [P]   (16-byte aligned vectors first)
  S* red = cvs + P;                         // [NW][P]
  S* Kt = red + OP_NW * P;                  // [n][P]
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
  // padding columns of the column-VJP vector stay 0 (the row dots read all M
  // slots; 0 * uninitialised shared memory could be NaN -- found by the
  // checked build's NaN-poisoned shared memory)
  if (threadIdx.x < P) cvs[threadIdx.x] = S(0);
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
    cvs[k] = vh[size_t(T) * P + k] * tot / mg.c(k);
  });
  // Per level t (SURVEY Appendix A with masses): cv = v~^t g_v / col,
  // g = [t=T] g_u - u~ (K~ cv), h = u~ g / row, G -= u~ cv' + h v~^{t-1}',
  // g_v = -v~^{t-1} (K~' h), replay u~^{t-1} = row / (K~ v~^{t-2}).
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
      const S h = mg.row ? u * gg / mg.row[i] : u * gg;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        g[k] = g[k] - u * cv[k] - h * vp[k];   // both softmax VJPs into gK
        c[k] = fma(row[k], h, c[k]);
      }
      if (t >= 2) ut[i] = mg.udiv(i, dotrow<S, M>(row, vpp));   // replay u~^{t-1}
    }
    if (t >= 2) {
      cta_reduce_cols<S, M, OP_NT, OpSum>(c, red, m, [&](int k, S tot) {
        const S vpk = vh[size_t(t - 1) * P + k];
        cvs[k] = vpk * (-(vpk * tot)) / mg.c(k);
      });
    }
  }
  for (int i = threadIdx.x; i < n; i += OP_NT)
    for (int k = 0; k < m; ++k) {
      const size_t o = size_t(i) * m + k;
      grad_kernel[size_t(b) * n * m + o] = fma(Kt[i * P + k], G[i * P + k], gp[o] * X[o]);
    }
}

template <typename S>
__global__ void cost_from_policy_op(const S* __restrict__ x, size_t count, S neg_eps, S* __restrict__ out,
                                    unsigned* __restrict__ bad) {
  bool ok = true;
  for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < count; q += size_t(gridDim.x) * blockDim.x) {
    const S v = x[q];
    ok &= v > S(0);
    out[q] = neg_eps * Fp<S>::log_(v);
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

}  // namespace
}  // namespace nsw
#include "nsw_ops_generic.cuh"
namespace nsw {
namespace {

template <typename S, int M>
size_t fwd_smem(int n) {
  constexpr int P = Pitch<S, M>::value;
  return sizeof(S) * (size_t(n) * P + 2 * size_t(n) + OP_NW * P + P + 2) + 8 * (2 * P + OP_NW) + 16;
}
template <typename S, int M>
size_t fin_smem(int n) {
  constexpr int P = Pitch<S, M>::value;
  return sizeof(S) * (size_t(n) * P + size_t(n) + OP_NW * P + 2 * P + 2) + 8 * (OP_NW + 1) + 16;
}
template <typename S, int M>
size_t bwd_smem(int n, int T) {
  constexpr int P = Pitch<S, M>::value;
  return sizeof(S) * (2 * size_t(n) * P + size_t(T + 1) * P + 3 * size_t(n) + OP_NW * P + P);
}

// Forward driver: fixed schedule (tol <= 0) = one chunk of T iterations;
// tolerance = chunks of OP_CHUNK with the lock-step test on the host.
template <typename S, int M>
nsw_status run_solve(const S* K, const S* row, const S* col, const S* lvi, int B, int n, int m, int T, double tol,
                     S* plan, S* lu, S* lv, S* hist, int32_t* iters_out, int32_t* conv_out, double* resid_out,
                     cudaStream_t st) {
  const size_t sf = fwd_smem<S, M>(n), sn = fin_smem<S, M>(n);
  if (std::max(sf, sn) > 227 * 1024) return NSW_ERR_UNSUPPORTED;
  auto f1 = fwd_chunk_op<S, M>;
  auto f2 = finish_op<S, M>;
  if (allow_smem((const void*)f1, size_t(sf)) != cudaSuccess ||
      allow_smem((const void*)f2, size_t(sn)) != cudaSuccess)
    return NSW_ERR_CUDA;
  const Marg<S> mg{row, col, n, m};
  const bool tolm = tol > 0.0;
  S* vt = nullptr;
  double* res = nullptr;
  double* rd = nullptr;
  nsw_status e = NSW_OK;
  if (private_malloc((void**)&vt, size_t(B) * (T + 1) * m * sizeof(S), st) != cudaSuccess ||
      private_malloc((void**)&rd, size_t(B) * sizeof(double), st) != cudaSuccess ||
      (tolm && private_malloc((void**)&res, size_t(B) * (T + 1) * sizeof(double), st) != cudaSuccess))
    e = NSW_ERR_CUDA;
  int ts = T;
  if (e == NSW_OK) {
    if (!tolm) {
      f1<<<B, OP_NT, sf, st>>>(K, lvi, mg, B, n, m, T, 0, T, hist, vt, nullptr);
    } else {
      std::vector<double> hres(size_t(B) * (T + 1));
      for (int t0 = 0; t0 < T; t0 += OP_CHUNK) {
        const int t1 = std::min(t0 + OP_CHUNK, T);
        f1<<<B, OP_NT, sf, st>>>(K, lvi, mg, B, n, m, T, t0, t1, hist, vt, res);
        if (cudaMemcpyAsync(hres.data(), res, hres.size() * sizeof(double), cudaMemcpyDeviceToHost, st) !=
                cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
          e = NSW_ERR_CUDA;
          break;
        }
        int found = 0;
        for (int t = t0 + 1; t <= t1 && !found; ++t) {
          double mx = 0.0;
          for (int b = 0; b < B; ++b) mx = std::max(mx, hres[size_t(b) * (T + 1) + t]);
          if (mx <= tol) found = t;   // residual.max() <= tol (sinkhorn.py:244)
        }
        if (found) {
          ts = found;
          break;
        }
      }
    }
  }
  if (e == NSW_OK) {
    f2<<<B, OP_NT, sn, st>>>(K, lvi, mg, B, n, m, T, ts, vt, plan, lu, lv, rd);
    if (cudaGetLastError() != cudaSuccess) e = NSW_ERR_CUDA;
  }
  std::vector<double> hr(B, 0.0);
  if (e == NSW_OK && (resid_out || conv_out)) {
    if (cudaMemcpyAsync(hr.data(), rd, B * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      e = NSW_ERR_CUDA;
  }
  if (vt) cudaFreeAsync(vt, st);
  if (res) cudaFreeAsync(res, st);
  if (rd) cudaFreeAsync(rd, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) e = NSW_ERR_CUDA;
  if (e != NSW_OK) return e;
  if (iters_out) *iters_out = ts;
  for (int b = 0; b < B; ++b) {
    if (resid_out) resid_out[b] = hr[b];
    if (conv_out) conv_out[b] = hr[b] <= tol;   // residual <= tol (sinkhorn.py:253)
  }
  return NSW_OK;
}

template <typename S, int M>
nsw_status launch_bwd(const S* K, const S* hist, const S* lvi, const S* row, const S* col, const S* gp, const S* X,
                      const S* lu, int B, int n, int m, int T, S* gk, cudaStream_t st) {
  const size_t smem = bwd_smem<S, M>(n, T);
  if (smem > 227 * 1024) return NSW_ERR_UNSUPPORTED;
  auto fn = sinkhorn_bwd_op<S, M>;
  if (allow_smem((const void*)fn, size_t(smem)) != cudaSuccess)
    return NSW_ERR_CUDA;
  fn<<<B, OP_NT, smem, st>>>(K, hist, lvi, Marg<S>{row, col, n, m}, gp, X, lu, B, n, m, T, gk);
  return cudaGetLastError() == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}

// Streaming drivers (nsw_ops_generic.cuh): same contract as run_solve / launch_bwd, any (n, m).
template <typename S>
nsw_status gen_run_solve(const S* K, const S* row, const S* col, const S* lvi, int B, int n, int m, int T, double tol,
                         S* plan, S* lu, S* lv, S* hist, int32_t* iters_out, int32_t* conv_out, double* resid_out,
                         cudaStream_t st) {
  const Marg<S> mg{row, col, n, m};
  const bool tolm = tol > 0.0;
  const size_t sm_f = 2 * size_t(m) * sizeof(S), sm_n = 3 * size_t(m) * sizeof(S);
  if (sm_n > 200 * 1024) return NSW_ERR_UNSUPPORTED;   // m beyond ~8000 (float64): no caller of this path
  auto f1 = gen_fwd_op<S, Marg<S>>;
  auto f2 = gen_finish_op<S, Marg<S>>;
  if (allow_smem((const void*)f1, size_t(sm_f)) != cudaSuccess ||
      allow_smem((const void*)f2, size_t(sm_n)) != cudaSuccess)
    return NSW_ERR_CUDA;
  double* res = nullptr;
  double* rd = nullptr;
  nsw_status e = NSW_OK;
  if (private_malloc((void**)&rd, size_t(B) * sizeof(double), st) != cudaSuccess ||
      (tolm && private_malloc((void**)&res, size_t(B) * (T + 1) * sizeof(double), st) != cudaSuccess))
    e = NSW_ERR_CUDA;
  int ts = T;
  if (e == NSW_OK) {
    if (!tolm) {
      f1<<<B, GOP_NT, sm_f, st>>>(K, lvi, mg, B, n, m, T, 0, T, hist, lu, nullptr);
    } else {
      std::vector<double> hres(size_t(B) * (T + 1));
      for (int t0 = 0; t0 < T; t0 += OP_CHUNK) {
        const int t1 = std::min(t0 + OP_CHUNK, T);
        f1<<<B, GOP_NT, sm_f, st>>>(K, lvi, mg, B, n, m, T, t0, t1, hist, lu, res);
        if (cudaMemcpyAsync(hres.data(), res, hres.size() * sizeof(double), cudaMemcpyDeviceToHost, st) !=
                cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
          e = NSW_ERR_CUDA;
          break;
        }
        int found = 0;
        for (int t = t0 + 1; t <= t1 && !found; ++t) {
          double mx = 0.0;
          for (int b = 0; b < B; ++b) mx = std::max(mx, hres[size_t(b) * (T + 1) + t]);
          if (mx <= tol) found = t;   // residual.max() <= tol (sinkhorn.py:244)
        }
        if (found) {
          ts = found;
          break;
        }
      }
    }
  }
  if (e == NSW_OK) {
    f2<<<B, GOP_NT, sm_n, st>>>(K, lvi, mg, B, n, m, ts, hist, plan, lu, lv, rd);
    if (cudaGetLastError() != cudaSuccess) e = NSW_ERR_CUDA;
  }
  std::vector<double> hr(B, 0.0);
  if (e == NSW_OK && (resid_out || conv_out)) {
    if (cudaMemcpyAsync(hr.data(), rd, B * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      e = NSW_ERR_CUDA;
  }
  if (res) cudaFreeAsync(res, st);
  if (rd) cudaFreeAsync(rd, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) e = NSW_ERR_CUDA;
  if (e != NSW_OK) return e;
  if (iters_out) *iters_out = ts;
  for (int b = 0; b < B; ++b) {
    if (resid_out) resid_out[b] = hr[b];
    if (conv_out) conv_out[b] = hr[b] <= tol;   // residual <= tol (sinkhorn.py:253)
  }
  return NSW_OK;
}

template <typename S>
nsw_status gen_launch_bwd(const S* K, const S* hist, const S* lvi, const S* row, const S* col, const S* gp, const S* X,
                          const S* lu, int B, int n, int m, int T, S* gk, cudaStream_t st) {
  const size_t smem = 4 * size_t(m) * sizeof(S);
  if (smem > 200 * 1024) return NSW_ERR_UNSUPPORTED;
  auto fn = gen_bwd_op<S, Marg<S>>;
  if (allow_smem((const void*)fn, size_t(smem)) != cudaSuccess)
    return NSW_ERR_CUDA;
  S* scratch = nullptr;
  if (private_malloc((void**)&scratch, size_t(B) * 2 * n * sizeof(S), st) != cudaSuccess) return NSW_ERR_CUDA;
  fn<<<B, GOP_NT, smem, st>>>(K, hist, lvi, Marg<S>{row, col, n, m}, gp, X, lu, B, n, m, T, gk, scratch);
  const cudaError_t ce = cudaGetLastError();
  cudaFreeAsync(scratch, st);
  return ce == cudaSuccess ? NSW_OK : NSW_ERR_CUDA;
}

template <typename S>
nsw_status dispatch_solve(const S* K, const S* row, const S* col, const S* lvi, int B, int n, int m, int T, double tol,
                          S* plan, S* lu, S* lv, S* hist, int32_t* iters, int32_t* conv, double* resid, void* stream) {
  if (!K || !lvi || !plan || !lu || !lv || !hist || B <= 0 || T <= 0) return NSW_ERR_ARG;
  if (m < 2 || n < 1) return NSW_ERR_SHAPE;
  if (!row && m > n) return NSW_ERR_SHAPE;   // ranking marginals need m <= n
  cudaStream_t st = (cudaStream_t)stream;
  // shared-memory tile if one holds the kernel (m <= 32 and n rows fit), else the streaming operators
  nsw_status e = NSW_ERR_UNSUPPORTED;
#define NSW_SOLVE(MM) e = run_solve<S, MM>(K, row, col, lvi, B, n, m, T, tol, plan, lu, lv, hist, iters, conv, resid, st)
  if (m <= 4) NSW_SOLVE(4);
  else if (m <= 8) NSW_SOLVE(8);
  else if (m <= 11) NSW_SOLVE(11);
  else if (m <= 16) NSW_SOLVE(16);
  else if (m <= 21) NSW_SOLVE(21);
  else if (m <= 32) NSW_SOLVE(32);
#undef NSW_SOLVE
  if (e == NSW_ERR_UNSUPPORTED)
    e = gen_run_solve<S>(K, row, col, lvi, B, n, m, T, tol, plan, lu, lv, hist, iters, conv, resid, st);
  return e;
}

template <typename S>
nsw_status dispatch_bwd(const S* K, const S* hist, const S* lvi, const S* row, const S* col, const S* gp, const S* X,
                        const S* lu, int B, int n, int m, int T, S* gk, void* stream) {
  if (!K || !hist || !lvi || !gp || !X || !lu || !gk || B <= 0 || T <= 0) return NSW_ERR_ARG;
  if (m < 2 || n < 1) return NSW_ERR_SHAPE;
  if (!row && m > n) return NSW_ERR_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  nsw_status e = NSW_ERR_UNSUPPORTED;
#define NSW_BWD(MM) e = launch_bwd<S, MM>(K, hist, lvi, row, col, gp, X, lu, B, n, m, T, gk, st)
  if (m <= 4) NSW_BWD(4);
  else if (m <= 8) NSW_BWD(8);
  else if (m <= 11) NSW_BWD(11);
  else if (m <= 16) NSW_BWD(16);
  else if (m <= 21) NSW_BWD(21);
  else if (m <= 32) NSW_BWD(32);
#undef NSW_BWD
  if (e == NSW_ERR_UNSUPPORTED) e = gen_launch_bwd<S>(K, hist, lvi, row, col, gp, X, lu, B, n, m, T, gk, st);
  return e;
}

template <typename S>
nsw_status cost_from_policy(const S* x, size_t count, double eps, S* out, void* stream) {
  if (!x || !out) return NSW_ERR_ARG;
  if (!(eps > 0)) return NSW_ERR_DOMAIN;
  if (count == 0) return NSW_ERR_DOMAIN;   // the reference rejects an empty plan (x.size == 0)
  cudaStream_t st = (cudaStream_t)stream;
  unsigned* bad = nullptr;
  unsigned hbad = 0;
  if (private_malloc((void**)&bad, sizeof(unsigned), st) != cudaSuccess) return NSW_ERR_CUDA;
  cudaMemsetAsync(bad, 0, sizeof(unsigned), st);
  cost_from_policy_op<S><<<sm_count() * 4, 256, 0, st>>>(x, count, S(-eps), out, bad);
  cudaMemcpyAsync(&hbad, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(bad, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return NSW_ERR_CUDA;
  return hbad ? NSW_ERR_DOMAIN : NSW_OK;   // "plan must be strictly positive" (sinkhorn.py:185-186)
}

}  // namespace
}  // namespace nsw

extern "C" {

nsw_status nsw_sinkhorn_solve_batch_f64(const double* log_kernel, const double* row, const double* col,
                                        const double* log_v_init, int32_t B, int32_t n, int32_t m, int32_t max_iters,
                                        double tol, double* plan, double* log_u, double* log_v, double* log_v_hist,
                                        int32_t* iterations, int32_t* converged, double* residual, void* stream) {
  return nsw::dispatch_solve<double>(log_kernel, row, col, log_v_init, B, n, m, max_iters, tol, plan, log_u, log_v,
                                     log_v_hist, iterations, converged, residual, stream);
}

nsw_status nsw_sinkhorn_solve_batch_f32(const float* log_kernel, const float* row, const float* col,
                                        const float* log_v_init, int32_t B, int32_t n, int32_t m, int32_t max_iters,
                                        double tol, float* plan, float* log_u, float* log_v, float* log_v_hist,
                                        int32_t* iterations, int32_t* converged, double* residual, void* stream) {
  return nsw::dispatch_solve<float>(log_kernel, row, col, log_v_init, B, n, m, max_iters, tol, plan, log_u, log_v,
                                    log_v_hist, iterations, converged, residual, stream);
}

nsw_status nsw_sinkhorn_batch_f64(const double* log_kernel, const double* log_v_init, int32_t B, int32_t n, int32_t m,
                                  int32_t iters, double* plan, double* log_u, double* log_v, double* log_v_hist,
                                  void* stream) {
  return nsw::dispatch_solve<double>(log_kernel, nullptr, nullptr, log_v_init, B, n, m, iters, -1.0, plan, log_u,
                                     log_v, log_v_hist, nullptr, nullptr, nullptr, stream);
}

nsw_status nsw_sinkhorn_batch_f32(const float* log_kernel, const float* log_v_init, int32_t B, int32_t n, int32_t m,
                                  int32_t iters, float* plan, float* log_u, float* log_v, float* log_v_hist,
                                  void* stream) {
  return nsw::dispatch_solve<float>(log_kernel, nullptr, nullptr, log_v_init, B, n, m, iters, -1.0, plan, log_u,
                                    log_v, log_v_hist, nullptr, nullptr, nullptr, stream);
}

nsw_status nsw_sinkhorn_backward_batch_f64(const double* log_kernel, const double* log_v_hist,
                                           const double* log_v_init, const double* grad_plan, const double* plan,
                                           const double* log_u_final, int32_t B, int32_t n, int32_t m, int32_t iters,
                                           double* grad_log_kernel, void* stream) {
  return nsw::dispatch_bwd<double>(log_kernel, log_v_hist, log_v_init, nullptr, nullptr, grad_plan, plan, log_u_final,
                                   B, n, m, iters, grad_log_kernel, stream);
}

nsw_status nsw_sinkhorn_backward_batch_f32(const float* log_kernel, const float* log_v_hist, const float* log_v_init,
                                           const float* grad_plan, const float* plan, const float* log_u_final,
                                           int32_t B, int32_t n, int32_t m, int32_t iters, float* grad_log_kernel,
                                           void* stream) {
  return nsw::dispatch_bwd<float>(log_kernel, log_v_hist, log_v_init, nullptr, nullptr, grad_plan, plan, log_u_final,
                                  B, n, m, iters, grad_log_kernel, stream);
}

nsw_status nsw_sinkhorn_backward_general_f64(const double* log_kernel, const double* row, const double* col,
                                             const double* log_v_hist, const double* log_v_init,
                                             const double* grad_plan, const double* plan, const double* log_u_final,
                                             int32_t B, int32_t n, int32_t m, int32_t iters, double* grad_log_kernel,
                                             void* stream) {
  return nsw::dispatch_bwd<double>(log_kernel, log_v_hist, log_v_init, row, col, grad_plan, plan, log_u_final, B, n,
                                   m, iters, grad_log_kernel, stream);
}

nsw_status nsw_sinkhorn_backward_general_f32(const float* log_kernel, const float* row, const float* col,
                                             const float* log_v_hist, const float* log_v_init, const float* grad_plan,
                                             const float* plan, const float* log_u_final, int32_t B, int32_t n,
                                             int32_t m, int32_t iters, float* grad_log_kernel, void* stream) {
  return nsw::dispatch_bwd<float>(log_kernel, log_v_hist, log_v_init, row, col, grad_plan, plan, log_u_final, B, n, m,
                                  iters, grad_log_kernel, stream);
}

nsw_status nsw_cost_from_policy_f64(const double* plan, size_t count, double epsilon, double* cost, void* stream) {
  return nsw::cost_from_policy<double>(plan, count, epsilon, cost, stream);
}

nsw_status nsw_cost_from_policy_f32(const float* plan, size_t count, double epsilon, float* cost, void* stream) {
  return nsw::cost_from_policy<float>(plan, count, epsilon, cost, stream);
}

}  // extern "C"
