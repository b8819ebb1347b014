// Streaming operator seam: the same three operators as nsw_ops.cu
// (_sinkhorn_batch forward in chunks, its finish, _sinkhorn_backward_batch)
// for shapes whose absorbed kernel does not fit one CTA's shared memory or
// whose m exceeds the compiled tile widths (m > 32) -- the reference accepts
// any (B, n, m) (sinkhorn.py:204-216).  One CTA per batch element, the log
// kernel read from global memory (L2) every pass, the reference's own
// log-domain recurrences (sinkhorn.py:219-243, :272-308) term by term:
// rows go to warps (lanes stride the columns, butterfly sums), column sums
// are thread-per-column over fixed row chunks combined in chunk order, so
// results are deterministic.  A fallback: several passes over K per
// iteration; the shared-memory tiles remain the fast path.
#pragma once

#include "nsw_device.cuh"

namespace nsw {
namespace {

constexpr int GOP_NT = 256;
constexpr int GOP_NW = GOP_NT / 32;

template <typename S>
__device__ __forceinline__ S warp_max(S x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
template <typename S>
__device__ __forceinline__ S warp_sum(S x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// The per-element context shared by the three kernels.
template <typename S, typename MG>
struct GenOp {
  using F = Fp<S>;
  const S* K;     // [n][m] log kernel of this element
  MG mg;
  int n, m;
  S* part;        // shared [GOP_NT] column-chunk partials
  S* part2;       // shared [GOP_NT]
  int tid, lane, warp;

  __device__ S log_row(int i) const { return F::log_(mg.r(i)); }
  __device__ S log_col(int k) const { return F::log_(mg.c(k)); }

  // log_u_i = log_row_i - LSE_k(K_ik + v_k)            (sinkhorn.py:219-226)
  __device__ void row_dual(const S* v, S* lu) const {
    for (int i = warp; i < n; i += GOP_NW) {
      const S* row = K + size_t(i) * m;
      S top = F::ninf();
      for (int k = lane; k < m; k += 32) top = fmax(top, row[k] + v[k]);
      top = warp_max(top);
      S acc = S(0);
      for (int k = lane; k < m; k += 32) acc += F::exp_(row[k] + v[k] - top);
      acc = warp_sum(acc);
      if (lane == 0) lu[i] = log_row(i) - (F::log_(acc) + top);
    }
  }

  // for every column k: fin(k, max_i f(i, k), sum_i exp(f(i, k) - that max)); two fixed-order
  // passes over the row chunks (the reference's max-then-sum LSE).  Ends with a barrier.
  template <class Fn, class Fin>
  __device__ void col_lse(Fn f, Fin fin) const {
    const int Q = max(1, GOP_NT / m);
    for (int k0 = 0; k0 < m; k0 += GOP_NT) {
      const int span = min(m - k0, GOP_NT);
      const int q = min(Q, GOP_NT / span);
      const int k = k0 + tid % span, qi = tid / span;
      const int i0 = int((long long)n * qi / q), i1 = int((long long)n * (qi + 1) / q);
      if (qi < q) {
        S top = F::ninf();
        for (int i = i0; i < i1; ++i) top = fmax(top, f(i, k));
        part[qi * span + (tid % span)] = top;
      }
      __syncthreads();
      S top = F::ninf();
      if (qi < q) {
        for (int j = 0; j < q; ++j) top = fmax(top, part[j * span + (tid % span)]);
        S acc = S(0);
        for (int i = i0; i < i1; ++i) acc += F::exp_(f(i, k) - top);
        part2[qi * span + (tid % span)] = acc;
      }
      __syncthreads();
      if (tid < span) {
        S tot = part2[tid];
        for (int j = 1; j < q; ++j) tot += part2[j * span + tid];
        fin(k0 + tid, top, tot);
      }
      __syncthreads();
    }
  }

  // for every column k: fin(k, sum_i f(i, k)) in fixed chunk order.  Ends with a barrier.
  template <class Fn, class Fin>
  __device__ void col_sum(Fn f, Fin fin) const {
    const int Q = max(1, GOP_NT / m);
    for (int k0 = 0; k0 < m; k0 += GOP_NT) {
      const int span = min(m - k0, GOP_NT);
      const int q = min(Q, GOP_NT / span);
      const int k = k0 + tid % span, qi = tid / span;
      if (qi < q) {
        const int i0 = int((long long)n * qi / q), i1 = int((long long)n * (qi + 1) / q);
        S acc = S(0);
        for (int i = i0; i < i1; ++i) acc += f(i, k);
        part[qi * span + (tid % span)] = acc;
      }
      __syncthreads();
      if (tid < span) {
        S tot = part[tid];
        for (int j = 1; j < q; ++j) tot += part[j * span + tid];
        fin(k0 + tid, tot);
      }
      __syncthreads();
    }
  }

};

// Iterations t0+1 .. t1 (1-based) of the lock-step forward for element b = blockIdx.x.
// hist: [T][B][m] log v after every iteration; lu: [B][n] (scratch here, final in finish);
// res (tolerance mode, else null): [B][T+1] residual after iteration t.
template <typename S, typename MG>
__global__ void __launch_bounds__(GOP_NT) gen_fwd_op(const S* __restrict__ log_kernel, const S* __restrict__ lvi_all,
                                                    MG mg, int B, int n, int m, int T, int t0, int t1, S* hist, S* lu_all,
                                                    double* res) {
  using F = Fp<S>;
  extern __shared__ __align__(16) unsigned char gop_smem[];
  S* lv = reinterpret_cast<S*>(gop_smem);   // [m]
  S* cres = lv + m;                         // [m] column residuals
  __shared__ S part[GOP_NT], part2[GOP_NT];
  __shared__ double red[GOP_NW + 1];
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  GenOp<S, MG> op{log_kernel + size_t(b) * n * m, mg, n, m, part, part2, tid, tid & 31, tid >> 5};
  S* lu = lu_all + size_t(b) * n;
  for (int k = tid; k < m; k += GOP_NT)
    lv[k] = t0 == 0 ? lvi_all[size_t(b) * m + k] : hist[(size_t(t0 - 1) * B + b) * m + k];
  __syncthreads();
  for (int t = t0; t < t1; ++t) {
    op.row_dual(lv, lu);
    __syncthreads();
    // log_v_k = log_col_k - LSE_i(K_ik + u_i)          (sinkhorn.py:227-234)
    op.col_lse([&](int i, int k) { return op.K[size_t(i) * m + k] + lu[i]; },
               [&](int k, S top, S tot) {
                 const S v = op.log_col(k) - (F::log_(tot) + top);
                 lv[k] = v;
                 hist[(size_t(t) * B + b) * m + k] = v;
               });
    if (res != nullptr) {
      double rmax = 0.0;
      for (int i = op.warp; i < n; i += GOP_NW) {
        const S* row = op.K + size_t(i) * m;
        S acc = S(0);
        for (int k = op.lane; k < m; k += 32) acc += F::exp_(row[k] + lu[i] + lv[k]);
        acc = warp_sum(acc);
        rmax = fmax(rmax, fabs(double(acc) - double(mg.r(i))));
      }
      if (op.lane == 0) red[op.warp] = rmax;
      op.col_sum([&](int i, int k) { return F::exp_(op.K[size_t(i) * m + k] + lu[i] + lv[k]); },
                 [&](int k, S tot) { cres[k] = S(fabs(double(tot) - double(mg.c(k)))); });
      if (tid == 0) {
        double r = 0.0;
        for (int w = 0; w < GOP_NW; ++w) r = fmax(r, red[w]);
        for (int k = 0; k < m; ++k) r = fmax(r, double(cres[k]));
        res[size_t(b) * (T + 1) + t + 1] = r;
      }
      __syncthreads();
    }
  }
}

// The plan and duals of iteration ts (1-based) from the recorded column duals.
template <typename S, typename MG>
__global__ void __launch_bounds__(GOP_NT) gen_finish_op(const S* __restrict__ log_kernel,
                                                       const S* __restrict__ lvi_all, MG mg, int B, int n, int m, int ts,
                                                       const S* __restrict__ hist, S* plan_all, S* lu_all, S* lv_all,
                                                       double* rd) {
  using F = Fp<S>;
  extern __shared__ __align__(16) unsigned char gop_smem[];
  S* lv = reinterpret_cast<S*>(gop_smem);   // [m] log v of iteration ts
  S* lvp = lv + m;                          // [m] log v of iteration ts - 1
  S* cres = lvp + m;                        // [m]
  __shared__ S part[GOP_NT], part2[GOP_NT];
  __shared__ double red[GOP_NW + 1];
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  GenOp<S, MG> op{log_kernel + size_t(b) * n * m, mg, n, m, part, part2, tid, tid & 31, tid >> 5};
  S* lu = lu_all + size_t(b) * n;
  S* plan = plan_all + size_t(b) * n * m;
  for (int k = tid; k < m; k += GOP_NT) {
    lv[k] = hist[(size_t(ts - 1) * B + b) * m + k];
    lvp[k] = ts >= 2 ? hist[(size_t(ts - 2) * B + b) * m + k] : lvi_all[size_t(b) * m + k];
    lv_all[size_t(b) * m + k] = lv[k];
  }
  __syncthreads();
  op.row_dual(lvp, lu);
  __syncthreads();
  double rmax = 0.0;
  for (int i = op.warp; i < n; i += GOP_NW) {
    const S* row = op.K + size_t(i) * m;
    S acc = S(0);
    for (int k = op.lane; k < m; k += 32) {
      const S x = F::exp_(row[k] + lu[i] + lv[k]);
      plan[size_t(i) * m + k] = x;
      acc += x;
    }
    acc = warp_sum(acc);
    rmax = fmax(rmax, fabs(double(acc) - double(mg.r(i))));
  }
  if (op.lane == 0) red[op.warp] = rmax;
  __syncthreads();   // the plan is complete
  op.col_sum([&](int i, int k) { return plan[size_t(i) * m + k]; },
             [&](int k, S tot) { cres[k] = S(fabs(double(tot) - double(mg.c(k)))); });
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < GOP_NW; ++w) r = fmax(r, red[w]);
    for (int k = 0; k < m; ++k) r = fmax(r, double(cres[k]));
    rd[b] = r;
  }
}

// Unrolled reverse mode (sinkhorn.py:258-309).  scratch: [B][2 n] (log u of the level, g_u).
template <typename S, typename MG>
__global__ void __launch_bounds__(GOP_NT) gen_bwd_op(const S* __restrict__ log_kernel, const S* __restrict__ hist,
                                                    const S* __restrict__ lvi_all, MG mg, const S* __restrict__ gp_all,
                                                    const S* __restrict__ X_all, const S* __restrict__ lu_final, int B,
                                                    int n, int m, int T, S* gk_all, S* scratch) {
  using F = Fp<S>;
  extern __shared__ __align__(16) unsigned char gop_smem[];
  S* vt = reinterpret_cast<S*>(gop_smem);   // [m] log v^t
  S* vp = vt + m;                           // [m] log v^{t-1}
  S* gv = vp + m;                           // [m] g_v
  S* lc = gv + m;                           // [m] log col
  __shared__ S part[GOP_NT], part2[GOP_NT];
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  GenOp<S, MG> op{log_kernel + size_t(b) * n * m, mg, n, m, part, part2, tid, tid & 31, tid >> 5};
  const S* gp = gp_all + size_t(b) * n * m;
  const S* X = X_all + size_t(b) * n * m;
  S* gk = gk_all + size_t(b) * n * m;
  S* ut = scratch + size_t(b) * 2 * n;
  S* gu = ut + n;
  auto vrow = [&](int t) -> const S* {   // log v^t, t = 0 is the warm start
    return t >= 1 ? hist + (size_t(t - 1) * B + b) * m : lvi_all + size_t(b) * m;
  };
  for (int k = tid; k < m; k += GOP_NT) lc[k] = op.log_col(k);
  for (int i = tid; i < n; i += GOP_NT) ut[i] = lu_final[size_t(b) * n + i];
  // w = grad_plan * plan; g_kernel = w; g_u = row sums; g_v = column sums   (sinkhorn.py:272-275)
  for (int i = op.warp; i < n; i += GOP_NW) {
    S acc = S(0);
    for (int k = op.lane; k < m; k += 32) {
      const S w = gp[size_t(i) * m + k] * X[size_t(i) * m + k];
      gk[size_t(i) * m + k] = w;
      acc += w;
    }
    acc = warp_sum(acc);
    if (op.lane == 0) gu[i] = acc;
  }
  __syncthreads();
  op.col_sum([&](int i, int k) { return gk[size_t(i) * m + k]; }, [&](int k, S tot) { gv[k] = tot; });
  for (int t = T; t >= 1; --t) {
    const S* v_t = vrow(t);
    const S* v_prev = vrow(t - 1);
    for (int k = tid; k < m; k += GOP_NT) {
      vt[k] = v_t[k];
      vp[k] = v_prev[k];
    }
    __syncthreads();
    const bool first = t == T;
    for (int i = op.warp; i < n; i += GOP_NW) {
      const S* row = op.K + size_t(i) * m;
      S* grow = gk + size_t(i) * m;
      const S ui = ut[i];
      // column softmax VJP (sinkhorn.py:281-289): s = exp(K + u + v_t - log_col) * g_v
      S acc = S(0);
      for (int k = op.lane; k < m; k += 32) {
        const S s = F::exp_(row[k] + ui + vt[k] - lc[k]) * gv[k];
        grow[k] -= s;
        acc += s;
      }
      acc = warp_sum(acc);
      const S g = (first ? gu[i] : S(0)) - acc;
      // row softmax VJP (sinkhorn.py:290-299): s = exp(K + v_prev + u - log_row) * g_u
      const S lr = op.log_row(i);
      for (int k = op.lane; k < m; k += 32) grow[k] -= F::exp_(row[k] + vp[k] + ui - lr) * g;
      if (op.lane == 0) gu[i] = g;
    }
    __syncthreads();
    // g_v = -column sums of the row term
    op.col_sum([&](int i, int k) { return F::exp_(op.K[size_t(i) * m + k] + vp[k] + ut[i] - op.log_row(i)) * gu[i]; },
               [&](int k, S tot) { gv[k] = -tot; });
    if (t >= 2) {   // log u of the previous level (sinkhorn.py:300-308)
      const S* v_pp = vrow(t - 2);
      for (int k = tid; k < m; k += GOP_NT) vt[k] = v_pp[k];
      __syncthreads();
      op.row_dual(vt, ut);
      __syncthreads();
    }
  }
}

}  // namespace
}  // namespace nsw
