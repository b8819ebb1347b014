// Fused outer-step kernel of the NSW ascent:  [backward of step k-1 +
// Adam ascent on the cost tile +] forward of step k + per-item impact terms.
//
// One CTA per user.  Replaces, per user, reference solver.py:186-240 minus
// the cross-user impact sum (solver.py:206), which is the only coupling
// between users and is done by impact_reduce_kernel / finalize_kernel.
//
// Register / shared-memory residency:
//   forward : K~ (R rows x M columns per thread) in registers; the column
//             scaling vector and the v~ history in shared memory.
//   backward: G (the K~-coordinates adjoint, R x M per thread) in registers,
//             K~ in shared memory (one 16-byte-vector row read per level).
#pragma once

#include "nsw_device.cuh"

namespace nsw {

template <typename S>
struct StepArgs {
  int U, n, m, T, outer_max, warm_start;
  S* C;          // [U][n][m] transport costs (the ascent variable)
  S* am;         // [U][n][m] Adam first moment
  S* av;         // [U][n][m] Adam second moment
  S* alpha;      // [U][n]    row dual after inner iteration 1 (absorption point)
  S* beta;       // [U][m]    column dual after inner iteration 1
  S* hist;       // [U][T+1][m] v~^t, t = 0..T  (v~^0 = exp(lvi - beta), v~^1 = 1)
  S* xbest;      // [U][n][m] best-F policy so far
  const S* rel;          // [U][n]
  const S* expo;         // [m-1]
  const double* expo_d;  // [m-1] (impact terms are accumulated in float64)
  double* partial;       // [U][n] sum_{k<m-1} r_ui e_k x_uik
  const double* imp;     // [n] Imp of the step being differentiated
  const int* state;      // device step state (ST_*)
  const double* bc;      // [2*(outer_max+1)] Adam bias corrections 1-b1^s, 1-b2^s
  S nie;                 // -1/eps (solver.py:188, :236)
  S lr, b1, b2, omb1, omb2, aeps;
  S c_real, c_dummy;     // initial costs -eps*log(1/n), -eps*log((n-m+1)/n)
  S mass_dummy, log_mass_dummy;
};

template <typename S>
__device__ __forceinline__ S mul_(S a, S b);
template <>
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
template <typename S>
__device__ __forceinline__ S add_(S a, S b);
template <>
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }

// Row dot product with two interleaved accumulators (halves the dependent
// FMA chain).  Every place that forms u~ = 1/(K~ v~) uses this one function,
// so the forward and the backward's replay produce bit-identical u~.
template <typename S, int M>
__device__ __forceinline__ S rdot(const S (&x)[M], const S (&y)[M]) {
  S s0 = S(0), s1 = S(0);
#pragma unroll
  for (int k = 0; k + 1 < M; k += 2) {
    s0 = fma(x[k], y[k], s0);
    s1 = fma(x[k + 1], y[k + 1], s1);
  }
  if constexpr (M % 2) s0 = fma(x[M - 1], y[M - 1], s0);
  return s0 + s1;
}

template <typename S, int M, int R, int NT>
__host__ __device__ constexpr size_t step_smem_bytes(int T) {
  constexpr int P = Pitch<S, M>::value;
  return sizeof(S) * (size_t(NT) * R * P + size_t(T + 1) * P + size_t(NT / 32) * P + 3 * P + 2 * size_t(NT) * R);
}

// Structure: the per-step phases that touch every cell once (K~ rebuild,
// seed, Adam, log-domain iteration 1) run as runtime loops over this
// thread's rows through the shared-memory tile Kt, so they add no register
// pressure; only the two hot loops (forward iterations 2..T and the T
// reverse levels) hold the R x M tile in registers.
template <typename S, int M, int R, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) step_kernel(const StepArgs<S> a) {
  using F = Fp<S>;
  constexpr int P = Pitch<S, M>::value;
  constexpr int NW = NT / 32;
  constexpr int PAIR = R >= 2 ? 2 : 1;
  static_assert(NT % 32 == 0 && M <= NT && P <= NT && R % PAIR == 0, "tile shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = a.T;
  S* Kt = reinterpret_cast<S*>(smem_raw);   // [NT*R][P]  K / K~ / gK rows
  S* vh = Kt + size_t(NT) * R * P;          // [T+1][P]   v~ history
  S* red = vh + size_t(T + 1) * P;          // [NW][P]    column partials
  S* vec0 = red + NW * P;                   // [P] scaling vector / cv
  S* vec1 = vec0 + P;                       // [P] beta / column max
  S* vec2 = vec1 + P;                       // [P] warm-start duals lvi
  S* rowA = vec2 + P;                       // [NT*R] u~^T per row, then u^1
  S* rowB = rowA + size_t(NT) * R;          // [NT*R] seed g_u per row

  const int phase = a.state[ST_PHASE];
  if (phase == PHASE_FINISHED) return;

  const int u = blockIdx.x;
  const int tid = threadIdx.x;
  const int n = a.n, m = a.m;
  const size_t ubase = size_t(u) * n * m;
  S* Cu = a.C + ubase;
  S* mu = a.am + ubase;
  S* vu = a.av + ubase;
  S* xb = a.xbest + ubase;
  S* hu = a.hist + size_t(u) * (T + 1) * m;
  const S* relu = a.rel + size_t(u) * n;
  auto ok = [&](int r) { return tid + r * NT < n; };
  auto mass = [&](int k) -> S { return k == m - 1 ? a.mass_dummy : S(1); };
  auto inv_mass = [&](int k) -> S { return k == m - 1 ? F::rcp(a.mass_dummy) : S(1); };

  if (tid < P) {
    vec0[tid] = S(0);
    vec1[tid] = S(0);
    vec2[tid] = S(0);
  }
  S ex[M];
#pragma unroll
  for (int k = 0; k < M; ++k) ex[k] = (k < m - 1) ? a.expo[(k < m - 1) ? k : 0] : S(0);

  if (phase == PHASE_RUNNING || phase == PHASE_DONE_PENDING) {
    // ---------------- rebuild K~ of step k-1 from C, alpha, beta ------------
    __syncthreads();
    if (tid < m) vec1[tid] = a.beta[size_t(u) * m + tid];
    for (int idx = tid; idx < (T + 1) * P; idx += NT) {
      const int t = idx / P, k = idx - t * P;
      vh[idx] = k < m ? hu[size_t(t) * m + k] : S(0);
    }
    __syncthreads();
    S vT[M];
    lds_vec<S, M>(vT, vh + size_t(T) * P);
    {
      S bt[M], vT1[M];
      lds_vec<S, M>(bt, vec1);
      lds_vec<S, M>(vT1, vh + size_t(T >= 2 ? T - 1 : 0) * P);
#pragma unroll 1
      for (int i = tid; i < NT * R; i += NT) {
        const bool v = i < n;
        S kr[M];
        const S al = v ? a.alpha[size_t(u) * n + i] : S(0);
#pragma unroll
        for (int k = 0; k < M; ++k)
          kr[k] = (v && k < m) ? F::exp_(add_(add_(mul_(Cu[size_t(i) * m + k], a.nie), al), bt[k])) : S(0);
        sts_vec<S, M>(Kt + size_t(i) * P, kr);
        rowA[i] = v ? ((T >= 2) ? F::rcp_fast(rdot<S, M>(kr, vT1)) : S(1)) : S(0);
      }
    }
    const int improved = a.state[ST_IMPROVED];
    if (phase == PHASE_DONE_PENDING) {
      // the stop fired after step k-1's forward: only its policy is still owed
      if (improved) {
#pragma unroll 1
        for (int i = tid; i < n; i += NT) {
          S kr[M];
          lds_vec<S, M>(kr, Kt + size_t(i) * P);
          const S uT = rowA[i];
#pragma unroll
          for (int k = 0; k < M; ++k)
            if (k < m) xb[size_t(i) * m + k] = mul_(mul_(kr[k], uT), vT[k]);
        }
      }
      return;
    }

    // ---------------- seed: W = gx .* X  (sinkhorn.py:272-275) --------------
    {
      S c[M];
#pragma unroll
      for (int k = 0; k < M; ++k) c[k] = S(0);
#pragma unroll 1
      for (int i = tid; i < NT * R; i += NT) {
        const bool v = i < n;
        S kr[M];
        lds_vec<S, M>(kr, Kt + size_t(i) * P);
        const S uT = rowA[i];
        const S rr = v ? relu[i] : S(0);
        const S imp_i = v ? S(a.imp[i]) : S(1);
        S gsum = S(0);
#pragma unroll
        for (int k = 0; k < M; ++k) {
          if (k >= m) continue;
          const S X = mul_(mul_(kr[k], uT), vT[k]);
          if (improved && v) xb[size_t(i) * m + k] = X;
          if (k < m - 1) {
            const S W = mul_(F::div(mul_(rr, ex[k]), imp_i), X);   // gx = r e / Imp, solver.py:86-89
            gsum += W;
            c[k] += W;
          }
        }
        rowB[i] = gsum;
      }
      cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
        vec0[k] = mul_(mul_(vh[size_t(T) * P + k], tot), inv_mass(k));   // cv^T = v~^T g_v / colmass
      });
    }

    // ---------------- unrolled reverse sweep  (sinkhorn.py:278-308) ---------
    // Per level t, per row i (u~ = u~^t_i, cv = v~^t g_v / colmass):
    //   g_u  <- [t==T] g_u^seed - u~ (K~ cv)_i                  column VJP
    //   h    <- u~ g_u
    //   G_ik <- G_ik - u~ cv_k - h v~^{t-1}_k                    both VJPs into gK
    //   g_v  <- -v~^{t-1} (K~' h)                                row VJP
    //   u~   <- 1/(K~ v~^{t-2})_i                                replay (t >= 3)
    {
      S A[R][M];  // adjoint G: gK = W + K~ .* G
      S ut[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ut[r] = rowA[tid + r * NT];
#pragma unroll
        for (int k = 0; k < M; ++k) A[r][k] = S(0);
      }
      for (int t = T; t >= 1; --t) {
        S cv[M], vp[M], vpp[M], c[M];
        lds_vec<S, M>(cv, vec0);
        lds_vec<S, M>(vp, vh + size_t(t - 1) * P);
        lds_vec<S, M>(vpp, vh + size_t(t >= 2 ? t - 2 : 0) * P);
        const bool first = t == T;
        const bool replay = t >= 3;
#pragma unroll
        for (int k = 0; k < M; ++k) c[k] = S(0);
#pragma unroll
        for (int r = 0; r < R; r += PAIR) {
          S kr[PAIR][M], h[PAIR];
#pragma unroll
          for (int q = 0; q < PAIR; ++q) lds_vec<S, M>(kr[q], Kt + size_t(tid + (r + q) * NT) * P);
#pragma unroll
          for (int q = 0; q < PAIR; ++q) {
            const S sig = rdot<S, M>(kr[q], cv);
            const S gs = first ? rowB[tid + (r + q) * NT] : S(0);
            h[q] = ut[r + q] * (gs - ut[r + q] * sig);
          }
#pragma unroll
          for (int q = 0; q < PAIR; ++q)
#pragma unroll
            for (int k = 0; k < M; ++k) {
              A[r + q][k] = fma(-ut[r + q], cv[k], A[r + q][k]);
              A[r + q][k] = fma(-h[q], vp[k], A[r + q][k]);
            }
#pragma unroll
          for (int k = 0; k < M; ++k)
#pragma unroll
            for (int q = 0; q < PAIR; ++q) c[k] = fma(kr[q][k], h[q], c[k]);
#pragma unroll
          for (int q = 0; q < PAIR; ++q) {
            const S rp = F::rcp_fast(rdot<S, M>(kr[q], vpp));
            ut[r + q] = ok(r + q) ? (replay ? rp : S(1)) : S(0);
          }
        }
        if (t >= 2) {
          cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
            const S vpk = vh[size_t(t - 1) * P + k];
            const S gv = -mul_(vpk, tot);
            vec0[k] = mul_(mul_(vpk, gv), inv_mass(k));
          });
        }
      }
      // gK = W + K~ .* G, written over K~ in the tile (W = gx .* X recomputed)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        S kr[M], gk[M];
        lds_vec<S, M>(kr, Kt + size_t(i) * P);
        const S uT = rowA[i];
        const S rr = ok(r) ? relu[i] : S(0);
        const S imp_i = ok(r) ? S(a.imp[i]) : S(1);
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const S X = mul_(mul_(kr[k], uT), vT[k]);
          const S W = (k < m - 1) ? mul_(F::div(mul_(rr, ex[k]), imp_i), X) : S(0);
          gk[k] = fma(kr[k], A[r][k], W);
        }
        sts_vec<S, M>(Kt + size_t(i) * P, gk);
      }
    }

    // ---------------- g_C = gK * (-1/eps); Adam ascent  (solver.py:105-122) -
    const int s = a.state[ST_STEP];
    const S bc1 = S(a.bc[2 * s]), bc2 = S(a.bc[2 * s + 1]);
    if (tid < m) vec2[tid] = a.warm_start ? add_(vec1[tid], F::log_(vh[size_t(T) * P + tid])) : S(0);
#pragma unroll 1
    for (int i = tid; i < n; i += NT) {
      S gk[M], kn[M];
      lds_vec<S, M>(gk, Kt + size_t(i) * P);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        kn[k] = S(0);
        if (k < m) {
          const S g = mul_(gk[k], a.nie);
          const size_t off = size_t(i) * m + k;
          const S m1 = add_(mul_(a.b1, mu[off]), mul_(a.omb1, g));
          const S v1 = add_(mul_(a.b2, vu[off]), mul_(mul_(a.omb2, g), g));
          const S mh = F::div(m1, bc1);
          const S vhat = F::div(v1, bc2);
          const S c1 = add_(Cu[off], F::div(mul_(a.lr, mh), add_(F::sqrt_(vhat), a.aeps)));
          mu[off] = m1;
          vu[off] = v1;
          Cu[off] = c1;
          kn[k] = mul_(c1, a.nie);
        }
      }
      sts_vec<S, M>(Kt + size_t(i) * P, kn);
    }
  } else {
    // INIT: initial cost C0 = -eps log(uniform) (solver.py:176-177), lvi = 0.
    // RESUME: caller-provided C (left as is), lvi taken from the beta buffer.
    const bool init = phase == PHASE_INIT;
    __syncthreads();
    if (!init && tid < m) vec2[tid] = a.beta[size_t(u) * m + tid];
#pragma unroll 1
    for (int i = tid; i < n; i += NT) {
      S kn[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        kn[k] = S(0);
        if (k < m) {
          const size_t off = size_t(i) * m + k;
          S c0;
          if (init) {
            c0 = (k == m - 1) ? a.c_dummy : a.c_real;
            Cu[off] = c0;
            mu[off] = S(0);
            vu[off] = S(0);
          } else {
            c0 = Cu[off];
          }
          kn[k] = mul_(c0, a.nie);
        }
      }
      sts_vec<S, M>(Kt + size_t(i) * P, kn);
    }
  }
  __syncthreads();

  // ======================= forward of step k =================================
  // inner iteration 1 in the log domain (sinkhorn.py:219-234), v^0 = lvi;
  // K = C * (-1/eps) is in the tile rows i < n.
  {
    S lv[M], c[M];
    lds_vec<S, M>(lv, vec2);
#pragma unroll
    for (int k = 0; k < M; ++k) c[k] = F::ninf();
#pragma unroll 1
    for (int i = tid; i < n; i += NT) {
      S kr[M];
      lds_vec<S, M>(kr, Kt + size_t(i) * P);
      S mx = F::ninf();
#pragma unroll
      for (int k = 0; k < M; ++k)
        if (k < m) mx = fmax(mx, add_(kr[k], lv[k]));
      S acc = S(0);
#pragma unroll
      for (int k = 0; k < M; ++k)
        if (k < m) acc += F::exp_(add_(kr[k], lv[k]) - mx);
      const S u1 = -(F::log_(acc) + mx);
      rowA[i] = u1;
#pragma unroll
      for (int k = 0; k < M; ++k)
        if (k < m) c[k] = fmax(c[k], add_(kr[k], u1));
    }
    cta_reduce_cols<S, M, NT, OpMax>(c, red, m, [&](int k, S tot) { vec1[k] = tot; });
    S cm[M];
    lds_vec<S, M>(cm, vec1);
#pragma unroll
    for (int k = 0; k < M; ++k) c[k] = S(0);
#pragma unroll 1
    for (int i = tid; i < n; i += NT) {
      S kr[M];
      lds_vec<S, M>(kr, Kt + size_t(i) * P);
      const S u1 = rowA[i];
#pragma unroll
      for (int k = 0; k < M; ++k)
        if (k < m) c[k] += F::exp_(add_(kr[k], u1) - cm[k]);
    }
    cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
      const S lc = (k == m - 1) ? a.log_mass_dummy : S(0);
      const S b = lc - (F::log_(tot) + vec1[k]);
      vec1[k] = b;
      a.beta[size_t(u) * m + k] = b;
      hu[k] = F::exp_(vec2[k] - b);  // v~^0
      if (T >= 1) hu[size_t(1) * m + k] = S(1);  // v~^1
      vec0[k] = S(1);
    });
    // absorb: K~ = exp(K + u^1 + v^1) = X^1 (rows >= n stay zero)
    S bt[M];
    lds_vec<S, M>(bt, vec1);
#pragma unroll 1
    for (int i = tid; i < NT * R; i += NT) {
      const bool v = i < n;
      S kr[M];
      lds_vec<S, M>(kr, Kt + size_t(i) * P);
      const S u1 = v ? rowA[i] : S(0);
      if (v) a.alpha[size_t(u) * n + i] = u1;
#pragma unroll
      for (int k = 0; k < M; ++k) kr[k] = (v && k < m) ? F::exp_(add_(add_(kr[k], u1), bt[k])) : S(0);
      sts_vec<S, M>(Kt + size_t(i) * P, kr);
    }
  }
  // inner iterations 2..T, multiplicative: u~ = 1/(K~ v~), v~ = colmass/(K~' u~)
  S A[R][M];  // K~, register resident
  S ut[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    lds_vec<S, M>(A[r], Kt + size_t(tid + r * NT) * P);
    ut[r] = ok(r) ? S(1) : S(0);
  }
  for (int t = 2; t <= T; ++t) {
    S vv[M], c[M];
    lds_vec<S, M>(vv, vec0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const S rp = F::rcp_fast(rdot<S, M>(A[r], vv));
      ut[r] = ok(r) ? rp : S(0);
    }
#pragma unroll
    for (int k = 0; k < M; ++k) {
      c[k] = A[0][k] * ut[0];
#pragma unroll
      for (int r = 1; r < R; ++r) c[k] = fma(A[r][k], ut[r], c[k]);
    }
    cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
      const S vn = F::div(mass(k), tot);
      vec0[k] = vn;
      hu[size_t(t) * m + k] = vn;
    });
  }
  // per-item impact terms of this user (solver.py:206), float64
  {
    S vv[M];
    lds_vec<S, M>(vv, vec0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = tid + r * NT;
      const double rr = ok(r) ? double(relu[i]) : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        if (k < m - 1) {
          const S X = mul_(mul_(A[r][k], ut[r]), vv[k]);
          acc = fma(rr * a.expo_d[(k < m - 1) ? k : 0], double(X), acc);
        }
      }
      if (ok(r)) a.partial[size_t(u) * n + i] = acc;
    }
  }
}

// --------------------------------------------------------------------------
// Impact reduction over this rank's users (deterministic, fixed order):
// split[y][i] = sum over user chunk y; the last CTA to finish sums the chunks.
// --------------------------------------------------------------------------
constexpr int IMP_THREADS = 256;
constexpr int IMP_ITEMS = 8;
__global__ void impact_reduce_kernel(const double* __restrict__ partial, int U, int n,
                                     double* __restrict__ imp_local, const int* __restrict__ state);

struct FinalizeArgs {
  int n, world, outer_max;
  const double* imp_all;   // [world][n]
  const double* rel_sq;    // [n] sum_u r_ui^2 over all users
  double exp_sq;           // sum_k e_k^2
  double grad_threshold;
  double* imp_cur;         // [n]
  double* best;            // [1]
  double* objective;       // [outer_max]
  double* grad_norm;       // [outer_max]
  unsigned long long* stamp;  // [outer_max+1] globaltimer ns
  int* state;
};

__global__ void finalize_kernel(FinalizeArgs f);
__global__ void stamp_kernel(unsigned long long* stamp);
__global__ void flush_kernel(float* buf, size_t n);

}  // namespace nsw
