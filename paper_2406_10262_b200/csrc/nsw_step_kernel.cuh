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

// 16-byte vector of scalars (float4 / double2) for coalesced tile traffic.
template <typename S>
union V16 {
  typename std::conditional<sizeof(S) == 4, float4, double2>::type v;
  S s[16 / sizeof(S)];
};

template <typename S, int M, int R, int NT>
__host__ __device__ constexpr size_t step_smem_bytes(int T) {
  constexpr int P = Pitch<S, M>::value;
  return sizeof(S) * (size_t(NT) * R * P + size_t(T + 1) * P + size_t(NT / 32) * P + 3 * P + 2 * size_t(NT) * R);
}

// Structure: the per-step phases that touch every cell once move the user's
// contiguous [n][m] tiles between HBM and the shared-memory tile Kt with
// coalesced 16-byte accesses (element-wise phases: K~ rebuild, Adam, the
// policy write) or as runtime loops over this thread's rows (seed, log-domain
// iteration 1); only the two hot loops (forward iterations 2..T and the T
// reverse levels) hold the R x M tile in registers.
template <typename S, int M, int R, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) step_kernel(const StepArgs<S> a) {
  using F = Fp<S>;
  constexpr int P = Pitch<S, M>::value;
  constexpr int NW = NT / 32;
  constexpr int V = 16 / sizeof(S);
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
  S* rowA = vec2 + P;                       // [NT*R] alpha, then u~^T, then u^1
  S* rowB = rowA + size_t(NT) * R;          // [NT*R] seed g_u per row

  const int phase = a.state[ST_PHASE];
  if (phase == PHASE_FINISHED) return;

  const int u = blockIdx.x;
  const int tid = threadIdx.x;
  const int n = a.n, m = a.m;
  const int nm = n * m;
  const bool vec_ok = (nm % V) == 0;   // user tiles are 16-byte aligned
  const size_t ubase = size_t(u) * nm;
  S* Cu = a.C + ubase;
  S* mu = a.am + ubase;
  S* vu = a.av + ubase;
  S* xb = a.xbest + ubase;
  S* hu = a.hist + size_t(u) * (T + 1) * m;
  const S* relu = a.rel + size_t(u) * n;
  auto ok = [&](int r) { return tid + r * NT < n; };
  auto mass = [&](int k) -> S { return k == m - 1 ? a.mass_dummy : S(1); };
  auto inv_mass = [&](int k) -> S { return k == m - 1 ? F::rcp(a.mass_dummy) : S(1); };
  auto kt = [&](int e) -> S& { const int i = e / m; return Kt[i * P + (e - i * m)]; };
  // element-wise, coalesced visit of the user's [n][m] tile: f(e, vector slot)
  auto foreach_cell = [&](auto&& f) {
    if (vec_ok) {
      for (int q = tid; q < nm / V; q += NT) f(q * V, q);
    } else {
      for (int e = tid; e < nm; e += NT) f(e, -1);
    }
  };

  // zero the tile (padding rows / columns must stay 0) and the small vectors
  for (int q = tid; q < NT * R * P / V; q += NT) reinterpret_cast<V16<S>*>(Kt)[q].v = V16<S>{}.v;
  if (tid < P) {
    vec0[tid] = S(0);
    vec1[tid] = S(0);
    vec2[tid] = S(0);
  }
  S ex[M];
#pragma unroll
  for (int k = 0; k < M; ++k) ex[k] = (k < m - 1) ? a.expo[(k < m - 1) ? k : 0] : S(0);
  __syncthreads();

  if (phase == PHASE_RUNNING || phase == PHASE_DONE_PENDING) {
    // ---------------- rebuild K~ of step k-1 from C, alpha, beta ------------
    if (tid < m) vec1[tid] = a.beta[size_t(u) * m + tid];
    for (int i = tid; i < n; i += NT) rowA[i] = a.alpha[size_t(u) * n + i];
    for (int idx = tid; idx < (T + 1) * P; idx += NT) {
      const int t = idx / P, k = idx - t * P;
      vh[idx] = k < m ? hu[size_t(t) * m + k] : S(0);
    }
    __syncthreads();
    foreach_cell([&](int e0, int q) {
      S c[V];
      const int cnt = q >= 0 ? V : 1;
      if (q >= 0) {
        V16<S> t;
        t.v = reinterpret_cast<const V16<S>*>(Cu)[q].v;
#pragma unroll
        for (int j = 0; j < V; ++j) c[j] = t.s[j];
      } else {
        c[0] = Cu[e0];
      }
      int i = e0 / m, k = e0 - i * m;
      for (int j = 0; j < cnt; ++j) {
        Kt[i * P + k] = F::exp_(add_(add_(mul_(c[j], a.nie), rowA[i]), vec1[k]));
        if (++k == m) { k = 0; ++i; }
      }
    });
    __syncthreads();
    S vT[M];
    lds_vec<S, M>(vT, vh + size_t(T) * P);
    {
      S vT1[M];
      lds_vec<S, M>(vT1, vh + size_t(T >= 2 ? T - 1 : 0) * P);
#pragma unroll 1
      for (int i = tid; i < NT * R; i += NT) {
        S kr[M];
        lds_vec<S, M>(kr, Kt + size_t(i) * P);
        rowA[i] = i < n ? ((T >= 2) ? F::rcp_fast(rdot<S, M>(kr, vT1)) : S(1)) : S(0);   // u~^T
      }
    }
    const int improved = a.state[ST_IMPROVED];
    auto write_policy = [&]() {   // X = diag(u~^T) K~ diag(v~^T), coalesced
      foreach_cell([&](int e0, int q) {
        int i = e0 / m, k = e0 - i * m;
        if (q >= 0) {
          V16<S> t;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            t.s[j] = mul_(mul_(Kt[i * P + k], rowA[i]), vh[size_t(T) * P + k]);
            if (++k == m) { k = 0; ++i; }
          }
          reinterpret_cast<V16<S>*>(xb)[q].v = t.v;
        } else {
          xb[e0] = mul_(mul_(Kt[i * P + k], rowA[i]), vh[size_t(T) * P + k]);
        }
      });
    };
    if (phase == PHASE_DONE_PENDING) {
      // the stop fired after step k-1's forward: only its policy is still owed
      if (improved) {
        __syncthreads();
        write_policy();
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
        S kr[M];
        lds_vec<S, M>(kr, Kt + size_t(i) * P);
        const S uT = rowA[i];
        const S rr = i < n ? relu[i] : S(0);
        const S imp_i = i < n ? S(a.imp[i]) : S(1);
        S gsum = S(0);
#pragma unroll
        for (int k = 0; k < M; ++k) {
          if (k < m - 1) {
            const S X = mul_(mul_(kr[k], uT), vT[k]);
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
    if (improved) write_policy();   // best-so-far policy is step k-1's (solver.py:217-219)

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
        S cv[M], c[M], h[R], un[R];
        lds_vec<S, M>(cv, vec0);
        const bool first = t == T;
        const bool replay = t >= 3;
#pragma unroll
        for (int k = 0; k < M; ++k) c[k] = S(0);
        {
          S vpp[M];
          lds_vec<S, M>(vpp, vh + size_t(t >= 2 ? t - 2 : 0) * P);
#pragma unroll
          for (int r = 0; r < R; r += PAIR) {
            S kr[PAIR][M];
#pragma unroll
            for (int q = 0; q < PAIR; ++q) lds_vec<S, M>(kr[q], Kt + size_t(tid + (r + q) * NT) * P);
#pragma unroll
            for (int q = 0; q < PAIR; ++q) {
              const S sig = rdot<S, M>(kr[q], cv);
              const S den = rdot<S, M>(kr[q], vpp);
              const S gs = first ? rowB[tid + (r + q) * NT] : S(0);
              h[r + q] = ut[r + q] * (gs - ut[r + q] * sig);
              un[r + q] = ok(r + q) ? (replay ? F::rcp_fast(den) : S(1)) : S(0);
            }
#pragma unroll
            for (int k = 0; k < M; ++k)
#pragma unroll
              for (int q = 0; q < PAIR; ++q) c[k] = fma(kr[q][k], h[r + q], c[k]);
          }
        }
        {
          S vp[M];
          lds_vec<S, M>(vp, vh + size_t(t - 1) * P);
#pragma unroll
          for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int k = 0; k < M; ++k) {
              A[r][k] = fma(-ut[r], cv[k], A[r][k]);
              A[r][k] = fma(-h[r], vp[k], A[r][k]);
            }
            ut[r] = un[r];
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
    if (tid < m) vec2[tid] = a.warm_start ? add_(vec1[tid], F::log_(vh[size_t(T) * P + tid])) : S(0);
    __syncthreads();

    // ---------------- g_C = gK * (-1/eps); Adam ascent  (solver.py:105-122) -
    const int s = a.state[ST_STEP];
    const S bc1 = S(a.bc[2 * s]), bc2 = S(a.bc[2 * s + 1]);
    auto adam = [&](S& cc, S& mm, S& vv, S gk) {
      const S g = mul_(gk, a.nie);
      mm = add_(mul_(a.b1, mm), mul_(a.omb1, g));
      vv = add_(mul_(a.b2, vv), mul_(mul_(a.omb2, g), g));
      const S mh = F::div(mm, bc1);
      const S vhat = F::div(vv, bc2);
      cc = add_(cc, F::div(mul_(a.lr, mh), add_(F::sqrt_(vhat), a.aeps)));
    };
    foreach_cell([&](int e0, int q) {
      int i = e0 / m, k = e0 - i * m;
      if (q >= 0) {
        V16<S> c, mm, vv;
        c.v = reinterpret_cast<const V16<S>*>(Cu)[q].v;
        mm.v = reinterpret_cast<const V16<S>*>(mu)[q].v;
        vv.v = reinterpret_cast<const V16<S>*>(vu)[q].v;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          S& slot = Kt[i * P + k];
          adam(c.s[j], mm.s[j], vv.s[j], slot);
          slot = mul_(c.s[j], a.nie);
          if (++k == m) { k = 0; ++i; }
        }
        reinterpret_cast<V16<S>*>(Cu)[q].v = c.v;
        reinterpret_cast<V16<S>*>(mu)[q].v = mm.v;
        reinterpret_cast<V16<S>*>(vu)[q].v = vv.v;
      } else {
        S c = Cu[e0], mm = mu[e0], vv = vu[e0];
        S& slot = Kt[i * P + k];
        adam(c, mm, vv, slot);
        slot = mul_(c, a.nie);
        Cu[e0] = c;
        mu[e0] = mm;
        vu[e0] = vv;
      }
    });
  } else {
    // INIT: initial cost C0 = -eps log(uniform) (solver.py:176-177), lvi = 0.
    // RESUME: caller-provided C (left as is), lvi taken from the beta buffer.
    const bool init = phase == PHASE_INIT;
    if (!init && tid < m) vec2[tid] = a.beta[size_t(u) * m + tid];
    foreach_cell([&](int e0, int q) {
      int i = e0 / m, k = e0 - i * m;
      if (q >= 0) {
        V16<S> c;
        if (init) {
#pragma unroll
          for (int j = 0; j < V; ++j) {
            c.s[j] = (k == m - 1) ? a.c_dummy : a.c_real;
            Kt[i * P + k] = mul_(c.s[j], a.nie);
            if (++k == m) { k = 0; ++i; }
          }
          reinterpret_cast<V16<S>*>(Cu)[q].v = c.v;
          reinterpret_cast<V16<S>*>(mu)[q].v = V16<S>{}.v;
          reinterpret_cast<V16<S>*>(vu)[q].v = V16<S>{}.v;
        } else {
          c.v = reinterpret_cast<const V16<S>*>(Cu)[q].v;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            Kt[i * P + k] = mul_(c.s[j], a.nie);
            if (++k == m) { k = 0; ++i; }
          }
        }
      } else {
        S c0;
        if (init) {
          c0 = (k == m - 1) ? a.c_dummy : a.c_real;
          Cu[e0] = c0;
          mu[e0] = S(0);
          vu[e0] = S(0);
        } else {
          c0 = Cu[e0];
        }
        Kt[i * P + k] = mul_(c0, a.nie);
      }
    });
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
    for (int i = tid; i < n; i += NT) {
      S kr[M];
      lds_vec<S, M>(kr, Kt + size_t(i) * P);
      const S u1 = rowA[i];
      a.alpha[size_t(u) * n + i] = u1;
#pragma unroll
      for (int k = 0; k < M; ++k) kr[k] = (k < m) ? F::exp_(add_(add_(kr[k], u1), bt[k])) : S(0);
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
      const S vn = F::div_fast(mass(k), tot);
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
