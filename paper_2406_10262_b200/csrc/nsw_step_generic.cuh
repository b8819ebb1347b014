// Streaming fused step for shapes no on-chip tile holds (any n, any m):
// float64 beyond the parity tiles (e.g. config 4's 4000 x 51 in float64),
// m > 52, n > 8192.  Same contract as step_kernel (StepArgs, device phase
// machine, per-item impact terms, tolerance residual records), so the impact
// reduction, finalize, tolerance and exchange kernels are shared.
//
// One CTA per user (persistent over users), the user's K~ and the adjoint G
// in a per-CTA global scratch (L2-resident while the CTA works on it).
// Rows go to warps (lanes stride the row's columns: coalesced, butterfly
// sums, bitwise identical in every lane); column totals are thread-per-column
// sums over fixed row chunks combined in chunk order.  Every reduction has a
// fixed order, so results are run-to-run deterministic, and the forward and
// the backward's replay form u~ with the same row-dot function, so the
// replayed u~ are bit-identical to the forward's (as in step_kernel).
// Reference: sinkhorn.py:204-309, solver.py:186-240 (one user's slice).
#pragma once

#include "nsw_generic.h"
#include "nsw_step_kernel.cuh"

namespace nsw {

#ifndef NSW_REABS_EVERY
#define NSW_REABS_EVERY 8   // inner iterations between re-absorption checks
#endif

template <typename S>
struct GenScratch {
  S* base;        // [ctas][scratch_elems(n, m)]
  int n, m;
  __host__ __device__ static size_t elems(int n, int m) {
    return 2 * size_t(n) * m + 4 * size_t(n) + 10 * size_t(m) + 8;
  }
};

template <typename S>
__device__ __forceinline__ S gen_row_dot(const S* __restrict__ row, const S* __restrict__ vec, int m, int lane) {
  S s = S(0);
  for (int k = lane; k < m; k += 32) s = fma(row[k], vec[k], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

template <typename S>
__global__ void __launch_bounds__(GEN_NT) step_kernel_gen(const StepArgs<S> a, const GenScratch<S> g) {
  using F = Fp<S>;
  constexpr int NT = GEN_NT;
  constexpr int NW = NT / 32;
  __shared__ S part[NT];        // column-chunk partial sums
  __shared__ S redmax[NW];      // per-warp row residual maxima (tolerance mode)
  const int phase = a.state[ST_PHASE];
  if (phase == PHASE_FINISHED) return;
  const bool tolm = a.tol_mode != 0;
  const int T = a.T;
  const int Tprev = tolm ? a.state[ST_TSTAR] : T;
  const int Th = phase == PHASE_FWD_CONT ? a.state[ST_T0] : (phase == PHASE_FWD_FIN ? a.state[ST_TSTAR] : Tprev);
  const int n = a.n, m = a.m;
  const size_t nm = size_t(n) * m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  S* scr = g.base + size_t(blockIdx.x) * GenScratch<S>::elems(n, m);
  S* Kt = scr;                  // [n][m] K / K~ / gK
  S* G = Kt + nm;               // [n][m] adjoint
  S* ut = G + nm;               // [n] current u~
  S* sA = ut + n;               // [n] alpha -> u~^T
  S* hb = sA + n;               // [n] h of the level / seed g_u
  S* rv = hb + n;               // [n] scratch row values
  S* v0 = rv + n;               // [m] scaling vector / cv
  S* v1 = v0 + m;               // [m] beta
  S* v2 = v1 + m;               // [m] lvi of the next forward
  S* cr = v2 + m;               // [2][m] column residuals
  S* vT = cr + 2 * m;           // [m] v~^T
  S* ex = vT + m;               // [m] exposures (0 from column m-1 on)
  S* vpc = ex + m;              // [m] v~^{t-1} in the coordinates of level t (re-absorption)
  S* vppc = vpc + m;            // [m] v~^{t-2} likewise
  __shared__ int ev_flag;
  // column chunks: Q row ranges per column, Q * m <= NT
  const int Q = max(1, NT / m);
  auto mass = [&](int k) -> S { return k == m - 1 ? a.mass_dummy : S(1); };
  auto inv_mass = [&](int k) -> S { return k == m - 1 ? a.inv_mass_dummy : S(1); };
  auto rcp_clamped = [&](S x) -> S { return F::rcp_fast(fmax(x, F::tiny())); };
  auto ktilde = [&](S c, S beta_k, S alpha_i) -> S {
    return F::exp_fast(add_(add_(mul_(c, a.nie), beta_k), alpha_i));
  };
  auto gx_of = [&](S rr, S e, double imp) -> S {
    if constexpr (sizeof(S) == 4) return mul_(mul_(rr, e), S(1.0 / imp));
    else return F::div(mul_(rr, e), S(imp));
  };
  // sum_i f(i, k) for every column k: thread (q, k) sums its row chunk in
  // row order, the chunks are combined in chunk order; fin(k, total) on
  // thread k < m.  Ends with a barrier.
  auto col_sum = [&](auto f, auto fin) {
    for (int k0 = 0; k0 < m; k0 += NT) {
      const int span = min(m - k0, NT);
      const int q = min(Q, NT / span);
      const int k = k0 + tid % span, qi = tid / span;
      if (qi < q) {
        const int i0 = int((long long)n * qi / q), i1 = int((long long)n * (qi + 1) / q);
        S acc = S(0);
        for (int i = i0; i < i1; ++i) acc = f(i, k, acc);
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
  };

  for (int u = blockIdx.x; u < a.U; u += gridDim.x) {
    const size_t ub = size_t(u) * nm;
    S* Cu = a.C + ub;
    S* mu = a.am + ub;
    S* vu = a.av + ub;
    S* xb = a.xbest + ub;
    S* hu = a.hist + size_t(u) * (T + 1) * m;
    const S* relu = a.rel + size_t(u) * n;
    const bool rebuild = phase == PHASE_RUNNING || phase == PHASE_DONE_PENDING || phase == PHASE_FWD_CONT ||
                         phase == PHASE_FWD_FIN;
    for (int k = tid; k < m; k += NT) {
      v0[k] = S(0);
      v1[k] = rebuild ? a.beta[size_t(u) * m + k] : S(0);
      v2[k] = S(0);
      ex[k] = k < m - 1 ? a.expo[k] : S(0);
    }
    __syncthreads();
    bool forward_from_absorb = true;
    int t_start = 1;
    // re-absorption events of the solve being differentiated (fixed schedule)
    const bool reabs = a.reabs_max > 0 && !tolm;
    const int nev = (reabs && (phase == PHASE_RUNNING || phase == PHASE_DONE_PENDING)) ? a.ev_count[u] : 0;
    const int* evt = reabs ? a.ev_t + size_t(u) * a.reabs_max : nullptr;
    const S* evab = reabs ? a.ev_ab + size_t(u) * a.reabs_max * (size_t(n) + m) : nullptr;
    if (rebuild) {
      // K~ of the solve being differentiated / continued
      for (size_t e = tid; e < nm; e += NT) {
        const int i = int(e / m), k = int(e - size_t(i) * m);
        Kt[e] = ktilde(Cu[e], v1[k], a.alpha[size_t(u) * n + i]);
      }
      for (int k = tid; k < m; k += NT) vT[k] = hu[size_t(Th) * m + k];
      __syncthreads();
      // u~^T = 1/(K~ v~^{T-1}) with the forward's own row dot
      for (int i = warp; i < n; i += NW) {
        const S d = gen_row_dot(Kt + size_t(i) * m, hu + size_t(Th - 1) * m, m, lane);
        if (lane == 0) sA[i] = F::rcp_fast(d);
      }
      __syncthreads();
      const int improved = a.state[ST_IMPROVED];
      auto write_policy = [&]() {
        for (size_t e = tid; e < nm; e += NT) {
          const int i = int(e / m), k = int(e - size_t(i) * m);
          xb[e] = mul_(mul_(Kt[e], sA[i]), vT[k]);
        }
      };
      if (phase == PHASE_DONE_PENDING) {
        if (improved) write_policy();
        __syncthreads();
        continue;
      }
      if (phase == PHASE_FWD_FIN) {
        for (int i = tid; i < n; i += NT) {
          const double rr = double(relu[i]);
          double acc = 0.0;
          for (int k = 0; k < m - 1; ++k)
            acc = fma(rr * a.expo_d[k], double(mul_(mul_(Kt[size_t(i) * m + k], sA[i]), vT[k])), acc);
          a.partial[size_t(u) * n + i] = acc;
        }
        __syncthreads();
        continue;
      }
      if (phase == PHASE_FWD_CONT) {
        for (int k = tid; k < m; k += NT) v0[k] = vT[k];
        for (int i = tid; i < n; i += NT) ut[i] = S(0);
        __syncthreads();
        forward_from_absorb = false;
        t_start = Th + 1;
      } else {
        if (improved) write_policy();
        // ---- seed W = gx .* X (sinkhorn.py:272-275): g_u = W 1, cv^T = v~^T (W' 1) / colmass
        for (int i = tid; i < n; i += NT) {
          const S rr = relu[i];
          const double imp = a.imp[i];
          S gsum = S(0);
          for (int k = 0; k < m - 1; ++k)
            gsum += mul_(gx_of(rr, ex[k], imp), mul_(mul_(Kt[size_t(i) * m + k], sA[i]), vT[k]));
          hb[i] = gsum;
          ut[i] = sA[i];
        }
        for (size_t e = tid; e < nm; e += NT) G[e] = S(0);
        col_sum(
            [&](int i, int k, S acc) -> S {
              if (k >= m - 1) return acc;
              return acc + mul_(gx_of(relu[i], ex[k], a.imp[i]), mul_(mul_(Kt[size_t(i) * m + k], sA[i]), vT[k]));
            },
            [&](int k, S tot) { v0[k] = mul_(mul_(vT[k], tot), inv_mass(k)); });
        // lvi of the next forward, from the final coordinates (before any crossing)
        for (int k = tid; k < m; k += NT) v2[k] = a.warm_start ? add_(v1[k], F::log_(vT[k])) : S(0);
        // ---- reverse levels t = Th..1 (sinkhorn.py:276-308), as in step_kernel
        for (int t = Th; t >= 1; --t) {
          const bool first = t == Th, last = t == 1;
          const S* vp = hu + size_t(t - 1) * m;                 // v~^{t-1}
          const S* vpp = hu + size_t(last ? 0 : t - 2) * m;     // v~^{t-2}
          if (nev > 0) {
            // history rows recorded before an event at t-1 / t-2 are in older
            // coordinates than level t's: v~ / b of every event in [row, t)
            bool cv1 = false, cv2 = false;
            for (int e = 0; e < nev; ++e) {
              cv1 |= evt[e] == t - 1;
              cv2 |= !last && (evt[e] == t - 1 || evt[e] == t - 2);
            }
            if (cv1 || cv2) {
              for (int k = tid; k < m; k += NT) {
                S x1 = vp[k], x2 = last ? S(1) : vpp[k];
                for (int e = 0; e < nev; ++e) {
                  const S b = evab[size_t(e) * (n + m) + n + k];
                  if (evt[e] == t - 1) {
                    x1 = F::div(x1, b);
                    if (!last) x2 = F::div(x2, b);
                  }
                  if (!last && evt[e] == t - 2) x2 = F::div(x2, b);
                }
                vpc[k] = x1;
                vppc[k] = x2;
              }
              __syncthreads();
              if (cv1) vp = vpc;
              if (cv2) vpp = vppc;
            }
          }
          for (int i = warp; i < n; i += NW) {
            const S* row = Kt + size_t(i) * m;
            const S sig = gen_row_dot(row, v0, m, lane);
            const S den = last ? S(1) : gen_row_dot(row, vpp, m, lane);
            const S uu = ut[i];
            const S h = uu * (first ? hb[i] - uu * sig : -(uu * sig));
            S* gr = G + size_t(i) * m;
            for (int k = lane; k < m; k += 32) {
              S x = fma(v0[k], -uu, gr[k]);
              gr[k] = fma(vp[k], -h, x);
            }
            __syncwarp();
            if (lane == 0) {
              rv[i] = h;
              if (!last) ut[i] = rcp_clamped(den);
            }
          }
          __syncthreads();
          if (!last) {
            col_sum([&](int i, int k, S acc) -> S { return fma(Kt[size_t(i) * m + k], rv[i], acc); },
                    [&](int k, S tot) {
                      const S vpk = vp[k];
                      const S gv = -mul_(vpk, tot);
                      v0[k] = mul_(mul_(vpk, gv), inv_mass(k));
                    });
          }
          // crossing an event at t-1 (going down): back to the older coordinates,
          // K~ / (a b'), G * (a b') (K~ .* G invariant), cv * b, u~ * a, and the
          // seed's u~^T / v~^T likewise (they end in the first solve coordinates)
          for (int e = 0; e < nev; ++e)
            if (evt[e] == t - 1 && t > 1) {
              const S* ea = evab + size_t(e) * (n + m);
              const S* eb = ea + n;
              for (size_t q = tid; q < nm; q += NT) {
                const int i = int(q / m), k = int(q - size_t(i) * m);
                const S f = mul_(ea[i], eb[k]);
                Kt[q] = F::div(Kt[q], f);
                G[q] = mul_(G[q], f);
              }
              for (int i = tid; i < n; i += NT) {
                ut[i] = mul_(ut[i], ea[i]);
                sA[i] = mul_(sA[i], ea[i]);
              }
              for (int k = tid; k < m; k += NT) {
                v0[k] = mul_(v0[k], eb[k]);
                vT[k] = mul_(vT[k], eb[k]);
              }
              __syncthreads();
            }
        }
        // ---- gK = W + K~ .* G (into G), lvi of the next forward
        for (size_t e = tid; e < nm; e += NT) {
          const int i = int(e / m), k = int(e - size_t(i) * m);
          const S kk = Kt[e];
          const S X = mul_(mul_(kk, sA[i]), vT[k]);
          const S W = k < m - 1 ? mul_(gx_of(relu[i], ex[k], a.imp[i]), X) : S(0);
          G[e] = fma(kk, G[e], W);
        }
        __syncthreads();
        // ---- g_C = gK (-1/eps); Adam ascent (solver.py:105-122); K = C (-1/eps)
        const int s = a.state[ST_STEP];
        const S bc1 = S(a.bc[2 * s]), bc2 = S(a.bc[2 * s + 1]);
        const S ibc1 = S(1.0 / a.bc[2 * s]), ibc2 = S(1.0 / a.bc[2 * s + 1]);
        for (size_t e = tid; e < nm; e += NT) {
          const S gg = mul_(G[e], a.nie);
          S mm = add_(mul_(a.b1, mu[e]), mul_(a.omb1, gg));
          S vv = add_(mul_(a.b2, vu[e]), mul_(mul_(a.omb2, gg), gg));
          S mh, vhat;
          if constexpr (sizeof(S) == 4) {
            mh = mul_(mm, ibc1);
            vhat = mul_(vv, ibc2);
          } else {
            mh = F::div(mm, bc1);
            vhat = F::div(vv, bc2);
          }
          const S c = add_(Cu[e], fdiv_<S>(mul_(a.lr, mh), add_(fsqrt_<S>(vhat), a.aeps)));
          Cu[e] = c;
          mu[e] = mm;
          vu[e] = vv;
          Kt[e] = mul_(c, a.nie);
        }
        __syncthreads();
      }
    } else {
      // INIT: C0 = -eps log(uniform) (solver.py:176-177), lvi = 0; RESUME: the caller's C and lvi
      const bool init = phase == PHASE_INIT;
      if (!init)
        for (int k = tid; k < m; k += NT) v2[k] = a.beta[size_t(u) * m + k];
      for (size_t e = tid; e < nm; e += NT) {
        const int k = int(e % size_t(m));
        S c;
        if (init) {
          c = k == m - 1 ? a.c_dummy : a.c_real;
          Cu[e] = c;
          mu[e] = S(0);
          vu[e] = S(0);
        } else {
          c = Cu[e];
        }
        Kt[e] = mul_(c, a.nie);
      }
      __syncthreads();
    }

    // ======================= forward ============================================
    if (forward_from_absorb) {
      for (int k = tid; k < m; k += NT) {
        a.beta[size_t(u) * m + k] = v2[k];
        hu[k] = S(1);
        v0[k] = S(1);
      }
      for (int i = tid; i < n; i += NT) {
        S* row = Kt + size_t(i) * m;
        S mx = F::ninf();
        for (int k = 0; k < m; ++k) mx = fmax(mx, add_(row[k], v2[k]));
        const S al = -mx;
        a.alpha[size_t(u) * n + i] = al;
        for (int k = 0; k < m; ++k) row[k] = F::exp_fast(add_(add_(row[k], v2[k]), al));
        ut[i] = S(0);
      }
      __syncthreads();
    }
    const int t_end = tolm ? min(t_start - 1 + a.chunk, T) : T;
    int nev_fwd = 0;
    for (int t = t_start; t <= t_end; ++t) {
      S wmax = S(0);
      for (int i = warp; i < n; i += NW) {
        const S sr = gen_row_dot(Kt + size_t(i) * m, v0, m, lane);
        if (tolm) wmax = fmax(wmax, fabs(ut[i] * sr - S(1)));
        __syncwarp();
        if (lane == 0) ut[i] = rcp_clamped(sr);
      }
      if (tolm && lane == 0) redmax[warp] = wmax;
      __syncthreads();
      col_sum([&](int i, int k, S acc) -> S { return fma(Kt[size_t(i) * m + k], ut[i], acc); },
              [&](int k, S tot) {
                const S vn = F::div_fast(mass(k), tot);
                v0[k] = vn;
                hu[size_t(t) * m + k] = vn;
                if (tolm) cr[(t & 1) * m + k] = sizeof(S) == 8 ? fabs(vn * tot - mass(k)) : S(0);
              });
      if (tolm && tid == 0 && t > t_start) {
        S r = S(0);
        for (int w = 0; w < NW; ++w) r = fmax(r, redmax[w]);
        for (int kk = 0; kk < m; ++kk) r = fmax(r, cr[((t - 1) & 1) * m + kk]);
        a.res[size_t(u) * (T + 1) + t - 1] = double(r);
      }
      // in-solve re-absorption: once the column scalings leave +-reabs_thr nats,
      // fold them into K~ (beta += log v~) and re-normalise the rows (alpha += log a);
      // v~^t stays recorded in the old coordinates, later iterations in the new
      if (reabs && (t % NSW_REABS_EVERY) == 0 && t >= 2 && t <= T - 2 && nev_fwd < a.reabs_max) {
        if (tid == 0) {
          S mx = S(0);
          for (int k = 0; k < m; ++k) mx = fmax(mx, fabs(F::log_(v0[k])));
          ev_flag = double(mx) > a.reabs_thr;
        }
        __syncthreads();
        if (ev_flag) {
          S* ea = a.ev_ab + (size_t(u) * a.reabs_max + nev_fwd) * (size_t(n) + m);
          for (int i = tid; i < n; i += NT) {
            S* row = Kt + size_t(i) * m;
            S mx = S(0);
            for (int k = 0; k < m; ++k) {
              row[k] = mul_(row[k], v0[k]);
              mx = fmax(mx, row[k]);
            }
            const S ai = F::rcp_fast(mx);
            for (int k = 0; k < m; ++k) row[k] = mul_(row[k], ai);
            ea[i] = ai;
            a.alpha[size_t(u) * n + i] = add_(a.alpha[size_t(u) * n + i], F::log_(ai));
          }
          __syncthreads();   // every row has used v~ before it is reset
          for (int k = tid; k < m; k += NT) {
            ea[n + k] = v0[k];
            a.beta[size_t(u) * m + k] = add_(a.beta[size_t(u) * m + k], F::log_(v0[k]));
            v0[k] = S(1);
          }
          if (tid == 0) a.ev_t[size_t(u) * a.reabs_max + nev_fwd] = t;
          ++nev_fwd;
          __syncthreads();
        }
      }
    }
    if (reabs && tid == 0) a.ev_count[u] = nev_fwd;
    if (tolm) {
      S wmax = S(0);
      for (int i = warp; i < n; i += NW) {
        const S sr = gen_row_dot(Kt + size_t(i) * m, v0, m, lane);
        wmax = fmax(wmax, fabs(ut[i] * sr - S(1)));
      }
      if (lane == 0) redmax[warp] = wmax;
      __syncthreads();
      if (tid == 0) {
        S r = S(0);
        for (int w = 0; w < NW; ++w) r = fmax(r, redmax[w]);
        for (int kk = 0; kk < m; ++kk) r = fmax(r, cr[(t_end & 1) * m + kk]);
        a.res[size_t(u) * (T + 1) + t_end] = double(r);
      }
      __syncthreads();
      continue;
    }
    // per-item impact terms (solver.py:206), float64
    for (int i = tid; i < n; i += NT) {
      const double rr = double(relu[i]);
      const S uu = ut[i];
      double acc = 0.0;
      for (int k = 0; k < m - 1; ++k)
        acc = fma(rr * a.expo_d[k], double(mul_(mul_(Kt[size_t(i) * m + k], uu), v0[k])), acc);
      a.partial[size_t(u) * n + i] = acc;
    }
    __syncthreads();
  }
}

}  // namespace nsw
