// Paired persistent cluster tile of the fused outer step (fixed schedule,
// float32, PHASE_RUNNING) -- an EXPERIMENT, opt-in with NSW_CL_PAIR=1: it
// hides the cluster tile's column exchange but runs config 4 5 % slower than
// step_kernel_cl (profiles/r02/ab_cluster_paired.txt has the numbers and why).
//
// step_kernel_cl spends about half of a config-4 step waiting for the 400
// DSMEM exchanges of one user's 2 x T serial reductions.  Here a cluster
// stays resident and walks its own list of users as a two-stage software
// pipeline: while user Y = users[s] runs its reverse sweep (level T+1-t),
// user X = users[s-1] -- whose backward and Adam finished one stage earlier
// -- runs forward iteration t.  The two chains are independent, so each one's
// exchange is in flight while the other computes:
//
//   F: row dots + column partials of X          collect Y's totals (posted one phase ago)
//   -- CTA barrier A --                          push X's CTA totals to every rank
//   B: level of Y (replay dots, adjoint update) collect X's totals
//   -- CTA barrier B --                          push Y's CTA totals
//
// Two CTA barriers per (iteration + level) instead of four, and no thread
// waits on an exchange younger than one compute phase.  Per SM: both users'
// K~ tiles in shared memory (2 x 93 KB at 448 items x 52 columns), Y's adjoint
// G in registers; X's K~ segments are re-read every iteration, because G and
// K~ of two users plus a level's working set do not fit 255 registers (that
// build spilled 176 bytes and ran 20 % slower).  This is what loses: the
// one-user kernel keeps K~ AND G in registers, and reading K~ from shared
// memory in both phases costs more issue time than the hidden exchange saves.
// Arithmetic, reduction orders and the exchange mechanism are those of
// step_kernel_cl: results are bit-identical to it (tests/test_gpu_cluster.py).
// Every other phase (INIT, RESUME, DONE_PENDING, the tolerance schedule) stays
// on step_kernel_cl, which skips PHASE_RUNNING when StepArgs::pair_mode is set.
#pragma once

#include "nsw_step_cluster.cuh"

namespace nsw {

template <typename S, int MC, int CG, int R, int NT, int CL>
struct Cl2Layout {
  using Tl = ClTile<S, MC, CG, R, NT, CL>;
  static constexpr int P = Tl::P, NR = Tl::NR, NW = Tl::NW;
  // one user's vectors (S elements from the slot base); every offset is a
  // whole number of 16-byte units
  static constexpr int O_VR = 0;                  // [4][P] ring of v~ history rows
  static constexpr int O_VTR = O_VR + 4 * P;      // [P] v~^T of the solve being differentiated
  static constexpr int O_RED = O_VTR + P;         // [NW][P] per-warp column partials
  static constexpr int O_VEC0 = O_RED + NW * P;   // [P] the chain's current column vector
  static constexpr int O_VEC1 = O_VEC0 + P;       // [P] beta of the previous step
  static constexpr int O_VEC2 = O_VEC1 + P;       // [P] beta of this step
  static constexpr int O_ROWA = O_VEC2 + P;       // [NR] alpha, then u~^T
  static constexpr int O_ROWB = O_ROWA + NR;      // [NR] seed row sums
  static constexpr int O_XCH = O_ROWB + NR;       // [2][CL][P] exchange slots
  static constexpr int SLOT = O_XCH + 2 * CL * P;
  static_assert(P % 4 == 0 && NR % 4 == 0 && Tl::KT % 4 == 0, "16-byte units");
  static constexpr size_t bytes() { return sizeof(S) * (2 * size_t(Tl::KT) + 2 * size_t(SLOT)) + 4 * 8 + 16; }
};

template <typename S, int MC, int CG, int R, int NT, int CL>
__host__ __device__ constexpr size_t cl2_smem_bytes(int) {
  return Cl2Layout<S, MC, CG, R, NT, CL>::bytes();
}

template <typename S, int MC, int CG, int R, int NT, int CL>
__global__ void __launch_bounds__(NT, 1) step_kernel_cl2(const StepArgs<S> a) {
  static_assert(sizeof(S) == 4 && CL > 1, "float32 cluster tiles only");
  using F = Fp<S>;
  using Tl = ClTile<S, MC, CG, R, NT, CL>;
  using L = Cl2Layout<S, MC, CG, R, NT, CL>;
  constexpr int P = Tl::P, RG = Tl::RG, NR = Tl::NR, NW = Tl::NW, SP = Tl::SP, KP = Tl::KP;
  constexpr int V = 16 / sizeof(S);
  namespace cg = cooperative_groups;
  if (a.state[ST_PHASE] != PHASE_RUNNING) return;   // every CTA of every cluster alike
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  nsw_poison_smem(smem_raw);
  S* const Kt0 = reinterpret_cast<S*>(smem_raw);
  S* const sl0 = Kt0 + 2 * size_t(Tl::KT);
  uint64_t* const xmb = reinterpret_cast<uint64_t*>(sl0 + 2 * size_t(L::SLOT));   // [slot][parity]
  auto Ktof = [&](int si) -> S* { return Kt0 + size_t(si) * Tl::KT; };
  auto slof = [&](int si) -> S* { return sl0 + size_t(si) * L::SLOT; };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(xmb + q)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int q = tid; q < 2 * Tl::KT + 2 * L::SLOT; q += NT) Kt0[q] = S(0);
  cluster.sync();   // every CTA's mbarriers exist before anyone pushes

  const int T = a.T;
  const int rank = int(cluster.block_rank());
  const int g = tid % CG, rg = tid / CG;
  const int n = a.n, m = a.m;
  const int r0 = rank * NR;                           // first item of this CTA
  const int nloc = max(0, min(NR, n - r0));           // items of this CTA
  const int ncell = nloc * m;
  const bool vec_ok = (size_t(n) * m % V == 0) && (size_t(NR) * m % V == 0);
  const int cid = int(blockIdx.x) / CL, NC = int(gridDim.x) / CL;
  const int nu = cid < a.U ? (a.U - cid + NC - 1) / NC : 0;   // users of this cluster: cid, cid + NC, ...
  auto user = [&](int k) { return a.user0 + cid + k * NC; };
  auto lrow = [&](int r) { return rg + r * RG; };
  auto kx = [&](int i, int k) {   // cell (item i, column k)
    const int gg = k / MC, j = k - gg * MC;
    return j < Tl::MCM ? i * KP + gg * SP + j : NR * KP + (i * CG + gg) * Tl::TL + (j - Tl::MCM);
  };
  auto ok = [&](int r) { return lrow(r) < nloc; };
  auto col = [&](int j) { return g * MC + j; };
  auto mass = [&](int k) -> S { return k == m - 1 ? a.mass_dummy : S(1); };
  auto inv_mass = [&](int k) -> S { return k == m - 1 ? a.inv_mass_dummy : S(1); };
  auto ktilde = [&](S c, S beta_k, S alpha_i) -> S {
    return F::exp_fast(add_(add_(mul_(c, a.nie), beta_k), alpha_i));
  };
  auto gx_of = [&](S rr, S e, S inv_imp) -> S { return mul_(mul_(rr, e), inv_imp); };
  auto ubase = [&](int u) { return size_t(u) * n * m + size_t(r0) * m; };

  // ---- column exchange, per slot si (its own slots, mbarriers, parity) ----
  uint32_t par = 0;   // bit si: buffer of slot si's next exchange
  uint32_t xph = 0;   // bit 2 si + p: mbarrier phase of slot si, buffer p
  // part 1 (before a CTA barrier): per-warp partials -> red
  auto stage_cols = [&](S (&v)[MC], S* sb) {
    int base = 0, lim = MC;
    rs_rows<S, MC, MC, 16, CG, OpSum>(v, lane, base, lim);
    constexpr int CF = rs_final_count<MC, 16, CG>();
    S* red = sb + L::O_RED;
#pragma unroll
    for (int j = 0; j < CF; ++j) {
      const int c = g * MC + base + j;
      if (base + j < lim && c < m) red[warp * P + c] = v[j];
    }
  };
  // part 2 (after it): thread q sums columns [4q, 4q+4) over the warps (warp
  // order) and pushes them as one 16-byte st.async to every CTA
  auto push_cols = [&](int si, S* sb) {
    const int p = (par >> si) & 1;
    const uint32_t mb = smem_u32(xmb + 2 * si + p);
    const int ng = (m + V - 1) / V;
    if (tid == 0) cl_expect_tx(mb, uint32_t(CL * ng * 16));
    if (tid < ng) {
      const S* red = sb + L::O_RED;
      V16<S> tot4;
      tot4.v = reinterpret_cast<const V16<S>*>(red + tid * V)->v;
#pragma unroll
      for (int w = 1; w < NW; ++w) {
        V16<S> x;
        x.v = reinterpret_cast<const V16<S>*>(red + w * P + tid * V)->v;
#pragma unroll
        for (int e = 0; e < V; ++e) tot4.s[e] += x.s[e];
      }
      S mine[V];
#pragma unroll
      for (int e = 0; e < V; ++e) mine[e] = (tid * V + e < m) ? tot4.s[e] : S(0);
      const uint32_t slot = smem_u32(sb + L::O_XCH + (size_t(p) * CL + rank) * P + tid * V);
#pragma unroll
      for (int q = 0; q < CL; ++q) cl_st_async16(cl_map(slot, q), mine, cl_map(mb, q));
    }
  };
  // part 3: wait for every rank's totals, fixed-order sum, fin(k, total) on
  // thread k < m (no trailing barrier: the caller's next CTA barrier publishes)
  auto collect_cols = [&](int si, S* sb, auto&& fin) {
    const int p = (par >> si) & 1;
    if (tid < m) {
      mbar_wait(smem_u32(xmb + 2 * si + p), (xph >> (2 * si + p)) & 1u);
      const S* xch = sb + L::O_XCH + size_t(p) * CL * P;
      S tot = S(0);
#pragma unroll
      for (int q = 0; q < CL; ++q) tot += xch[q * P + tid];   // rank order
      fin(tid, tot);
    }
    xph ^= 1u << (2 * si + p);
    par ^= 1u << si;
  };
  auto reduce_cols = [&](S (&v)[MC], int si, S* sb, auto&& fin) {
    stage_cols(v, sb);
    __syncthreads();
    push_cols(si, sb);
    collect_cols(si, sb, fin);
    __syncthreads();
  };

  // exposure and v~^T segments are re-read where the seed and the gK pass need them
  auto load_ex = [&](S (&ex)[MC]) {
#pragma unroll
    for (int j = 0; j < MC; ++j) ex[j] = (col(j) < m - 1) ? a.expo[min(col(j), m - 2)] : S(0);
  };
  const int improved = a.state[ST_IMPROVED];
  const int step = a.state[ST_STEP];
  const S ibc1 = S(1.0 / a.bc[2 * step]), ibc2 = S(1.0 / a.bc[2 * step + 1]);

  for (int k0 = 0; k0 < nu; k0 += 2) {
    const bool hasB = k0 + 1 < nu;

    // ================= backward + Adam, one user after the other =================
    for (int w = 0; w < (hasB ? 2 : 1); ++w) {
      const int si = w;
      const int uY = user(k0 + w);
      S* const KtY = Ktof(si);
      S* const sbY = slof(si);
      S* const huY = a.hist + size_t(uY) * (T + 1) * m;
      const S* const reluY = a.rel + size_t(uY) * n + r0;
      S* const vrY = sbY + L::O_VR;
      S* const vTrY = sbY + L::O_VTR;
      S* const vec0Y = sbY + L::O_VEC0;
      S* const vec1 = sbY + L::O_VEC1;
      S* const vec2 = sbY + L::O_VEC2;
      S* const rowAY = sbY + L::O_ROWA;
      S* const rowBY = sbY + L::O_ROWB;
      S* const Cu = a.C + ubase(uY);
      auto vrow = [&](int t) -> S* { return vrY + (t & 3) * P; };
      auto load_row = [&](S* dst, int t) {
        for (int k = tid; k < P; k += NT) cp_async_zfill(dst + k, huY + size_t(t) * m + (k < m ? k : 0), k < m);
        cp_async_commit();
      };
      auto foreach_cell = [&](auto&& f) {
        if (vec_ok) {
          for (int q = tid; q < ncell / V; q += NT) f(q * V, q);
        } else {
          for (int e = tid; e < ncell; e += NT) f(e, -1);
        }
      };
      // ---- rebuild the previous step's K~, u~^T, policy, seed ----
      if (tid < m) vec1[tid] = a.beta[size_t(uY) * m + tid];
      for (int i = tid; i < nloc; i += NT) rowAY[i] = a.alpha[size_t(uY) * n + r0 + i];
      load_row(vTrY, T);
      load_row(vrow(T - 1), T - 1);
      if (T >= 2) load_row(vrow(T - 2), T - 2);
      cp_async_wait_all();
      __syncthreads();
      foreach_cell([&](int e0, int q) {
        int i = e0 / m, k = e0 - i * m;
        if (q >= 0) {
          V16<S> c;
          c.v = reinterpret_cast<const V16<S>*>(Cu)[q].v;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            KtY[kx(i, k)] = ktilde(c.s[j], vec1[k], rowAY[i]);
            if (++k == m) { k = 0; ++i; }
          }
        } else {
          KtY[kx(i, k)] = ktilde(Cu[e0], vec1[k], rowAY[i]);
        }
      });
      __syncthreads();
      {
        S vT1[MC];
#pragma unroll
        for (int j = 0; j < MC; ++j) vT1[j] = vrow(T - 1)[col(j)];
        for (int r = 0; r < R; ++r) {   // u~^T (all lanes of the group agree)
          S kr[MC];
          ld_seg<Tl, S, MC>(kr, KtY, lrow(r), g);
          const S uT = F::rcp_fast(rdot_g<S, MC, CG>(kr, vT1));
          __syncwarp();
          if (g == 0) rowAY[lrow(r)] = ok(r) ? uT : S(0);
        }
      }
      __syncthreads();
      if (improved) {
        S* const xb = a.xbest + ubase(uY);
        foreach_cell([&](int e0, int q) {
          int i = e0 / m, k = e0 - i * m;
          if (q >= 0) {
            V16<S> t;
#pragma unroll
            for (int j = 0; j < V; ++j) {
              t.s[j] = mul_(mul_(KtY[kx(i, k)], rowAY[i]), vTrY[k]);
              if (++k == m) { k = 0; ++i; }
            }
            reinterpret_cast<V16<S>*>(xb)[q].v = t.v;
          } else {
            xb[e0] = mul_(mul_(KtY[kx(i, k)], rowAY[i]), vTrY[k]);
          }
        });
      }
      S G[R][MC];    // adjoint of K~
      S Kr[R][MC];   // K~ row segments, register-resident for the whole sweep
      S ut[R];
      {
        // seed W = gx .* X
        S c[MC], ex[MC], vT[MC];
        load_ex(ex);
#pragma unroll
        for (int j = 0; j < MC; ++j) {
          c[j] = S(0);
          vT[j] = vTrY[col(j)];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int il = lrow(r);
          ld_seg<Tl, S, MC>(Kr[r], KtY, il, g);
          ut[r] = rowAY[il];
          const S rr = ok(r) ? reluY[il] : S(0);
          const S imp_i = ok(r) ? S(a.imp[r0 + il]) : S(1);
          const S inv_imp = S(1.0 / double(imp_i));
          S gsum = S(0);
#pragma unroll
          for (int j = 0; j < MC; ++j) {
            G[r][j] = S(0);
            if (col(j) < m - 1) {
              const S W = mul_(gx_of(rr, ex[j], inv_imp), mul_(mul_(Kr[r][j], ut[r]), vT[j]));
              gsum += W;
              c[j] += W;
            }
          }
          gsum = group_sum<S, CG>(gsum);
          if (g == 0) rowBY[il] = gsum;
        }
        reduce_cols(c, si, sbY, [&](int k, S tot) { vec0Y[k] = mul_(mul_(vTrY[k], tot), inv_mass(k)); });
      }
      // ---- reverse sweep (as step_kernel_cl: the exchange is exposed here) ----
      for (int t = T; t >= 1; --t) {
        if (t >= 3) load_row(vrow(t - 3), t - 3);
        S cv[MC], vp[MC], vpp[MC], c[MC];
        const S* rp = vrow(t - 1);
        const S* rpp = vrow(t >= 2 ? t - 2 : 0);
        const bool first = t == T;
#pragma unroll
        for (int j = 0; j < MC; ++j) {
          cv[j] = vec0Y[col(j)];
          vp[j] = rp[col(j)];
          vpp[j] = rpp[col(j)];
          c[j] = S(0);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int il = lrow(r);
          const S sig = rdot_g<S, MC, CG>(Kr[r], cv);
          const S den = rdot_g<S, MC, CG>(Kr[r], vpp);
          const S gs = first ? rowBY[il] : S(0);
          const S h = ut[r] * (gs - ut[r] * sig);
          axpy_<S, MC, true>(G[r], cv, -ut[r]);
          axpy_<S, MC, true>(G[r], vp, -h);
          axpy_<S, MC, true>(c, Kr[r], h);
          ut[r] = (ok(r) && t >= 2) ? F::rcp_fast(den) : S(0);
        }
        if (t >= 2) {
          cp_async_wait_all();   // row t-3 lands before the reduction's barrier publishes it
          reduce_cols(c, si, sbY, [&](int k, S tot) {
            const S vpk = rp[k];
            vec0Y[k] = mul_(mul_(vpk, -mul_(vpk, tot)), inv_mass(k));
          });
        }
      }
      // ---- gK = W + K~ .* G over the tile, then the Adam ascent ----
      {
        S ex[MC], vT[MC];
        load_ex(ex);
#pragma unroll
        for (int j = 0; j < MC; ++j) vT[j] = vTrY[col(j)];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int il = lrow(r);
          S gk[MC];
          const S uT = rowAY[il];
          const S rr = ok(r) ? reluY[il] : S(0);
          const S imp_i = ok(r) ? S(a.imp[r0 + il]) : S(1);
          const S inv_imp = S(1.0 / double(imp_i));
#pragma unroll
          for (int j = 0; j < MC; ++j) {
            const S W = (col(j) < m - 1) ? mul_(gx_of(rr, ex[j], inv_imp), mul_(mul_(Kr[r][j], uT), vT[j])) : S(0);
            gk[j] = fma(Kr[r][j], G[r][j], W);
          }
          st_seg<Tl, S, MC>(KtY, il, g, gk);
        }
      }
      if (tid < m) vec2[tid] = a.warm_start ? add_(vec1[tid], F::log_(vTrY[tid])) : S(0);
      __syncthreads();
      S* const mu = a.am + ubase(uY);
      S* const vu = a.av + ubase(uY);
      auto adam = [&](S& cc, S& mm, S& vv, S gk) {
        const S gg = mul_(gk, a.nie);
        mm = add_(mul_(a.b1, mm), mul_(a.omb1, gg));
        vv = add_(mul_(a.b2, vv), mul_(mul_(a.omb2, gg), gg));
        const S mh = mul_(mm, ibc1);
        const S vhat = mul_(vv, ibc2);
        cc = add_(cc, fdiv_<S>(mul_(a.lr, mh), add_(fsqrt_<S>(vhat), a.aeps)));
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
            S& slot = KtY[kx(i, k)];
            adam(c.s[j], mm.s[j], vv.s[j], slot);
            slot = mul_(c.s[j], a.nie);
            if (++k == m) { k = 0; ++i; }
          }
          reinterpret_cast<V16<S>*>(Cu)[q].v = c.v;
          reinterpret_cast<V16<S>*>(mu)[q].v = mm.v;
          reinterpret_cast<V16<S>*>(vu)[q].v = vv.v;
        } else {
          S c = Cu[e0], mm = mu[e0], vv = vu[e0];
          S& slot = KtY[kx(i, k)];
          adam(c, mm, vv, slot);
          slot = mul_(c, a.nie);
          Cu[e0] = c;
          mu[e0] = mm;
          vu[e0] = vv;
        }
      });
      __syncthreads();   // the tile now holds K = -C/eps of this user's forward
    }

    // ================= the two forwards, interleaved =================
    const int uA = user(k0), uB = hasB ? user(k0 + 1) : uA;
    S* const sbA = slof(0);
    S* const sbB = slof(1);
    S* const vec0A = sbA + L::O_VEC0;
    S* const vec0B = sbB + L::O_VEC0;
    S* const huA = a.hist + size_t(uA) * (T + 1) * m;
    S* const huB = a.hist + size_t(uB) * (T + 1) * m;
    S KA[R][MC], KB[R][MC];   // K~ row segments of the two users
    S utA[R], utB[R];
    // absorb beta = lvi, alpha = -rowmax(K + beta)
    auto absorb = [&](S (&K)[R][MC], S (&ut)[R], int u, const S* Kt, S* sb, S* hu) {
      const S* const vec2 = sb + L::O_VEC2;
      if (rank == 0 && tid < m) {
        a.beta[size_t(u) * m + tid] = vec2[tid];
        hu[tid] = S(1);
      }
      if (tid < m) sb[L::O_VEC0 + tid] = S(1);
      S bt[MC];
#pragma unroll
      for (int j = 0; j < MC; ++j) bt[j] = vec2[col(j)];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int il = lrow(r);
        ld_seg<Tl, S, MC>(K[r], Kt, il, g);
        S mx = F::ninf();
#pragma unroll
        for (int j = 0; j < MC; ++j)
          if (col(j) < m) mx = fmax(mx, add_(K[r][j], bt[j]));
        mx = group_max<S, CG>(mx);
        const S al = -mx;
        if (g == 0 && ok(r)) a.alpha[size_t(u) * n + r0 + il] = al;
#pragma unroll
        for (int j = 0; j < MC; ++j)
          K[r][j] = (ok(r) && col(j) < m) ? F::exp_fast(add_(add_(K[r][j], bt[j]), al)) : S(0);
        ut[r] = S(0);
      }
    };
    absorb(KA, utA, uA, Ktof(0), sbA, huA);
    if (hasB) {
      absorb(KB, utB, uB, Ktof(1), sbB, huB);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        utB[r] = S(0);
#pragma unroll
        for (int j = 0; j < MC; ++j) KB[r][j] = S(0);
      }
    }
    __syncthreads();
    // one forward iteration's compute: row dots, u~, column partials -> red
    auto fwd_compute = [&](const S (&K)[R][MC], S (&ut)[R], S* sb) {
      S vv[MC], c[MC];
      const S* vec0 = sb + L::O_VEC0;
#pragma unroll
      for (int j = 0; j < MC; ++j) vv[j] = vec0[col(j)];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const S rp = F::rcp_fast(rdot_g<S, MC, CG>(K[r], vv));
        ut[r] = ok(r) ? rp : S(0);
      }
#pragma unroll
      for (int j = 0; j < MC; ++j) c[j] = S(0);
#pragma unroll
      for (int r = 0; r < R; ++r) axpy_<S, MC, true>(c, K[r], ut[r]);
      stage_cols(c, sb);
    };
    auto fwd_collect = [&](int si, S* sb, S* hu, int t) {
      S* vec0 = sb + L::O_VEC0;
      collect_cols(si, sb, [&](int k, S tot) {
        const S vn = F::div_fast(mass(k), tot);
        vec0[k] = vn;
        if (rank == 0) hu[size_t(t) * m + k] = vn;
      });
    };
    // A's totals travel while B computes and vice versa: every collect comes
    // one compute phase after its push
    for (int t = 1; t <= T; ++t) {
      fwd_compute(KA, utA, sbA);
      if (hasB && t > 1) fwd_collect(1, sbB, huB, t - 1);
      __syncthreads();   // A's partials and B's v~ are published
      push_cols(0, sbA);
      if (hasB) fwd_compute(KB, utB, sbB);
      fwd_collect(0, sbA, huA, t);
      __syncthreads();   // B's partials and A's v~ are published
      if (hasB) push_cols(1, sbB);
    }
    if (hasB) fwd_collect(1, sbB, huB, T);
    __syncthreads();
    // per-item impact terms, float64, completed across the group
    auto impact = [&](const S (&K)[R][MC], const S (&ut)[R], int u, const S* sb) {
      S vv[MC];
#pragma unroll
      for (int j = 0; j < MC; ++j) vv[j] = sb[L::O_VEC0 + col(j)];
      const S* const relu = a.rel + size_t(u) * n + r0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int il = lrow(r);
        const double rr = ok(r) ? double(relu[il]) : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < MC; ++j)
          if (col(j) < m - 1)
            acc = fma(rr * a.expo_d[min(col(j), m - 2)], double(mul_(mul_(K[r][j], ut[r]), vv[j])), acc);
        acc = group_sum<double, CG>(acc);
        if (g == 0 && ok(r)) a.partial[size_t(u) * n + r0 + il] = acc;
      }
    };
    impact(KA, utA, uA, sbA);
    if (hasB) impact(KB, utB, uB, sbB);
    __syncthreads();   // the slots are free for the next two users
  }
  cluster.sync();   // keep every CTA's shared memory alive until remote pushes have landed
}

}  // namespace nsw
