// Cluster tile of the fused outer step, for users whose n x m tile does not
// fit one SM (BASELINE config 4: n = 4000, m = 51 -> 204k cells per user).
//
// A user is split over a thread-block cluster of CL CTAs (one per SM), each
// owning NR = (NT / CG) * R consecutive items.  Inside a CTA the mapping is
// two-dimensional: CG consecutive lanes share a row group and each owns MC of
// the (padded) MC * CG columns, so every per-thread vector has MC entries --
// a 1-D row-per-thread mapping would need 5 * 51 registers of vectors at
// m = 51.  Row sums finish with a log2(CG)-step xor butterfly across the
// group; column sums with a reduce-scatter over the row-group lanes, a
// fixed-order cross-warp sum and a fixed-order sum of the CL CTA totals read
// through distributed shared memory (every CTA computes the same bits).
// Numerics are identical in form to step_kernel (nsw_step_kernel.cuh).
// Fixed schedule only.
#pragma once

#include <cooperative_groups.h>

#include "nsw_step_kernel.cuh"

namespace nsw {

template <typename S, int MC, int CG, int R, int NT, int CL>
struct ClTile {
  static constexpr int MP = MC * CG;                                  // padded columns
  // column-vector pitch: >= MP + 1 (tolerance slot), whole 16-byte units
  static constexpr int P = (MP + 1 + 16 / int(sizeof(S)) - 1) / (16 / int(sizeof(S))) * (16 / int(sizeof(S)));
  static constexpr int RG = NT / CG;                                  // row groups per CTA
  static constexpr int NR = RG * R;                                   // items per CTA
  static constexpr int NW = NT / 32;
  // K~ tile layout: a lane's MC-column segment is split into its MCM = MC -
  // MC % VE leading columns, stored 16-byte aligned with an odd number of
  // 16-byte units per segment (the 8 lanes of a 128-bit load phase -- 2 row
  // groups x 4 segments -- hit distinct bank quads; KP = CG * SP per item
  // row), and its TL trailing columns, stored densely after the main block
  // ([NR][CG][TL]: the 32 lanes' scalar loads hit 32 consecutive words).
  static constexpr int VE = 16 / sizeof(S);
  static constexpr int MCM = MC / VE * VE;                            // vector-loaded columns
  static constexpr int TL = MC - MCM;                                 // trailing columns
  static constexpr int SPV = MCM / VE;                                // 16-byte units holding MCM
  static constexpr int SP = (SPV % 2 ? SPV : SPV + 1) * VE;           // segment pitch
  static constexpr int KP = CG * SP;                                  // item-row pitch (main block)
  static constexpr int KT = NR * KP + NR * CG * TL;                   // K~ tile elements
  static_assert(MCM > 0, "segment narrower than a 16-byte unit");
};

template <typename S, int MC, int CG, int R, int NT, int CL>
__host__ __device__ constexpr size_t cl_smem_bytes(int T) {
  using Tl = ClTile<S, MC, CG, R, NT, CL>;
  (void)T;   // the v~ history is streamed through a 4-row ring: shared memory does not grow with T
  return sizeof(S) * (size_t(Tl::KT) + 5 * size_t(Tl::P) + size_t(Tl::NW) * Tl::P + 3 * Tl::P +
                      2 * size_t(Tl::NR) + 2 * Tl::P + 4 + 2 * size_t(CL) * Tl::P + 2 * Tl::P + Tl::NW) +
         48;   // exchange slots [2][CL][P] + two mbarriers (8-byte aligned) + residual scratch
}

#ifndef NSW_EXP_XTIME
#define NSW_EXP_XTIME 0   // diagnostics only (see xstamp)
#endif

// DSMEM push exchange of the per-CTA column totals: every CTA stores its
// totals into slot [parity][its rank] of every CTA of the cluster with
// st.async, which completes bytes on the receiver's mbarrier; a receiver
// waits on its own mbarrier (no cluster-wide barrier per reduction).
__device__ __forceinline__ uint32_t cl_map(uint32_t local_saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_st_async(uint32_t raddr, float v, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rmbar)
               : "memory");
}
__device__ __forceinline__ void cl_st_async(uint32_t raddr, double v, uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rmbar)
               : "memory");
}
// 16-byte push (4 floats / 2 doubles of consecutive columns)
__device__ __forceinline__ void cl_st_async16(uint32_t raddr, const float (&v)[4], uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(rmbar)
               : "memory");
}
__device__ __forceinline__ void cl_st_async16(uint32_t raddr, const double (&v)[2], uint32_t rmbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "l"(__double_as_longlong(v[0])), "l"(__double_as_longlong(v[1])), "r"(rmbar)
               : "memory");
}
__device__ __forceinline__ void cl_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(mbar),
               "r"(bytes)
               : "memory");
}

// Reduce-scatter across the row-group lanes (xor offsets 16 .. CG).
template <typename S, int N, int CNT, int OFF, int CGM, class Op>
__device__ __forceinline__ void rs_rows(S (&v)[N], int lane, int& base, int& lim) {
  if constexpr (OFF >= CGM) {
    constexpr int H = (CNT + 1) / 2;
    const bool up = (lane & OFF) != 0;
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const S lo = v[j];
      const S hi = (j + H < CNT) ? v[(j + H < CNT) ? (j + H) : 0] : Op::template identity<S>();
      const S send = up ? lo : hi;
      const S keep = up ? hi : lo;
      v[j] = Op{}(keep, __shfl_xor_sync(0xffffffffu, send, OFF));
    }
    if (up) {
      base += H;
    } else {
      lim = min(lim, base + H);
    }
    rs_rows<S, N, H, OFF / 2, CGM, Op>(v, lane, base, lim);
  }
}

template <int CNT, int OFF, int CGM>
__host__ __device__ constexpr int rs_final_count() {
  if constexpr (OFF >= CGM) return rs_final_count<(CNT + 1) / 2, OFF / 2, CGM>();
  else return CNT;
}

template <typename S, int CG>
__device__ __forceinline__ S group_sum(S x) {
#pragma unroll
  for (int o = 1; o < CG; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <typename S, int CG>
__device__ __forceinline__ S group_max(S x) {
#pragma unroll
  for (int o = 1; o < CG; o <<= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Row dot of this lane's MC-column segment, completed across the group.
template <typename S, int MC, int CG>
__device__ __forceinline__ S rdot_g(const S (&x)[MC], const S (&y)[MC]) {
  return group_sum<S, CG>(rdot<S, MC, 2, true>(x, y));
}

// A lane's MC-column segment of one item row (16-byte aligned): vector
// loads / stores, the padding past MC ignored on load and left untouched.
// A lane's MC-column segment of item row il (main block: 16-byte vectors;
// trailing columns: scalars from the dense tail block).
template <typename Tl, typename S, int MC>
__device__ __forceinline__ void ld_seg(S (&dst)[MC], const S* Kt, int il, int g) {
  constexpr int VE = Tl::VE, MCM = Tl::MCM, TL = Tl::TL;
  const S* src = Kt + size_t(il) * Tl::KP + g * Tl::SP;
#pragma unroll
  for (int q = 0; q < MCM / VE; ++q) {
    V16<S> t;
    t.v = reinterpret_cast<const V16<S>*>(src)[q].v;
#pragma unroll
    for (int e = 0; e < VE; ++e) dst[q * VE + e] = t.s[e];
  }
  if constexpr (TL > 0) {
    const S* tl = Kt + size_t(Tl::NR) * Tl::KP + (size_t(il) * (Tl::KP / Tl::SP) + g) * TL;
#pragma unroll
    for (int e = 0; e < TL; ++e) dst[MCM + e] = tl[e];
  }
}

template <typename Tl, typename S, int MC>
__device__ __forceinline__ void st_seg(S* Kt, int il, int g, const S (&src)[MC]) {
  constexpr int VE = Tl::VE, MCM = Tl::MCM, TL = Tl::TL;
  S* dst = Kt + size_t(il) * Tl::KP + g * Tl::SP;
#pragma unroll
  for (int q = 0; q < MCM / VE; ++q) {
    V16<S> t;
#pragma unroll
    for (int e = 0; e < VE; ++e) t.s[e] = src[q * VE + e];
    reinterpret_cast<V16<S>*>(dst)[q].v = t.v;
  }
  if constexpr (TL > 0) {
    S* tl = Kt + size_t(Tl::NR) * Tl::KP + (size_t(il) * (Tl::KP / Tl::SP) + g) * TL;
#pragma unroll
    for (int e = 0; e < TL; ++e) tl[e] = src[MCM + e];
  }
}

template <typename S, int MC, int CG, int R, int NT, int CL, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) step_kernel_cl(const StepArgs<S> a) {
  using F = Fp<S>;
  using Tl = ClTile<S, MC, CG, R, NT, CL>;
  constexpr int P = Tl::P, RG = Tl::RG, NR = Tl::NR, NW = Tl::NW, SP = Tl::SP, KP = Tl::KP;
  constexpr int V = 16 / sizeof(S);
  static_assert(32 % CG == 0 && NT % 32 == 0, "tile shape");
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  nsw_poison_smem(smem_raw);
  const int T = a.T;
  S* Kt = reinterpret_cast<S*>(smem_raw);   // [NR][CG][SP] lane segments + [NR][CG][TL] tails
  S* vr = Kt + size_t(Tl::KT);             // [4][P] ring of v~ history rows (row t in slot t & 3)
  S* vTr = vr + 4 * P;                      // [P] row Th of the history (v~ of the solve being differentiated)
  S* red = vTr + P;                         // [NW][P]
  S* vec0 = red + NW * P;
  S* vec1 = vec0 + P;
  S* vec2 = vec1 + P;
  S* rowA = vec2 + P;                       // [NR]
  S* rowB = rowA + NR;                      // [NR]
  S* clred = rowB + NR;                     // [2][P] this CTA's column totals
  S* xch = clred + 2 * P;                   // [2][CL][P] exchange slots (pushed by every rank)
  uint64_t* xmb = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(xch + 2 * CL * P) + 7) & ~uintptr_t(7));
  S* colres = reinterpret_cast<S*>(xmb + 2);   // [2][P] column residuals (tolerance mode)
  S* rmw = colres + 2 * P;                      // [NW] per-warp row-residual maxima

  const int phase = a.state[ST_PHASE];
  if (phase == PHASE_FINISHED) {
    cluster.sync();
    return;
  }
  uint32_t xph = 0;   // mbarrier phase bit per exchange buffer
  if constexpr (CL > 1) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(xmb)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(xmb + 1)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();   // every CTA's mbarriers exist before anyone pushes
  }
  const bool tolm = a.tol_mode != 0;
  // length of the v~ history of the K~ this launch rebuilds (see step_kernel)
  const int Tprev = tolm ? a.state[ST_TSTAR] : T;
  const int Th = phase == PHASE_FWD_CONT ? a.state[ST_T0] : (phase == PHASE_FWD_FIN ? a.state[ST_TSTAR] : Tprev);
  const int rank = int(cluster.block_rank());
  const int u = a.user0 + int(blockIdx.x) / CL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = tid % CG, rg = tid / CG;
  const int n = a.n, m = a.m;
  const int r0 = rank * NR;                           // first item of this CTA
  const int nloc = max(0, min(NR, n - r0));           // items of this CTA
  const int ncell = nloc * m;
  const size_t ubase = size_t(u) * n * m + size_t(r0) * m;
  S* Cu = a.C + ubase;
  S* mu = a.am + ubase;
  S* vu = a.av + ubase;
  S* xb = a.xbest + ubase;
  S* hu = a.hist + size_t(u) * (T + 1) * m;
  const S* relu = a.rel + size_t(u) * n + r0;
  const bool vec_ok = (size_t(n) * m % V == 0) && (size_t(NR) * m % V == 0);
  int parity = 0;
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
  auto gx_of = [&](S rr, S e, S imp_i, S inv_imp) -> S {
    if constexpr (sizeof(S) == 4) return mul_(mul_(rr, e), inv_imp);
    else return F::div(mul_(rr, e), imp_i);
  };
  // column reduction over the whole cluster; fin(k, total) on thread k < m
  // of every CTA (identical bits everywhere)
  // xval: this CTA's row-residual max (tolerance mode) travels in slot m of
  // the exchange; the cluster maximum is returned in *xmax on thread m
  // split in two so independent work can run while the exchange is in
  // flight: post_cols (partials -> barrier -> warp sums -> DSMEM pushes) and
  // collect_cols (wait for every rank's totals -> fin -> barrier)
  // diagnostics (NSW_EXP_XTIME builds, scripts/cluster_skew.py): thread 0 of
  // every rank stamps its arrival at / completion of 24 exchanges of the
  // launch's first user into phase_ns
  int xcnt = 0;
  auto xstamp = [&](int which) {
    if constexpr (NSW_EXP_XTIME) {
      constexpr int E0 = 100, E = 24;
      if (tid == 0 && u == a.user0 && a.phase_ns != nullptr && xcnt >= E0 && xcnt < E0 + E)
        a.phase_ns[size_t(rank) * 2 * E + 2 * (xcnt - E0) + which] = globaltimer_ns();
    }
  };
  auto post_cols = [&](S (&v)[MC], bool xon = false, S xval = S(0)) {
    int base = 0, lim = MC;
    rs_rows<S, MC, MC, 16, CG, OpSum>(v, lane, base, lim);
    constexpr int CF = rs_final_count<MC, 16, CG>();
#pragma unroll
    for (int j = 0; j < CF; ++j) {
      const int c = g * MC + base + j;
      if (base + j < lim && c < m) red[warp * P + c] = v[j];
    }
    __syncthreads();
    xstamp(0);
    if constexpr (CL > 1) {
      // thread q sums columns [VE q, VE q + VE) over the warps (warp order,
      // the same bits as a per-column sum) and pushes them as one 16-byte
      // st.async to every CTA of the cluster
      constexpr int VE = 16 / sizeof(S);
      const uint32_t mb = smem_u32(xmb + parity);
      const int nx = m + (xon ? 1 : 0);
      const int ng = (nx + VE - 1) / VE;
      if (tid == 0) cl_expect_tx(mb, uint32_t(CL * ng * 16));
      if (tid < ng) {
        V16<S> tot4;
        tot4.v = reinterpret_cast<const V16<S>*>(red + tid * VE)->v;
#pragma unroll
        for (int w = 1; w < NW; ++w) {
          V16<S> x;
          x.v = reinterpret_cast<const V16<S>*>(red + w * P + tid * VE)->v;
#pragma unroll
          for (int e = 0; e < VE; ++e) tot4.s[e] += x.s[e];
        }
        S mine[VE];
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          const int c = tid * VE + e;
          mine[e] = c < m ? tot4.s[e] : (c == m && xon ? xval : S(0));
        }
        const uint32_t slot = smem_u32(xch + (size_t(parity) * CL + rank) * P + tid * VE);
#pragma unroll
        for (int q = 0; q < CL; ++q) cl_st_async16(cl_map(slot, q), mine, cl_map(mb, q));
      }
    }
  };
  auto collect_cols = [&](auto&& fin, bool xon = false, S xval = S(0), S* xmax = nullptr) {
    if constexpr (CL > 1) {
      const uint32_t mb = smem_u32(xmb + parity);
      const int nx = m + (xon ? 1 : 0);
      if (tid < nx) {
        mbar_wait(mb, (xph >> parity) & 1u);
        if (tid < m) {
          S tot = S(0);
#pragma unroll
          for (int q = 0; q < CL; ++q) tot += xch[(size_t(parity) * CL + q) * P + tid];   // rank order
          fin(tid, tot);
        } else {
          S mx = S(0);
#pragma unroll
          for (int q = 0; q < CL; ++q) mx = fmax(mx, xch[(size_t(parity) * CL + q) * P + tid]);
          *xmax = mx;
        }
      }
      xph ^= 1u << parity;
      parity ^= 1;
    } else {
      S acc = S(0);
      if (tid < m) {
        acc = red[tid];
#pragma unroll
        for (int w = 1; w < NW; ++w) acc += red[w * P + tid];
      }
      if (tid < m) fin(tid, acc);
      if (xon && tid == m) *xmax = xval;
    }
    __syncthreads();
    xstamp(1);
    ++xcnt;
  };
  auto reduce_cols = [&](S (&v)[MC], auto&& fin, bool xon = false, S xval = S(0), S* xmax = nullptr) {
    post_cols(v, xon, xval);
    collect_cols(fin, xon, xval, xmax);
  };
  // v~ history rows: global (written by the forward) -> shared slots by
  // cp.async, zero-filled past column m-1
  auto vrow = [&](int t) -> S* { return vr + (t & 3) * P; };
  auto load_row = [&](S* dst, int t) {
    for (int k = tid; k < P; k += NT) cp_async_zfill(dst + k, hu + size_t(t) * m + (k < m ? k : 0), k < m);
    cp_async_commit();
  };
  // coalesced element-wise visit of this CTA's cells: f(local cell e, vector slot or -1)
  auto foreach_cell = [&](auto&& f) {
    if (vec_ok) {
      for (int q = tid; q < ncell / V; q += NT) f(q * V, q);
    } else {
      for (int e = tid; e < ncell; e += NT) f(e, -1);
    }
  };

  for (int q = tid; q < Tl::KT; q += NT) Kt[q] = S(0);
  if (tid < P) {
    vec0[tid] = S(0);
    vec1[tid] = S(0);
    vec2[tid] = S(0);
    clred[tid] = S(0);
    clred[P + tid] = S(0);
  }
  S ex[MC];
#pragma unroll
  for (int j = 0; j < MC; ++j) ex[j] = (col(j) < m - 1) ? a.expo[min(col(j), m - 2)] : S(0);
  __syncthreads();

  if (phase == PHASE_RUNNING || phase == PHASE_DONE_PENDING || phase == PHASE_FWD_CONT || phase == PHASE_FWD_FIN) {
    // ---- rebuild K~ (step k-1's for the backward; this step's for a
    // tolerance-mode continuation / finish) of this CTA's items ----
    if (tid < m) vec1[tid] = a.beta[size_t(u) * m + tid];
    for (int i = tid; i < nloc; i += NT) rowA[i] = a.alpha[size_t(u) * n + r0 + i];
    load_row(vTr, Th);
    load_row(vrow(Th - 1), Th - 1);
    if (Th >= 2) load_row(vrow(Th - 2), Th - 2);
    cp_async_wait_all();
    __syncthreads();
    foreach_cell([&](int e0, int q) {
      int i = e0 / m, k = e0 - i * m;
      if (q >= 0) {
        V16<S> c;
        c.v = reinterpret_cast<const V16<S>*>(Cu)[q].v;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          Kt[kx(i, k)] = ktilde(c.s[j], vec1[k], rowA[i]);
          if (++k == m) { k = 0; ++i; }
        }
      } else {
        Kt[kx(i, k)] = ktilde(Cu[e0], vec1[k], rowA[i]);
      }
    });
    __syncthreads();
    S vT[MC];
#pragma unroll
    for (int j = 0; j < MC; ++j) vT[j] = vTr[col(j)];
    {
      S vT1[MC];
#pragma unroll
      for (int j = 0; j < MC; ++j) vT1[j] = vrow(Th - 1)[col(j)];
      for (int r = 0; r < R; ++r) {   // u~^T (all lanes of the group agree)
        S kr[MC];
        ld_seg<Tl, S, MC>(kr, Kt, lrow(r), g);
        const S uT = F::rcp_fast(rdot_g<S, MC, CG>(kr, vT1));
        __syncwarp();
        if (g == 0) rowA[lrow(r)] = ok(r) ? uT : S(0);
      }
    }
    __syncthreads();
    const int improved = a.state[ST_IMPROVED];
    auto write_policy = [&]() {
      foreach_cell([&](int e0, int q) {
        int i = e0 / m, k = e0 - i * m;
        if (q >= 0) {
          V16<S> t;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            t.s[j] = mul_(mul_(Kt[kx(i, k)], rowA[i]), vTr[k]);
            if (++k == m) { k = 0; ++i; }
          }
          reinterpret_cast<V16<S>*>(xb)[q].v = t.v;
        } else {
          xb[e0] = mul_(mul_(Kt[kx(i, k)], rowA[i]), vTr[k]);
        }
      });
    };
    if (phase == PHASE_DONE_PENDING) {
      if (improved) write_policy();
      cluster.sync();
      return;
    }
    if (phase == PHASE_FWD_FIN) {
      // tolerance mode: the forward stopped at t* = Th; impact terms of X^{t*}
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        const int il = lrow(r);
        S kr[MC];
        ld_seg<Tl, S, MC>(kr, Kt, il, g);
        const double rr = ok(r) ? double(relu[il]) : 0.0;
        const S uT = rowA[il];
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < MC; ++j)
          if (col(j) < m - 1) acc = fma(rr * a.expo_d[min(col(j), m - 2)], double(mul_(mul_(kr[j], uT), vT[j])), acc);
        acc = group_sum<double, CG>(acc);
        if (g == 0 && ok(r)) a.partial[size_t(u) * n + r0 + il] = acc;
      }
      cluster.sync();
      return;
    }
    if (phase == PHASE_FWD_CONT) {
      // tolerance mode: continue this step's forward from v~^{t0}, t0 = Th
      if (tid < P) vec0[tid] = vTr[tid];
      __syncthreads();
      goto forward_iterations;
    }
    if (improved) write_policy();

    // ---- seed W = gx .* X, reverse sweep (see step_kernel) ----
    S A[R][MC];
    S ut[R];
    {
      S c[MC];
#pragma unroll
      for (int j = 0; j < MC; ++j) c[j] = S(0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int il = lrow(r);
        S kr[MC];
        ld_seg<Tl, S, MC>(kr, Kt, il, g);
        ut[r] = rowA[il];
        const S rr = ok(r) ? relu[il] : S(0);
        const S imp_i = ok(r) ? S(a.imp[r0 + il]) : S(1);
        const S inv_imp = S(1.0 / double(imp_i));
        S gsum = S(0);
#pragma unroll
        for (int j = 0; j < MC; ++j) {
          A[r][j] = S(0);
          if (col(j) < m - 1) {
            const S W = mul_(gx_of(rr, ex[j], imp_i, inv_imp), mul_(mul_(kr[j], ut[r]), vT[j]));
            gsum += W;
            c[j] += W;
          }
        }
        gsum = group_sum<S, CG>(gsum);
        if (g == 0) rowB[il] = gsum;
      }
      reduce_cols(c, [&](int k, S tot) { vec0[k] = mul_(mul_(vTr[k], tot), inv_mass(k)); });
    }
#ifndef NSW_KREG_CL
#define NSW_KREG_CL 1   // +1.5 % on the config-4 shard (profiles/r02/ab_kreg_cluster.txt)
#endif
    // KREG: the K~ row segments stay in registers for the whole sweep
    constexpr bool KREG = NSW_KREG_CL && sizeof(S) == 4 && R <= 7;   // R = 8 tiles would spill
    S Kr[KREG ? R : 1][MC];
    if constexpr (KREG) {
#pragma unroll
      for (int r = 0; r < R; ++r) ld_seg<Tl, S, MC>(Kr[r], Kt, lrow(r), g);
    }
    for (int t = Th; t >= 1; --t) {
      // stream row t-3 into the slot row t+1 held (last read at level t+2)
      if (t >= 3) load_row(vrow(t - 3), t - 3);
      S cv[MC], vp[MC], vpp[MC], c[MC];
      const S* rp = vrow(t - 1);
      const S* rpp = vrow(t >= 2 ? t - 2 : 0);
      const bool first = t == Th;
#pragma unroll
      for (int j = 0; j < MC; ++j) {
        cv[j] = vec0[col(j)];
        vp[j] = rp[col(j)];
        vpp[j] = rpp[col(j)];
        c[j] = S(0);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int il = lrow(r);
        S kr[MC];
        if constexpr (KREG) {
#pragma unroll
          for (int j = 0; j < MC; ++j) kr[j] = Kr[r][j];
        } else {
          ld_seg<Tl, S, MC>(kr, Kt, il, g);
        }
        const S sig = rdot_g<S, MC, CG>(kr, cv);
        const S den = rdot_g<S, MC, CG>(kr, vpp);
        const S gs = first ? rowB[il] : S(0);
        const S h = ut[r] * (gs - ut[r] * sig);
        axpy_<S, MC, true>(A[r], cv, -ut[r]);
        axpy_<S, MC, true>(A[r], vp, -h);
        axpy_<S, MC, true>(c, kr, h);
        ut[r] = (ok(r) && t >= 2) ? F::rcp_fast(den) : S(0);
      }
      if (t >= 2) {
        cp_async_wait_all();   // row t-3 lands before the reduction's barrier publishes it
        reduce_cols(c, [&](int k, S tot) {
          const S vpk = rp[k];
          vec0[k] = mul_(mul_(vpk, -mul_(vpk, tot)), inv_mass(k));
        });
      }
    }
    // gK = W + K~ .* G over the tile
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int il = lrow(r);
      S kr[MC], gk[MC];
      ld_seg<Tl, S, MC>(kr, Kt, il, g);
      const S uT = rowA[il];
      const S rr = ok(r) ? relu[il] : S(0);
      const S imp_i = ok(r) ? S(a.imp[r0 + il]) : S(1);
      const S inv_imp = S(1.0 / double(imp_i));
#pragma unroll
      for (int j = 0; j < MC; ++j) {
        const S W = (col(j) < m - 1) ? mul_(gx_of(rr, ex[j], imp_i, inv_imp), mul_(mul_(kr[j], uT), vT[j])) : S(0);
        gk[j] = fma(kr[j], A[r][j], W);
      }
      st_seg<Tl, S, MC>(Kt, il, g, gk);
    }
    if (tid < m) vec2[tid] = a.warm_start ? add_(vec1[tid], F::log_(vTr[tid])) : S(0);
    __syncthreads();
    // ---- Adam ascent on this CTA's cells ----
    const int s = a.state[ST_STEP];
    const S bc1 = S(a.bc[2 * s]), bc2 = S(a.bc[2 * s + 1]);
    const S ibc1 = S(1.0 / a.bc[2 * s]), ibc2 = S(1.0 / a.bc[2 * s + 1]);
    auto adam = [&](S& cc, S& mm, S& vv, S gk) {
      const S gg = mul_(gk, a.nie);
      mm = add_(mul_(a.b1, mm), mul_(a.omb1, gg));
      vv = add_(mul_(a.b2, vv), mul_(mul_(a.omb2, gg), gg));
      S mh, vhat;
      if constexpr (sizeof(S) == 4) {
        mh = mul_(mm, ibc1);
        vhat = mul_(vv, ibc2);
      } else {
        mh = F::div(mm, bc1);
        vhat = F::div(vv, bc2);
      }
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
          S& slot = Kt[kx(i, k)];
          adam(c.s[j], mm.s[j], vv.s[j], slot);
          slot = mul_(c.s[j], a.nie);
          if (++k == m) { k = 0; ++i; }
        }
        reinterpret_cast<V16<S>*>(Cu)[q].v = c.v;
        reinterpret_cast<V16<S>*>(mu)[q].v = mm.v;
        reinterpret_cast<V16<S>*>(vu)[q].v = vv.v;
      } else {
        S c = Cu[e0], mm = mu[e0], vv = vu[e0];
        S& slot = Kt[kx(i, k)];
        adam(c, mm, vv, slot);
        slot = mul_(c, a.nie);
        Cu[e0] = c;
        mu[e0] = mm;
        vu[e0] = vv;
      }
    });
  } else {
    // INIT (C0 = -eps log uniform, lvi = 0) or RESUME (given C, lvi in beta)
    const bool init = phase == PHASE_INIT;
    if (!init && tid < m) vec2[tid] = a.beta[size_t(u) * m + tid];
    for (int e = tid; e < ncell; e += NT) {
      const int i = e / m, k = e - i * m;
      S c0;
      if (init) {
        c0 = (k == m - 1) ? a.c_dummy : a.c_real;
        Cu[e] = c0;
        mu[e] = S(0);
        vu[e] = S(0);
      } else {
        c0 = Cu[e];
      }
      Kt[kx(i, k)] = mul_(c0, a.nie);
    }
  }
  __syncthreads();

  // ---- forward: absorb beta = lvi, alpha = -rowmax(K + beta); T iterations ----
  if (rank == 0 && tid < m) {
    a.beta[size_t(u) * m + tid] = vec2[tid];
    hu[tid] = S(1);
  }
  if (tid < m) vec0[tid] = S(1);
  {
    S bt[MC];
#pragma unroll
    for (int j = 0; j < MC; ++j) bt[j] = vec2[col(j)];
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      const int il = lrow(r);
      S kr[MC];
      ld_seg<Tl, S, MC>(kr, Kt, il, g);
      S mx = F::ninf();
#pragma unroll
      for (int j = 0; j < MC; ++j)
        if (col(j) < m) mx = fmax(mx, add_(kr[j], bt[j]));
      mx = group_max<S, CG>(mx);
      const S al = -mx;
      if (g == 0 && ok(r)) a.alpha[size_t(u) * n + r0 + il] = al;
#pragma unroll
      for (int j = 0; j < MC; ++j) kr[j] = (ok(r) && col(j) < m) ? F::exp_fast(add_(add_(kr[j], bt[j]), al)) : S(0);
      st_seg<Tl, S, MC>(Kt, il, g, kr);
    }
  }
  __syncthreads();
forward_iterations:
  S A[R][MC];
  S ut[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    ld_seg<Tl, S, MC>(A[r], Kt, lrow(r), g);
    ut[r] = S(0);
  }
  const int t_start = phase == PHASE_FWD_CONT ? Th + 1 : 1;
  const int t_end = tolm ? min(t_start - 1 + a.chunk, T) : T;
  // tolerance mode also records the reference's L-inf marginal residual of
  // every iteration (sinkhorn.py:237-243), as step_kernel does: the row
  // residual of iteration t-1 from iteration t's own row dot (max over the
  // cluster through the exchange), the column residual (fp64) in fin
  auto row_res_max = [&](S rm) -> S {   // CTA maximum, valid on every thread after the barrier
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rm = fmax(rm, __shfl_xor_sync(0xffffffffu, rm, o));
    if (lane == 0) rmw[warp] = rm;
    __syncthreads();
    S r = S(0);
    for (int w = 0; w < NW; ++w) r = fmax(r, rmw[w]);
    return r;
  };
  // the iteration body is instantiated twice so the fixed schedule carries
  // no residual bookkeeping at all
  auto iterate = [&](auto tol_c) {
    constexpr bool TOLM = decltype(tol_c)::value;
    for (int t = t_start; t <= t_end; ++t) {
      S vv[MC], c[MC];
#pragma unroll
      for (int j = 0; j < MC; ++j) vv[j] = vec0[col(j)];
      S rmax = S(0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const S sr = rdot_g<S, MC, CG>(A[r], vv);
        if (TOLM && ok(r)) rmax = fmax(rmax, fabs(ut[r] * sr - S(1)));
        const S rp = F::rcp_fast(sr);
        ut[r] = ok(r) ? rp : S(0);
      }
#pragma unroll
      for (int j = 0; j < MC; ++j) c[j] = S(0);
#pragma unroll
      for (int r = 0; r < R; ++r) axpy_<S, MC, true>(c, A[r], ut[r]);
      if constexpr (TOLM) {
        const bool rec = t > t_start;   // residual of iteration t-1 completes here
        S rcta = S(0), rall = S(0);
        if (rec) rcta = row_res_max(rmax);
        reduce_cols(
            c,
            [&](int k, S tot) {
              const S vn = F::div_fast(mass(k), tot);
              vec0[k] = vn;
              if (rank == 0) hu[size_t(t) * m + k] = vn;
              colres[(t & 1) * P + k] = sizeof(S) == 8 ? S(fabs(vn * tot - mass(k))) : S(0);
            },
            rec, rcta, &rall);
        if (rec && rank == 0 && tid == m) {
          S r = rall;
          for (int kk = 0; kk < m; ++kk) r = fmax(r, colres[((t - 1) & 1) * P + kk]);
          a.res[size_t(u) * (T + 1) + t - 1] = double(r);
        }
      } else {
        reduce_cols(c, [&](int k, S tot) {
          const S vn = F::div_fast(mass(k), tot);
          vec0[k] = vn;
          if (rank == 0) hu[size_t(t) * m + k] = vn;
        });
      }
    }
  };
  if (tolm) {
    iterate(std::true_type{});
  } else {
    iterate(std::false_type{});
  }
  if (tolm) {
    // residual of the chunk's last iteration: one more row pass; cluster max
    // through distributed shared memory (once per chunk)
    S vv[MC];
#pragma unroll
    for (int j = 0; j < MC; ++j) vv[j] = vec0[col(j)];
    S rmax = S(0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const S sr = rdot_g<S, MC, CG>(A[r], vv);
      if (ok(r)) rmax = fmax(rmax, fabs(ut[r] * sr - S(1)));
    }
    const S rcta = row_res_max(rmax);
    if (tid == 0) clred[0] = rcta;
    cluster.sync();
    if (rank == 0 && tid == 0) {
      S r = S(0);
      for (int q = 0; q < CL; ++q) r = fmax(r, *cluster.map_shared_rank(clred, q));
      for (int kk = 0; kk < m; ++kk) r = fmax(r, colres[(t_end & 1) * P + kk]);
      a.res[size_t(u) * (T + 1) + t_end] = double(r);
    }
    cluster.sync();   // remote reads done before any CTA exits
    return;           // impact terms come from the finish launch once t* is known
  }
  // per-item impact terms, float64, completed across the group
  {
    S vv[MC];
#pragma unroll
    for (int j = 0; j < MC; ++j) vv[j] = vec0[col(j)];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int il = lrow(r);
      const double rr = ok(r) ? double(relu[il]) : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < MC; ++j)
        if (col(j) < m - 1) acc = fma(rr * a.expo_d[min(col(j), m - 2)], double(mul_(mul_(A[r][j], ut[r]), vv[j])), acc);
      acc = group_sum<double, CG>(acc);
      if (g == 0 && ok(r)) a.partial[size_t(u) * n + r0 + il] = acc;
    }
  }
  cluster.sync();   // keep every CTA's shared memory alive until remote reads are done
}

}  // namespace nsw
