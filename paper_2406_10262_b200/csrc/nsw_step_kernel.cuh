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
  int user0;     // first user of this launch (the tail launch uses another tile)
  int tol_mode;  // 0: fixed schedule; 1: reference tolerance mode (chunked forward)
  int chunk;     // tolerance mode: inner iterations per forward launch
  double* res;   // tolerance mode: [U][T+1] L-inf marginal residual after iteration t
  S* C;          // [U][n][m] transport costs (the ascent variable)
  S* am;         // [U][n][m] Adam first moment
  S* av;         // [U][n][m] Adam second moment
  S* alpha;      // [U][n]    row absorption point -max_k(K_ik + beta_k)
  S* beta;       // [U][m]    column absorption point = warm-start duals lvi
  S* hist;       // [U][T+1][m] v~^t = exp(v^t - beta), t = 0..T (v~^0 = 1)
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
  S inv_mass_dummy;              // 1/(n-m+1), correctly rounded on the host
  unsigned long long* phase_ns;  // [U][16] diagnostics: phase-boundary timestamps (nullptr: off)
  // in-solve re-absorption (streaming step only; reabs_thr > 0): per user up
  // to reabs_max events of the last forward, event e at iteration ev_t[u][e]
  // with row factors a (n) and column factors b (m) in ev_ab[u][e][n + m]
  double reabs_thr;
  int reabs_max;
  int* ev_count;   // [U]
  int* ev_t;       // [U][reabs_max]
  S* ev_ab;        // [U][reabs_max][n + m]
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
// CH = 2: two interleaved FMA chains (short latency for tiles with few rows
// per thread); CH = 1: one chain (tiles with >= 4 independent rows per thread
// have ILP to spare, and the chains' final add is saved).
#ifndef NSW_PK_ALL
#define NSW_PK_ALL 0   // A/B builds: packed FMAs in every fp32 tile
#endif

// PK (fp32): two chains packed into one FFMA2 per column pair.
template <typename S, int M, int CH = 2, bool PK = false>
__device__ __forceinline__ S rdot(const S (&x)[M], const S (&y)[M]) {
  if constexpr (sizeof(S) == 4 && NSW_FFMA2 && PK) {
    S s0 = S(0), s1 = S(0);
#pragma unroll
    for (int k = 0; k + 1 < M; k += 2) ffma2(s0, s1, x[k], x[k + 1], y[k], y[k + 1], s0, s1);
    if constexpr (M % 2) s0 = fmaf(x[M - 1], y[M - 1], s0);
    return s0 + s1;
  }
  if constexpr (CH == 1) {
    S s0 = S(0);
#pragma unroll
    for (int k = 0; k < M; ++k) s0 = fma(x[k], y[k], s0);
    return s0;
  }
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

// Per-row scalars (alpha, u~^T, seed g_u, u^1) live in the tile's padding
// column when the row pitch has one (P > M), else in two row buffers.
template <typename S, int M>
struct RowSlots {
  static constexpr int P = RowPitch<S, M>::value;
  static constexpr bool kPad = P > M;
};

// fp32 tiles of >= 2 warps stage relevance and 1/Imp per row in shared
// memory; fp64, one-warp and 7-per-SM tiles keep that shared memory free
// (7 x 34 KB would not fit an SM).
template <typename S, int NT, int MINB>
__host__ __device__ constexpr bool stage_inputs() {
  return sizeof(S) == 4 && NT >= 64 && MINB < 7;
}

// Tensor-core adjoint tile shape: the accumulator's N (the m columns padded to
// a multiple of 16), TMEM columns allocated (a power of two >= 32) and the
// K~-tile region, which must also hold the A operand (64 B per row: 8 K slots
// x hi/lo) that the sweep stages over it.
template <int M, int R, int NT>
struct TcShape {
  static constexpr int kNPC = M <= 16 ? 16 : 32;
  static constexpr int kNeed = NT * R / 128 * kNPC;
  static constexpr int kCols = kNeed <= 32 ? 32 : kNeed <= 64 ? 64 : kNeed <= 128 ? 128 : kNeed <= 256 ? 256 : 512;
};
template <typename S, int M, int R, int NT, bool TC>
__host__ __device__ constexpr size_t tile_elems() {
  constexpr size_t kt = size_t(NT) * R * RowPitch<S, M>::value;
  constexpr size_t ta = size_t(NT) * R * 64 / sizeof(S);
  return TC && ta > kt ? ta : kt;
}

template <typename S, int M, int R, int NT, int MINB, bool TC = false>
__host__ __device__ constexpr size_t step_smem_bytes(int T) {
  constexpr int P = RowPitch<S, M>::value;
  constexpr size_t rows = RowSlots<S, M>::kPad ? 0 : 2 * size_t(NT) * R;
  return sizeof(S) * (tile_elems<S, M, R, NT, TC>() + size_t(T + 1) * P + 2 * size_t(NT / 32) * P + 3 * P + rows + 2 * P +
                      size_t(NT / 32) + 4 + (stage_inputs<S, NT, MINB>() ? 2 * size_t(NT) * R : 0) + P) +
         32 + 8 * size_t(P) +   // staged inputs (relevance, Imp, exposures in S and float64)
         16 +                   // mbarrier of the cost tile's bulk copy
         (TC ? size_t(2) * 2 * TcShape<M, R, NT>::kNPC * 32 + 64 + 128 : 0);   // tensor-core path: 2 x (hi, lo) B operands + mbarrier
}

// ---------------------------------------------------------------------------
// tcgen05 / TMEM helpers (sm_100a) for the tensor-core adjoint accumulation
#ifndef NSW_TC_EXP
#define NSW_TC_EXP 0   // diagnostics only: 1 = no A/B staging stores, 2 = no MMAs / waits, 4 = no proxy
                       // fence, 8 = no waits (wrong results); 16 = one thread issues every block's MMAs
#endif
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// K-major, no-swizzle UMMA shared-memory descriptor: core matrices of
// 8 rows x 16 bytes; LBO = stride between the two 16-byte K chunks, SBO =
// stride between 8-row groups (both >> 4), version 1 (Blackwell).
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M=128, N=16
constexpr uint32_t kIdescTf32_128x16 = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(accum), "r"(kIdescTf32_128x16), "r"(0u));
}
// both operands from shared memory (K-major descriptors), D in TMEM
template <int N>
__device__ __forceinline__ void umma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t accum) {
  constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | ((128u >> 4) << 24);
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(accum), "r"(idesc));
}
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  [[maybe_unused]] unsigned polls = 0;
  while (!done) {
    if constexpr (NSW_CHECKS) {
      if (++polls > (1u << 28)) nsw_check_fail("mbarrier wait timed out", mbar, parity);
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(mbar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr)
      : "memory");
}

// fp32 throughput path: divisions / square roots off the hot path use the
// fast (MUFU) forms; the fp64 parity path keeps IEEE-rounded operations in
// the reference's order (solver.py:86-89, :115-121).
template <typename S>
__device__ __forceinline__ S fdiv_(S a, S b) {
  if constexpr (sizeof(S) == 4) return Fp<float>::div_fast(a, b);
  else return Fp<double>::div(a, b);
}
template <typename S>
__device__ __forceinline__ S fsqrt_(S x) {
  if constexpr (sizeof(S) == 4) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  } else {
    return Fp<double>::sqrt_(x);
  }
}

// Structure: the per-step phases that touch every cell once move the user's
// contiguous [n][m] tiles between HBM and the shared-memory tile Kt with
// coalesced 16-byte accesses (element-wise phases: K~ rebuild, Adam, the
// policy write) or as loops over this thread's rows (seed, log-domain
// iteration 1); only the two hot loops (forward iterations 2..T and the T
// reverse levels) hold the R x M tile in registers.
template <typename S, int M, int R, int NT, int MINB, bool TC = false>
__global__ void __launch_bounds__(NT, MINB) step_kernel(const StepArgs<S> a) {
  // TC: the backward's adjoint G accumulates in tensor memory through tcgen05
  // MMAs (fp32 path, 4-warp CTAs, M <= 16) instead of 2 FFMAs per cell-level.
  static_assert(!TC || (sizeof(S) == 4 && NT % 128 == 0 && M <= 32 && TcShape<M, R, NT>::kNeed <= 512 / MINB),
                "tensor-core tile shape");
  using F = Fp<S>;
  constexpr int P = RowPitch<S, M>::value;
  constexpr bool PAD = RowSlots<S, M>::kPad;
  constexpr int NW = NT / 32;
  constexpr int V = 16 / sizeof(S);
  constexpr int CH = R >= 4 ? 1 : 2;   // row-dot chains; one value for every u~ (forward, replay, u~^T)
  // Packed FFMA2 in the hot loops for tiles of >= 12 warps per SM (issue-
  // bound: config 1 main wave) and the 2-row latency tiles (config-1 tail);
  // the 4- and 8-row tiles at one CTA per SM lose 5-8 % with it (configs 2,
  // 3; profiles/r01/r01d_ab_ffma2.txt).
  constexpr bool PK = sizeof(S) == 4 && (NT * MINB >= 384 || R <= 2 || NSW_PK_ALL);
  // the row dot's form (forward, replay and u~^T share it, so replays are
  // bit-exact) and the forward's column axpy, separately
#ifndef NSW_PK_DOT
#define NSW_PK_DOT 0
#endif
#ifndef NSW_PK_FWD_AXPY
#define NSW_PK_FWD_AXPY 1   // the forward's column axpy packed (broadcast u~): config 3 +1.5 %, configs 1-2 neutral
#endif                      // (profiles/r02/ab_pk_fwd_axpy.txt); FFMA2 rounds like two FFMAs: same bits
  constexpr bool PKD = PK || (NSW_PK_DOT && sizeof(S) == 4);
  constexpr bool PKF = PK || (NSW_PK_FWD_AXPY && sizeof(S) == 4);
  // register-lean backward (tiles packed 7 per SM): the v~ history rows are
  // re-read from shared memory per row instead of held across the row loop
  constexpr bool LEAN = MINB >= 7;
  // fp32: the seed's W is folded into the adjoint as its rank-1 start value
  constexpr bool RANK1 = sizeof(S) == 4;
  static_assert(NT % 32 == 0 && M <= NT && P <= NT, "tile shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  nsw_poison_smem(smem_raw);
  const int T = a.T;
  S* Kt = reinterpret_cast<S*>(smem_raw);   // [NT*R][P]  K / K~ / gK rows
  S* vh = Kt + tile_elems<S, M, R, NT, TC>();   // [T+1][P]   v~ history
  S* red = vh + size_t(T + 1) * P;          // [2][NW][P] column partials (double-buffered)
  S* vec0 = red + 2 * NW * P;               // [P] scaling vector / cv
  S* vec1 = vec0 + P;                       // [P] beta / column max
  S* vec2 = vec1 + P;                       // [P] warm-start duals lvi
  S* rowA = vec2 + P;                       // [NT*R] (no padding column only)
  S* rowB = rowA + (PAD ? 0 : size_t(NT) * R);
  S* colres = rowB + (PAD ? 0 : size_t(NT) * R);  // [2][P] column residuals (tolerance mode)
  S* redmax = colres + 2 * P;                     // [NW] per-warp row-residual maxima
  // per-item / per-position inputs staged once per launch (the seed, the gK
  // epilogue and the impact terms read them from here, not from global)
  S* relS = reinterpret_cast<S*>((reinterpret_cast<uintptr_t>(redmax + NW) + 15) & ~uintptr_t(15));  // [NT*R] relevance (0 on padding rows)
  constexpr bool STAGE = stage_inputs<S, NT, MINB>();
  S* impS = relS + (STAGE ? size_t(NT) * R : 0);   // [NT*R] 1/Imp of the step being differentiated (fp32)
  S* exS = impS + (STAGE ? size_t(NT) * R : 0);   // [P] exposures (0 from column m-1 on)
  double* exD = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(exS + P) + 15) & ~uintptr_t(15));  // [P]
  // tensor-core path: B operands (2 buffers x hi/lo x NPC rows x 8 tf32) and the MMA mbarrier
  constexpr int NPC = TcShape<M, R, NT>::kNPC;
  uint64_t* bmb = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(exD + P) + 7) & ~uintptr_t(7));
  unsigned char* tc_base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(bmb + 1) + 127) & ~uintptr_t(127));
  float* Bop = reinterpret_cast<float*>(tc_base);            // [2][2][NPC x 8]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tc_base + 4 * NPC * 32);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tc_base + 4 * NPC * 32 + 8);
  // slotA: alpha -> u~^T -> u^1 ; slotB: seed g_u (shares slotA's storage
  // when PAD: written after u~^T is in registers, u~^T restored at level T)
  auto slotA = [&](int i) -> S& { return PAD ? Kt[size_t(i) * P + M] : rowA[i]; };
  auto slotB = [&](int i) -> S& { return PAD ? Kt[size_t(i) * P + M] : rowB[i]; };

  const int phase = a.state[ST_PHASE];
  if (phase == PHASE_FINISHED) return;
  const bool tolm = a.tol_mode != 0;
  // Length of the v~ history of the K~ this launch rebuilds: the previous
  // solve's iteration count for the backward / owed policy, the iterations
  // done so far for a forward continuation, the stopping iteration t* for
  // the forward's finish (tolerance mode; the fixed schedule always has T).
  const int Tprev = tolm ? a.state[ST_TSTAR] : T;
  const int Th = phase == PHASE_FWD_CONT ? a.state[ST_T0] : (phase == PHASE_FWD_FIN ? a.state[ST_TSTAR] : Tprev);

  const int u = a.user0 + blockIdx.x;
  const int tid = threadIdx.x;
  // diagnostics: global-timer stamp of phase boundary p (thread 0; off unless
  // the solver was created with NSW_PHASE_TIMING set)
  auto mark = [&](int p) {
    if (a.phase_ns != nullptr && tid == 0) a.phase_ns[size_t(u) * 16 + p] = globaltimer_ns();
  };
  mark(0);
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
  // 1/x on live rows, 0 on padding rows, as arithmetic (no branch): a select
  // lets the compiler branch around the whole row dot, which splits the row
  // loop into basic blocks and serialises the rows' FMA chains.
  auto masked_rcp = [&](S x, bool live) -> S {
    const S on = live ? S(1) : S(0);
    return F::rcp_fast(x + (S(1) - on)) * on;
  };
  // 1/x clamped away from 0: padding rows (all-zero K~ rows, x = 0) get a
  // large finite value instead of inf, so u~ * 0 stays 0 without a mask.
  auto rcp_clamped = [&](S x) -> S { return F::rcp_fast(fmax(x, F::tiny())); };
  // K~ = exp(K + beta_k + alpha_i), K = C * (-1/eps) (solver.py:188); the one
  // expression used by both the forward and the backward's rebuild, so K~ is
  // bit-identical in both.
  auto ktilde = [&](S c, S beta_k, S alpha_i) -> S {
    return F::exp_fast(add_(add_(mul_(c, a.nie), beta_k), alpha_i));
  };
  auto mass = [&](int k) -> S { return k == m - 1 ? a.mass_dummy : S(1); };
  auto inv_mass = [&](int k) -> S { return k == m - 1 ? a.inv_mass_dummy : S(1); };
  // gx = r e / Imp (solver.py:86-89); fp32 uses a per-row reciprocal
  // (impv = impv_of(i): 1/Imp_i on the fp32 path, Imp_i on the fp64 path)
  auto gx_of = [&](S rr, S e, S impv) -> S {
    if constexpr (sizeof(S) == 4) return mul_(mul_(rr, e), impv);
    else return F::div(mul_(rr, e), impv);
  };

  const bool rebuild = phase == PHASE_RUNNING || phase == PHASE_DONE_PENDING || phase == PHASE_FWD_CONT ||
                       phase == PHASE_FWD_FIN;
  // All of this launch's small per-user inputs are requested up front, so
  // their latencies overlap: the v~ history goes global -> shared memory
  // asynchronously (cp.async, zero-filled past column m-1); alpha, beta,
  // relevance and Imp go through registers and are stored after the tile is
  // zeroed.
  // The user's cost tile (contiguous [n][m], 16-byte multiple) comes in as one
  // TMA bulk copy (cp.async.bulk, completion on an mbarrier) into the top of
  // the K~ tile region, issued before anything else; the rebuild expands it
  // in place into padded K~ rows.
  // fp32: only the 2048-row tiles (config 3: +1.8 %); on the smaller fp32
  // tiles the extra code perturbs the hot loops' register allocation for a
  // -0.3..-0.8 % net (profiles/r01/r01f_ab_tma.txt).  fp64 tiles always use it.
  constexpr bool BULK_TILE = sizeof(S) == 8 || NT * R >= 2048;
  const bool bulk = BULK_TILE && rebuild && vec_ok && !TC;
  const int stage_off = (NT * R * P - nm) / V * V;   // first staged element (16-byte aligned)
  if (BULK_TILE && bulk && tid == 0) {
    const uint32_t mb = smem_u32(bmb);
    const uint32_t bytes = uint32_t(nm) * sizeof(S);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(mb),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(Kt + stage_off)),
        "l"(Cu), "r"(bytes), "r"(mb)
        : "memory");
  }
  if (rebuild) {
    for (int idx = tid; idx < (Th + 1) * P; idx += NT) {
      const int t = idx / P, k = idx - t * P;
      cp_async_zfill(vh + idx, hu + size_t(t) * m + (k < m ? k : 0), k < m);
    }
  }
  cp_async_commit();
  S al[R], rv[R];
  double iv[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = tid + r * NT;
    al[r] = (rebuild && i < n) ? a.alpha[size_t(u) * n + i] : S(0);
    if constexpr (STAGE) {
      rv[r] = i < n ? relu[i] : S(0);
      iv[r] = i < n ? a.imp[i] : 1.0;
    }
  }
  const S bt0 = (rebuild && tid < m) ? a.beta[size_t(u) * m + tid] : S(0);
  // warm L2 with this user's big tiles (C, Adam moments): one prefetch per
  // 128-byte line, spread over the CTA.
  {
    auto pf = [&](const void* base, size_t bytes) {
      const char* b = reinterpret_cast<const char*>(base);
      for (size_t off = size_t(tid) * 128; off < bytes; off += size_t(NT) * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(b + off));
    };
    if (!bulk) pf(Cu, size_t(nm) * sizeof(S));
    if (phase == PHASE_RUNNING) {
      pf(mu, size_t(nm) * sizeof(S));
      pf(vu, size_t(nm) * sizeof(S));
    }
  }

  // zero the tile (padding rows / columns must stay 0) and the small vectors;
  // a bulk-copied tile is rebuilt as whole padded rows instead
  if (!bulk)
    for (int q = tid; q < NT * R * P / V; q += NT) reinterpret_cast<V16<S>*>(Kt)[q].v = V16<S>{}.v;
  if (tid < P) {
    vec0[tid] = S(0);
    vec1[tid] = bt0;
    vec2[tid] = S(0);
    exS[tid] = tid < m - 1 ? a.expo[tid < m - 1 ? tid : 0] : S(0);
    exD[tid] = tid < m - 1 ? a.expo_d[tid < m - 1 ? tid : 0] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = tid + r * NT;
    if (rebuild && !bulk) slotA(i) = al[r];   // (bulk: the staged tile occupies the slots)
    if constexpr (STAGE) {
      relS[i] = rv[r];
      impS[i] = S(1.0 / iv[r]);   // reciprocal: gx is two multiplies
    }
  }
  // relevance and Imp (fp32: 1/Imp) of item i; fp64 reads them from global
  // and divides by Imp in the reference's order
  auto rel_of = [&](int i) -> S {
    if constexpr (STAGE) return relS[i];
    else return i < n ? relu[i] : S(0);
  };
  auto impv_of = [&](int i) -> S {
    if constexpr (STAGE) return impS[i];
    else if constexpr (sizeof(S) == 4) return i < n ? F::rcp_fast(S(a.imp[i])) : S(1);
    else return i < n ? S(a.imp[i]) : S(1);
  };
  // exposures, loaded where used so they are not live across the loops
  auto load_ex = [&](S (&e)[M]) { lds_vec<S, M>(e, exS); };
  cp_async_wait_all();
  __syncthreads();
  mark(1);

  if (rebuild) {
    // ---------------- rebuild K~ from C, alpha, beta (step k-1's for the
    // backward; this step's for a tolerance-mode continuation / finish) ------
    if (BULK_TILE && bulk) {
      // this thread's rows from the staged tile into registers, a barrier
      // (rows expand in place), then whole padded rows; the row's alpha
      // goes to its padding slot afterwards
      mbar_wait(smem_u32(bmb), 0u);
      S cr[R][M];
      const S* stg = Kt + stage_off;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
#pragma unroll
        for (int k = 0; k < M; ++k) cr[r][k] = (i < n && k < m) ? stg[i * m + k] : S(0);
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        S kr[M];
#pragma unroll
        for (int k = 0; k < M; ++k) kr[k] = (i < n && k < m) ? ktilde(cr[r][k], vec1[k], al[r]) : S(0);
        sts_vec<S, M>(Kt + size_t(i) * P, kr);
        slotA(i) = al[r];
      }
    } else if (vec_ok) {
      const int nq = nm / V;
      for (int q0 = tid; q0 < nq; q0 += 8 * NT) {
        V16<S> c[8];
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (q0 + b * NT < nq) c[b].v = reinterpret_cast<const V16<S>*>(Cu)[q0 + b * NT].v;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int q = q0 + b * NT;
          if (q >= nq) break;
          int i = q * V / m, k = q * V - i * m;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            Kt[i * P + k] = ktilde(c[b].s[j], vec1[k], slotA(i));
            if (++k == m) { k = 0; ++i; }
          }
        }
      }
    } else {
      for (int e = tid; e < nm; e += NT) {
        const int i = e / m, k = e - i * m;
        Kt[i * P + k] = ktilde(Cu[e], vec1[k], slotA(i));
      }
    }
    __syncthreads();
    mark(2);
    S vT[M];
    lds_vec<S, M>(vT, vh + size_t(Th) * P);
    {
      S vT1[M];
      lds_vec<S, M>(vT1, vh + size_t(Th - 1) * P);
#pragma unroll 1
      for (int i = tid; i < NT * R; i += NT) {
        S kr[M];
        lds_vec<S, M>(kr, Kt + size_t(i) * P);
        slotA(i) = i < n ? F::rcp_fast(rdot<S, M, CH, PKD>(kr, vT1)) : S(0);   // u~^T
      }
    }
    const int improved = a.state[ST_IMPROVED];
    auto write_policy = [&]() {   // X = diag(u~^T) K~ diag(v~^T), coalesced
      for (int q = tid; q < (vec_ok ? nm / V : nm); q += NT) {
        const int e0 = vec_ok ? q * V : q;
        int i = e0 / m, k = e0 - i * m;
        if (vec_ok) {
          V16<S> t;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            t.s[j] = mul_(mul_(Kt[i * P + k], slotA(i)), vh[size_t(Th) * P + k]);
            if (++k == m) { k = 0; ++i; }
          }
          reinterpret_cast<V16<S>*>(xb)[q].v = t.v;
        } else {
          xb[e0] = mul_(mul_(Kt[i * P + k], slotA(i)), vh[size_t(Th) * P + k]);
        }
      }
    };
    if (phase == PHASE_DONE_PENDING) {
      // the stop fired after step k-1's forward: only its policy is still owed
      if (improved) {
        __syncthreads();
        write_policy();
      }
      return;
    }
    if (phase == PHASE_FWD_FIN) {
      // tolerance mode: the forward stopped at t* = Th; impact terms of X^{t*}
#pragma unroll 1
      for (int i = tid; i < n; i += NT) {
        S kr[M];
        lds_vec<S, M>(kr, Kt + size_t(i) * P);
        const S uT = slotA(i);
        const double rr = double(rel_of(i));
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < M; ++k)
          if (k < m - 1) acc = fma(rr * exD[k], double(mul_(mul_(kr[k], uT), vT[k])), acc);
        a.partial[size_t(u) * n + i] = acc;
      }
      return;
    }
    if (phase == PHASE_FWD_CONT) {
      // tolerance mode: continue this step's forward from v~^{t0}, t0 = Th
      if (tid < P) vec0[tid] = vh[size_t(Th) * P + tid];
      __syncthreads();
      goto forward_iterations;
    }
    __syncthreads();
    mark(3);
    if (improved) write_policy();   // best-so-far policy is step k-1's (solver.py:217-219)
    __syncthreads();
    mark(4);

    // ---------------- seed: W = gx .* X  (sinkhorn.py:272-275) --------------
    if constexpr (TC) {
      // ---------------- tensor-core adjoint (tcgen05 + TMEM) ----------------
      // The adjoint G (gK = K~ .* G) is only ever accumulated during the sweep
      // -- the levels read K~, never G -- so its 2T rank-1 terms
      //   G = a b' - sum_t (u~^t cv^t' + h^t v~^{t-1}')     (sinkhorn.py:288, :297)
      // are one [rows x 2T] x [2T x m] product: every 4 levels (K = 8) one
      // 128 x NPC x 8 tf32 MMA per 128-row block accumulates into TMEM, split
      // 3xTF32 (hi*hi + hi*lo + lo*hi) for fp32 accuracy.  A (u~, h of each
      // row, two levels per 16-byte store) and B (-cv, -v~^{t-1} per column)
      // are staged in shared memory in the canonical K-major no-swizzle layout
      // (8-row x 16-byte core matrices, LBO 128 B between the two K halves,
      // SBO 256 B between 8-row groups); A lies over the K~ tile, which the
      // register-resident sweep does not read.  The seed W = K~ .* (a b') is
      // added in the epilogue.  Row i = tid + r*NT is TMEM lane i % 128 of
      // block i / 128: the lanes warp (tid / 32) % 4 may access.
      // The FP32 pipe keeps 3 of the 5 FMAs per cell-level (two row dots and
      // the column dot); the rank-2 update moves to the tensor pipe.
      constexpr int NB = NT * R / 128;
      constexpr int NI = NB < NW ? NB : NW;   // issuing warps (one commit each)
      constexpr bool PKR_TC = sizeof(S) == 4;  // packed replay dot, as the register-resident sweep
      const int warp_id = tid >> 5;
      const int lane_id = tid & 31;
      const uint32_t lane_base = uint32_t(32 * (warp_id & 3)) << 16;
      unsigned char* Abuf = reinterpret_cast<unsigned char*>(Kt);   // [NB][hi, lo][128 rows x 32 B]
      if (warp_id == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TcShape<M, R, NT>::kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
      }
      if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "n"((NSW_TC_EXP & 16) ? 1 : NI));
      for (int q = tid; q < 4 * NPC * 8; q += NT) Bop[q] = 0.f;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tmem = *tmem_slot;
      const uint32_t mb = smem_u32(mbar);
      // tf32 split x = hi + lo: hi = x rounded to tf32, lo = x - hi exact in
      // fp32 (the MMA reads its top 19 bits)
      auto split = [](float x, float& hi, float& lo) {
        hi = to_tf32(x);   // round to nearest: |lo| <= 2^-11 |x| (truncation doubles it: 10x worse dC)
        lo = x - hi;
      };
      // A: this thread's rows; row i = tid + r*NT -> block (tid >> 7) + r*NT/128,
      // row p = tid & 127 of the block; (x0..x3) at K slots 4q..4q+3, hi / lo
      unsigned char* const a_base = Abuf + size_t(tid >> 7) * 8192 + ((tid & 127) >> 3) * 256 + (tid & 7) * 16;
      auto put_a = [&](int r, float x0, float x1, float x2, float x3, int q) {
        if constexpr (NSW_TC_EXP & 1) return;   // timing-only diagnostics build
        unsigned char* dst = a_base + size_t(r) * (NT / 128) * 8192 + q * 128;
        float4 hi, lo;
        split(x0, hi.x, lo.x);
        split(x1, hi.y, lo.y);
        split(x2, hi.z, lo.z);
        split(x3, hi.w, lo.w);
        *reinterpret_cast<float4*>(dst) = hi;
        *reinterpret_cast<float4*>(dst + 4096) = lo;
      };
      // B: written by the last warp (warp 0 finishes the column reductions):
      // column n = tid - (NT - 32) < NPC, (x0, x1) at K slots 2j, 2j+1
      const int bn = tid - (NT - 32);
      float* const b_base = Bop + (bn >> 3) * 64 + (bn & 7) * 4;
      auto put_b = [&](int bb, int j, float x0, float x1) {
        if constexpr (NSW_TC_EXP & 1) return;
        float* bh = b_base + bb * 2 * NPC * 8 + (j >> 1) * 32 + (j & 1) * 2;
        float h0, l0, h1, l1;
        split(x0, h0, l0);
        split(x1, h1, l1);
        *reinterpret_cast<float2*>(bh) = make_float2(h0, h1);
        *reinterpret_cast<float2*>(bh + NPC * 8) = make_float2(l0, l1);
      };
      int chunk = 0;   // chunks issued so far; B buffer of the current chunk = chunk & 1
      auto issue = [&]() {
        if (!(NSW_TC_EXP & 2) && lane_id == 0 && ((NSW_TC_EXP & 16) ? warp_id == NW - 1 : warp_id < NI)) {
          asm volatile("tcgen05.fence::after_thread_sync;");
          const float* bb = Bop + (chunk & 1) * 2 * NPC * 8;
          const uint64_t bh = umma_desc_kmajor(smem_u32(bb), 128, 256);
          const uint64_t bl = umma_desc_kmajor(smem_u32(bb + NPC * 8), 128, 256);
#pragma unroll
          for (int b = (NSW_TC_EXP & 16) ? 0 : warp_id; b < NB; b += (NSW_TC_EXP & 16) ? 1 : NI) {
            const uint32_t d = tmem + uint32_t(b * NPC);
            const uint64_t ah = umma_desc_kmajor(smem_u32(Abuf + size_t(2 * b) * 4096), 128, 256);
            const uint64_t al = umma_desc_kmajor(smem_u32(Abuf + size_t(2 * b + 1) * 4096), 128, 256);
            umma_tf32_ss<NPC>(d, ah, bh, chunk > 0 ? 1u : 0u);
            umma_tf32_ss<NPC>(d, ah, bl, 1u);
            umma_tf32_ss<NPC>(d, al, bh, 1u);
          }
          umma_commit(mb);
        }
        __syncwarp();
        ++chunk;
      };

      S Kr[R][M];
      S ut[R];
      S gs[R];   // seed g_u (row sums of W), live only until the first level
      S ai[R];   // seed row factor a_i = u~^T_i r_i / Imp_i
      {
        S c[M], ex[M];
        load_ex(ex);
#pragma unroll
        for (int k = 0; k < M; ++k) c[k] = S(0);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid + r * NT;
          lds_vec<S, M>(Kr[r], Kt + size_t(i) * P);
          ut[r] = slotA(i);
          const S rr = rel_of(i);
          ai[r] = mul_(mul_(rr, impv_of(i)), ut[r]);
          S gsum = S(0);
#pragma unroll
          for (int k = 0; k < M; ++k) {
            const S W = mul_(Kr[r][k], mul_(ai[r], mul_(ex[k], vT[k])));
            gsum += W;
            c[k] += W;
          }
          gs[r] = gsum;
        }
        cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
          vec0[k] = mul_(mul_(vh[size_t(Th) * P + k], tot), inv_mass(k));   // cv^T = v~^T g_v / colmass
        });
      }
      mark(5);
      S up[R], hp[R];   // (u~, h) of the even level of the current pair
      S live[R];        // 1 on real rows, 0 on padding rows (finite MMA inputs)
#pragma unroll
      for (int r = 0; r < R; ++r) live[r] = ok(r) ? S(1) : S(0);
      // ODD: the level's K slot pair j = (Th - t) & 3 is odd (it completes a
      // 16-byte A store); the first level (t = Th) has j = 0
      auto level_tc = [&](const int t, auto first_c, auto last_c, auto odd_c) {
        constexpr bool FIRST = decltype(first_c)::value;
        constexpr bool LAST = decltype(last_c)::value;
        constexpr bool ODD = decltype(odd_c)::value;
        const int j = (Th - t) & 3;
        S cv[M], c[M];
        lds_vec<S, M>(cv, vec0);
        const S* vpp1 = vh + size_t(t - 1) * P;
        const S* vppp = vh + size_t(LAST ? 0 : t - 2) * P;
        if (bn >= 0 && bn < NPC) {
          const float x0 = bn < m ? -vec0[bn] : 0.f;
          const float x1 = bn < m ? -vpp1[bn] : 0.f;
          put_b(chunk & 1, j, x0, x1);
          if constexpr (LAST)
            for (int jj = j + 1; jj < 4; ++jj) put_b(chunk & 1, jj, 0.f, 0.f);   // short final chunk
        }
#pragma unroll
        for (int k = 0; k < M; ++k) c[k] = S(0);
        S uc[R], hc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const S sig = rdot<S, M, CH, true>(Kr[r], cv);
          S den = S(1);
          if constexpr (!LAST) {
            S vpp[M];
            lds_vec<S, M>(vpp, vppp);
            den = rdot<S, M, CH, PKR_TC>(Kr[r], vpp);
          }
          const S h = ut[r] * (FIRST ? gs[r] - ut[r] * sig : -(ut[r] * sig));
          uc[r] = ut[r] * live[r];
          hc[r] = h;
          if constexpr (!LAST) axpy_<S, M, true>(c, Kr[r], h);
          if constexpr (!LAST) ut[r] = rcp_clamped(den);
        }
        if constexpr (ODD || LAST) {
          // the chunk's first A store waits for the previous chunk's MMAs
          if (!(NSW_TC_EXP & 10) && (j == 1 || (LAST && j == 0)) && chunk > 0) mbar_wait(mb, uint32_t((chunk - 1) & 1));
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if constexpr (ODD) put_a(r, up[r], hp[r], uc[r], hc[r], j >> 1);
            else put_a(r, uc[r], hc[r], 0.f, 0.f, j >> 1);
          }
          // generic-proxy stores -> the MMA (async proxy), before the barrier
          // that precedes the issue
          if (!(NSW_TC_EXP & 4) && (j == 3 || LAST)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            up[r] = uc[r];
            hp[r] = hc[r];
          }
        }
        if constexpr (!LAST) {
          cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
            const S vpk = vh[size_t(t - 1) * P + k];
            const S gv = -mul_(vpk, tot);
            vec0[k] = mul_(mul_(vpk, gv), inv_mass(k));
          });
        } else {
          __syncthreads();
        }
        if (LAST || (ODD && j == 3)) issue();
      };
      using TT = std::true_type;
      using FF = std::false_type;
      if (Th == 1) {
        level_tc(1, TT{}, TT{}, FF{});
      } else {
        level_tc(Th, TT{}, FF{}, FF{});
        int t = Th - 1;   // always an odd-slot level here
        for (; t >= 3; t -= 2) {
          level_tc(t, FF{}, FF{}, TT{});
          level_tc(t - 1, FF{}, FF{}, FF{});
        }
        if (t == 2) {
          level_tc(2, FF{}, FF{}, TT{});
          level_tc(1, FF{}, TT{}, FF{});
        } else {
          level_tc(1, FF{}, TT{}, TT{});
        }
      }
      mark(6);
      if constexpr (!(NSW_TC_EXP & 2)) mbar_wait(mb, uint32_t((chunk - 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      // gK = K~ .* (a b' + G), G read back from TMEM, over the tile
      {
        S ex[M], vTe[M];
        load_ex(ex);
        lds_vec<S, M>(vTe, vh + size_t(Th) * P);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid + r * NT;
          const int b = i >> 7;
          float g[NPC];
#pragma unroll
          for (int q = 0; q < NPC / 16; ++q) {
            float g16[16];
            tmem_ld16(tmem + lane_base + uint32_t(b * NPC + 16 * q), g16);
#pragma unroll
            for (int e = 0; e < 16; ++e) g[16 * q + e] = g16[e];
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          S gk[M];
#pragma unroll
          for (int k = 0; k < M; ++k) gk[k] = ok(r) ? mul_(Kr[r][k], fma(ai[r], mul_(ex[k], vTe[k]), S(g[k]))) : S(0);
          sts_vec<S, M>(Kt + size_t(i) * P, gk);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      if (warp_id == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TcShape<M, R, NT>::kCols));
      }
    } else {
    S A[R][M];  // adjoint G: gK = W + K~ .* G
      S ut[R];
      S gs[R];    // seed g_u (row sums of W), live only until the first level
      {
        S c[M], ex[M];
        load_ex(ex);
  #pragma unroll
        for (int k = 0; k < M; ++k) c[k] = S(0);
  #pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid + r * NT;
          S kr[M];
          lds_vec<S, M>(kr, Kt + size_t(i) * P);
          ut[r] = slotA(i);
          const S rr = rel_of(i);
          S gsum = S(0);
          if constexpr (RANK1) {
            // W = K~ .* (a b'), a_i = u~^T_i r_i / Imp_i, b_k = e_k v~^T_k:
            // G starts at a b', so gK = K~ .* G at the end needs no W
            const S ai = mul_(mul_(rr, impv_of(i)), ut[r]);
  #pragma unroll
            for (int k = 0; k < M; ++k) {
              A[r][k] = mul_(ai, mul_(ex[k], vT[k]));
              const S W = mul_(kr[k], A[r][k]);
              gsum += W;
              c[k] += W;
            }
          } else {
  #pragma unroll
            for (int k = 0; k < M; ++k) {
              A[r][k] = S(0);
              if (k < m - 1) {
                const S X = mul_(mul_(kr[k], ut[r]), vT[k]);
                const S W = mul_(gx_of(rr, ex[k], impv_of(i)), X);
                gsum += W;
                c[k] += W;
              }
            }
          }
          gs[r] = gsum;
        }
        cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
          vec0[k] = mul_(mul_(vh[size_t(Th) * P + k], tot), inv_mass(k));   // cv^T = v~^T g_v / colmass
        });
      }
      mark(5);

      // Per level t, per row i (u~ = u~^t_i, cv = v~^t g_v / colmass):
      //   g_u  <- [t==T] g_u^seed - u~ (K~ cv)_i                  column VJP
      //   h    <- u~ g_u
      //   G_ik <- G_ik - u~ cv_k - h v~^{t-1}_k                    both VJPs into gK
      //   g_v  <- -v~^{t-1} (K~' h)                                row VJP (t >= 2)
      //   u~   <- 1/(K~ v~^{t-2})_i                                replay (t >= 2)
      // The first level (seed g_u) and the last (t = 1: v^0 = lvi is held
      // constant, so neither g_v nor a replay is needed) are peeled, so the
      // steady-state body is branch-free.  Padding rows (K~ row = 0) get a
      // finite u~ from the clamped reciprocal, hence h = 0 and no column
      // contribution; their G is discarded in the epilogue.
      // cv of the current level: in registers of every thread, delivered by
      // the previous level's broadcast reduction (NSW_BCAST) or from vec0
      S cvr[M];
      if constexpr (NSW_BCAST) lds_vec<S, M>(cvr, vec0);
      // KREG: the K~ rows stay in registers for the whole sweep
      // (next to the adjoint) instead of one shared-memory row read per level
#ifndef NSW_KREG_BWD
#define NSW_KREG_BWD 1   // +12 % config 2, +3 % config 3 (profiles/r02/ab_kreg_backward.txt)
#endif
#ifndef NSW_KREG_MINR
#define NSW_KREG_MINR 2   // R = 2 tail tiles: +2.7 % config 1 (profiles/r02/ab_kreg_tail_tiles.txt)
#endif
      // (only where the two R x M tiles and the level vectors fit the register cap)
      constexpr int REG_CAP = (65536 / (NT * MINB)) < 255 ? (65536 / (NT * MINB)) : 255;
      constexpr bool KREG = NSW_KREG_BWD && sizeof(S) == 4 && MINB == 1 && R >= NSW_KREG_MINR &&
                            2 * R * M + 3 * M + 24 <= REG_CAP;
      // packed FFMA2 (fma.rn.f32x2) in the register-resident backward's sig
      // dot and rank-1 updates: its issue rate is bound by register-bank reads
      // (a 3-register FFMA needs two cycles unless an operand comes from the
      // reuse cache), and a packed FMA with a broadcast operand halves the
      // instructions for the same reads
#ifndef NSW_PK_BWD
#define NSW_PK_BWD 1
#endif
      constexpr bool PKB = PK || (NSW_PK_BWD && sizeof(S) == 4 && KREG);
      // the replay dot packed too (backward -5 %, config 2): fp32 replays then
      // differ from the forward's u~ in the last bits (fp64 never packs); the
      // forward's own dot stays scalar (packed it is 10 % slower: latency-bound)
#ifndef NSW_PK_REPLAY
#define NSW_PK_REPLAY 1
#endif
      constexpr bool PKR = PKD || (NSW_PK_REPLAY && PKB);
      S Kr[KREG ? R : 1][M];
      if constexpr (KREG) {
#pragma unroll
        for (int r = 0; r < R; ++r) lds_vec<S, M>(Kr[r], Kt + size_t(tid + r * NT) * P);
      }
      auto level = [&](const int t, auto first_c, auto last_c) {
        constexpr bool FIRST = decltype(first_c)::value;
        constexpr bool LAST = decltype(last_c)::value;
        S cv[M], vp[M], c[M];
        if constexpr (NSW_BCAST) {
#pragma unroll
          for (int k = 0; k < M; ++k) cv[k] = cvr[k];
        } else {
          lds_vec<S, M>(cv, vec0);
        }
        const S* vpp1 = vh + size_t(t - 1) * P;
        if constexpr (!LEAN) lds_vec<S, M>(vp, vpp1);
        const S* vppp = vh + size_t(LAST ? 0 : t - 2) * P;
  #pragma unroll
        for (int k = 0; k < M; ++k) c[k] = S(0);
  #pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid + r * NT;
          S kr[M];
          if constexpr (KREG) {
#pragma unroll
            for (int k = 0; k < M; ++k) kr[k] = Kr[r][k];
          } else {
            lds_vec<S, M>(kr, Kt + size_t(i) * P);
          }
          const S sig = rdot<S, M, CH, PKB>(kr, cv);
          S den = S(1);
          if constexpr (!LAST) {
            S vpp[M];
            if constexpr (LEAN) lds_vec_nc<S, M>(vpp, vppp);
            else lds_vec<S, M>(vpp, vppp);
            den = rdot<S, M, CH, PKR>(kr, vpp);
          }
          const S h = ut[r] * (FIRST ? gs[r] - ut[r] * sig : -(ut[r] * sig));
          if constexpr (LEAN) lds_vec_nc<S, M>(vp, vpp1);
          axpy_<S, M, PKB>(A[r], cv, -ut[r]);
          axpy_<S, M, PKB>(A[r], vp, -h);
          if constexpr (!LAST) axpy_<S, M, PKB>(c, kr, h);
          if constexpr (!LAST) ut[r] = rcp_clamped(den);
        }
        if constexpr (!LAST) {
          if constexpr (NSW_BCAST) {
            cta_reduce_cols_bcast<S, M, NT>(
                c, red + (t & 1) * NW * M, m,
                [&](int k, S tot) -> S {
                  const S vpk = vh[size_t(t - 1) * P + k];
                  const S gv = -mul_(vpk, tot);
                  return mul_(mul_(vpk, gv), inv_mass(k));
                },
                cvr);
          } else {
            cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
              const S vpk = vh[size_t(t - 1) * P + k];
              const S gv = -mul_(vpk, tot);
              vec0[k] = mul_(mul_(vpk, gv), inv_mass(k));
            });
          }
        }
      };
      if (Th == 1) {
        level(1, std::true_type{}, std::true_type{});
      } else {
        level(Th, std::true_type{}, std::false_type{});
        for (int t = Th - 1; t >= 2; --t) level(t, std::false_type{}, std::false_type{});
        level(1, std::false_type{}, std::true_type{});
      }
      mark(6);
      // gK = W + K~ .* G, written over K~ in the tile (fp64: W = gx .* X
      // recomputed in the reference's operation order; fp32: folded into G
      // at the seed).  v~^T and the exposures are reloaded here rather than
      // held across the levels.
      if constexpr (RANK1) {
  #pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid + r * NT;
          S kr[M], gk[M];
          lds_vec<S, M>(kr, Kt + size_t(i) * P);
  #pragma unroll
          for (int k = 0; k < M; ++k) gk[k] = ok(r) ? mul_(kr[k], A[r][k]) : S(0);   // padding rows stay 0
          sts_vec<S, M>(Kt + size_t(i) * P, gk);
        }
      } else {
        S ex[M], vTe[M];
        load_ex(ex);
        lds_vec<S, M>(vTe, vh + size_t(Th) * P);
  #pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid + r * NT;
          S kr[M], gk[M];
          lds_vec<S, M>(kr, Kt + size_t(i) * P);
          const S uT = slotA(i);
          const S rr = rel_of(i);
  #pragma unroll
          for (int k = 0; k < M; ++k) {
            const S X = mul_(mul_(kr[k], uT), vTe[k]);
            const S W = (k < m - 1) ? mul_(gx_of(rr, ex[k], impv_of(i)), X) : S(0);
            gk[k] = ok(r) ? fma(kr[k], A[r][k], W) : S(0);   // padding rows stay 0 for the forward
          }
          sts_vec<S, M>(Kt + size_t(i) * P, gk);
        }
      }
    }
    if (tid < m) vec2[tid] = a.warm_start ? add_(vec1[tid], F::log_(vh[size_t(Th) * P + tid])) : S(0);
    __syncthreads();
    mark(7);

    // ---------------- g_C = gK * (-1/eps); Adam ascent  (solver.py:105-122) -
    const int s = a.state[ST_STEP];
    const S bc1 = S(a.bc[2 * s]), bc2 = S(a.bc[2 * s + 1]);
    const S ibc1 = S(1.0 / a.bc[2 * s]), ibc2 = S(1.0 / a.bc[2 * s + 1]);
    auto adam = [&](S& cc, S& mm, S& vv, S gk) {
      const S g = mul_(gk, a.nie);
      mm = add_(mul_(a.b1, mm), mul_(a.omb1, g));
      vv = add_(mul_(a.b2, vv), mul_(mul_(a.omb2, g), g));
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
    if (vec_ok) {
      const int nq = nm / V;
      for (int q0 = tid; q0 < nq; q0 += 6 * NT) {
        V16<S> c[6], mm[6], vv[6];
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          const int q = q0 + b * NT;
          if (q < nq) {
            c[b].v = reinterpret_cast<const V16<S>*>(Cu)[q].v;
            mm[b].v = reinterpret_cast<const V16<S>*>(mu)[q].v;
            vv[b].v = reinterpret_cast<const V16<S>*>(vu)[q].v;
          }
        }
#pragma unroll
        for (int b = 0; b < 6; ++b) {
          const int q = q0 + b * NT;
          if (q >= nq) break;
          int i = q * V / m, k = q * V - i * m;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            S& slot = Kt[i * P + k];
            adam(c[b].s[j], mm[b].s[j], vv[b].s[j], slot);
            slot = mul_(c[b].s[j], a.nie);
            if (++k == m) { k = 0; ++i; }
          }
          reinterpret_cast<V16<S>*>(Cu)[q].v = c[b].v;
          reinterpret_cast<V16<S>*>(mu)[q].v = mm[b].v;
          reinterpret_cast<V16<S>*>(vu)[q].v = vv[b].v;
        }
      }
    } else {
      for (int e = tid; e < nm; e += NT) {
        const int i = e / m, k = e - i * m;
        S c = Cu[e], mm = mu[e], vv = vu[e];
        S& slot = Kt[i * P + k];
        adam(c, mm, vv, slot);
        slot = mul_(c, a.nie);
        Cu[e] = c;
        mu[e] = mm;
        vu[e] = vv;
      }
    }
  } else {
    // INIT: initial cost C0 = -eps log(uniform) (solver.py:176-177), lvi = 0.
    // RESUME: caller-provided C (left as is), lvi taken from the beta buffer.
    const bool init = phase == PHASE_INIT;
    if (!init && tid < m) vec2[tid] = a.beta[size_t(u) * m + tid];
    for (int q = tid; q < (vec_ok ? nm / V : nm); q += NT) {
      const int e0 = vec_ok ? q * V : q;
      int i = e0 / m, k = e0 - i * m;
      if (vec_ok) {
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
    }
  }
  __syncthreads();
  mark(8);

  // ======================= forward of step k =================================
  // Absorption point: beta = lvi (the warm-start column duals, so v~^0 = 1)
  // and alpha_i = -max_k (K_ik + beta_k), so every K~ row peaks at exactly 1.
  // Then iterations t = 1..T are the multiplicative Sinkhorn updates, the
  // same fixed point as the log-domain iterations of sinkhorn.py:219-234:
  //   u~^t = 1 / (K~ v~^{t-1}),   v~^t = colmass / (K~' u~^t),
  //   u^t = alpha + log u~^t,     v^t = beta + log v~^t.
  if (tid < m) {
    a.beta[size_t(u) * m + tid] = vec2[tid];
    hu[tid] = S(1);                       // v~^0
    vec0[tid] = S(1);
  }
  {
    S bt[M];
    lds_vec<S, M>(bt, vec2);
#pragma unroll 1
    for (int i = tid; i < n; i += NT) {
      S kr[M];
      lds_vec<S, M>(kr, Kt + size_t(i) * P);   // K = C * (-1/eps)
      S mx = F::ninf();
#pragma unroll
      for (int k = 0; k < M; ++k)
        if (k < m) mx = fmax(mx, add_(kr[k], bt[k]));
      const S al = -mx;
      a.alpha[size_t(u) * n + i] = al;
#pragma unroll
      for (int k = 0; k < M; ++k) kr[k] = (k < m) ? F::exp_fast(add_(add_(kr[k], bt[k]), al)) : S(0);
      sts_vec<S, M>(Kt + size_t(i) * P, kr);
    }
  }
  __syncthreads();
  mark(9);
forward_iterations:
  // Wide-row forward (fixed schedule, one-CTA-per-SM fp32 tiles whose
  // doubled row tile fits the register file): half the warps each hold 2R
  // K~ rows; the column reduction's shuffle and barrier work is per warp, so
  // it halves, and the rows supply the FMA chains' independence (config 2:
  // the reduce-scatter and its barriers were ~40 % of the forward).
#ifndef NSW_WIDE_FWD
#define NSW_WIDE_FWD 1
#endif
  if constexpr (NSW_WIDE_FWD && sizeof(S) == 4 && MINB == 1 && NT >= 256 && R <= 4 && M <= 32 &&
                2 * R * M + 2 * M + 2 * R + 24 <= (65536 / NT < 255 ? 65536 / NT : 255)) {
    if (!tolm) {
      constexpr int NTA = NT / 2, RA = 2 * R;
      if (tid >= NTA) return;   // nothing after the forward needs the idle warps
      S A[RA][M];
      S ut[RA];
#pragma unroll
      for (int r = 0; r < RA; ++r) lds_vec<S, M>(A[r], Kt + size_t(tid + r * NTA) * P);
      S vv[M];
      for (int t = 1; t <= T; ++t) {
        lds_vec<S, M>(vv, vec0);
        S c[M];
#pragma unroll
        for (int r = 0; r < RA; ++r) ut[r] = rcp_clamped(rdot<S, M, 1, PKD>(A[r], vv));
#pragma unroll
        for (int k = 0; k < M; ++k) c[k] = S(0);
#pragma unroll
        for (int r = 0; r < RA; ++r) axpy_<S, M, PKF>(c, A[r], ut[r]);
        cta_reduce_cols_part<S, M, NTA, OpSum>(c, red, m, [&](int k, S tot) {
          const S vn = F::div_fast(mass(k), tot);
          vec0[k] = vn;
          hu[size_t(t) * m + k] = vn;
        });
      }
      mark(10);
      lds_vec<S, M>(vv, vec0);
#pragma unroll
      for (int r = 0; r < RA; ++r) {
        const int i = tid + r * NTA;
        const double rr = double(rel_of(i));
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          if (k < m - 1) {
            const S X = mul_(mul_(A[r][k], ut[r]), vv[k]);
            acc = fma(rr * exD[k], double(X), acc);
          }
        }
        if (i < n) a.partial[size_t(u) * n + i] = acc;
      }
      mark(11);
      return;
    }
  }
  {
    S A[R][M];  // K~, register resident
    S ut[R];
    const int t_start = phase == PHASE_FWD_CONT ? Th + 1 : 1;
    const int t_end = tolm ? min(t_start - 1 + a.chunk, T) : T;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      lds_vec<S, M>(A[r], Kt + size_t(tid + r * NT) * P);
      ut[r] = S(0);
    }
    // tolerance mode also records the reference's L-inf marginal residual of
    // every iteration (sinkhorn.py:237-243): the row sums of X^{t-1} are
    // u~^{t-1} (K~ v~^{t-1}) -- the next iteration's own row dot -- and the
    // column sums are v~ times the column totals.
    auto warp_max = [&](S x) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      return x;
    };
    // the iteration body is instantiated twice so the fixed schedule carries
    // no residual bookkeeping at all
    auto iterate = [&](auto tol_c) {
      constexpr bool TOLM = decltype(tol_c)::value;
      if constexpr (!TOLM && NSW_BCAST) {
        // fixed schedule: v~ stays in registers; one barrier per iteration
        S vv[M];
        lds_vec<S, M>(vv, vec0);
        for (int t = t_start; t <= t_end; ++t) {
          S c[M];
#pragma unroll
          for (int r = 0; r < R; ++r) ut[r] = rcp_clamped(rdot<S, M, CH, PKD>(A[r], vv));
#pragma unroll
          for (int k = 0; k < M; ++k) c[k] = S(0);
#pragma unroll
          for (int r = 0; r < R; ++r) axpy_<S, M, PKF>(c, A[r], ut[r]);
          cta_reduce_cols_bcast<S, M, NT>(
              c, red + (t & 1) * NW * M, m,
              [&](int k, S tot) -> S {
                const S vn = F::div_fast(mass(k), tot);
                if (warp == 0) {
                  vec0[k] = vn;
                  hu[size_t(t) * m + k] = vn;
                }
                return vn;
              },
              vv);
        }
        __syncthreads();   // warp 0's last vec0 before the impact terms read it
        return;
      }
      for (int t = t_start; t <= t_end; ++t) {
        S vv[M], c[M];
        lds_vec<S, M>(vv, vec0);
        S rmax = S(0);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const S sr = rdot<S, M, CH, PKD>(A[r], vv);
          if (TOLM && ok(r)) rmax = fmax(rmax, fabs(ut[r] * sr - S(1)));
          ut[r] = rcp_clamped(sr);
        }
        if constexpr (TOLM) {
          rmax = warp_max(rmax);
          if (lane == 0) redmax[warp] = rmax;
        }
#pragma unroll
        for (int k = 0; k < M; ++k) c[k] = S(0);
#pragma unroll
        for (int r = 0; r < R; ++r) axpy_<S, M, PKF>(c, A[r], ut[r]);
        cta_reduce_cols<S, M, NT, OpSum>(c, red, m, [&](int k, S tot) {
          const S vn = F::div_fast(mass(k), tot);
          vec0[k] = vn;
          hu[size_t(t) * m + k] = vn;
          if constexpr (TOLM) {
            // fp64: |v~ (K~' u~) - colmass| as the reference measures it; fp32
            // cannot resolve 1e-6 against the dummy mass, and the columns are
            // normalised exactly by construction, so it counts as 0 there.
            colres[(t & 1) * P + k] = sizeof(S) == 8 ? fabs(vn * tot - mass(k)) : S(0);
            if (k == 0 && t > t_start) {
              S r = S(0);
              for (int w = 0; w < NW; ++w) r = fmax(r, redmax[w]);
              for (int kk = 0; kk < m; ++kk) r = fmax(r, colres[((t - 1) & 1) * P + kk]);
              a.res[size_t(u) * (T + 1) + t - 1] = double(r);
            }
          }
        });
      }
    };
    if (tolm) {
      iterate(std::true_type{});
    } else {
      iterate(std::false_type{});
    }
    mark(10);
    if (tolm) {
      // residual of the chunk's last iteration needs one more row pass
      S vv[M];
      lds_vec<S, M>(vv, vec0);
      S rmax = S(0);
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (ok(r)) rmax = fmax(rmax, fabs(ut[r] * rdot<S, M, CH, PKD>(A[r], vv) - S(1)));
      rmax = warp_max(rmax);
      if (lane == 0) redmax[warp] = rmax;
      __syncthreads();
      if (tid == 0) {
        S r = S(0);
        for (int w = 0; w < NW; ++w) r = fmax(r, redmax[w]);
        for (int kk = 0; kk < m; ++kk) r = fmax(r, colres[(t_end & 1) * P + kk]);
        a.res[size_t(u) * (T + 1) + t_end] = double(r);
      }
      return;  // impact terms come from the finish launch once t* is known
    }
  // per-item impact terms of this user (solver.py:206), float64
  {
    S vv[M];
    lds_vec<S, M>(vv, vec0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = tid + r * NT;
      const double rr = double(rel_of(i));
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        if (k < m - 1) {
          const S X = mul_(mul_(A[r][k], ut[r]), vv[k]);
          acc = fma(rr * exD[k], double(X), acc);
        }
      }
      if (ok(r)) a.partial[size_t(u) * n + i] = acc;
    }
  }
  mark(11);
  }
}

// --------------------------------------------------------------------------
// Impact reduction over this rank's users (deterministic, fixed order):
// split[y][i] = sum over user chunk y; the last CTA to finish sums the chunks.
// --------------------------------------------------------------------------
constexpr int IMP_THREADS = 256;
constexpr int IMP_ITEMS = 8;
struct FinalizeArgs {
  int n, world, outer_max;
  const double* imp_all;   // [world][n + 1]: impacts + converged-user count per rank
  const double* rel_sq;    // [n] sum_u r_ui^2 over all users
  double exp_sq;           // sum_k e_k^2
  double grad_threshold;
  double* imp_cur;         // [n]
  double* best;            // [1]
  double* objective;       // [outer_max]
  double* grad_norm;       // [outer_max]
  unsigned long long* stamp;  // [outer_max+1] globaltimer ns
  int* state;
  int tol_mode, U, T;
  int U_total;             // users over all ranks (SolverError fraction)
  double tol;
  const double* res;       // [U][T+1] residuals (tolerance mode)
  int* iters;              // [outer_max] inner iterations per step (trace)
};

// imp_local has n + 1 slots: the n impacts and, in tolerance mode, this
// shard's count of users whose residual at t* is <= tol (the exchange
// carries it to every rank for the SolverError guard).
__global__ void impact_reduce_kernel(const double* __restrict__ partial, int U, int n, int chunks,
                                     double* __restrict__ split, unsigned int* counter,
                                     double* __restrict__ imp_local, const int* __restrict__ state, int tol_mode,
                                     const double* __restrict__ res, int T, double tol, int fuse_finalize,
                                     FinalizeArgs fin);

// Tolerance mode, after each forward chunk, the lock-step stopping test of
// sinkhorn.py:244 in two parts so the ranks of a sharded solve can combine
// their maxima in between (all-reduce MAX, in place):
//   tol_chunk_max_kernel: cmax[j] = max over this shard's users of the
//     residual after iteration t0+1+j of the chunk;
//   tol_decide_kernel: t* = first iteration whose (global) max is <= tol;
//     sets PHASE_FWD_FIN (t* found or the budget is spent) or PHASE_FWD_CONT.
__global__ void tol_chunk_max_kernel(const double* __restrict__ res, int U, int T, int chunk, const int* state,
                                     double* __restrict__ cmax);
__global__ void tol_decide_kernel(const double* __restrict__ cmax, int T, int chunk, double tol, int* state,
                                  unsigned long long cond = 0);


__global__ void finalize_kernel(FinalizeArgs f);
__global__ void stamp_kernel(unsigned long long* stamp);
__global__ void flush_kernel(float* buf, size_t n);
__global__ void discard_kernel(float* buf, size_t n);
__global__ void widen_kernel(const float* __restrict__ src, double* __restrict__ dst, size_t n, unsigned* bad);
__global__ void narrow_kernel(const double* __restrict__ src, float* __restrict__ dst, size_t n);
__global__ void rel_check_kernel(const double* __restrict__ rel, size_t count, unsigned* __restrict__ flags);
__global__ void rel_sq_kernel(const double* __restrict__ rel, int U, int n, double* __restrict__ rsq);

}  // namespace nsw
