// Device building blocks of the NSW ascent path (sm_100a).
//
// Data layout in HBM (per GPU, users are this rank's contiguous block):
//   C, adam_m, adam_v, xbest : [U][n][m]   reference layout (solver.py:176-185)
//   alpha                    : [U][n]      row absorption point
//   beta                     : [U][m]      column absorption point (= lvi)
//   hist                     : [U][T+1][m] v~^t = exp(v^t - beta), t = 0..T
//   partial                  : [U][n] f64  per-user impact terms
//
// Numerical form ("stabilised multiplicative"):
// every solve absorbs beta = lvi (the warm-start column duals of
// sinkhorn.py:213, so v~^0 = 1) and alpha_i = -max_k (K_ik + beta_k) into
// K~ = exp(K + alpha 1' + 1 beta') <= 1, then runs the T iterations of
// sinkhorn.py:218-236 as u~ = 1/(K~ v~), v~ = colmass/(K~' u~) -- two FMAs
// per cell and one reciprocal per row / column, with K~ held in registers;
// u = alpha + log u~, v = beta + log v~ are the reference's log-domain duals.
// The unrolled reverse mode (sinkhorn.py:258-309) is restated in the same
// coordinates (see step_kernel in nsw_step_kernel.cuh).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <cstdio>

#include <type_traits>

namespace nsw {

// PHASE_RESUME: forward of step k from a caller-provided cost tensor, with the
// warm-start duals lvi supplied in the `beta` buffer (checkpoint / resume,
// and one-step parity from an oracle state).
// Tolerance mode (the reference's default stopping rule, sinkhorn.py:237-246)
// runs each forward in chunks: PHASE_FWD_CONT = continue this step's forward,
// PHASE_FWD_FIN = the lock-step stop t* is known, emit X^{t*}'s impact terms.
enum : int {
  PHASE_INIT = 0,
  PHASE_RUNNING = 1,
  PHASE_DONE_PENDING = 2,
  PHASE_FINISHED = 3,
  PHASE_RESUME = 4,
  PHASE_FWD_CONT = 5,
  PHASE_FWD_FIN = 6
};
// ST_T0: inner iterations done in the current forward; ST_TSTAR: iterations of
// the last finished forward (the next backward's depth); ST_CONV: users within
// tolerance at t* (for the > 50 % guard of solver.py:200-205).
enum : int { ST_PHASE = 0, ST_STEP = 1, ST_IMPROVED = 2, ST_ERR = 3, ST_T0 = 4, ST_TSTAR = 5, ST_CONV = 6 };
constexpr int ST_WORDS = 8;
enum : int { ERR_IMPACT = 1, ERR_NONFINITE = 2, ERR_SOLVER = 4 };

// ---------------------------------------------------------------------------
// Checked build (-DNSW_CHECKS=1, `build.py --tag checked -D NSW_CHECKS=1`):
// the tests run against it in place of compute-sanitizer (closed on the GPU
// pool).  Every vector shared-memory access of the tiles is bounds-checked
// against the CTA's shared-memory size, the dynamic shared memory is poisoned
// with NaN at kernel entry (a read of a never-written slot propagates NaN into
// the parity comparisons), mbarrier waits trap after ~2^28 polls instead of
// hanging, and every solver buffer gets 64 KB canary guard bands that are
// verified when it is freed (nsw_capi.cu).
// ---------------------------------------------------------------------------
#ifndef NSW_CHECKS
#define NSW_CHECKS 0
#endif

__device__ __forceinline__ void nsw_check_fail(const char* what, unsigned a, unsigned b) {
  printf("NSW_CHECKS: %s (block %d thread %d: %u vs %u)\n", what, int(blockIdx.x), int(threadIdx.x), a, b);
  __trap();
}

// shared-memory window [p, p + bytes) lies inside this CTA's shared memory
__device__ __forceinline__ void nsw_check_smem(const void* p, unsigned bytes) {
  if constexpr (NSW_CHECKS) {
    if (!__isShared(p)) nsw_check_fail("vector access outside shared memory", 0u, 0u);
    unsigned total, dyn;
    asm("mov.u32 %0, %%total_smem_size;" : "=r"(total));
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    extern __shared__ __align__(16) unsigned char nsw_dyn_base[];
    // the dynamic window [base, base + dyn) ends the CTA's shared memory
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(nsw_dyn_base));
    const unsigned off = static_cast<unsigned>(__cvta_generic_to_shared(p));
    if (off + bytes > base + dyn)
      nsw_check_fail("shared-memory access past the CTA's allocation", off + bytes - base, dyn);
    (void)total;
  }
}

// fill the dynamic shared memory with quiet NaNs (checked builds)
__device__ __forceinline__ void nsw_poison_smem(unsigned char* base) {
  if constexpr (NSW_CHECKS) {
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    for (unsigned q = threadIdx.x; q < dyn / 4; q += blockDim.x) reinterpret_cast<unsigned*>(base)[q] = 0x7fffffffu;
    __syncthreads();
  }
}

template <typename S>
struct Fp;

template <>
struct Fp<float> {
  static __device__ __forceinline__ float exp_(float x) { return expf(x); }
  // exp(x) = 2^(x log2 e) on the SFU: 2 instructions, ~2 ulp + |x| 2^-24
  static __device__ __forceinline__ float exp_fast(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
    return y;
  }
  static __device__ __forceinline__ float log_(float x) { return logf(x); }
  static __device__ __forceinline__ float rcp(float x) { return __frcp_rn(x); }
  // hot-loop reciprocal: one MUFU.RCP (<= 1 ulp), no IEEE fix-up branch.
  // volatile: executed unconditionally, so a select on its result is an
  // FSEL rather than a branch around the asm block.
  static __device__ __forceinline__ float rcp_fast(float x) {
    float y;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float div_fast(float a, float b) { return a * rcp_fast(b); }
  static __device__ __forceinline__ float sqrt_(float x) { return __fsqrt_rn(x); }
  static __device__ __forceinline__ float ninf() { return -CUDART_INF_F; }
  static __device__ __forceinline__ float tiny() { return 1.17549435e-38f; }  // FLT_MIN
  static constexpr int kVec = 4;  // elements per 16-byte vector
};

template <>
struct Fp<double> {
  static __device__ __forceinline__ double exp_(double x) { return exp(x); }
  static __device__ __forceinline__ double exp_fast(double x) { return exp(x); }
  static __device__ __forceinline__ double log_(double x) { return log(x); }
  static __device__ __forceinline__ double rcp(double x) { return __drcp_rn(x); }
  static __device__ __forceinline__ double rcp_fast(double x) { return __drcp_rn(x); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double div_fast(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt_(double x) { return __dsqrt_rn(x); }
  static __device__ __forceinline__ double ninf() { return -CUDART_INF; }
  static __device__ __forceinline__ double tiny() { return 2.2250738585072014e-308; }  // DBL_MIN
  static constexpr int kVec = 2;
};

// Packed fp32 FMA (sm_100 FFMA2, fma.rn.f32x2): two independent IEEE fmas
// per instruction, d = a * b + c lane-wise -- the same rounding as two FFMAs,
// half the issue slots.  A scalar b (b0 == b1) becomes FFMA2's broadcast
// operand form.
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0,
                                      float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}

// NSW_FFMA2=0 builds the scalar-FFMA form of the same loops (A/B experiments).
#ifndef NSW_FFMA2
#define NSW_FFMA2 1
#endif

// c[k] += x[k] * s over an M-vector (IEEE fma each; PK: fp32 pairs packed
// into FFMA2).
template <typename S, int M, bool PK = false>
__device__ __forceinline__ void axpy_(S (&c)[M], const S (&x)[M], S s) {
  if constexpr (sizeof(S) == 4 && NSW_FFMA2 && PK) {
#pragma unroll
    for (int k = 0; k + 1 < M; k += 2) ffma2(c[k], c[k + 1], x[k], x[k + 1], s, s, c[k], c[k + 1]);
    if constexpr (M % 2) c[M - 1] = fmaf(x[M - 1], s, c[M - 1]);
  } else {
#pragma unroll
    for (int k = 0; k < M; ++k) c[k] = fma(x[k], s, c[k]);
  }
}

// Padded row pitch (elements) of a K~ row in shared memory: 16-byte multiple.
template <typename S, int M>
struct Pitch {
  static constexpr int value = (M + Fp<S>::kVec - 1) / Fp<S>::kVec * Fp<S>::kVec;
};

// Row pitch of the fused step kernel's K~ tile: fp32 rows span an odd number
// of 16-byte units, so the 8 lanes of a 128-bit load phase (8 consecutive
// rows) hit 8 distinct bank quads (M = 21 with a 24-float pitch was 2-way
// conflicted; M = 16 / 32 4- / 8-way).  fp64 keeps the tight pitch (its
// 2048-item parity tiles need the shared memory).
template <typename S, int M>
struct RowPitch {
  static constexpr int U = (M + Fp<S>::kVec - 1) / Fp<S>::kVec;
  static constexpr int value = sizeof(S) == 4 ? ((U % 2) ? U : U + 1) * Fp<S>::kVec : Pitch<S, M>::value;
};

struct OpSum {
  template <typename S>
  __device__ __forceinline__ S operator()(S a, S b) const { return a + b; }
  template <typename S>
  static __device__ __forceinline__ S identity() { return S(0); }
};

struct OpMax {
  template <typename S>
  __device__ __forceinline__ S operator()(S a, S b) const { return a > b ? a : b; }
  template <typename S>
  static __device__ __forceinline__ S identity() { return Fp<S>::ninf(); }
};

// Warp reduce-scatter of an M-vector held by every lane.  Stage OFF halves
// the live range: the lane with bit OFF clear keeps the lower half, its
// partner the upper half, each receiving the other's copy of its half.
// Cost ~ M shuffles instead of 5*M for a full butterfly.  After the five
// stages lane L holds the warp totals of columns [base, base+ceil(M/32))
// clipped at `lim` (columns past `lim` are padding of an uneven split).
template <typename S, int M, int CNT, int OFF, class Op>
__device__ __forceinline__ void reduce_scatter(S (&v)[M], int lane, int& base, int& lim) {
  if constexpr (OFF > 0) {
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
    reduce_scatter<S, M, H, OFF / 2, Op>(v, lane, base, lim);
  }
}

// Column reduction of per-thread M-vectors over the whole CTA, in a fixed
// order (warp reduce-scatter, then warps summed in index order by thread k),
// so results are bitwise deterministic.  fin(k, total) runs on thread k < m
// between the two barriers.  `v` is destroyed.
template <typename S, int M, int NT, class Op, class Fin>
__device__ __forceinline__ void cta_reduce_cols(S (&v)[M], S* red, int m, Fin fin) {
  constexpr int NW = NT / 32;
  constexpr int CF = (M + 31) / 32;
  // lane id re-read per reduction (volatile: not hoisted out of the hot
  // loops, where a loop-invariant copy would only be spilled)
  int lane;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
  const int warp = threadIdx.x >> 5;
  int base = 0, lim = M;
  reduce_scatter<S, M, M, 16, Op>(v, lane, base, lim);
  if constexpr (NW == 1) {
    // one-warp CTA: the owning lane finishes its column; warp barriers order
    // fin's shared-memory writes after every lane's reads of the previous
    // values and publish them
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CF; ++j) {
      const int col = base + j;
      if (col < lim && col < m) fin(col, v[j]);
    }
    __syncwarp();
    return;
  }
#pragma unroll
  for (int j = 0; j < CF; ++j) {
    const int col = base + j;
    if (col < lim && col < m) red[warp * M + col] = v[j];
  }
  __syncthreads();
  if (threadIdx.x < m) {
    const int k = threadIdx.x;
    S acc = red[k];
#pragma unroll
    for (int w = 1; w < NW; ++w) acc = Op{}(acc, red[w * M + k]);
    fin(k, acc);
  }
  __syncthreads();
}

// The same column reduction over the first NTA threads of the CTA only
// (named barrier 1): the forward of the wide-row tiles runs on half the warps.
template <int NTA>
__device__ __forceinline__ void bar_part() {
  asm volatile("bar.sync 1, %0;" ::"n"(NTA) : "memory");
}
template <typename S, int M, int NTA, class Op, class Fin>
__device__ __forceinline__ void cta_reduce_cols_part(S (&v)[M], S* red, int m, Fin fin) {
  constexpr int NW = NTA / 32;
  constexpr int CF = (M + 31) / 32;
  int lane;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
  const int warp = threadIdx.x >> 5;
  int base = 0, lim = M;
  reduce_scatter<S, M, M, 16, Op>(v, lane, base, lim);
#pragma unroll
  for (int j = 0; j < CF; ++j) {
    const int col = base + j;
    if (col < lim && col < m) red[warp * M + col] = v[j];
  }
  bar_part<NTA>();
  if (threadIdx.x < m) {
    const int k = threadIdx.x;
    S acc = red[k];
#pragma unroll
    for (int w = 1; w < NW; ++w) acc = Op{}(acc, red[w * M + k]);
    fin(k, acc);
  }
  bar_part<NTA>();
}

// Same reduction with the finished vector delivered to EVERY thread in
// registers (M <= 32): after the warp reduce-scatter and one barrier, every
// warp sums the per-warp partials in warp order itself (lane k: column k) and
// applies fval(k, total), and the values are spread over the warp by shuffles.
// One barrier instead of two and no shared-memory round trip of the result;
// the same summation order, so bitwise identical to cta_reduce_cols.  `red`
// must be double-buffered by the caller across consecutive calls ([2][NW][M]:
// a warp may store the next call's partials while a slower one still reads).
#ifndef NSW_BCAST
#define NSW_BCAST 0   // measured slower on configs 1-3 (profiles/r02/ab_bcast_reduce.txt)
#endif
template <typename S, int M, int NT, class FVal>
__device__ __forceinline__ void cta_reduce_cols_bcast(S (&v)[M], S* red, int m, FVal fval, S (&out)[M]) {
  static_assert(M <= 32, "one column per lane");
  constexpr int NW = NT / 32;
  int lane;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
  const int warp = threadIdx.x >> 5;
  int base = 0, lim = M;
  reduce_scatter<S, M, M, 16, OpSum>(v, lane, base, lim);
  if (base < lim && base < m) red[warp * M + base] = v[0];
  if constexpr (NW == 1) {
    __syncwarp();
  } else {
    __syncthreads();
  }
  S val = S(0);
  if (lane < m) {
    S acc = red[lane];
#pragma unroll
    for (int w = 1; w < NW; ++w) acc = acc + red[w * M + lane];
    val = fval(lane, acc);
  }
#pragma unroll
  for (int k = 0; k < M; ++k) out[k] = __shfl_sync(0xffffffffu, val, k);
}

// Load an M-vector from shared memory (16-byte vector loads; pitch padded).
template <typename S, int M>
__device__ __forceinline__ void lds_vec(S (&dst)[M], const S* src) {
  constexpr int V = Fp<S>::kVec;
  nsw_check_smem(src, unsigned((M + V - 1) / V * 16));
  if constexpr (V == 4) {
#pragma unroll
    for (int q = 0; q < (M + 3) / 4; ++q) {
      const float4 t = reinterpret_cast<const float4*>(src)[q];
      if (4 * q + 0 < M) dst[(4 * q + 0 < M) ? 4 * q + 0 : 0] = t.x;
      if (4 * q + 1 < M) dst[(4 * q + 1 < M) ? 4 * q + 1 : 0] = t.y;
      if (4 * q + 2 < M) dst[(4 * q + 2 < M) ? 4 * q + 2 : 0] = t.z;
      if (4 * q + 3 < M) dst[(4 * q + 3 < M) ? 4 * q + 3 : 0] = t.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < (M + 1) / 2; ++q) {
      const double2 t = reinterpret_cast<const double2*>(src)[q];
      if (2 * q + 0 < M) dst[(2 * q + 0 < M) ? 2 * q + 0 : 0] = t.x;
      if (2 * q + 1 < M) dst[(2 * q + 1 < M) ? 2 * q + 1 : 0] = t.y;
    }
  }
}

// Same, through volatile shared loads: re-read at every use instead of being
// kept live in registers (for register-lean loops that fetch a broadcast
// vector once per row).
template <typename S, int M>
__device__ __forceinline__ void lds_vec_nc(S (&dst)[M], const S* src) {
  nsw_check_smem(src, unsigned((M * sizeof(S) + 15) / 16 * 16));
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(src));
  if constexpr (sizeof(S) == 4) {
#pragma unroll
    for (int q = 0; q < (M + 3) / 4; ++q) {
      float x, y, z, w;
      asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(x), "=f"(y), "=f"(z), "=f"(w)
                   : "r"(a + 16 * q));
      if (4 * q + 0 < M) dst[(4 * q + 0 < M) ? 4 * q + 0 : 0] = x;
      if (4 * q + 1 < M) dst[(4 * q + 1 < M) ? 4 * q + 1 : 0] = y;
      if (4 * q + 2 < M) dst[(4 * q + 2 < M) ? 4 * q + 2 : 0] = z;
      if (4 * q + 3 < M) dst[(4 * q + 3 < M) ? 4 * q + 3 : 0] = w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < (M + 1) / 2; ++q) {
      double x, y;
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a + 16 * q));
      if (2 * q + 0 < M) dst[(2 * q + 0 < M) ? 2 * q + 0 : 0] = x;
      if (2 * q + 1 < M) dst[(2 * q + 1 < M) ? 2 * q + 1 : 0] = y;
    }
  }
}

template <typename S, int M>
__device__ __forceinline__ void sts_vec(S* dst, const S (&src)[M]) {
  constexpr int V = Fp<S>::kVec;
  constexpr int P = Pitch<S, M>::value;
  nsw_check_smem(dst, unsigned(P * sizeof(S)));
  if constexpr (V == 4) {
#pragma unroll
    for (int q = 0; q < P / 4; ++q) {
      float4 t;
      t.x = (4 * q + 0 < M) ? src[(4 * q + 0 < M) ? 4 * q + 0 : 0] : 0.f;
      t.y = (4 * q + 1 < M) ? src[(4 * q + 1 < M) ? 4 * q + 1 : 0] : 0.f;
      t.z = (4 * q + 2 < M) ? src[(4 * q + 2 < M) ? 4 * q + 2 : 0] : 0.f;
      t.w = (4 * q + 3 < M) ? src[(4 * q + 3 < M) ? 4 * q + 3 : 0] : 0.f;
      reinterpret_cast<float4*>(dst)[q] = t;
    }
  } else {
#pragma unroll
    for (int q = 0; q < P / 2; ++q) {
      double2 t;
      t.x = (2 * q + 0 < M) ? src[(2 * q + 0 < M) ? 2 * q + 0 : 0] : 0.0;
      t.y = (2 * q + 1 < M) ? src[(2 * q + 1 < M) ? 2 * q + 1 : 0] : 0.0;
      reinterpret_cast<double2*>(dst)[q] = t;
    }
  }
}

// Host: SM count of the current device (grid sizing of the streaming
// kernels: a few CTAs per SM), cached per host thread.
inline int sm_count() {
  thread_local int dev = -1, sms = 148;
  int d = 0;
  if (cudaGetDevice(&d) == cudaSuccess && d != dev) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) sms = 148;
    dev = d;
  }
  return sms;
}

// Asynchronous global -> shared copy of one scalar (cp.async, Ampere-style);
// valid == false zero-fills the destination without reading the source.
template <typename S>
__device__ __forceinline__ void cp_async_zfill(S* smem_dst, const S* gsrc, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(gsrc), "n"(int(sizeof(S))),
               "r"(valid ? int(sizeof(S)) : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

}  // namespace nsw
