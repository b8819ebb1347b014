// C ABI of libnswrank_b200.so (declared in include/nswrank_b200.h).
//
// Host runtime of the drop-in: owns the device state of one user shard,
// chooses the fused-step tile variant, issues the per-step kernel sequence
// (fused step -> impact reduction -> [caller's exchange] -> finalize),
// captures it in a CUDA graph, and copies results back in the reference's
// layouts.  Mirrors solve_fair_ranking (reference solver.py:138-241).
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nswrank_b200.h"
#include "nsw_generic.h"
#ifndef NSW_REABS_EVERY
#define NSW_REABS_EVERY 8
#endif
#include "nsw_pool.h"
#include "nsw_registry.h"
#include "nsw_step_kernel.cuh"

namespace nsw {
std::vector<Variant>& variant_registry() {
  static std::vector<Variant> v;
  return v;
}
}  // namespace nsw

using namespace nsw;

namespace {

// NVTX ranges (header-only nvtx3: a no-op unless a profiler is attached) mark
// the phases of the C ABI on the timeline: setup, stepping, result download.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

thread_local std::string g_err;

nsw_status fail(nsw_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return fail(NSW_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
  } while (0)

constexpr size_t kMaxSmem = 227 * 1024;

nsw_status pool_malloc(void** p, size_t bytes, cudaStream_t st);   // private device pool (below)
void pool_free(void* p, cudaStream_t st);

// Every entry point that touches a solver runs on the solver's device and
// gives the caller its current device back on return (a sharded caller's
// rank r keeps its own device current).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

int sizeof_dtype(int dt) { return dt == NSW_F64 ? 8 : 4; }

// Pick the tile variant for (dtype, n, m, T): smallest M >= m, then the
// smallest row capacity R*NT >= n (least padding), ties -> more rows per
// thread (amortises the per-iteration column reduction).
const Variant* choose_variant(int dtype, int n, int m, int T, int forced) {
  auto& reg = variant_registry();
  std::vector<const Variant*> c;
  if (forced == -2 && dtype == NSW_F32) {
    // tensor-core adjoint tiles (registered under dtype 2), smallest fitting
    const Variant* best = nullptr;
    for (auto& v : reg)
      if (v.dtype == 2 && v.M >= m && v.rows >= n && v.smem(T) <= kMaxSmem)
        if (!best || v.M < best->M || (v.M == best->M && v.rows < best->rows)) best = &v;
    if (best) return best;
    forced = -1;
  }
  // one-CTA-per-user tiles first; cluster tiles (CL > 1 CTAs per user) only
  // when no single-CTA tile holds the user's n x m tile
  for (int pass = 0; pass < 2 && c.empty(); ++pass)
    for (auto& v : reg)
      if (v.dtype == dtype && v.M >= m && v.CL * v.rows >= n && v.smem(T) <= kMaxSmem && (v.CL > 1) == (pass == 1))
        c.push_back(&v);
  if (c.empty()) return nullptr;
  std::sort(c.begin(), c.end(), [](const Variant* a, const Variant* b) {
    if (a->M != b->M) return a->M < b->M;
    if (a->CL != b->CL) return a->CL < b->CL;
    if (a->rows != b->rows) return a->rows < b->rows;
    // one-warp tiles (NT = 32: 7 single-wave CTAs per SM, but less latency
    // hiding and slower once-per-step phases) only by explicit choice
    if ((a->NT >= 64) != (b->NT >= 64)) return a->NT >= 64;
    if (a->R != b->R) return a->R > b->R;
    return a->minb < b->minb;
  });
  if (forced >= 0) {
    // forced index counts over the candidates with the chosen M
    std::vector<const Variant*> same;
    for (auto* v : c)
      if (v->M == c[0]->M) same.push_back(v);
    if (forced < int(same.size())) return same[forced];
  }
  return c[0];
}

// Latency-oriented tile for a launch with at most one user per SM: same M,
// about two rows per thread (short serial chains, cheap cross-warp sums),
// then the fewest threads that cover n.
const Variant* choose_wide_variant(const Variant* base, int n, int T) {
  const Variant* best = nullptr;
  auto score = [](const Variant* v) { return std::abs(v->R - 2) * 4096 + v->NT; };
  for (auto& v : variant_registry())
    if (v.dtype == (base->dtype == 2 ? 0 : base->dtype) && v.M == base->M && v.CL == 1 && v.rows >= n &&
        v.smem(T) <= kMaxSmem)
      if (!best || score(&v) < score(best)) best = &v;
  return best;
}

}  // namespace

struct nsw_solver {
  int dtype = 0;
  int device = 0;                 // CUDA device the solver's memory and stream live on
  int U = 0, n = 0, m = 0, T = 0, outer_max = 0, world = 1;
  nsw_solver_config cfg{};
  nsw_device_options opt{};
  const Variant* var = nullptr;   // tile of the main launch (users [0, U1)); nullptr: streaming path
  bool generic = false;           // streaming fused step (no on-chip tile holds the user)
  int gen_ctas = 0;               // its CTAs (persistent over users)
  void* gen_scratch = nullptr;    // [gen_ctas][gen_scratch_elems] K~ / adjoint / row + column vectors
  int reabs_max = 0;              // in-solve re-absorption events per user (0: off)
  int* ev_count = nullptr;        // [U]
  int* ev_t = nullptr;            // [U][reabs_max]
  void* ev_ab = nullptr;          // [U][reabs_max][n + m]
  size_t smem = 0;
  const Variant* var2 = nullptr;  // wide, latency-oriented tile of the tail launch
  size_t smem2 = 0;
  cudaStream_t ext = nullptr;     // last caller-provided stream that carried this solver's work (sharded drivers)
  int U1 = 0;                     // users in the main launch (U1 == U: no tail launch)
  int imp_chunks = 1;             // user chunks of the impact reduction
  // device state
  void *C = nullptr, *am = nullptr, *av = nullptr, *alpha = nullptr, *beta = nullptr, *hist = nullptr,
       *xbest = nullptr, *rel = nullptr, *expo = nullptr;
  double *expo_d = nullptr, *partial = nullptr, *split = nullptr, *imp_local = nullptr,
         *imp_all = nullptr, *imp_cur = nullptr, *rel_sq = nullptr, *best = nullptr,
         *objective = nullptr, *grad_norm = nullptr, *bc = nullptr;
  unsigned long long* stamp = nullptr;
  unsigned int* counter = nullptr;
  int* state = nullptr;
  double* res = nullptr;   // tolerance mode: [U][T+1] residuals
  int* iters = nullptr;    // [outer_max] inner iterations per step
  int tol = 0;             // tolerance-mode schedule
  int* state_host = nullptr;  // pinned
  bool own_exchange = true;
  double* own_imp_local = nullptr;   // [n + 1]
  double* own_imp_all = nullptr;     // [world][n + 1]
  double* own_tol = nullptr;         // [chunk] per-iteration residual maxima (tolerance mode)
  double* tolbuf = nullptr;          // bound exchange buffer for them (all-reduce MAX in place)
  int U_total = 0;                   // users over all ranks
  std::vector<double> expo_host;     // exposures [m-1] (metrics)
  cudaStream_t stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraphExec_t tol_gexec = nullptr;   // tolerance schedule, single shard: one graph per outer step
  cudaStream_t body_stream = nullptr;    // capture stream of its while-loop body
  bool graph_dirty = true;
  int64_t launches = 0;
  StepArgs<float> a32{}, b32{};   // main / tail launch arguments
  StepArgs<double> a64{}, b64{};
  FinalizeArgs fin{};
  float* flush_buf = nullptr;
  size_t flush_n = 0;
  cudaStream_t side = nullptr;              // tail launch stream (concurrent with the main wave)
  cudaEvent_t fork = nullptr, join = nullptr;
  unsigned long long* phase_ns = nullptr;  // [U][16] phase stamps (NSW_PHASE_TIMING diagnostics)
};

namespace {

template <typename S>
void fill_step_args(nsw_solver* s, StepArgs<S>& a) {
  a.U = s->U;
  a.n = s->n;
  a.m = s->m;
  a.T = s->T;
  a.outer_max = s->outer_max;
  a.warm_start = s->cfg.warm_start;
  a.C = (S*)s->C;
  a.am = (S*)s->am;
  a.av = (S*)s->av;
  a.alpha = (S*)s->alpha;
  a.beta = (S*)s->beta;
  a.hist = (S*)s->hist;
  a.xbest = (S*)s->xbest;
  a.rel = (const S*)s->rel;
  a.expo = (const S*)s->expo;
  a.expo_d = s->expo_d;
  a.partial = s->partial;
  a.imp = s->imp_cur;
  a.state = s->state;
  a.bc = s->bc;
  a.tol_mode = s->tol;
  a.chunk = s->opt.tol_chunk > 0 ? s->opt.tol_chunk : 16;
  a.res = s->res;
  const double eps = s->cfg.epsilon;
  a.nie = S(-1.0 / eps);
  a.lr = S(s->cfg.adam_lr);
  a.b1 = S(s->cfg.adam_beta1);
  a.b2 = S(s->cfg.adam_beta2);
  a.omb1 = S(1.0 - s->cfg.adam_beta1);
  a.omb2 = S(1.0 - s->cfg.adam_beta2);
  a.aeps = S(s->cfg.adam_eps);
  const int n = s->n, m = s->m;
  a.c_real = S(-eps * std::log(1.0 / n));
  a.c_dummy = S(-eps * std::log(double(n - m + 1) / n));
  a.mass_dummy = S(n - m + 1);
  a.log_mass_dummy = S(std::log(double(n - m + 1)));
  a.inv_mass_dummy = S(1.0 / double(n - m + 1));
  a.phase_ns = s->phase_ns;
  a.reabs_thr = s->reabs_max > 0 ? s->opt.reabsorb : 0.0;
  a.reabs_max = s->reabs_max;
  a.ev_count = s->ev_count;
  a.ev_t = s->ev_t;
  a.ev_ab = (S*)s->ev_ab;
}

template <typename S>
nsw_status upload_converted(void* dst, const double* src, size_t count) {
  if constexpr (sizeof(S) == 8) {
    CUDA_TRY(cudaMemcpy(dst, src, count * 8, cudaMemcpyHostToDevice));
  } else {
    std::vector<float> tmp(count);
    for (size_t i = 0; i < count; ++i) tmp[i] = float(src[i]);
    CUDA_TRY(cudaMemcpy(dst, tmp.data(), count * 4, cudaMemcpyHostToDevice));
  }
  return NSW_OK;
}

nsw_status download_converted(int dtype, const void* src, double* dst, size_t count, cudaStream_t st,
                              bool* nonfinite = nullptr) {
  if (dtype == NSW_F64) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, count * 8, cudaMemcpyDeviceToHost, st));
  } else {
    // widen on the device, then one copy straight into the caller's buffer
    double* wide = nullptr;
    if (nsw_status pe = pool_malloc((void**)&wide, count * 8 + 16, st); pe != NSW_OK) return pe;
    unsigned* bad = reinterpret_cast<unsigned*>(wide + count);   // one word past the values
    CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned), st));
    widen_kernel<<<sm_count() * 4, 256, 0, st>>>(static_cast<const float*>(src), wide, count, bad);
    cudaError_t ce = cudaGetLastError();
    unsigned bad_h = 0;
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(dst, wide, count * 8, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&bad_h, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    pool_free(wide, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return fail(NSW_ERR_CUDA, std::string("download: ") + cudaGetErrorString(ce));
    if (nonfinite) *nonfinite = bad_h != 0;
    return NSW_OK;
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return NSW_OK;
}

nsw_status validate_config(const nsw_solver_config* c) {
  if (!c) return fail(NSW_ERR_ARG, "config is NULL");
  if (!(c->epsilon > 0)) return fail(NSW_ERR_DOMAIN, "epsilon must be > 0");
  if (!(c->sinkhorn_tol > 0)) return fail(NSW_ERR_DOMAIN, "sinkhorn_tol must be > 0");
  if (!(c->grad_threshold > 0)) return fail(NSW_ERR_DOMAIN, "grad_threshold must be > 0");
  if (c->sinkhorn_max_iters <= 0 || c->outer_max_iters <= 0)
    return fail(NSW_ERR_DOMAIN, "iteration budgets must be positive");
  return NSW_OK;
}

// Work of a solver runs on its own stream (+ the side stream of the tail
// launch) or on a stream the caller passed to the step-level entry points.
// Waiting for it never uses cudaDeviceSynchronize: a device-wide wait from one
// host thread invalidates a CUDA-graph capture another thread has open (every
// solver captures its step), so concurrent solvers in one process would break.
cudaStream_t pick_stream(nsw_solver* s, void* stream) {
  if (!stream) return s->stream;
  s->ext = (cudaStream_t)stream;
  return s->ext;
}
cudaError_t sync_solver(nsw_solver* s) {
  cudaError_t ce = cudaStreamSynchronize(s->stream);
  if (ce == cudaSuccess && s->side) ce = cudaStreamSynchronize(s->side);
  if (ce == cudaSuccess && s->ext && s->ext != s->stream) ce = cudaStreamSynchronize(s->ext);
  return ce;
}

// The fused step over all users: the main launch covers users [0, U1) with
// the occupancy-oriented tile; a tail of at most one user per SM (what is
// left after whole waves) runs as a second launch with the wide tile, which
// finishes a lone user several times faster.
// allow_side = false keeps the tail launch on `st` itself: the body of the
// tolerance schedule's while-node is its own capture, and the side stream
// already belongs to the enclosing one (a stream cannot join two captures).
nsw_status launch_fused(nsw_solver* s, cudaStream_t st, bool allow_side = true) {
  void* args32[] = {&s->a32};
  void* args64[] = {&s->a64};
  if (s->generic) {
    const cudaError_t ce = s->dtype == NSW_F64
                               ? gen_launch(s->a64, static_cast<double*>(s->gen_scratch), s->gen_ctas, st)
                               : gen_launch(s->a32, static_cast<float*>(s->gen_scratch), s->gen_ctas, st);
    if (ce != cudaSuccess) return fail(NSW_ERR_CUDA, std::string("streaming step launch: ") + cudaGetErrorString(ce));
    s->launches += 1;
    return NSW_OK;
  }
  if (s->var->CL > 1) {
    // thread-block cluster of CL CTAs per user (DSMEM column reductions)
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(s->var->CL);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.gridDim = dim3(unsigned(s->U) * s->var->CL);
    lc.blockDim = dim3(s->var->NT);
    lc.dynamicSmemBytes = s->smem;
    lc.stream = st;
    lc.attrs = at;
    lc.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelExC(&lc, s->var->fn, s->dtype == NSW_F64 ? args64 : args32));
    s->launches += 1;
    return NSW_OK;
  }
  // The tail users are independent of the main launch's users within a step:
  // the tail goes on a side stream forked after the main launch, so its CTAs
  // start on SMs as soon as the main wave frees them (joined before the
  // impact reduction).
  const bool both = s->U1 > 0 && s->U1 < s->U;
  const bool side = both && s->side != nullptr && allow_side;
  if (side) {
    CUDA_TRY(cudaEventRecord(s->fork, st));
    CUDA_TRY(cudaStreamWaitEvent(s->side, s->fork, 0));
  }
  if (s->U1 > 0)
    CUDA_TRY(cudaLaunchKernel(s->var->fn, dim3(s->U1), dim3(s->var->NT), s->dtype == NSW_F64 ? args64 : args32,
                              s->smem, st));
  if (s->U1 < s->U) {
    void* brgs32[] = {&s->b32};
    void* brgs64[] = {&s->b64};
    CUDA_TRY(cudaLaunchKernel(s->var2->fn, dim3(s->U - s->U1), dim3(s->var2->NT),
                              s->dtype == NSW_F64 ? brgs64 : brgs32, s->smem2, side ? s->side : st));
    s->launches += 1;
  }
  if (side) {
    CUDA_TRY(cudaEventRecord(s->join, s->side));
    CUDA_TRY(cudaStreamWaitEvent(st, s->join, 0));
  }
  s->launches += 1;
  return NSW_OK;
}

// Single shard with its own exchange buffers: the finalize runs in the
// impact reduction's last CTA (one launch and one dependency less per step).
bool fuse_finalize(const nsw_solver* s) { return s->world == 1 && s->imp_all == s->imp_local; }

nsw_status launch_impact_reduce(nsw_solver* s, cudaStream_t st, bool fuse = false) {
  const dim3 grid((s->n + IMP_ITEMS - 1) / IMP_ITEMS, s->imp_chunks);
  impact_reduce_kernel<<<grid, IMP_THREADS, 0, st>>>(s->partial, s->U, s->n, s->imp_chunks, s->split, s->counter,
                                                     s->imp_local, s->state, s->tol, s->res, s->T,
                                                     s->cfg.sinkhorn_tol, fuse ? 1 : 0, s->fin);
  CUDA_TRY(cudaGetLastError());
  s->launches += 1;
  return NSW_OK;
}

nsw_status launch_step(nsw_solver* s, cudaStream_t st, bool fuse = false) {
  nsw_status e = launch_fused(s, st);
  if (e != NSW_OK) return e;
  return launch_impact_reduce(s, st, fuse);
}

nsw_status launch_finalize(nsw_solver* s, cudaStream_t st) {
  finalize_kernel<<<1, 512, 0, st>>>(s->fin);
  CUDA_TRY(cudaGetLastError());
  s->launches += 1;
  return NSW_OK;
}

nsw_status refresh_args(nsw_solver* s) {
  fill_step_args(s, s->a32);
  fill_step_args(s, s->a64);
  s->b32 = s->a32;
  s->b64 = s->a64;
  s->b32.user0 = s->b64.user0 = s->U1;
  s->fin.n = s->n;
  s->fin.world = s->world;
  s->fin.outer_max = s->outer_max;
  s->fin.imp_all = s->imp_all;
  s->fin.rel_sq = s->rel_sq;
  s->fin.grad_threshold = s->cfg.grad_threshold;
  s->fin.imp_cur = s->imp_cur;
  s->fin.best = s->best;
  s->fin.objective = s->objective;
  s->fin.grad_norm = s->grad_norm;
  s->fin.stamp = s->stamp;
  s->fin.state = s->state;
  s->fin.tol_mode = s->tol;
  s->fin.U = s->U;
  s->fin.U_total = s->U_total;
  s->fin.T = s->T;
  s->fin.tol = s->cfg.sinkhorn_tol;
  s->fin.res = s->res;
  s->fin.iters = s->iters;
  s->graph_dirty = true;
  return NSW_OK;
}

nsw_status read_state(nsw_solver* s) {
  CUDA_TRY(cudaMemcpyAsync(s->state_host, s->state, ST_WORDS * sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return NSW_OK;
}

// Device memory of the solvers comes from the library's private pool
// (nsw_pool.h).
cudaMemPool_t solver_pool(int device) { return private_pool(device); }

#if NSW_CHECKS
// checked builds: 64 KB canary bands on both sides of every solver buffer,
// verified when the buffer is freed (an out-of-bounds write aborts loudly)
constexpr size_t kGuard = size_t(64) << 10;
std::mutex g_guard_mu;
std::map<void*, std::pair<void*, size_t>> g_guarded;   // user pointer -> (base, bytes)
#endif

nsw_status pool_malloc(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  cudaMemPool_t pool = solver_pool(dev);
  if (!pool) return fail(NSW_ERR_CUDA, "cudaMemPoolCreate failed");
  bytes = std::max<size_t>(bytes, 16);
#if NSW_CHECKS
  void* base = nullptr;
  CUDA_TRY(cudaMallocFromPoolAsync(&base, bytes + 2 * kGuard, pool, st));
  CUDA_TRY(cudaMemsetAsync(base, 0xA5, kGuard, st));
  CUDA_TRY(cudaMemsetAsync(static_cast<char*>(base) + kGuard + bytes, 0xA5, kGuard, st));
  *p = static_cast<char*>(base) + kGuard;
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guarded[*p] = {base, bytes};
#else
  CUDA_TRY(cudaMallocFromPoolAsync(p, bytes, pool, st));
#endif
  return NSW_OK;
}

void pool_free(void* p, cudaStream_t st) {
  if (!p) return;
#if NSW_CHECKS
  std::pair<void*, size_t> e{nullptr, 0};
  {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    auto it = g_guarded.find(p);
    if (it != g_guarded.end()) {
      e = it->second;
      g_guarded.erase(it);
    }
  }
  if (!e.first) {
    cudaFreeAsync(p, st);
    return;
  }
  std::vector<unsigned char> lo(kGuard), hi(kGuard);
  cudaError_t ce = cudaStreamSynchronize(st);
  if (ce == cudaSuccess) ce = cudaMemcpy(lo.data(), e.first, kGuard, cudaMemcpyDeviceToHost);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(hi.data(), static_cast<char*>(e.first) + kGuard + e.second, kGuard, cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) {   // a dead context (e.g. a trapped kernel) cannot be checked
    std::fprintf(stderr, "NSW_CHECKS: guard bands not verifiable: %s\n", cudaGetErrorString(ce));
    return;
  }
  size_t bad_lo = 0, bad_hi = 0, first_lo = kGuard, last_lo = 0, first_hi = kGuard, last_hi = 0;
  for (size_t i = 0; i < kGuard; ++i) {
    if (lo[i] != 0xA5) {
      ++bad_lo;
      first_lo = std::min(first_lo, i);
      last_lo = i;
    }
    if (hi[i] != 0xA5) {
      ++bad_hi;
      first_hi = std::min(first_hi, i);
      last_hi = i;
    }
  }
  if (bad_lo || bad_hi) {
    std::fprintf(stderr,
                 "NSW_CHECKS: guard bands of a %zu-byte solver buffer at %p overwritten: low %zu bytes "
                 "[%zu, %zu] (offsets from 64 KB below the buffer), high %zu bytes [%zu, %zu]\n",
                 e.second, p, bad_lo, first_lo, last_lo, bad_hi, first_hi, last_hi);
    std::fflush(stderr);
    std::abort();
  }
  cudaFreeAsync(e.first, st);
#else
  cudaFreeAsync(p, st);
#endif
}

template <typename T>
nsw_status dmalloc(T** p, size_t bytes, cudaStream_t st) {
  nsw_status e = pool_malloc((void**)p, bytes, st);
  if (e != NSW_OK) return e;
  CUDA_TRY(cudaMemsetAsync(*p, 0, std::max<size_t>(bytes, 16), st));
  return NSW_OK;
}

// Pinned state words: a process-wide free list (cudaMallocHost costs
// milliseconds; solvers come and go per solve call).
std::mutex g_pinned_mu;
std::vector<int*> g_pinned_free;

int* pinned_state_get() {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      int* p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  int* p = nullptr;
  return cudaMallocHost((void**)&p, 64) == cudaSuccess ? p : nullptr;
}

void pinned_state_put(int* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(p);
}

// Page-locked host blocks for results (the policy tensor): a small
// process-wide cache keyed by size, so repeated solves neither pay
// cudaHostAlloc nor fault fresh pageable memory.
std::mutex g_host_mu;
std::multimap<size_t, void*> g_host_free;
std::map<void*, size_t> g_host_size;
constexpr size_t kHostCacheBytes = size_t(4) << 30;   // cached (free) page-locked bytes at most
size_t g_host_cached = 0;


}  // namespace

extern "C" {

const char* nsw_last_error(void) { return g_err.c_str(); }
void* nsw_host_alloc(size_t bytes) {
  if (bytes == 0) bytes = 16;
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = g_host_free.find(bytes);
    if (it != g_host_free.end()) {
      void* p = it->second;
      g_host_cached -= it->first;
      g_host_free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_host_mu);
  g_host_size[p] = bytes;
  return p;
}

void nsw_host_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_host_mu);
  auto it = g_host_size.find(p);
  if (it == g_host_size.end()) return;
  if (g_host_cached + it->second <= kHostCacheBytes) {
    g_host_free.emplace(it->second, p);
    g_host_cached += it->second;
    return;
  }
  g_host_size.erase(it);
  cudaFreeHost(p);
}

void nsw_release_cached(void) {
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    for (auto& kv : g_host_free) {
      g_host_size.erase(kv.second);
      cudaFreeHost(kv.second);
    }
    g_host_free.clear();
    g_host_cached = 0;
  }
  PoolTable& t = pool_table();
  std::lock_guard<std::mutex> lk(t.mu);
  for (int d = 0; d < 64; ++d)
    if (t.pool[d]) {
      DeviceGuard guard(d);
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(t.pool[d], 0);
    }
}

const char* nsw_version(void) { return "nswrank_b200 0.1.0 (sm_100a)"; }

int32_t nsw_supported(int32_t dtype, int32_t n, int32_t m, int32_t iters) {
  // every shape the reference accepts (2 <= m <= n, core.py:60-66): an
  // on-chip tile when one holds it, else the streaming fused step
  if ((dtype != NSW_F32 && dtype != NSW_F64) || m < 2 || m > n || iters <= 0) return 0;
  return 1;
}

int32_t nsw_tiled(int32_t dtype, int32_t n, int32_t m, int32_t iters) {
  return choose_variant(dtype, n, m, iters, -1) != nullptr;
}

nsw_status nsw_solver_create(const double* relevance_local, const double* exposure, int32_t users_local,
                             int32_t n, int32_t m, const double* rel_sq_sum, int32_t world,
                             const nsw_solver_config* config, const nsw_device_options* options,
                             nsw_solver** out) {
  if (!out || !relevance_local || !exposure || !options) return fail(NSW_ERR_ARG, "NULL argument");
  NvtxRange nvtx("nsw_solver_create");
  *out = nullptr;
  nsw_status st = validate_config(config);
  if (st != NSW_OK) return st;
  if (users_local <= 0 || n <= 0 || m < 2 || m > n)
    return fail(NSW_ERR_SHAPE, "need users > 0 and 2 <= num_positions <= num_items");
  if (world < 1) return fail(NSW_ERR_ARG, "world must be >= 1");
  // the value checks of the reference's ExposureModel (core.py:113-123), same
  // order and messages: a C caller gets the DomainError the reference would
  // have raised (the relevance is checked on the device after its upload)
  {
    bool finite = true, rising = false;
    double lo = INFINITY, hi = -INFINITY;
    for (int k = 0; k < m - 1; ++k) {
      const double v = exposure[k];
      finite = finite && std::isfinite(v);
      lo = std::min(lo, v);
      hi = std::max(hi, v);
      if (k > 0 && v > exposure[k - 1]) rising = true;
    }
    if (!finite) return fail(NSW_ERR_DOMAIN, "exposure contains non-finite entries");
    if (lo <= 0.0 || hi > 1.0) return fail(NSW_ERR_DOMAIN, "exposure entries must lie in (0, 1]");
    if (rising) return fail(NSW_ERR_DOMAIN, "exposure must be non-increasing in position");
  }
  if (options->dtype != NSW_F32 && options->dtype != NSW_F64) return fail(NSW_ERR_ARG, "bad dtype");
  if (options->schedule != NSW_SCHEDULE_FIXED && options->schedule != NSW_SCHEDULE_TOLERANCE)
    return fail(NSW_ERR_ARG, "bad schedule");
  const int T = config->sinkhorn_max_iters;
  const Variant* var = choose_variant(options->dtype, n, m, T, options->variant);
  if (const char* e = std::getenv("NSW_TC"); e && std::atoi(e) && var && var->dtype == NSW_F32 && var->CL == 1)
    for (auto& v : variant_registry())   // experiments: the same tile with the tensor-core adjoint
      if (v.dtype == 2 && v.M == var->M && v.R == var->R && v.NT == var->NT && v.minb == var->minb &&
          v.smem(T) <= kMaxSmem) {
        var = &v;
        break;
      }
  if (const char* e = std::getenv("NSW_MAIN_TILE"); e && var && var->CL == 1) {   // experiments: "R,NT[,MINB]"
    int r = 0, nt = 0, mb = 0;
    if (std::sscanf(e, "%d,%d,%d", &r, &nt, &mb) >= 2)
      for (auto& v : variant_registry())
        if (v.dtype == var->dtype && v.M == var->M && v.CL == 1 && v.R == r && v.NT == nt && v.rows >= n &&
            (mb == 0 || v.minb == mb))
          var = &v;
  }
  if (const char* e = std::getenv("NSW_CL_TILE"); e && var) {   // experiments: "M,R,NT,CL"
    int mm = 0, r = 0, nt = 0, cl = 0;
    if (std::sscanf(e, "%d,%d,%d,%d", &mm, &r, &nt, &cl) == 4)
      for (auto& v : variant_registry())
        if (v.dtype == var->dtype && v.M == mm && v.M >= m && v.R == r && v.NT == nt && v.CL == cl &&
            v.CL * v.rows >= n)
          var = &v;
  }
  // no on-chip tile holds the user's n x m tile (or forced with variant -3):
  // the streaming fused step, any shape
  const bool reabsorb = options->reabsorb > 0.0;
  if (reabsorb && options->schedule != NSW_SCHEDULE_FIXED)
    return fail(NSW_ERR_UNSUPPORTED, "in-solve re-absorption runs the fixed schedule");
  const bool generic = !var || options->variant == -3 || reabsorb;
  if (generic) var = nullptr;
  // device < 0: the caller's current device
  int dev = options->device;
  if (dev < 0) CUDA_TRY(cudaGetDevice(&dev));
  DeviceGuard guard(dev);
  // Cluster tiles: the GPU's GPC layout decides how many clusters of each size
  // can be resident (B200: 15 clusters of 8 or 9 CTAs, 7 of 16), so among the
  // tiles that hold n items pick the most users in flight per unit of per-user
  // time: resident clusters / (rows per thread x CTAs sharing an SM).
  if (var && var->CL > 1 && options->variant == -1 && !std::getenv("NSW_CL_TILE")) {
    const Variant* best = nullptr;
    double best_score = 0.0;
    for (auto& v : variant_registry()) {
      if (v.dtype != var->dtype || v.M != var->M || v.CL < 2 || v.CL * v.rows < n || v.smem(T) > kMaxSmem) continue;
      if (v.CL > 8 && cudaFuncSetAttribute(v.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        continue;
      if (allow_smem((const void*)v.fn, size_t(v.smem(T))) != cudaSuccess)
        continue;
      cudaLaunchConfig_t lc = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = unsigned(v.CL);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.gridDim = dim3(unsigned(v.CL) * 64u);
      lc.blockDim = dim3(unsigned(v.NT));
      lc.dynamicSmemBytes = v.smem(T);
      lc.attrs = at;
      lc.numAttrs = 1;
      int clusters = 0;
      if (cudaOccupancyMaxActiveClusters(&clusters, v.fn, &lc) != cudaSuccess || clusters <= 0) continue;
      int per_sm = 1;   // CTAs sharing an SM run their rows at a fraction of its issue rate
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v.fn, v.NT, v.smem(T)) != cudaSuccess || per_sm < 1)
        per_sm = 1;
      const double score = double(clusters) / (double(v.R) * per_sm);
      if (!best || score > best_score * 1.0001) {
        best = &v;
        best_score = score;
      }
    }
    cudaGetLastError();   // a rejected candidate must not leave a sticky error behind
    if (best) var = best;
  }
  auto* s = new nsw_solver();
  if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete s;
    return fail(NSW_ERR_CUDA, "cudaStreamCreate failed");
  }
  s->dtype = options->dtype;
  s->device = dev;
  s->U = users_local;
  s->n = n;
  s->m = m;
  s->T = T;
  s->outer_max = config->outer_max_iters;
  s->world = world;
  s->cfg = *config;
  s->opt = *options;
  s->opt.device = dev;
  if (s->opt.check_every <= 0) s->opt.check_every = 8;
  s->var = var;
  s->generic = generic;
  s->smem = generic ? 0 : var->smem(T);
  const size_t es = sizeof_dtype(s->dtype);
  const size_t cells = size_t(users_local) * n * m;
  nsw_status e = NSW_OK;
#define ALLOC(p, bytes)                       \
  do {                                        \
    e = dmalloc(&(p), (bytes), s->stream);    \
    if (e != NSW_OK) {                        \
      nsw_solver_destroy(s);                  \
      return e;                               \
    }                                         \
  } while (0)
  ALLOC(s->C, cells * es);
  ALLOC(s->am, cells * es);
  ALLOC(s->av, cells * es);
  ALLOC(s->xbest, cells * es);
  ALLOC(s->alpha, size_t(users_local) * n * es);
  ALLOC(s->beta, size_t(users_local) * m * es);
  ALLOC(s->hist, size_t(users_local) * (T + 1) * m * es);
  ALLOC(s->rel, size_t(users_local) * n * es);
  ALLOC(s->expo, size_t(m) * es);
  ALLOC(s->expo_d, size_t(m) * 8);
  ALLOC(s->partial, size_t(users_local) * n * 8);
  // impact reduction: ~2 CTAs per SM of (8 items x user chunk)
  s->imp_chunks = std::max(1, std::min(std::min(users_local, 64), (2 * sm_count() * IMP_ITEMS + n - 1) / n));
  if (const char* e = std::getenv("NSW_IMP_CHUNKS"))   // experiments
    s->imp_chunks = std::max(1, std::min(users_local, std::atoi(e)));
  ALLOC(s->split, size_t(s->imp_chunks) * n * 8);
  ALLOC(s->own_imp_local, size_t(n + 1) * 8);
  ALLOC(s->own_imp_all, size_t(world) * (n + 1) * 8);
  ALLOC(s->imp_cur, size_t(n) * 8);
  ALLOC(s->rel_sq, size_t(n) * 8);
  ALLOC(s->best, 8);
  ALLOC(s->objective, size_t(s->outer_max) * 8);
  ALLOC(s->grad_norm, size_t(s->outer_max) * 8);
  ALLOC(s->bc, size_t(2) * (s->outer_max + 1) * 8);
  ALLOC(s->stamp, size_t(s->outer_max + 1) * 8);
  ALLOC(s->counter, 16);
  ALLOC(s->state, ST_WORDS * sizeof(int));
  ALLOC(s->iters, size_t(s->outer_max) * sizeof(int));
  if (generic) {
    // CTAs of the streaming step: occupancy-bound, and their scratch (a K~
    // and an adjoint tile each) within a quarter of the free device memory
    s->gen_ctas = gen_ctas(s->dtype, users_local);
    const size_t per_cta = gen_scratch_elems(n, m) * es;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && per_cta > 0)
      s->gen_ctas = int(std::max<size_t>(1, std::min<size_t>(size_t(s->gen_ctas), free_b / 4 / per_cta)));
    ALLOC(s->gen_scratch, size_t(s->gen_ctas) * per_cta);
  }
  if (reabsorb) {
    s->reabs_max = std::min((T + NSW_REABS_EVERY - 1) / NSW_REABS_EVERY, 64);
    ALLOC(s->ev_count, size_t(users_local) * sizeof(int));
    ALLOC(s->ev_t, size_t(users_local) * s->reabs_max * sizeof(int));
    ALLOC(s->ev_ab, size_t(users_local) * s->reabs_max * (size_t(n) + m) * es);
  }
  if (const char* pt = std::getenv("NSW_PHASE_TIMING"); pt && *pt && *pt != '0') {
    ALLOC(s->phase_ns, size_t(users_local) * 16 * 8);
    CUDA_TRY(cudaMemset(s->phase_ns, 0, size_t(users_local) * 16 * 8));
  }
  s->tol = options->schedule == NSW_SCHEDULE_TOLERANCE;
  if (s->tol) {
    ALLOC(s->res, size_t(users_local) * (T + 1) * 8);
    ALLOC(s->own_tol, size_t(std::max(1, options->tol_chunk > 0 ? options->tol_chunk : 16)) * 8);
  }
  s->tolbuf = s->own_tol;
  s->U_total = users_local;
#undef ALLOC
  // the pool allocations and their zero fills are ordered on the solver's
  // stream; the synchronous uploads below must not overtake them
  if (cudaStreamSynchronize(s->stream) != cudaSuccess) {
    nsw_solver_destroy(s);
    return fail(NSW_ERR_CUDA, "allocation failed");
  }
  s->imp_local = s->own_imp_local;
  s->imp_all = world == 1 ? s->own_imp_local : s->own_imp_all;
  static_assert(ST_WORDS * sizeof(int) <= 64, "pinned state block");
  if ((s->state_host = pinned_state_get()) == nullptr) {
    nsw_solver_destroy(s);
    return fail(NSW_ERR_CUDA, "cudaMallocHost failed");
  }
  if (!generic && var->CL > 8 &&
      cudaFuncSetAttribute(var->fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    nsw_solver_destroy(s);
    return fail(NSW_ERR_UNSUPPORTED, "16-CTA clusters are not available on this device");
  }
  if (!generic && allow_smem((const void*)var->fn, size_t(s->smem)) !=
                      cudaSuccess) {
    nsw_solver_destroy(s);
    return fail(NSW_ERR_CUDA, "cudaFuncSetAttribute(smem) failed");
  }
  // Wave split: whole waves of the main tile, then (if what is left is at
  // most one user per SM) a tail launch with the wide tile.
  s->U1 = users_local;
  if (!generic && options->variant == -1 && var->CL == 1) {
    int sms = 148, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // Fewer users than one wave of the throughput tile (e.g. a strong-scaling
    // shard): the tile with the fewest rows per thread (R >= 2) that still
    // holds every user in one wave has the shortest per-user latency
    // (config 1 at 149..444 users per GPU: R=4/NT=128 is 28 % faster than
    // R=8/NT=64).  At most one user per SM goes to the wide tile below.
    if (!std::getenv("NSW_MAIN_TILE") && users_local > sms) {
      const Variant* low = nullptr;
      for (auto& v : variant_registry()) {
        if (v.dtype != var->dtype || v.M != var->M || v.CL != 1 || v.rows < n || v.R < 2 ||
            v.smem(T) > kMaxSmem || v.R >= var->R)
          continue;
        int ps = 0;
        if (allow_smem((const void*)v.fn, size_t(v.smem(T))) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, v.fn, v.NT, v.smem(T)) != cudaSuccess)
          continue;
        if (ps * sms >= users_local &&
            (!low || v.R < low->R || (v.R == low->R && (v.NT < low->NT || (v.NT == low->NT && v.minb < low->minb)))))
          low = &v;
      }
      if (low) {
        var = low;
        s->var = low;
        s->smem = low->smem(T);
      }
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, var->fn, var->NT, s->smem);
    const Variant* wide = choose_wide_variant(var, n, T);
    if (const char* e = std::getenv("NSW_TAIL_TILE")) {   // experiments: "R,NT[,MINB]" of the tail tile
      int r = 0, nt = 0, mb = 0;
      if (std::sscanf(e, "%d,%d,%d", &r, &nt, &mb) >= 2)
        for (auto& v : variant_registry())
          if (v.dtype == var->dtype && v.M == var->M && v.CL == 1 && v.R == r && v.NT == nt && v.rows >= n &&
              (mb == 0 || v.minb == mb))
            wide = &v;
    }
    const int slots = per_sm * sms;
    if (wide && wide != var && slots > 0) {
      const int rem = users_local % slots;
      if (users_local <= sms) {
        s->U1 = 0;  // at most one user per SM: all users on the wide tile
      } else if (users_local > slots && rem > 0 && rem <= sms) {
        s->U1 = users_local - rem;
      }
    }
    // tests / experiments: force the main/tail split at user k (both tiles
    // run, the tail on the side stream as in production)
    if (const char* e = std::getenv("NSW_SPLIT_USERS"); e && wide && wide != var) {
      const int k = std::atoi(e);
      if (k >= 0 && k < users_local) s->U1 = k;
    }
    if (s->U1 < users_local) {
      s->var2 = wide;
      s->smem2 = wide->smem(T);
      const char* tc = std::getenv("NSW_TAIL_CONCURRENT");
      if (s->U1 > 0 && !(tc && *tc == '0')) {
        if (cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming) != cudaSuccess) {
          nsw_solver_destroy(s);
          return fail(NSW_ERR_CUDA, "side stream creation failed");
        }
      }
      if (allow_smem((const void*)wide->fn, size_t(s->smem2)) !=
          cudaSuccess) {
        nsw_solver_destroy(s);
        return fail(NSW_ERR_CUDA, "cudaFuncSetAttribute(smem, tail) failed");
      }
    }
  }
  // inputs: the float64 relevance goes to the device as is; the fp32 copy
  // and sum_u r^2 (when the caller does not pass it) are formed there
  {
    const size_t cells_r = size_t(users_local) * n;
    double* r64 = nullptr;
    if (s->dtype == NSW_F64) {
      r64 = static_cast<double*>(s->rel);
    } else if ((e = pool_malloc((void**)&r64, cells_r * 8, s->stream)) != NSW_OK ||
               cudaStreamSynchronize(s->stream) != cudaSuccess) {
      nsw_solver_destroy(s);
      return e != NSW_OK ? e : fail(NSW_ERR_CUDA, "relevance staging failed");
    }
    cudaError_t ce = cudaMemcpyAsync(r64, relevance_local, cells_r * 8, cudaMemcpyHostToDevice, s->stream);
    if (ce == cudaSuccess && s->dtype == NSW_F32) {
      narrow_kernel<<<sm_count() * 4, 256, 0, s->stream>>>(r64, static_cast<float*>(s->rel), cells_r);
      ce = cudaGetLastError();
    }
    if (ce == cudaSuccess && !rel_sq_sum) {
      rel_sq_kernel<<<(n + 127) / 128, 128, 0, s->stream>>>(r64, users_local, n, s->rel_sq);
      ce = cudaGetLastError();
    }
    // RelevanceMatrix's value checks (core.py:85-93) on the uploaded float64 copy
    unsigned* flags = nullptr;
    unsigned hflags = 0;
    if (ce == cudaSuccess && pool_malloc((void**)&flags, sizeof(unsigned), s->stream) != NSW_OK) ce = cudaErrorMemoryAllocation;
    if (ce == cudaSuccess) ce = cudaMemsetAsync(flags, 0, sizeof(unsigned), s->stream);
    if (ce == cudaSuccess) {
      rel_check_kernel<<<sm_count() * 4, 256, 0, s->stream>>>(r64, cells_r, flags);
      ce = cudaGetLastError();
    }
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&hflags, flags, sizeof(unsigned), cudaMemcpyDeviceToHost, s->stream);
    if (flags) pool_free(flags, s->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s->stream);
    if (s->dtype == NSW_F32) pool_free(r64, s->stream);
    if (ce == cudaSuccess && hflags != 0) {
      nsw_solver_destroy(s);
      return fail(NSW_ERR_DOMAIN, (hflags & 1u) ? "relevance contains non-finite entries"
                                                : "relevance entries must lie in (0, 1]");
    }
    if (ce != cudaSuccess) {
      nsw_solver_destroy(s);
      return fail(NSW_ERR_CUDA, std::string("relevance upload: ") + cudaGetErrorString(ce));
    }
  }
  s->expo_host.assign(exposure, exposure + (m - 1));
  std::vector<double> ex(m, 0.0);
  double exp_sq = 0.0;
  for (int k = 0; k < m - 1; ++k) {
    ex[k] = exposure[k];
    exp_sq += exposure[k] * exposure[k];
  }
  if ((e = s->dtype == NSW_F64 ? upload_converted<double>(s->expo, ex.data(), m)
                              : upload_converted<float>(s->expo, ex.data(), m)) != NSW_OK) {
    nsw_solver_destroy(s);
    return e;
  }

  // Adam bias corrections exactly as the reference computes them (Python
  // floats: 1.0 - b1**step, solver.py:118-119).
  std::vector<double> bc(size_t(2) * (s->outer_max + 1), 1.0);
  for (int st2 = 1; st2 <= s->outer_max; ++st2) {
    bc[2 * st2] = 1.0 - std::pow(config->adam_beta1, double(st2));
    bc[2 * st2 + 1] = 1.0 - std::pow(config->adam_beta2, double(st2));
  }
  const double neg_inf = -INFINITY;
  int init_state[ST_WORDS] = {PHASE_INIT, 0, 0, 0, 0, 0, 0, 0};
  if (cudaMemcpy(s->expo_d, ex.data(), m * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      (rel_sq_sum && cudaMemcpy(s->rel_sq, rel_sq_sum, n * 8, cudaMemcpyHostToDevice) != cudaSuccess) ||
      cudaMemcpy(s->bc, bc.data(), bc.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(s->best, &neg_inf, 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(s->state, init_state, sizeof(init_state), cudaMemcpyHostToDevice) != cudaSuccess) {
    nsw_solver_destroy(s);
    return fail(NSW_ERR_CUDA, "initial upload failed");
  }
  s->fin.exp_sq = exp_sq;
  refresh_args(s);
  stamp_kernel<<<1, 1, 0, s->stream>>>(s->stamp);
  s->launches += 1;
  if (cudaStreamSynchronize(s->stream) != cudaSuccess) {
    nsw_solver_destroy(s);
    return fail(NSW_ERR_CUDA, "stream sync failed");
  }
  *out = s;
  return NSW_OK;
}

nsw_status nsw_solver_destroy(nsw_solver* s) {
  if (!s) return NSW_OK;
  DeviceGuard guard(s->device);
  if (s->gexec) cudaGraphExecDestroy(s->gexec);
  if (s->tol_gexec) cudaGraphExecDestroy(s->tol_gexec);
  if (s->body_stream) cudaStreamDestroy(s->body_stream);
  void* bufs[] = {s->C, s->am, s->av, s->alpha, s->beta, s->hist, s->xbest, s->rel, s->expo, s->expo_d,
                  s->partial, s->split, s->own_imp_local, s->own_imp_all, s->imp_cur, s->rel_sq, s->best,
                  s->objective, s->grad_norm, s->bc, s->stamp, s->counter, s->state, s->res, s->iters,
                  s->phase_ns, s->own_tol, s->gen_scratch, s->ev_count, s->ev_t, s->ev_ab};
  if (s->stream) {
    for (void* p : bufs)
      if (p) pool_free(p, s->stream);   // back to the pool, stream-ordered
    cudaStreamSynchronize(s->stream);
  }
  if (s->flush_buf) cudaFree(s->flush_buf);
  if (s->fork) cudaEventDestroy(s->fork);
  if (s->join) cudaEventDestroy(s->join);
  if (s->side) cudaStreamDestroy(s->side);
  pinned_state_put(s->state_host);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return NSW_OK;
}

nsw_status nsw_solver_exchange_buffers(nsw_solver* s, void** local_dev, void** gathered_dev) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  DeviceGuard guard(s->device);
  if (local_dev) *local_dev = s->imp_local;
  if (gathered_dev) *gathered_dev = s->imp_all;
  return NSW_OK;
}

nsw_status nsw_solver_bind_exchange(nsw_solver* s, void* local_dev, void* gathered_dev) {
  if (!s || !local_dev || !gathered_dev) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  s->imp_local = (double*)local_dev;
  s->imp_all = (double*)gathered_dev;
  return refresh_args(s);
}

static nsw_status tol_local(nsw_solver* s, cudaStream_t st);
static nsw_status tol_decide(nsw_solver* s, cudaStream_t st, int* phase);

nsw_status nsw_solver_bind_tol_exchange(nsw_solver* s, void* cmax_dev) {
  if (!s || !cmax_dev) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  if (!s->tol) return fail(NSW_ERR_STATE, "solver is not in the tolerance schedule");
  s->tolbuf = (double*)cmax_dev;
  return NSW_OK;
}

nsw_status nsw_solver_tol_local(nsw_solver* s, void* stream) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  DeviceGuard guard(s->device);
  if (!s->tol) return fail(NSW_ERR_STATE, "solver is not in the tolerance schedule");
  return tol_local(s, pick_stream(s, stream));
}

nsw_status nsw_solver_tol_decide(nsw_solver* s, void* stream, int32_t* phase) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  DeviceGuard guard(s->device);
  if (!s->tol) return fail(NSW_ERR_STATE, "solver is not in the tolerance schedule");
  int ph = 0;
  nsw_status e = tol_decide(s, pick_stream(s, stream), &ph);
  if (phase) *phase = ph;
  return e;
}

nsw_status nsw_solver_local_step(nsw_solver* s, void* stream) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  NvtxRange nvtx("nsw_solver_local_step");
  DeviceGuard guard(s->device);
  return launch_step(s, pick_stream(s, stream));
}

nsw_status nsw_solver_finalize(nsw_solver* s, void* stream) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  NvtxRange nvtx("nsw_solver_finalize");
  DeviceGuard guard(s->device);
  return launch_finalize(s, pick_stream(s, stream));
}

static nsw_status ensure_graph(nsw_solver* s) {
  if (!s->graph_dirty && s->gexec) return NSW_OK;
  if (s->gexec) {
    cudaGraphExecDestroy(s->gexec);
    s->gexec = nullptr;
  }
  cudaGraph_t g;
  CUDA_TRY(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
  const int64_t before = s->launches;
  const bool fuse = fuse_finalize(s);
  nsw_status e = launch_step(s, s->stream, fuse);
  if (e == NSW_OK && !fuse) e = launch_finalize(s, s->stream);
  s->launches = before;
  cudaError_t ce = cudaStreamEndCapture(s->stream, &g);
  if (e != NSW_OK) return e;
  if (ce != cudaSuccess) return fail(NSW_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
  ce = cudaGraphInstantiate(&s->gexec, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return fail(NSW_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
  s->graph_dirty = false;
  return NSW_OK;
}

// Tolerance mode: the forward of a step runs in chunks until the lock-step
// test (tol_check_kernel) finds t*; the host reads the device phase after
// each chunk (the number of chunks is data dependent), then the finish
// launch emits X^{t*}'s impact terms.
static nsw_status tol_local(nsw_solver* s, cudaStream_t st) {
  const int chunk = s->opt.tol_chunk > 0 ? s->opt.tol_chunk : 16;
  tol_chunk_max_kernel<<<1, 256, 0, st>>>(s->res, s->U, s->T, chunk, s->state, s->tolbuf);
  CUDA_TRY(cudaGetLastError());
  s->launches += 1;
  return NSW_OK;
}

// Single-shard tolerance schedule as ONE graph per outer step, no host
// round trip per chunk: [fused launch] -> while (cond) { chunk maxima ->
// decide (sets cond = another chunk follows) -> fused launch (next chunk, or
// the finish launch once t* is known) } -> impact reduction + finalize.
static nsw_status ensure_tol_graph(nsw_solver* s) {
  if (s->tol_gexec && !s->graph_dirty) return NSW_OK;
  if (s->tol_gexec) {
    cudaGraphExecDestroy(s->tol_gexec);
    s->tol_gexec = nullptr;
  }
  if (!s->body_stream) CUDA_TRY(cudaStreamCreateWithFlags(&s->body_stream, cudaStreamNonBlocking));
  const int chunk = s->opt.tol_chunk > 0 ? s->opt.tol_chunk : 16;
  const int64_t before = s->launches;
  cudaStream_t st = s->stream;
  CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  nsw_status e = launch_fused(s, st);
  cudaGraph_t capg = nullptr, g = nullptr;
  cudaGraphNode_t cnode = nullptr;
  cudaGraphConditionalHandle h = 0;
  cudaError_t ce = cudaSuccess;
  if (e == NSW_OK) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    ce = cudaStreamGetCaptureInfo(st, &cs, nullptr, &capg, &deps, &ndeps);
    if (ce == cudaSuccess) ce = cudaGraphConditionalHandleCreate(&h, capg, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (ce == cudaSuccess) ce = cudaGraphAddNode(&cnode, capg, deps, ndeps, &cp);
    if (ce == cudaSuccess) ce = cudaStreamUpdateCaptureDependencies(st, &cnode, 1, cudaStreamSetCaptureDependencies);
    if (ce == cudaSuccess) {
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      ce = cudaStreamBeginCaptureToGraph(s->body_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
      if (ce == cudaSuccess) {
        tol_chunk_max_kernel<<<1, 256, 0, s->body_stream>>>(s->res, s->U, s->T, chunk, s->state, s->tolbuf);
        tol_decide_kernel<<<1, 32, 0, s->body_stream>>>(s->tolbuf, s->T, chunk, s->cfg.sinkhorn_tol, s->state,
                                                         static_cast<unsigned long long>(h));
        e = launch_fused(s, s->body_stream, /*allow_side=*/false);
        cudaGraph_t bg = nullptr;
        const cudaError_t ce2 = cudaStreamEndCapture(s->body_stream, &bg);
        if (ce == cudaSuccess) ce = ce2;
      }
    }
  }
  if (e == NSW_OK && ce == cudaSuccess) e = launch_impact_reduce(s, st, true);
  const cudaError_t ce3 = cudaStreamEndCapture(st, &g);
  s->launches = before;
  if (e != NSW_OK) {
    if (g) cudaGraphDestroy(g);
    return e;
  }
  if (ce != cudaSuccess || ce3 != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return fail(NSW_ERR_CUDA, std::string("tolerance graph capture: ") +
                                  cudaGetErrorString(ce != cudaSuccess ? ce : ce3));
  }
  ce = cudaGraphInstantiate(&s->tol_gexec, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return fail(NSW_ERR_CUDA, std::string("tolerance graph instantiate: ") + cudaGetErrorString(ce));
  s->graph_dirty = false;
  return NSW_OK;
}

static nsw_status tol_decide(nsw_solver* s, cudaStream_t st, int* phase) {
  const int chunk = s->opt.tol_chunk > 0 ? s->opt.tol_chunk : 16;
  tol_decide_kernel<<<1, 32, 0, st>>>(s->tolbuf, s->T, chunk, s->cfg.sinkhorn_tol, s->state);
  CUDA_TRY(cudaGetLastError());
  s->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(s->state_host, s->state, ST_WORDS * sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (phase) *phase = s->state_host[ST_PHASE];
  return NSW_OK;
}

static nsw_status one_step_tolerance(nsw_solver* s) {
  if (s->opt.use_graph && fuse_finalize(s)) {
    nsw_status ge = ensure_tol_graph(s);
    if (ge != NSW_OK) return ge;
    CUDA_TRY(cudaGraphLaunch(s->tol_gexec, s->stream));
    s->launches += 4;   // at least: fused, chunk maxima, decide, finish + impact reduction (data-dependent)
    return NSW_OK;
  }
  nsw_status e = launch_fused(s, s->stream);
  if (e != NSW_OK) return e;
  for (;;) {
    int ph = 0;
    if ((e = tol_local(s, s->stream)) != NSW_OK) return e;
    if ((e = tol_decide(s, s->stream, &ph)) != NSW_OK) return e;
    if (ph == PHASE_FWD_CONT) {
      e = launch_fused(s, s->stream);
      if (e != NSW_OK) return e;
      continue;
    }
    if (ph == PHASE_FWD_FIN) {
      const bool fuse = fuse_finalize(s);
      e = launch_step(s, s->stream, fuse);  // finish launch + impact reduction (+ finalize)
      if (e != NSW_OK || fuse) return e;
    }
    return launch_finalize(s, s->stream);
  }
}

static nsw_status one_step(nsw_solver* s) {
  if (s->tol) return one_step_tolerance(s);
  if (s->opt.use_graph) {
    nsw_status e = ensure_graph(s);
    if (e != NSW_OK) return e;
    CUDA_TRY(cudaGraphLaunch(s->gexec, s->stream));
    s->launches += (s->U1 > 0 && s->U1 < s->U ? 2 : 1) + (fuse_finalize(s) ? 1 : 2);
    return NSW_OK;
  }
  const bool fuse = fuse_finalize(s);
  nsw_status e = launch_step(s, s->stream, fuse);
  if (e != NSW_OK || fuse) return e;
  return launch_finalize(s, s->stream);
}

nsw_status nsw_solver_run(nsw_solver* s, int32_t max_steps, int32_t* done) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  NvtxRange nvtx("nsw_solver_run");
  DeviceGuard guard(s->device);
  if (s->world != 1) return fail(NSW_ERR_ARG, "nsw_solver_run drives a single shard (world == 1)");
  if (done) *done = 0;
  for (int it = 0; it < max_steps; ++it) {
    nsw_status e = one_step(s);
    if (e != NSW_OK) return e;
    if ((it + 1) % s->opt.check_every == 0 || it + 1 == max_steps) {
      e = read_state(s);
      if (e != NSW_OK) return e;
      if (s->state_host[ST_PHASE] == PHASE_FINISHED) {
        if (done) *done = 1;
        break;
      }
    }
  }
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return NSW_OK;
}

nsw_status nsw_solver_status(nsw_solver* s, int32_t* phase, int32_t* steps, int32_t* errors) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  DeviceGuard guard(s->device);
  nsw_status e = read_state(s);
  if (e != NSW_OK) return e;
  if (phase) *phase = s->state_host[ST_PHASE];
  if (steps) *steps = s->state_host[ST_STEP];
  if (errors) *errors = s->state_host[ST_ERR];
  return NSW_OK;
}

nsw_status nsw_solver_stream(nsw_solver* s, void** stream) {
  if (!s || !stream) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  *stream = s->stream;
  return NSW_OK;
}

nsw_status nsw_solver_result(nsw_solver* s, double* policy_out, nsw_trace* trace) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  NvtxRange nvtx("nsw_solver_result");
  DeviceGuard guard(s->device);
  CUDA_TRY(sync_solver(s));
  nsw_status e = read_state(s);
  if (e != NSW_OK) return e;
  const int steps = s->state_host[ST_STEP];
  if (policy_out) {
    bool nonfinite = false;
    e = download_converted(s->dtype, s->xbest, policy_out, size_t(s->U) * s->n * s->m, s->stream, &nonfinite);
    if (e != NSW_OK) return e;
    // the reference's RankingPolicy rejects non-finite entries (core.py:131-148);
    // the fp32 path checks them on the device while widening
    if (nonfinite) return fail(NSW_ERR_DOMAIN, "policy contains non-finite entries");
  }
  if (trace) {
    trace->steps = steps;
    std::vector<unsigned long long> st(steps + 1);
    if (steps > 0) {
      if (trace->objective) CUDA_TRY(cudaMemcpy(trace->objective, s->objective, steps * 8, cudaMemcpyDeviceToHost));
      if (trace->grad_norm) CUDA_TRY(cudaMemcpy(trace->grad_norm, s->grad_norm, steps * 8, cudaMemcpyDeviceToHost));
      CUDA_TRY(cudaMemcpy(st.data(), s->stamp, (steps + 1) * 8, cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < steps; ++k) {
      if (trace->wall_time) trace->wall_time[k] = double(st[k + 1] - st[k]) * 1e-9;
    }
  }
  if (trace && trace->sinkhorn_iterations && steps > 0)
    CUDA_TRY(cudaMemcpy(trace->sinkhorn_iterations, s->iters, steps * sizeof(int), cudaMemcpyDeviceToHost));
  const int err = s->state_host[ST_ERR];
  if (err & ERR_SOLVER) {
    const double failed = 1.0 - double(s->state_host[ST_CONV]) / double(s->U_total);
    char msg[160];
    snprintf(msg, sizeof(msg), "Sinkhorn failed to converge for %.0f%% of users within %d iterations", failed * 100.0,
             s->T);
    return fail(NSW_ERR_SOLVER, msg);
  }
  if (err & ERR_IMPACT) {
    if (s->dtype == NSW_F32)
      return fail(NSW_ERR_DOMAIN,
                  "item impact became nonpositive during the solve: the float32 Sinkhorn scalings left the fp32 "
                  "exponent range (small epsilon" + std::string(s->cfg.warm_start ? "" : " with warm_start=False") +
                      "); use DeviceOptions(dtype='float64') or warm_start=True");
    return fail(NSW_ERR_DOMAIN, "item impact became nonpositive during the solve");
  }
  return NSW_OK;
}

static nsw_status field_ptr(nsw_solver* s, const char* f, void** p, size_t* count, bool* typed) {
  const size_t cells = size_t(s->U) * s->n * s->m;
  *typed = true;
  if (!strcmp(f, "cost")) { *p = s->C; *count = cells; }
  else if (!strcmp(f, "adam_m")) { *p = s->am; *count = cells; }
  else if (!strcmp(f, "adam_v")) { *p = s->av; *count = cells; }
  else if (!strcmp(f, "xbest")) { *p = s->xbest; *count = cells; }
  else if (!strcmp(f, "alpha")) { *p = s->alpha; *count = size_t(s->U) * s->n; }
  else if (!strcmp(f, "beta") || !strcmp(f, "lvi")) { *p = s->beta; *count = size_t(s->U) * s->m; }
  else if (!strcmp(f, "hist")) { *p = s->hist; *count = size_t(s->U) * (s->T + 1) * s->m; }
  else if (!strcmp(f, "partial")) { *p = s->partial; *count = size_t(s->U) * s->n; *typed = false; }
  else if (!strcmp(f, "imp")) { *p = s->imp_cur; *count = s->n; *typed = false; }
  else if (!strcmp(f, "imp_local")) { *p = s->imp_local; *count = s->n; *typed = false; }
  else if (!strcmp(f, "objective")) { *p = s->objective; *count = s->outer_max; *typed = false; }
  else if (!strcmp(f, "grad_norm")) { *p = s->grad_norm; *count = s->outer_max; *typed = false; }
  else return fail(NSW_ERR_ARG, std::string("unknown field ") + f);
  return NSW_OK;
}

nsw_status nsw_solver_get(nsw_solver* s, const char* field, double* host, size_t count) {
  if (!s || !field || !host) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  void* p;
  size_t c;
  bool typed;
  nsw_status e = field_ptr(s, field, &p, &c, &typed);
  if (e != NSW_OK) return e;
  if (count != c) return fail(NSW_ERR_SHAPE, std::string("field ") + field + " has " + std::to_string(c) + " elements");
  CUDA_TRY(sync_solver(s));
  if (!typed) {
    CUDA_TRY(cudaMemcpy(host, p, c * 8, cudaMemcpyDeviceToHost));
    return NSW_OK;
  }
  return download_converted(s->dtype, p, host, c, s->stream);
}

nsw_status nsw_solver_set(nsw_solver* s, const char* field, const double* host, size_t count) {
  if (!s || !field || !host) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  void* p;
  size_t c;
  bool typed;
  nsw_status e = field_ptr(s, field, &p, &c, &typed);
  if (e != NSW_OK) return e;
  if (count != c) return fail(NSW_ERR_SHAPE, std::string("field ") + field + " has " + std::to_string(c) + " elements");
  CUDA_TRY(sync_solver(s));
  if (!typed) {
    CUDA_TRY(cudaMemcpy(p, host, c * 8, cudaMemcpyHostToDevice));
    return NSW_OK;
  }
  return s->dtype == NSW_F64 ? upload_converted<double>(p, host, c) : upload_converted<float>(p, host, c);
}

nsw_status nsw_solver_set_scalar(nsw_solver* s, const char* field, int64_t value) {
  if (!s || !field) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  CUDA_TRY(sync_solver(s));
  int idx = -1;
  if (!strcmp(field, "phase")) idx = ST_PHASE;
  else if (!strcmp(field, "step")) idx = ST_STEP;
  else if (!strcmp(field, "improved")) idx = ST_IMPROVED;
  if (idx >= 0) {
    // the step indexes the per-step trace arrays and the Adam bias-correction
    // table on the device: an out-of-range value would write past them
    if (idx == ST_STEP && (value < 0 || value >= s->outer_max))
      return fail(NSW_ERR_DOMAIN, "step must lie in [0, outer_max_iters)");
    if (idx == ST_PHASE && (value < PHASE_INIT || value > PHASE_FWD_FIN))
      return fail(NSW_ERR_DOMAIN, "unknown phase");
    if (idx == ST_IMPROVED && value != 0 && value != 1) return fail(NSW_ERR_DOMAIN, "improved is 0 or 1");
    int v = int(value);
    CUDA_TRY(cudaMemcpy(s->state + idx, &v, 4, cudaMemcpyHostToDevice));
    return NSW_OK;
  }
  if (!strcmp(field, "users_total")) {   // sharded solve: users over all ranks
    if (value < s->U) return fail(NSW_ERR_ARG, "users_total < local users");
    s->U_total = int(value);
    return refresh_args(s);
  }
  if (!strcmp(field, "best_is_neg_inf")) {
    const double neg_inf = -INFINITY;
    CUDA_TRY(cudaMemcpy(s->best, &neg_inf, 8, cudaMemcpyHostToDevice));
    return NSW_OK;
  }
  return fail(NSW_ERR_ARG, std::string("unknown scalar ") + field);
}

int64_t nsw_solver_launch_count(nsw_solver* s) { return s ? s->launches : -1; }

nsw_status nsw_solver_variant(nsw_solver* s, int32_t* M, int32_t* R, int32_t* NT, int32_t* smem) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  // main tile; when a tail launch exists its shape is reported in the upper
  // 16 bits of R and NT (R | R2 << 16, NT | NT2 << 16) and *smem is the main one
  if (s->generic) {   // streaming path: M = 0, R = CTAs of the launch
    if (M) *M = 0;
    if (R) *R = s->gen_ctas;
    if (NT) *NT = GEN_NT;
    if (smem) *smem = 0;
    return NSW_OK;
  }
  if (M) *M = s->var->M;
  if (R) *R = s->var->R | (s->var2 && s->U1 < s->U ? s->var2->R << 16 : 0);
  if (NT) *NT = s->var->NT | (s->var2 && s->U1 < s->U ? s->var2->NT << 16 : 0);
  if (smem) *smem = int(s->smem);
  return NSW_OK;
}

int32_t nsw_solver_tail_users(nsw_solver* s) { return s ? s->U - s->U1 : -1; }

static nsw_status ensure_flush_buffer(nsw_solver* s) {
  if (s->flush_buf) return NSW_OK;
  s->flush_n = size_t(256) << 20;  // 1 GiB of floats > 126 MB L2
  CUDA_TRY(cudaMalloc((void**)&s->flush_buf, s->flush_n * 4));
  CUDA_TRY(cudaMemset(s->flush_buf, 0, s->flush_n * 4));
  return NSW_OK;
}

// Write 1 GiB (evicts everything from the 126 MB L2), then drop those dirty
// lines without writing them back: the next step starts from a cold, clean L2
// instead of paying the flush's own write-backs.
static nsw_status launch_l2_flush(nsw_solver* s, cudaStream_t st) {
  flush_kernel<<<sm_count() * 8, 512, 0, st>>>(s->flush_buf, s->flush_n);
  CUDA_TRY(cudaGetLastError());
  discard_kernel<<<sm_count() * 8, 512, 0, st>>>(s->flush_buf, s->flush_n);
  CUDA_TRY(cudaGetLastError());
  return NSW_OK;
}

nsw_status nsw_solver_flush_l2(nsw_solver* s, void* stream) {
  if (!s) return fail(NSW_ERR_ARG, "NULL solver");
  DeviceGuard guard(s->device);
  nsw_status e = ensure_flush_buffer(s);
  if (e != NSW_OK) return e;
  return launch_l2_flush(s, pick_stream(s, stream));
}

nsw_status nsw_solver_time_steps(nsw_solver* s, int32_t steps, int32_t flush_l2, float* ms_total,
                                 float* ms_fused) {
  if (!s || steps <= 0) return fail(NSW_ERR_ARG, "bad arguments");
  DeviceGuard guard(s->device);
  if (s->world != 1) return fail(NSW_ERR_ARG, "timing helper drives a single shard");
  if (s->tol) return fail(NSW_ERR_ARG, "timing helper runs the fixed schedule");
  if (flush_l2) {
    nsw_status fe = ensure_flush_buffer(s);
    if (fe != NSW_OK) return fe;
  }
  // One step as the solve runs it, as CUDA graphs: [fused launch(es)] and
  // [impact reduction + finalize], with events between them so the fused
  // kernels' share is measured on the same replay.
  std::vector<cudaEvent_t> ev(size_t(3) * steps);
  for (auto& x : ev) CUDA_TRY(cudaEventCreate(&x));
  const bool fuse = fuse_finalize(s);
  const int64_t before = s->launches;
  nsw_status e = NSW_OK;
  auto capture = [&](cudaGraphExec_t* out, bool fused_part) -> nsw_status {
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    nsw_status r = NSW_OK;
    if (fused_part) {
      r = launch_fused(s, s->stream);
    } else {
      r = launch_impact_reduce(s, s->stream, fuse);
      if (r == NSW_OK && !fuse) r = launch_finalize(s, s->stream);
    }
    cudaError_t ce = cudaStreamEndCapture(s->stream, &g);
    if (r == NSW_OK && ce != cudaSuccess) r = fail(NSW_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    if (r == NSW_OK && cudaGraphInstantiate(out, g, 0) != cudaSuccess) r = fail(NSW_ERR_CUDA, "graph instantiate");
    if (g) cudaGraphDestroy(g);
    return r;
  };
  cudaGraphExec_t gx = nullptr, gy = nullptr;
  e = capture(&gx, true);
  if (e == NSW_OK) e = capture(&gy, false);
  const int64_t per_step = s->launches - before;
  s->launches = before;
  // all steps enqueued ahead (the host never waits inside the timed region)
  for (int i = 0; i < steps && e == NSW_OK; ++i) {
    if (flush_l2 && (e = launch_l2_flush(s, s->stream)) != NSW_OK) break;
    if (cudaEventRecord(ev[3 * i], s->stream) != cudaSuccess || cudaGraphLaunch(gx, s->stream) != cudaSuccess ||
        cudaEventRecord(ev[3 * i + 1], s->stream) != cudaSuccess || cudaGraphLaunch(gy, s->stream) != cudaSuccess ||
        cudaEventRecord(ev[3 * i + 2], s->stream) != cudaSuccess) {
      e = fail(NSW_ERR_CUDA, "timed step failed");
      break;
    }
    s->launches += per_step;
  }
  if (e == NSW_OK && cudaStreamSynchronize(s->stream) != cudaSuccess) e = fail(NSW_ERR_CUDA, "timed steps failed");
  float tot = 0.f, fus = 0.f;
  for (int i = 0; i < steps && e == NSW_OK; ++i) {
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 2]);
    cudaEventElapsedTime(&b, ev[3 * i], ev[3 * i + 1]);
    tot += a;
    fus += b;
  }
  if (gy) cudaGraphExecDestroy(gy);
  if (gx) cudaGraphExecDestroy(gx);
  for (auto& x : ev) cudaEventDestroy(x);
  if (e != NSW_OK) return e;
  if (ms_total) *ms_total = tot;
  if (ms_fused) *ms_fused = fus;
  return NSW_OK;
}

// Measurement helper for any shard (world >= 1): device time of the fused
// launch(es) alone -- no impact reduction, exchange or finalize, so the device
// state machine does not advance; the iterate (C, Adam moments) does, without
// a trace entry.  For timing at the end of a measurement only.
nsw_status nsw_solver_time_fused(nsw_solver* s, int32_t steps, int32_t flush_l2, float* ms_fused) {
  if (!s || steps <= 0) return fail(NSW_ERR_ARG, "bad arguments");
  DeviceGuard guard(s->device);
  if (s->tol) return fail(NSW_ERR_ARG, "timing helper runs the fixed schedule");
  if (flush_l2) {
    nsw_status fe = ensure_flush_buffer(s);
    if (fe != NSW_OK) return fe;
  }
  std::vector<cudaEvent_t> ev(size_t(2) * steps);
  for (auto& x : ev) CUDA_TRY(cudaEventCreate(&x));
  const int64_t before = s->launches;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t gx = nullptr;
  nsw_status e = NSW_OK;
  if (cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    e = fail(NSW_ERR_CUDA, "graph capture");
  } else {
    e = launch_fused(s, s->stream);
    cudaError_t ce = cudaStreamEndCapture(s->stream, &g);
    if (e == NSW_OK && ce != cudaSuccess) e = fail(NSW_ERR_CUDA, "graph capture");
    if (e == NSW_OK && cudaGraphInstantiate(&gx, g, 0) != cudaSuccess) e = fail(NSW_ERR_CUDA, "graph instantiate");
    if (g) cudaGraphDestroy(g);
  }
  const int64_t per_step = s->launches - before;
  s->launches = before;
  for (int i = 0; i < steps && e == NSW_OK; ++i) {
    if (flush_l2 && (e = launch_l2_flush(s, s->stream)) != NSW_OK) break;
    if (cudaEventRecord(ev[2 * i], s->stream) != cudaSuccess || cudaGraphLaunch(gx, s->stream) != cudaSuccess ||
        cudaEventRecord(ev[2 * i + 1], s->stream) != cudaSuccess) {
      e = fail(NSW_ERR_CUDA, "timed launch failed");
      break;
    }
    s->launches += per_step;
  }
  if (e == NSW_OK && cudaStreamSynchronize(s->stream) != cudaSuccess) e = fail(NSW_ERR_CUDA, "timed launches failed");
  float tot = 0.f;
  for (int i = 0; i < steps && e == NSW_OK; ++i) {
    float a = 0.f;
    cudaEventElapsedTime(&a, ev[2 * i], ev[2 * i + 1]);
    tot += a;
  }
  if (gx) cudaGraphExecDestroy(gx);
  for (auto& x : ev) cudaEventDestroy(x);
  if (e != NSW_OK) return e;
  if (ms_fused) *ms_fused = tot;
  return NSW_OK;
}

nsw_status nsw_solver_top_positions(nsw_solver* s, int32_t* out_host) {
  if (!s || !out_host) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  int32_t* d = nullptr;
  const size_t count = size_t(s->U) * (s->m - 1);
  CUDA_TRY(cudaMalloc(&d, count * sizeof(int32_t)));
  nsw_status e = s->dtype == NSW_F64
                     ? nsw_top_positions_f64((const double*)s->xbest, s->U, s->n, s->m, d, s->stream)
                     : nsw_top_positions_f32((const float*)s->xbest, s->U, s->n, s->m, d, s->stream);
  if (e == NSW_OK) {
    s->launches += 1;
    if (cudaMemcpyAsync(out_host, d, count * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
        cudaStreamSynchronize(s->stream) != cudaSuccess)
      e = fail(NSW_ERR_CUDA, "top_positions copy failed");
  }
  cudaFree(d);
  return e;
}

nsw_status nsw_solver_metrics(nsw_solver* s, double threshold, double* out_host) {
  if (!s || !out_host) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  const nsw_status e =
      s->dtype == NSW_F64
          ? nsw_policy_metrics_f64((const double*)s->xbest, (const double*)s->rel, s->expo_host.data(), s->U, s->n,
                                   s->m, threshold, out_host, s->stream)
          : nsw_policy_metrics_f32((const float*)s->xbest, (const float*)s->rel, s->expo_host.data(), s->U, s->n,
                                   s->m, threshold, out_host, s->stream);
  if (e != NSW_OK) return fail(e, "policy metrics failed");
  s->launches += 6;   // masses, impact partials + combine, envy GEMM + combine, finish
  return NSW_OK;
}

nsw_status nsw_solver_phase_times(nsw_solver* s, uint64_t* out, int32_t count) {
  if (!s || !out) return fail(NSW_ERR_ARG, "NULL argument");
  DeviceGuard guard(s->device);
  if (!s->phase_ns) return fail(NSW_ERR_UNSUPPORTED, "phase timing is off (set NSW_PHASE_TIMING=1 before creating the solver)");
  const size_t words = size_t(std::min(count, s->U)) * 16;
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  CUDA_TRY(cudaMemcpy(out, s->phase_ns, words * 8, cudaMemcpyDeviceToHost));
  return NSW_OK;
}

nsw_status nsw_solve_fair_ranking(const double* relevance, const double* exposure, int32_t U, int32_t n,
                                  int32_t m, const nsw_solver_config* config,
                                  const nsw_device_options* options, double* policy_out, nsw_trace* trace) {
  if (!relevance || !exposure || !config || !options) return fail(NSW_ERR_ARG, "NULL argument");
  NvtxRange nvtx("nsw_solve_fair_ranking");
  nsw_solver* s = nullptr;
  nsw_status e = nsw_solver_create(relevance, exposure, U, n, m, nullptr, 1, config, options, &s);
  if (e != NSW_OK) return e;
  // at most outer_max forwards + one materialisation step
  int32_t done = 0;
  e = nsw_solver_run(s, config->outer_max_iters + 1, &done);
  if (e == NSW_OK) e = nsw_solver_result(s, policy_out, trace);
  if (e == NSW_OK && !done) e = fail(NSW_ERR_STATE, "solver did not reach its stop state");
  nsw_solver_destroy(s);
  return e;
}

}  // extern "C"
