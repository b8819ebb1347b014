/*
 * nswrank_b200 -- B200-native drop-in for the NSW fair-ranking ascent path.
 *
 * C ABI of libnswrank_b200.so: plain pointers and sizes, no torch types.
 * Every entry point names the reference interface it replaces
 * (/root/reference/pkg/src/nswrank, version 0.1.0).  The reference is pure
 * Python/numpy, so the binding a maintainer would add on the reference side
 * is a ctypes stub; it is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Host pointers are float64 row-major arrays in the reference's layouts:
 *     relevance [U][n], exposure [m-1], policy [U][n][m].
 *   - Device pointers (the *_dev / operator entry points) are stream-ordered;
 *     `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Every function returns an nsw_status; nsw_last_error() gives the text.
 *     The Python host layer maps the codes onto the reference's exception
 *     classes (reference core.py:20-33): SHAPE -> ShapeError,
 *     DOMAIN -> DomainError, SOLVER -> SolverError, STATE -> StateError.
 */
#ifndef NSWRANK_B200_H
#define NSWRANK_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NSW_OK = 0,
  NSW_ERR_SHAPE = 1,        /* ShapeError   (reference core.py:20)          */
  NSW_ERR_DOMAIN = 2,       /* DomainError  (reference core.py:24)          */
  NSW_ERR_STATE = 3,        /* StateError   (reference core.py:28)          */
  NSW_ERR_SOLVER = 4,       /* SolverError  (reference core.py:32)          */
  NSW_ERR_UNSUPPORTED = 5,  /* shape/dtype has no compiled kernel variant   */
  NSW_ERR_CUDA = 6,         /* CUDA runtime failure                         */
  NSW_ERR_ARG = 7           /* bad argument (null pointer, bad enum)        */
} nsw_status;

typedef enum { NSW_F32 = 0, NSW_F64 = 1 } nsw_dtype;

typedef enum {
  NSW_SCHEDULE_FIXED = 0,     /* exactly sinkhorn_max_iters inner iterations per solve */
  NSW_SCHEDULE_TOLERANCE = 1  /* reference default: lock-step stop at residual <= tol  */
} nsw_schedule;

/* Mirrors SolverConfig (reference core.py:171-201) field for field. */
typedef struct {
  double epsilon;
  int32_t sinkhorn_max_iters;
  double sinkhorn_tol;
  int32_t outer_max_iters;
  double grad_threshold;
  double adam_lr;
  double adam_beta1;
  double adam_beta2;
  double adam_eps;
  int32_t warm_start;
} nsw_solver_config;

/* Device-side options (not part of the reference config). */
typedef struct {
  int32_t dtype;          /* nsw_dtype: F32 throughput path, F64 parity path        */
  int32_t schedule;       /* nsw_schedule                                           */
  int32_t device;         /* CUDA device ordinal; -1 = the caller's current device  */
  int32_t variant;        /* -1 = automatic tile choice, else index into the table  */
  int32_t use_graph;      /* capture the outer step in a CUDA graph (1) or not (0)  */
  int32_t check_every;    /* host polls the stop flag every N outer steps           */
  int32_t tol_chunk;      /* tolerance schedule: inner iterations per forward chunk */
  double reabsorb;        /* > 0: in-solve re-absorption -- every 8 inner iterations,
                             once max_k |log v~_k| exceeds this many nats, the
                             scalings are folded into K~ (beta += log v~, alpha
                             re-normalised) and the backward crosses back; runs the
                             streaming fused step, fixed schedule.  0 = off.       */
} nsw_device_options;

/* Returned trace; mirrors SolveTrace (reference solver.py:125-135). */
typedef struct {
  int32_t steps;            /* number of recorded outer iterations               */
  double* objective;        /* caller-allocated [outer_max_iters]                */
  double* grad_norm;        /* caller-allocated [outer_max_iters]                */
  int32_t* sinkhorn_iterations;  /* caller-allocated [outer_max_iters]           */
  double* wall_time;        /* caller-allocated [outer_max_iters], seconds/step  */
} nsw_trace;

const char* nsw_last_error(void);
const char* nsw_version(void);

/* ------------------------------------------------------------------------ *
 * 1. Whole solve, host buffers.                                           *
 *    Replaces solve_fair_ranking (reference solver.py:138-241).  The best  *
 *    iterate's policy (solver.py:217-219, 241) is written to policy_out    *
 *    [U][n][m] float64; the trace to *trace.                               *
 * ------------------------------------------------------------------------ */
nsw_status nsw_solve_fair_ranking(const double* relevance, const double* exposure,
                                  int32_t num_users, int32_t num_items, int32_t num_positions,
                                  const nsw_solver_config* config, const nsw_device_options* options,
                                  double* policy_out, nsw_trace* trace);

/* ------------------------------------------------------------------------ *
 * 2. Step-level solver handle: the same solve split into stream-ordered    *
 *    pieces so a caller can shard users over GPUs and run the per-step     *
 *    impact exchange (reference solver.py:206) itself.                     *
 * ------------------------------------------------------------------------ */
typedef struct nsw_solver nsw_solver;

/* users_local: this rank's contiguous user block; relevance_local [users_local][n]
 * float64 host; rel_sq_sum [n] = sum over ALL users of r_ui^2 (closed-form
 * gradient norm, solver.py:211); world = number of impact partials the
 * finalize step sums (1 for a single GPU). */
nsw_status nsw_solver_create(const double* relevance_local, const double* exposure,
                             int32_t users_local, int32_t num_items, int32_t num_positions,
                             const double* rel_sq_sum, int32_t world,
                             const nsw_solver_config* config, const nsw_device_options* options,
                             nsw_solver** out);
nsw_status nsw_solver_destroy(nsw_solver* s);

/* Device pointers of the impact exchange: local [n + 1] float64 (written by
 * nsw_solver_local_step: the n item impacts, then -- tolerance schedule --
 * this shard's count of converged users), gathered [world][n + 1] float64
 * (read by nsw_solver_finalize).  May be rebound to caller-owned buffers. */
nsw_status nsw_solver_exchange_buffers(nsw_solver* s, void** local_dev, void** gathered_dev);
nsw_status nsw_solver_bind_exchange(nsw_solver* s, void* local_dev, void* gathered_dev);

/* One outer step minus the exchange: [backward of step k-1 + Adam +]
 * forward of step k + local impact reduction.  No-op once finished. */
nsw_status nsw_solver_local_step(nsw_solver* s, void* stream);
/* Objective, gradient norm, best-iterate and stop decisions from the
 * gathered impacts (solver.py:206-223).  No-op once finished. */
nsw_status nsw_solver_finalize(nsw_solver* s, void* stream);
/* Tolerance schedule across shards (sinkhorn.py:237-246 over all users):
 * after each forward chunk, nsw_solver_tol_local writes this shard's
 * per-iteration residual maxima [tol_chunk] float64 into the bound buffer;
 * the caller all-reduces it (MAX, in place); nsw_solver_tol_decide picks t*
 * and returns the device phase (host-synchronising): 5 = next chunk (call
 * nsw_solver_local_step again), 6 = t* found (call nsw_solver_local_step for
 * the finish launch), anything else = no forward pending.  Pass the total
 * user count with nsw_solver_set_scalar(s, "users_total", U) so the
 * SolverError fraction (solver.py:200-205) is over all ranks. */
nsw_status nsw_solver_bind_tol_exchange(nsw_solver* s, void* cmax_dev);
nsw_status nsw_solver_tol_local(nsw_solver* s, void* stream);
nsw_status nsw_solver_tol_decide(nsw_solver* s, void* stream, int32_t* phase);
/* local_step + finalize, world must be 1; uses the solver's own stream and
 * CUDA graph.  Runs at most max_steps outer steps; *done = 1 when finished. */
nsw_status nsw_solver_run(nsw_solver* s, int32_t max_steps, int32_t* done);
/* Host view of the device state: phase (0 init, 1 running, 2 stop pending,
 * 3 finished), recorded steps, error bits. */
nsw_status nsw_solver_status(nsw_solver* s, int32_t* phase, int32_t* steps, int32_t* errors);
nsw_status nsw_solver_stream(nsw_solver* s, void** stream);
/* Best policy [users_local][n][m] float64 and the trace (host). */
nsw_status nsw_solver_result(nsw_solver* s, double* policy_out, nsw_trace* trace);
/* Top-m ranking of the returned (best-F) policy, computed on the device:
 * out_host[u][k] = argmax_i X[u][i][k] for k < m-1, lowest index on ties
 * ([U][m-1] int32).  The reference has no ranking extraction; this is the
 * definition of SURVEY.md 8(a) (numpy argmax over items). */
nsw_status nsw_solver_top_positions(nsw_solver* s, int32_t* out_host);
/* Evaluation metrics (reference metrics.py) of the best policy, on the
 * device where it lives: out_host[4] as nsw_policy_metrics_*.  This
 * shard's users only (a sharded solve evaluates its block). */
nsw_status nsw_solver_metrics(nsw_solver* s, double threshold, double* out_host);

/* Raw state access for tests and one-step parity (host float64 buffers):
 * field = "cost" | "adam_m" | "adam_v" [U][n][m], "alpha" [U][n], "beta" [U][m],
 * "hist" [U][T+1][m], "partial" [U][n], "imp" [n], "xbest" [U][n][m].
 * nsw_solver_set_state also takes "adam_step" / "phase" through `scalar`. */
nsw_status nsw_solver_get(nsw_solver* s, const char* field, double* host, size_t count);
nsw_status nsw_solver_set(nsw_solver* s, const char* field, const double* host, size_t count);
nsw_status nsw_solver_set_scalar(nsw_solver* s, const char* field, int64_t value);
/* Number of kernel launches issued by the solver so far (evidence counter). */
int64_t nsw_solver_launch_count(nsw_solver* s);
/* Kernel variant chosen for the fused step: M, rows/thread, threads/CTA of the
 * main launch; a tail launch's R / NT (if any) are packed in bits 16..31. */
nsw_status nsw_solver_variant(nsw_solver* s, int32_t* M, int32_t* R, int32_t* NT, int32_t* smem_bytes);
/* Users handled by the tail launch (the wide, latency-oriented tile). */
int32_t nsw_solver_tail_users(nsw_solver* s);
/* Measurement helper: evict the L2 (1 GiB write, then discard of those
 * lines) on `stream` (NULL = the solver's stream). */
nsw_status nsw_solver_flush_l2(nsw_solver* s, void* stream);
/* Device time (ms) of the last N fused step kernels, CUDA events. */
nsw_status nsw_solver_time_steps(nsw_solver* s, int32_t steps, int32_t flush_l2, float* ms_total,
                                 float* ms_fused_kernel);
/* Measurement helper for any shard (also world > 1): device time (ms, summed)
 * of N replays of the fused step launch(es) alone, the L2 evicted before each;
 * the state machine does not advance (no impact reduction / finalize), the
 * iterate does.  Call at the end of a measurement. */
nsw_status nsw_solver_time_fused(nsw_solver* s, int32_t steps, int32_t flush_l2, float* ms_fused_kernel);
/* Diagnostics: global-timer stamps (ns) of the fused kernel's phase
 * boundaries, [count users][16], of the last step the solver ran.  Only when
 * the environment had NSW_PHASE_TIMING=1 at nsw_solver_create. */
nsw_status nsw_solver_phase_times(nsw_solver* s, uint64_t* out, int32_t count);

/* Top-m ranking of a device policy tensor X [U][n][m] (float32 / float64)
 * into device int32 out [U][m-1], on `stream` (cudaStream_t, 0 = default). */
nsw_status nsw_top_positions_f32(const float* X, int32_t U, int32_t n, int32_t m, int32_t* out, void* stream);
nsw_status nsw_top_positions_f64(const double* X, int32_t U, int32_t n, int32_t m, int32_t* out, void* stream);

/* Policy evaluation metrics (reference metrics.py:16-69) of a device policy
 * X [U][n][m] with device relevance [U][n] (same scalar type) and host
 * exposures [m-1] float64: out_host[0..3] = user_utility, mean_max_envy,
 * items_better_off(threshold), items_worse_off(threshold).  float64
 * accumulation; the n x n x U envy product is a cuBLAS DGEMM. */
nsw_status nsw_policy_metrics_f32(const float* X, const float* rel, const double* expo, int32_t U, int32_t n,
                                  int32_t m, double threshold, double* out_host, void* stream);
nsw_status nsw_policy_metrics_f64(const double* X, const double* rel, const double* expo, int32_t U, int32_t n,
                                  int32_t m, double threshold, double* out_host, void* stream);

/* Building blocks of the ascent as standalone device ops (reference
 * solver.py:46-122), for callers that compose their own loop:
 *   nsw_policy_impact_*     Imp_i = sum_{u,k<m-1} r_ui e_k x_uik -> host imp[n]
 *   nsw_welfare_gradient_*  grad [U][n][m] = r_ui e_k / Imp_i (0 at the dummy)
 *   nsw_adam_update_*       one Adam ascent step in place on count entries,
 *                           bias1/bias2 = 1 - beta^step as the caller computes
 *                           them; IEEE operations in the reference's order. */
nsw_status nsw_policy_impact_f32(const float* X, const float* rel, const double* expo, int32_t U, int32_t n,
                                 int32_t m, double* imp_host, void* stream);
nsw_status nsw_policy_impact_f64(const double* X, const double* rel, const double* expo, int32_t U, int32_t n,
                                 int32_t m, double* imp_host, void* stream);
nsw_status nsw_welfare_gradient_f32(const float* rel, const double* expo, const double* imp, int32_t U,
                                    int32_t n, int32_t m, float* grad, void* stream);
nsw_status nsw_welfare_gradient_f64(const double* rel, const double* expo, const double* imp, int32_t U,
                                    int32_t n, int32_t m, double* grad, void* stream);
nsw_status nsw_adam_update_f32(float* params, const float* grads, float* adam_m, float* adam_v, size_t count,
                               double lr, double beta1, double beta2, double eps, double bias1, double bias2,
                               void* stream);
nsw_status nsw_adam_update_f64(double* params, const double* grads, double* adam_m, double* adam_v,
                               size_t count, double lr, double beta1, double beta2, double eps, double bias1,
                               double bias2, void* stream);

/* ------------------------------------------------------------------------ *
 * 3. Inner operator seam (device pointers; one CTA per batch element).     *
 *    nsw_sinkhorn_solve_batch_* replaces _sinkhorn_batch (reference         *
 *        sinkhorn.py:204-255) with its full contract: log_kernel [B][n][m], *
 *        row [n] and col [m] masses (NULL, NULL = the ranking marginals of  *
 *        sinkhorn.py:55-60), log_v_init [B][m], tol (<= 0: exactly         *
 *        max_iters iterations; > 0: lock-step stop over the batch when the  *
 *        largest L-inf marginal residual is <= tol, sinkhorn.py:237-246)   *
 *        -> plan [B][n][m], log_u [B][n], log_v [B][m], log_v_hist          *
 *        [max_iters][B][m] (first *iterations rows valid), host outputs     *
 *        *iterations, converged[B] (0/1), residual[B] (float64).            *
 *    nsw_sinkhorn_batch_*: the fixed-schedule, ranking-marginal form.       *
 *    nsw_sinkhorn_backward_batch_* / _general_* replace                     *
 *        _sinkhorn_backward_batch (reference sinkhorn.py:258-309)           *
 *        -> grad_log_kernel [B][n][m]; _general_ takes the masses.          *
 *    nsw_cost_from_policy_* replaces cost_from_policy (sinkhorn.py:176-188):*
 *        cost = -epsilon log(plan) elementwise; NSW_ERR_DOMAIN unless every *
 *        entry is > 0 and epsilon > 0.                                      *
 * ------------------------------------------------------------------------ */
nsw_status nsw_sinkhorn_solve_batch_f64(const double* log_kernel, const double* row, const double* col,
                                        const double* log_v_init, int32_t B, int32_t n, int32_t m,
                                        int32_t max_iters, double tol, double* plan, double* log_u,
                                        double* log_v, double* log_v_hist, int32_t* iterations,
                                        int32_t* converged, double* residual, void* stream);
nsw_status nsw_sinkhorn_solve_batch_f32(const float* log_kernel, const float* row, const float* col,
                                        const float* log_v_init, int32_t B, int32_t n, int32_t m,
                                        int32_t max_iters, double tol, float* plan, float* log_u,
                                        float* log_v, float* log_v_hist, int32_t* iterations,
                                        int32_t* converged, double* residual, void* stream);
nsw_status nsw_sinkhorn_batch_f64(const double* log_kernel, const double* log_v_init, int32_t B,
                                  int32_t n, int32_t m, int32_t iters, double* plan, double* log_u,
                                  double* log_v, double* log_v_hist, void* stream);
nsw_status nsw_sinkhorn_batch_f32(const float* log_kernel, const float* log_v_init, int32_t B,
                                  int32_t n, int32_t m, int32_t iters, float* plan, float* log_u,
                                  float* log_v, float* log_v_hist, void* stream);
nsw_status nsw_sinkhorn_backward_batch_f64(const double* log_kernel, const double* log_v_hist,
                                           const double* log_v_init, const double* grad_plan,
                                           const double* plan, const double* log_u_final, int32_t B,
                                           int32_t n, int32_t m, int32_t iters,
                                           double* grad_log_kernel, void* stream);
nsw_status nsw_sinkhorn_backward_batch_f32(const float* log_kernel, const float* log_v_hist,
                                           const float* log_v_init, const float* grad_plan,
                                           const float* plan, const float* log_u_final, int32_t B,
                                           int32_t n, int32_t m, int32_t iters,
                                           float* grad_log_kernel, void* stream);
nsw_status nsw_sinkhorn_backward_general_f64(const double* log_kernel, const double* row, const double* col,
                                             const double* log_v_hist, const double* log_v_init,
                                             const double* grad_plan, const double* plan,
                                             const double* log_u_final, int32_t B, int32_t n, int32_t m,
                                             int32_t iters, double* grad_log_kernel, void* stream);
nsw_status nsw_sinkhorn_backward_general_f32(const float* log_kernel, const float* row, const float* col,
                                             const float* log_v_hist, const float* log_v_init,
                                             const float* grad_plan, const float* plan,
                                             const float* log_u_final, int32_t B, int32_t n, int32_t m,
                                             int32_t iters, float* grad_log_kernel, void* stream);
nsw_status nsw_cost_from_policy_f64(const double* plan, size_t count, double epsilon, double* cost,
                                    void* stream);
nsw_status nsw_cost_from_policy_f32(const float* plan, size_t count, double epsilon, float* cost,
                                    void* stream);

/* Page-locked host memory for results, from a small process-wide cache
 * (at most 4 GiB of free blocks are kept; NULL on failure).  Free with
 * nsw_host_free. */
void* nsw_host_alloc(size_t bytes);
void nsw_host_free(void* ptr);
/* Return cached memory: the free page-locked host blocks, and the unused
 * part of the solvers' private device pools (trimmed to zero). */
void nsw_release_cached(void);

/* On-device generation of the BASELINE synthetic relevance (counter-based
 * Philox4x32-10: every value a pure function of (seed, stream, index), so a
 * rank generates exactly its user shard [user0, user0 + users)); out is a
 * device [users][n] array of `dtype` (fp32 values are rounded once, clamped
 * to [1e-6, 1]).  Replaces the host generators for configs 1-4
 * (the reference's own generator is data.py:30-52).
 *   latent: r = sigmoid(<p_u, q_i> + b_i), p, q ~ N(0, I/d); bias_kind 0 none,
 *           1 N(0, bias_scale), 2 LogNormal(0, bias_scale) mean-centred.
 *   sparse: per_user distinct items ~ rank^-zipf_s (Gumbel-top-k), r ~ Beta(2, 5),
 *           every other entry floor_value. */
nsw_status nsw_datagen_latent(int64_t user0, int32_t users, int32_t n, int32_t d, int32_t bias_kind,
                              double bias_scale, uint64_t seed, int32_t dtype, void* out, void* stream);
nsw_status nsw_datagen_sparse(int64_t user0, int32_t users, int32_t n, int32_t per_user, double zipf_s,
                              double floor_value, uint64_t seed, int32_t dtype, void* out, void* stream);

/* Whether a (dtype, n, m, iters) problem runs on the device: every shape the
 * reference accepts (2 <= m <= n, reference core.py:60-66) does. */
int32_t nsw_supported(int32_t dtype, int32_t num_items, int32_t num_positions, int32_t iters);
/* Whether it runs on a compiled on-chip tile (register / shared-memory /
 * cluster resident); otherwise the streaming fused step (K~ and the adjoint
 * in an L2-resident per-CTA scratch) runs it. */
int32_t nsw_tiled(int32_t dtype, int32_t num_items, int32_t num_positions, int32_t iters);

#ifdef __cplusplus
}
#endif
#endif /* NSWRANK_B200_H */
