"""CPU oracle for the NSW fair-ranking ascent path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import it.  The shipped solver
(``paper_2406_10262_b200``) never imports, links or executes anything under
``oracle/``.

It is a dtype-parametric numpy restatement of the reference algorithm
(``/root/reference/pkg/src/nswrank``, version 0.1.0).  Every function names the
reference lines it restates.  In float64 it reproduces the reference
bit-for-bit (pinned by ``tests/test_oracle.py`` against the golden fixtures in
``tests/golden/`` that ``oracle/gen_golden.py`` produced by running the real
reference with the fixed-schedule shim).  In float32 it is the "same algorithm,
fp32 arithmetic" yard-stick used for one-step parity of the fp32 device path.

Parity pinned: yes (golden fixtures generated from the imported reference).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np


# --------------------------------------------------------------------------
# marginals and initial cost
# --------------------------------------------------------------------------
def ranking_marginals(n: int, m: int, dtype=np.float64):
    """Row masses 1, column masses (1,...,1, n-m+1).

    Restates ``Marginals.for_shape`` (sinkhorn.py:55-60) and the log-marginals
    of ``solve_fair_ranking`` (solver.py:172-174)."""
    row = np.ones(n, dtype=dtype)
    col = np.ones(m, dtype=dtype)
    col[m - 1] = n - m + 1
    return row, col, np.log(row), np.log(col)


def initial_cost(U: int, n: int, m: int, eps: float, dtype=np.float64):
    """C0 = -eps * log(uniform policy).

    Restates ``uniform_policy`` (core.py:220-231) and solver.py:176-177."""
    x = np.empty((U, n, m), dtype=np.float64)
    x[:, :, : m - 1] = 1.0 / n
    x[:, :, m - 1] = (n - m + 1) / n
    return (-eps * np.log(x)).astype(dtype)


# --------------------------------------------------------------------------
# batched Sinkhorn forward  (sinkhorn.py:204-255)
# --------------------------------------------------------------------------
@dataclass
class ForwardResult:
    plan: np.ndarray      # (B, n, m)
    log_u: np.ndarray     # (B, n)
    log_v: np.ndarray     # (B, m)
    hist: np.ndarray      # (T, B, m) column duals after each iteration
    iterations: int
    converged: np.ndarray
    residual: np.ndarray
    residual_trace: list  # max-over-users residual after every iteration


def _row_dual(log_kernel, log_v, log_row):
    # u = log_row - LSE_k(K + v)                       sinkhorn.py:219-226
    z = log_kernel + log_v[:, None, :]
    top = z.max(axis=2)
    z -= top[:, :, None]
    np.exp(z, out=z)
    acc = z.sum(axis=2)
    np.log(acc, out=acc)
    return log_row[None, :] - (acc + top)


def _col_dual(log_kernel, log_u, log_col):
    # v = log_col - LSE_i(K + u)                       sinkhorn.py:227-234
    z = log_kernel + log_u[:, :, None]
    top = z.max(axis=1)
    z -= top[:, None, :]
    np.exp(z, out=z)
    acc = z.sum(axis=1)
    np.log(acc, out=acc)
    return log_col[None, :] - (acc + top)


def sinkhorn_forward(log_kernel, log_row, log_col, row, col, tol, max_iters, log_v_init):
    """Lock-step log-domain Sinkhorn with the every-iteration residual test.

    ``tol < 0`` gives the fixed schedule (exactly ``max_iters`` iterations),
    which is what the reference does when the shim forces ``tol=-1``."""
    B, n, m = log_kernel.shape
    log_v = log_v_init.copy()
    log_u = np.zeros((B, n), dtype=log_kernel.dtype)
    hist = np.empty((max_iters, B, m), dtype=log_kernel.dtype)
    plan = None
    residual = np.full(B, np.inf)
    res_trace = []
    used = max_iters
    for t in range(max_iters):
        log_u = _row_dual(log_kernel, log_v, log_row)
        log_v = _col_dual(log_kernel, log_u, log_col)
        hist[t] = log_v
        # reconstructed plan and L-inf marginal residual     sinkhorn.py:237-243
        plan = log_kernel + log_u[:, :, None]
        plan += log_v[:, None, :]
        np.exp(plan, out=plan)
        r_res = np.abs(plan.sum(axis=2) - row[None, :]).max(axis=1)
        c_res = np.abs(plan.sum(axis=1) - col[None, :]).max(axis=1)
        residual = np.maximum(r_res, c_res)
        res_trace.append(float(residual.max()))
        if residual.max() <= tol:                          # sinkhorn.py:244-246
            used = t + 1
            break
    return ForwardResult(plan, log_u, log_v, hist[:used].copy(), used,
                         residual <= tol, residual, res_trace)


# --------------------------------------------------------------------------
# unrolled reverse mode  (sinkhorn.py:258-309)
# --------------------------------------------------------------------------
def sinkhorn_backward(log_kernel, log_row, log_col, hist, log_v_init, grad_plan, plan, log_u_final):
    """Exact reverse-mode derivative of the recorded iteration sequence with
    respect to ``log_kernel`` (warm-start duals are constants)."""
    T = hist.shape[0]
    w = grad_plan * plan                                   # sinkhorn.py:272
    g_kernel = w.copy()
    g_u = w.sum(axis=2)
    g_v = w.sum(axis=1)
    log_u_t = log_u_final
    for t in range(T, 0, -1):
        v_t = hist[t - 1]
        v_prev = hist[t - 2] if t >= 2 else log_v_init
        # column softmax VJP                               sinkhorn.py:281-289
        s = log_kernel + log_u_t[:, :, None]
        s += v_t[:, None, :]
        s -= log_col[None, None, :]
        np.exp(s, out=s)
        s *= g_v[:, None, :]
        g_kernel -= s
        g_u = g_u - s.sum(axis=2)
        # row softmax VJP                                  sinkhorn.py:290-299
        s = log_kernel + v_prev[:, None, :]
        s += log_u_t[:, :, None]
        s -= log_row[None, :, None]
        np.exp(s, out=s)
        s *= g_u[:, :, None]
        g_kernel -= s
        g_v = -s.sum(axis=1)
        g_u = np.zeros_like(g_u)
        if t >= 2:                                         # sinkhorn.py:300-308
            v_pp = hist[t - 3] if t >= 3 else log_v_init
            log_u_t = _row_dual(log_kernel, v_pp, log_row)
    return g_kernel


# --------------------------------------------------------------------------
# objective pieces  (solver.py:46-122)
# --------------------------------------------------------------------------
def impact(rel, expo, plan):
    """Imp_i = sum_u sum_{k<m-1} r_ui e_k x_uik  (solver.py:206, :46-53)."""
    m1 = expo.shape[0]
    return np.einsum("ui,k,uik->i", rel, expo, plan[:, :, :m1])


def welfare_gradient(rel, expo, imp, out):
    """gx = r e / Imp on real positions, dummy untouched (solver.py:86-89)."""
    m1 = expo.shape[0]
    np.multiply(rel[:, :, None], expo[None, None, :], out=out[:, :, :m1])
    out[:, :, :m1] /= imp[None, :, None]


def adam_ascent(params, grads, m, v, step, lr, b1, b2, eps):
    """One Adam *ascent* step (solver.py:105-122); returns (p, m, v, step)."""
    step = step + 1
    m_new = b1 * m + (1.0 - b1) * grads
    v_new = b2 * v + (1.0 - b2) * grads * grads
    m_hat = m_new / (1.0 - b1 ** step)
    v_hat = v_new / (1.0 - b2 ** step)
    return params + lr * m_hat / (np.sqrt(v_hat) + eps), m_new, v_new, step


# --------------------------------------------------------------------------
# the outer ascent loop  (solver.py:138-241)
# --------------------------------------------------------------------------
@dataclass
class SolverParams:
    epsilon: float = 0.1
    sinkhorn_max_iters: int = 500
    sinkhorn_tol: float = 1e-6
    outer_max_iters: int = 300
    grad_threshold: float = 1e-3
    adam_lr: float = 0.05
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    warm_start: bool = True
    fixed_schedule: bool = True   # True = the shimmed reference (tol=-1, guard off)


class OracleSolverError(RuntimeError):
    pass


class OracleDomainError(ValueError):
    pass


@dataclass
class OracleTrace:
    objective: list = field(default_factory=list)
    grad_norm: list = field(default_factory=list)
    sinkhorn_iterations: list = field(default_factory=list)
    wall_time: list = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.objective)


def solve(rel, expo, p: SolverParams, dtype=np.float64, record_states=(), on_step=None):
    """Restatement of ``solve_fair_ranking`` (solver.py:138-241).

    ``p.fixed_schedule`` reproduces the reference under the fixed-schedule shim
    (``_sinkhorn_batch`` called with tol=-1 and every user marked converged;
    SURVEY.md section 8(c)).  ``record_states`` is a set of outer-step indices
    at whose *start* (C, adam m, adam v, adam step, lvi) is captured, for
    one-step parity checks.  Returns (best_plan, trace, states).
    """
    rel = np.asarray(rel, dtype=dtype)
    expo = np.asarray(expo, dtype=dtype)
    U, n = rel.shape
    m = expo.shape[0] + 1
    row, col, log_row, log_col = ranking_marginals(n, m, dtype)
    cost = initial_cost(U, n, m, p.epsilon, dtype)
    am = np.zeros_like(cost)
    av = np.zeros_like(cost)
    astep = 0
    lvi = np.zeros((U, m), dtype=dtype)
    gx = np.zeros_like(cost)
    tol = -1.0 if p.fixed_schedule else p.sinkhorn_tol
    trace = OracleTrace()
    states = {}
    best = -np.inf
    best_plan = None
    neg_inv_eps = dtype(-1.0 / p.epsilon) if dtype is not np.float64 else -1.0 / p.epsilon
    for it in range(p.outer_max_iters):
        tic = time.perf_counter()
        if it in record_states:
            states[it] = dict(cost=cost.copy(), m=am.copy(), v=av.copy(), step=astep, lvi=lvi.copy())
        log_kernel = cost * neg_inv_eps                          # solver.py:188
        fwd = sinkhorn_forward(log_kernel, log_row, log_col, row, col, tol,
                               p.sinkhorn_max_iters, lvi)
        if not p.fixed_schedule:
            failed = 1.0 - float(fwd.converged.mean())            # solver.py:200-205
            if failed > 0.5:
                raise OracleSolverError(
                    f"Sinkhorn failed to converge for {failed:.0%} of users "
                    f"within {p.sinkhorn_max_iters} iterations (outer step {it})")
        imp = impact(rel, expo, fwd.plan)
        if imp.min() <= 0.0:
            raise OracleDomainError("item impact became nonpositive during the solve")
        objective = float(np.log(imp.astype(np.float64)).sum())
        welfare_gradient(rel, expo, imp, gx)
        grad_norm = float(np.linalg.norm(gx[:, :, : m - 1]))
        trace.objective.append(objective)
        trace.grad_norm.append(grad_norm)
        trace.sinkhorn_iterations.append(fwd.iterations)
        trace.wall_time.append(time.perf_counter() - tic)
        if it in record_states:
            states[it].update(plan=fwd.plan.copy(), log_u=fwd.log_u.copy(), log_v=fwd.log_v.copy(),
                              hist=fwd.hist.copy(), imp=imp.copy(), objective=objective)
        if objective >= best:                                    # solver.py:217-219
            best = objective
            best_plan = fwd.plan
        if on_step is not None:
            on_step(it, fwd, imp)
        if grad_norm <= p.grad_threshold or len(trace.objective) == p.outer_max_iters:
            break
        g_kernel = sinkhorn_backward(log_kernel, log_row, log_col, fwd.hist, lvi, gx,
                                     fwd.plan, fwd.log_u)
        g_kernel *= neg_inv_eps                                  # solver.py:235-236
        if it in record_states:
            states[it]["grad_cost"] = g_kernel.copy()
        cost, am, av, astep = adam_ascent(cost, g_kernel, am, av, astep, p.adam_lr,
                                          p.adam_beta1, p.adam_beta2, p.adam_eps)
        trace.wall_time[-1] = time.perf_counter() - tic
        if p.warm_start:
            lvi = fwd.log_v
    return best_plan, trace, states


def one_step(rel, expo, state, p: SolverParams, dtype=np.float64):
    """Run one full outer step (forward, impact, gradient, backward, Adam) from
    a captured state.  Used for fp32 one-step parity."""
    rel = np.asarray(rel, dtype=dtype)
    expo = np.asarray(expo, dtype=dtype)
    U, n = rel.shape
    m = expo.shape[0] + 1
    row, col, log_row, log_col = ranking_marginals(n, m, dtype)
    cost = state["cost"].astype(dtype)
    lvi = state["lvi"].astype(dtype)
    neg_inv_eps = dtype(-1.0 / p.epsilon) if dtype is not np.float64 else -1.0 / p.epsilon
    log_kernel = cost * neg_inv_eps
    fwd = sinkhorn_forward(log_kernel, log_row, log_col, row, col, -1.0, p.sinkhorn_max_iters, lvi)
    imp = impact(rel.astype(np.float64), expo.astype(np.float64), fwd.plan.astype(np.float64))
    gx = np.zeros_like(cost)
    welfare_gradient(rel, expo, imp.astype(dtype), gx)
    g_kernel = sinkhorn_backward(log_kernel, log_row, log_col, fwd.hist, lvi, gx, fwd.plan, fwd.log_u)
    g_kernel *= neg_inv_eps
    c1, m1, v1, s1 = adam_ascent(cost, g_kernel, state["m"].astype(dtype), state["v"].astype(dtype),
                                 state["step"], p.adam_lr, p.adam_beta1, p.adam_beta2, p.adam_eps)
    return dict(plan=fwd.plan, imp=imp, grad_cost=g_kernel, cost=c1, m=m1, v=v1, step=s1,
                log_v=fwd.log_v, log_u=fwd.log_u)


# --------------------------------------------------------------------------
# evaluation metrics  (metrics.py:16-69)
# --------------------------------------------------------------------------
def policy_metrics(policy, rel, expo, threshold=0.10):
    """user_utility, mean_max_envy, items_better_off, items_worse_off of a
    policy (metrics.py:16-22, :25-41, :44-52, :55-63; uniform reference
    policy core.py:220-231)."""
    U, n, m = policy.shape
    x = policy[:, :, : m - 1]
    util = float(np.einsum("ui,k,uik->", rel, expo, x) / U)               # metrics.py:20-22
    alloc = np.einsum("ujk,k->uj", x, expo)                               # metrics.py:37
    cross = rel.T @ alloc                                                  # metrics.py:39
    envy = float((cross.max(axis=1) - np.diagonal(cross)).mean())         # metrics.py:40-41
    imp = impact(rel, expo, policy)
    unif = np.empty((U, n, m))
    unif[:, :, : m - 1] = 1.0 / n
    unif[:, :, m - 1] = (n - m + 1) / n
    imp_u = impact(rel, expo, unif)                                        # metrics.py:66-68
    better = float(np.mean(imp > (1.0 + threshold) * imp_u))
    worse = float(np.mean(imp < (1.0 - threshold) * imp_u))
    return util, envy, better, worse


def top_positions(policy):
    """Top-m ranking used for the bit-exact ranking check: for every user and
    real position k, argmax_i X[u, i, k] (numpy first-index tie-break).

    The reference defines no ranking extraction; this is the
    recommended definition it names."""
    return np.argmax(policy[:, :, :-1], axis=1).astype(np.int32)
