"""Inner operator seam and per-user API on the device, with the reference's
log-domain inputs and outputs (reference nswrank/sinkhorn.py):

    Marginals, SinkhornState                                 ~ sinkhorn.py:28-82
    sinkhorn_solve(cost, marginals, config, record_iterates) ~ sinkhorn.py:85-148 (tolerance stop)
    sinkhorn_backward(state, grad_plan)                      ~ sinkhorn.py:151-173
    cost_from_policy(plan, epsilon)                          ~ sinkhorn.py:176-188 (Theorem-1 map)
    sinkhorn_batch_solve(log_kernel, log_row, log_col, row, col, tol, max_iters, log_v_init, record)
                                                             ~ _sinkhorn_batch (sinkhorn.py:204-255)
    sinkhorn_batch(log_kernel, log_v_init, iters)            ~ _sinkhorn_batch(..., tol=-1), ranking marginals
    sinkhorn_backward_batch(log_kernel, log_v_hist, log_v_init, grad_plan, plan, log_u_final[, row, col])
                                                             ~ _sinkhorn_backward_batch (sinkhorn.py:258-309)

Arrays may be numpy (copied to the device, results returned as numpy) or
CUDA torch tensors (results returned as CUDA tensors on the same device).
float32 / float64 select the kernel instantiation.  No CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import DomainError, ShapeError, StateError

import ctypes as C

from . import _lib
from .solver import check

__all__ = ["sinkhorn_batch", "sinkhorn_backward_batch", "sinkhorn_batch_solve", "BatchResult", "Marginals",
           "SinkhornState", "sinkhorn_solve", "sinkhorn_backward", "cost_from_policy"]


def _to_dev(x, dtype):
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(dtype=dtype).contiguous(), True
    a = np.asarray(x)
    if not a.flags.writeable or not a.flags.c_contiguous:
        a = np.array(a, copy=True, order="C")
    return torch.as_tensor(a, dtype=dtype, device="cuda"), False


def _dtype_of(x):
    import torch
    if isinstance(x, torch.Tensor):
        return torch.float64 if x.dtype == torch.float64 else torch.float32
    return torch.float64 if np.asarray(x).dtype == np.float64 else torch.float32


def _out(t, as_torch):
    return t if as_torch else t.cpu().numpy()


def sinkhorn_batch(log_kernel, log_v_init, iters: int):
    """Returns (plan (B,n,m), log_u (B,n), log_v (B,m), log_v_hist (T,B,m))."""
    import torch
    dt = _dtype_of(log_kernel)
    K, is_t = _to_dev(log_kernel, dt)
    lvi, _ = _to_dev(log_v_init, dt)
    B, n, m = K.shape
    plan = torch.empty_like(K)
    lu = torch.empty((B, n), dtype=dt, device=K.device)
    lv = torch.empty((B, m), dtype=dt, device=K.device)
    hist = torch.empty((iters, B, m), dtype=dt, device=K.device)
    fn = _lib.load().nsw_sinkhorn_batch_f64 if dt == torch.float64 else _lib.load().nsw_sinkhorn_batch_f32
    stream = torch.cuda.current_stream(K.device).cuda_stream
    check(fn(K.data_ptr(), lvi.data_ptr(), B, n, m, int(iters), plan.data_ptr(), lu.data_ptr(), lv.data_ptr(),
             hist.data_ptr(), stream), "sinkhorn_batch")
    torch.cuda.current_stream(K.device).synchronize()
    return tuple(_out(t, is_t) for t in (plan, lu, lv, hist))


def sinkhorn_backward_batch(log_kernel, log_v_hist, log_v_init, grad_plan, plan, log_u_final, row=None, col=None):
    """Gradient with respect to log_kernel (B,n,m); ``row``/``col`` masses
    (default: the ranking marginals)."""
    if row is not None or col is not None:
        return _backward_general(log_kernel, log_v_hist, log_v_init, grad_plan, plan, log_u_final, row, col)
    import torch
    dt = _dtype_of(log_kernel)
    K, is_t = _to_dev(log_kernel, dt)
    hist, _ = _to_dev(log_v_hist, dt)
    lvi, _ = _to_dev(log_v_init, dt)
    gp, _ = _to_dev(grad_plan, dt)
    X, _ = _to_dev(plan, dt)
    lu, _ = _to_dev(log_u_final, dt)
    B, n, m = K.shape
    T = hist.shape[0]
    gk = torch.empty_like(K)
    lib = _lib.load()
    fn = lib.nsw_sinkhorn_backward_batch_f64 if dt == torch.float64 else lib.nsw_sinkhorn_backward_batch_f32
    stream = torch.cuda.current_stream(K.device).cuda_stream
    check(fn(K.data_ptr(), hist.data_ptr(), lvi.data_ptr(), gp.data_ptr(), X.data_ptr(), lu.data_ptr(), B, n, m, T,
             gk.data_ptr(), stream), "sinkhorn_backward_batch")
    torch.cuda.current_stream(K.device).synchronize()
    return _out(gk, is_t)


# ---------------------------------------------------------------------------
# full _sinkhorn_batch contract and the per-user API
# ---------------------------------------------------------------------------
@dataclass
class BatchResult:
    """Output of a batched solve (reference _BatchResult, sinkhorn.py:191-200)."""
    plan: object          # (B, n, m)
    log_u: object         # (B, n)
    log_v: object         # (B, m)
    log_v_hist: object    # (T, B, m) or None
    iterations: int
    converged: np.ndarray  # (B,) bool
    residual: np.ndarray   # (B,)


def sinkhorn_batch_solve(log_kernel, log_row, log_col, row, col, tol, max_iters, log_v_init, record=True):
    """Lock-step Sinkhorn over a stack of kernels with shared marginals
    (reference _sinkhorn_batch, sinkhorn.py:204-255): iterates until every
    element's L-inf marginal residual is <= tol (tol <= 0: exactly
    max_iters iterations).  ``log_row``/``log_col`` are accepted for
    signature parity; the device uses the linear masses ``row``/``col``."""
    import torch
    dt = _dtype_of(log_kernel)
    K, is_t = _to_dev(log_kernel, dt)
    lvi, _ = _to_dev(log_v_init, dt)
    r, _ = _to_dev(row, dt)
    c, _ = _to_dev(col, dt)
    B, n, m = K.shape
    if r.numel() != n or c.numel() != m:
        raise ShapeError(f"marginals ({r.numel()}, {c.numel()}) do not match kernel shape {(n, m)}")
    T = int(max_iters)
    plan = torch.empty_like(K)
    lu = torch.empty((B, n), dtype=dt, device=K.device)
    lv = torch.empty((B, m), dtype=dt, device=K.device)
    hist = torch.empty((T, B, m), dtype=dt, device=K.device)
    its = C.c_int32()
    conv = np.zeros(B, dtype=np.int32)
    res = np.zeros(B)
    lib = _lib.load()
    fn = lib.nsw_sinkhorn_solve_batch_f64 if dt == torch.float64 else lib.nsw_sinkhorn_solve_batch_f32
    stream = torch.cuda.current_stream(K.device).cuda_stream
    check(fn(K.data_ptr(), r.data_ptr(), c.data_ptr(), lvi.data_ptr(), B, n, m, T, float(tol), plan.data_ptr(),
             lu.data_ptr(), lv.data_ptr(), hist.data_ptr(), C.byref(its), conv.ctypes.data_as(C.POINTER(C.c_int32)),
             res.ctypes.data_as(C.POINTER(C.c_double)), stream), "sinkhorn_batch_solve")
    used = its.value
    return BatchResult(plan=_out(plan, is_t), log_u=_out(lu, is_t), log_v=_out(lv, is_t),
                       log_v_hist=_out(hist[:used], is_t) if record else None, iterations=used,
                       converged=conv.astype(bool), residual=res)


def _backward_general(log_kernel, log_v_hist, log_v_init, grad_plan, plan, log_u_final, row, col):
    import torch
    dt = _dtype_of(log_kernel)
    K, is_t = _to_dev(log_kernel, dt)
    hist, _ = _to_dev(log_v_hist, dt)
    lvi, _ = _to_dev(log_v_init, dt)
    gp, _ = _to_dev(grad_plan, dt)
    X, _ = _to_dev(plan, dt)
    lu, _ = _to_dev(log_u_final, dt)
    B, n, m = K.shape
    r, _ = _to_dev(np.ones(n) if row is None else row, dt)
    c, _ = _to_dev(col if col is not None else np.r_[np.ones(m - 1), n - m + 1.0], dt)
    T = hist.shape[0]
    gk = torch.empty_like(K)
    lib = _lib.load()
    fn = lib.nsw_sinkhorn_backward_general_f64 if dt == torch.float64 else lib.nsw_sinkhorn_backward_general_f32
    stream = torch.cuda.current_stream(K.device).cuda_stream
    check(fn(K.data_ptr(), r.data_ptr(), c.data_ptr(), hist.data_ptr(), lvi.data_ptr(), gp.data_ptr(), X.data_ptr(),
             lu.data_ptr(), B, n, m, T, gk.data_ptr(), stream), "sinkhorn_backward_general")
    torch.cuda.current_stream(K.device).synchronize()
    return _out(gk, is_t)


@dataclass(frozen=True)
class Marginals:
    """Prescribed row and column masses of a transport plan (reference
    sinkhorn.py:28-60): strictly positive, equal totals."""

    row: np.ndarray
    col: np.ndarray

    def __post_init__(self):
        row = np.array(self.row, dtype=np.float64, copy=True)
        col = np.array(self.col, dtype=np.float64, copy=True)
        if row.ndim != 1 or col.ndim != 1:
            raise ShapeError("marginals must be 1-d vectors")
        if row.min() <= 0.0 or col.min() <= 0.0:
            raise DomainError("marginals must be strictly positive")
        total = row.sum()
        if abs(col.sum() - total) > 1e-9 * max(1.0, total):
            raise DomainError("row and column marginals must have equal total mass")
        row.setflags(write=False)
        col.setflags(write=False)
        object.__setattr__(self, "row", row)
        object.__setattr__(self, "col", col)

    @classmethod
    def for_shape(cls, num_items: int, num_positions: int) -> "Marginals":
        """Ranking marginals: unit item rows, unit real positions, dummy remainder."""
        col = np.ones(num_positions)
        col[-1] = num_items - num_positions + 1
        return cls(np.ones(num_items), col)


@dataclass(frozen=True)
class SinkhornState:
    """Forward record of a solve (reference sinkhorn.py:63-82)."""

    epsilon: float
    log_kernel: np.ndarray
    log_row: np.ndarray
    log_col: np.ndarray
    log_u: np.ndarray
    log_v: np.ndarray
    log_v_init: np.ndarray
    log_v_iterates: np.ndarray | None
    iterations_used: int
    converged: bool
    final_residual: float


def sinkhorn_solve(cost, marginals: Marginals, config, record_iterates: bool = True):
    """One entropic transport solve on the device (reference sinkhorn.py:85-148):
    log-domain kernel -C/eps, the config's tolerance stop and iteration budget,
    warm start v^0 = 0.  Returns (plan (n, m) float64, SinkhornState)."""
    c = np.asarray(cost, dtype=np.float64)
    if c.ndim != 2:
        raise ShapeError(f"cost must be 2-d, got ndim={c.ndim}")
    if not np.all(np.isfinite(c)):
        raise DomainError("cost contains non-finite entries")
    n, m = c.shape
    if marginals.row.size != n or marginals.col.size != m:
        raise ShapeError(f"marginals ({marginals.row.size}, {marginals.col.size}) do not match cost shape {(n, m)}")
    log_kernel = -c / config.epsilon
    log_row = np.log(marginals.row)
    log_col = np.log(marginals.col)
    log_v0 = np.zeros((1, m))
    res = sinkhorn_batch_solve(log_kernel[None], log_row, log_col, marginals.row, marginals.col,
                               config.sinkhorn_tol, config.sinkhorn_max_iters, log_v0, record_iterates)
    state = SinkhornState(epsilon=config.epsilon, log_kernel=log_kernel, log_row=log_row, log_col=log_col,
                          log_u=res.log_u[0], log_v=res.log_v[0], log_v_init=log_v0[0],
                          log_v_iterates=None if res.log_v_hist is None else res.log_v_hist[:, 0, :],
                          iterations_used=res.iterations, converged=bool(res.converged[0]),
                          final_residual=float(res.residual[0]))
    return res.plan[0], state


def sinkhorn_backward(state: SinkhornState, grad_plan) -> np.ndarray:
    """Gradient of a recorded solve with respect to the cost matrix
    (reference sinkhorn.py:151-173)."""
    if state.log_v_iterates is None:
        raise StateError("solve was run without iterate recording; cannot differentiate")
    g = np.asarray(grad_plan, dtype=np.float64)
    if g.shape != state.log_kernel.shape:
        raise ShapeError(f"grad_plan has shape {g.shape}, expected {state.log_kernel.shape}")
    plan = np.exp(state.log_u[:, None] + state.log_kernel + state.log_v[None, :])
    gk = _backward_general(state.log_kernel[None], state.log_v_iterates[:, None, :], state.log_v_init[None],
                           g[None], plan[None], state.log_u[None], np.exp(state.log_row), np.exp(state.log_col))
    return gk[0] / (-state.epsilon)


def cost_from_policy(plan, epsilon: float):
    """Cost whose entropic transport solution is ``plan``: -epsilon log(plan),
    elementwise, for a matrix or a stacked policy tensor (reference
    sinkhorn.py:176-188; Theorem 1).  numpy in -> numpy out (float64); a CUDA
    torch tensor stays on the device."""
    import torch
    if epsilon <= 0:
        raise DomainError("epsilon must be > 0")
    as_t = isinstance(plan, torch.Tensor)
    x = plan.contiguous() if as_t else _lib.host_to_cuda(np.asarray(plan, dtype=np.float64))
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    out = torch.empty_like(x)
    lib = _lib.load()
    fn = lib.nsw_cost_from_policy_f64 if x.dtype == torch.float64 else lib.nsw_cost_from_policy_f32
    st = fn(x.data_ptr(), x.numel(), float(epsilon), out.data_ptr(), torch.cuda.current_stream(x.device).cuda_stream)
    if st == 2:
        raise DomainError("plan must be strictly positive to take its logarithm")
    check(st, "cost_from_policy")
    return out if as_t else out.cpu().numpy()
