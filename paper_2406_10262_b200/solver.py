"""Drop-in ``solve_fair_ranking`` backed by the sm_100a kernels.

Same signature, argument meaning, return layout and exception classes as the
reference entry point (``nswrank.solver.solve_fair_ranking``, reference
solver.py:138-241):

    policy, trace = solve_fair_ranking(relevance, exposure, shape, config)

``policy`` is a ``RankingPolicy`` holding the best-objective iterate
(solver.py:217-219, 241) as a read-only float64 [U][n][m] array; ``trace`` is a
``SolveTrace`` with per-outer-step objective, gradient norm, Sinkhorn
iterations and wall time (solver.py:125-135).

Device-side knobs that the reference does not have live in a separate
``DeviceOptions`` object so ``SolverConfig`` keeps the reference defaults.
There is no CPU fallback: every call goes through libnswrank_b200.so.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import (DomainError, ExposureModel, ProblemShape, RankingPolicy, RelevanceMatrix, ShapeError,
                   SolverConfig, SolverError, StateError)

__all__ = ["DeviceOptions", "SolveTrace", "DeviceSolver", "solve_fair_ranking", "NativeLibraryError"]

NativeLibraryError = _lib.NativeLibraryError


@dataclass
class SolveTrace:
    """Per-outer-iteration diagnostics (reference solver.py:125-135)."""

    objective: list = field(default_factory=list)
    grad_norm: list = field(default_factory=list)
    sinkhorn_iterations: list = field(default_factory=list)
    wall_time: list = field(default_factory=list)

    def __len__(self) -> int:
        return len(self.objective)


@dataclass(frozen=True)
class DeviceOptions:
    """Device-only options.

    dtype     "float64" (parity instantiation, default: matches the float64
              reference) or "float32" (throughput instantiation).
    schedule  "tolerance" (default, the reference's own stopping rule,
              sinkhorn.py:237-246: lock-step stop once every user's marginal
              residual is <= sinkhorn_tol, SolverError if > 50 % of users miss
              it, solver.py:200-205) or "fixed": every Sinkhorn solve runs
              exactly ``config.sinkhorn_max_iters`` iterations (the reference
              with the fixed-schedule shim; what BASELINE.json
              measures).
    device    CUDA device ordinal; None (default) = the caller's current
              device.  The library runs every call on the solver's device and
              restores the caller's current device before returning.
    variant   -1 = automatic tile choice; >= 0 forces a compiled tile shape;
              -3 forces the streaming fused step (any shape; what runs when
              no on-chip tile holds the user's n x m tile).
    use_graph capture the outer step in a CUDA graph (fixed schedule).
    check_every  poll the device stop flag every N outer steps.
    tol_chunk inner iterations per forward launch in the tolerance schedule.
    reabsorb  None (default) or a threshold in nats: in-solve re-absorption of
              the Sinkhorn scalings (every 8 inner iterations, once
              max |log v~| exceeds it, v~ is folded into K~ and alpha re-
              normalised; the backward crosses back).  Needed only when one
              solve's duals travel beyond the float32 exponent range (cold
              start, warm_start=False, at small eps); runs the streaming fused
              step, fixed schedule.
    """

    dtype: str = "float64"
    schedule: str = "tolerance"
    device: int | None = None
    variant: int = -1
    use_graph: bool = True
    check_every: int = 16
    tol_chunk: int = 16
    reabsorb: float | None = None

    def to_c(self) -> _lib.DeviceOptionsC:
        if self.dtype not in ("float32", "float64"):
            raise DomainError(f"dtype must be 'float32' or 'float64', got {self.dtype!r}")
        if self.schedule not in ("fixed", "tolerance"):
            raise DomainError(f"schedule must be 'fixed' or 'tolerance', got {self.schedule!r}")
        return _lib.DeviceOptionsC(
            _lib.NSW_F64 if self.dtype == "float64" else _lib.NSW_F32,
            _lib.NSW_SCHEDULE_FIXED if self.schedule == "fixed" else _lib.NSW_SCHEDULE_TOLERANCE,
            -1 if self.device is None else int(self.device), int(self.variant), int(bool(self.use_graph)), int(self.check_every),
            int(self.tol_chunk), float(self.reabsorb or 0.0))


def _config_c(cfg) -> _lib.SolverConfigC:
    return _lib.SolverConfigC(float(cfg.epsilon), int(cfg.sinkhorn_max_iters), float(cfg.sinkhorn_tol),
                              int(cfg.outer_max_iters), float(cfg.grad_threshold), float(cfg.adam_lr),
                              float(cfg.adam_beta1), float(cfg.adam_beta2), float(cfg.adam_eps),
                              int(bool(cfg.warm_start)))


_ERRORS = {
    _lib.NSW_ERR_SHAPE: ShapeError,
    _lib.NSW_ERR_DOMAIN: DomainError,
    _lib.NSW_ERR_STATE: StateError,
    _lib.NSW_ERR_SOLVER: SolverError,
    _lib.NSW_ERR_UNSUPPORTED: NotImplementedError,
    _lib.NSW_ERR_CUDA: RuntimeError,
    _lib.NSW_ERR_ARG: ValueError,
}


def check(status: int, what: str = ""):
    if status != _lib.NSW_OK:
        msg = _lib.last_error()
        raise _ERRORS.get(status, RuntimeError)(f"{what}: {msg}" if what else msg)


def _values(obj, name):
    return np.ascontiguousarray(getattr(obj, "values", obj), dtype=np.float64)


def _check_instance(rel: np.ndarray, expo: np.ndarray, shape) -> None:
    """Shape checks of reference solver.py:34-43 (same messages)."""
    U, n, m = shape.num_users, shape.num_items, shape.num_positions
    if rel.shape != (U, n):
        raise ShapeError(f"relevance shape {rel.shape} does not match ({U}, {n})")
    if expo.size + 1 != m:
        raise ShapeError(f"exposure is for m={expo.size + 1}, shape has m={m}")


def _coerce(relevance, exposure, shape, config):
    """Accept this package's types, the reference's own types (duck typing),
    or plain arrays; validate like the reference's constructors."""
    if not isinstance(relevance, RelevanceMatrix):
        relevance = RelevanceMatrix(_values(relevance, "relevance"))
    if not isinstance(exposure, ExposureModel):
        exposure = ExposureModel(_values(exposure, "exposure"))
    if not isinstance(shape, ProblemShape):
        shape = ProblemShape(int(shape.num_users), int(shape.num_items), int(shape.num_positions))
    if not isinstance(config, SolverConfig):
        fields = SolverConfig.__dataclass_fields__
        config = SolverConfig(**{k: getattr(config, k) for k in fields if hasattr(config, k)})
    return relevance, exposure, shape, config


class DeviceSolver:
    """Step-level handle over one user shard (C ABI ``nsw_solver_*``).

    ``relevance_local`` are this shard's rows; ``rel_sq_sum`` is sum_u r_ui^2
    over ALL users (closed-form gradient norm); ``world`` is how many impact
    partials the finalize step sums.
    """

    def __init__(self, relevance_local, exposure, num_items, num_positions, config, options=None,
                 rel_sq_sum=None, world=1):
        self.lib = _lib.load()
        self.options = options or DeviceOptions()
        self.config = config
        rel = np.ascontiguousarray(relevance_local, dtype=np.float64)
        expo = np.ascontiguousarray(exposure, dtype=np.float64)
        self.U, self.n = rel.shape
        self.m = int(num_positions)
        assert self.n == num_items
        self.T = int(config.sinkhorn_max_iters)
        self.world = int(world)
        rsq = None if rel_sq_sum is None else np.ascontiguousarray(rel_sq_sum, dtype=np.float64)
        h = C.c_void_p()
        cfg = _config_c(config)
        opt = self.options.to_c()
        check(self.lib.nsw_solver_create(_lib.dptr(rel), _lib.dptr(expo), self.U, self.n, self.m,
                                         None if rsq is None else _lib.dptr(rsq), self.world,
                                         C.byref(cfg), C.byref(opt), C.byref(h)), "nsw_solver_create")
        self.h = h

    # -- lifecycle ---------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            self.lib.nsw_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- stepping ----------------------------------------------------------------
    def run(self, max_steps: int) -> bool:
        done = C.c_int32(0)
        check(self.lib.nsw_solver_run(self.h, int(max_steps), C.byref(done)), "nsw_solver_run")
        return bool(done.value)

    def local_step(self, stream: int | None = None):
        check(self.lib.nsw_solver_local_step(self.h, C.c_void_p(stream)), "nsw_solver_local_step")

    def finalize(self, stream: int | None = None):
        check(self.lib.nsw_solver_finalize(self.h, C.c_void_p(stream)), "nsw_solver_finalize")

    def exchange_buffers(self):
        a, b = C.c_void_p(), C.c_void_p()
        check(self.lib.nsw_solver_exchange_buffers(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def bind_exchange(self, local_ptr: int, gathered_ptr: int):
        check(self.lib.nsw_solver_bind_exchange(self.h, C.c_void_p(local_ptr), C.c_void_p(gathered_ptr)))

    # tolerance schedule across shards (all-reduce MAX between local and decide)
    def bind_tol_exchange(self, cmax_ptr: int):
        check(self.lib.nsw_solver_bind_tol_exchange(self.h, C.c_void_p(cmax_ptr)), "bind_tol_exchange")

    def tol_local(self, stream: int | None = None):
        check(self.lib.nsw_solver_tol_local(self.h, C.c_void_p(stream)), "nsw_solver_tol_local")

    def tol_decide(self, stream: int | None = None) -> int:
        ph = C.c_int32()
        check(self.lib.nsw_solver_tol_decide(self.h, C.c_void_p(stream), C.byref(ph)), "nsw_solver_tol_decide")
        return ph.value

    def stream(self) -> int:
        s = C.c_void_p()
        check(self.lib.nsw_solver_stream(self.h, C.byref(s)))
        return s.value or 0

    def status(self):
        p, s, e = C.c_int32(), C.c_int32(), C.c_int32()
        check(self.lib.nsw_solver_status(self.h, C.byref(p), C.byref(s), C.byref(e)))
        return p.value, s.value, e.value

    def variant(self):
        M, R, NT, sm = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        check(self.lib.nsw_solver_variant(self.h, C.byref(M), C.byref(R), C.byref(NT), C.byref(sm)))
        if M.value == 0:   # streaming fused step (no on-chip tile holds the user)
            return dict(M=0, generic=True, ctas=R.value, NT=NT.value, smem=0)
        out = dict(M=M.value, R=R.value & 0xFFFF, NT=NT.value & 0xFFFF, smem=sm.value)
        tail = int(self.lib.nsw_solver_tail_users(self.h))
        if tail > 0:
            out.update(tail_users=tail, tail_R=R.value >> 16, tail_NT=NT.value >> 16)
        return out

    def launch_count(self) -> int:
        return int(self.lib.nsw_solver_launch_count(self.h))

    def flush_l2(self, stream: int | None = None):
        """Measurement helper: evict the L2 on ``stream`` (1 GiB write + discard)."""
        check(self.lib.nsw_solver_flush_l2(self.h, C.c_void_p(stream)), "flush_l2")

    def time_steps(self, steps: int, flush_l2: bool = True):
        tot, fus = C.c_float(), C.c_float()
        check(self.lib.nsw_solver_time_steps(self.h, int(steps), int(flush_l2), C.byref(tot), C.byref(fus)))
        return tot.value, fus.value

    def time_fused(self, steps: int, flush_l2: bool = True) -> float:
        """Device ms of ``steps`` replays of the fused launch(es) alone (any
        world size; advances the iterate without a trace entry: call last)."""
        ms = C.c_float()
        check(self.lib.nsw_solver_time_fused(self.h, int(steps), int(flush_l2), C.byref(ms)), "time_fused")
        return ms.value

    def phase_times(self) -> np.ndarray:
        """Diagnostics: [U][16] global-timer stamps (ns) of the fused kernel's
        phase boundaries in the last step (solver created with NSW_PHASE_TIMING=1)."""
        out = np.zeros((self.U, 16), dtype=np.uint64)
        check(self.lib.nsw_solver_phase_times(self.h, out.ctypes.data_as(C.POINTER(C.c_uint64)), self.U))
        return out

    # -- state access ------------------------------------------------------------
    _FIELD_SHAPES = {
        "cost": lambda s: (s.U, s.n, s.m), "adam_m": lambda s: (s.U, s.n, s.m),
        "adam_v": lambda s: (s.U, s.n, s.m), "xbest": lambda s: (s.U, s.n, s.m),
        "alpha": lambda s: (s.U, s.n), "beta": lambda s: (s.U, s.m), "lvi": lambda s: (s.U, s.m),
        "hist": lambda s: (s.U, s.T + 1, s.m), "partial": lambda s: (s.U, s.n),
        "imp": lambda s: (s.n,), "imp_local": lambda s: (s.n,),
        "objective": lambda s: (s.config.outer_max_iters,), "grad_norm": lambda s: (s.config.outer_max_iters,),
    }

    def get(self, name: str) -> np.ndarray:
        out = np.empty(self._FIELD_SHAPES[name](self), dtype=np.float64)
        check(self.lib.nsw_solver_get(self.h, name.encode(), _lib.dptr(out), out.size), f"get {name}")
        return out

    def set(self, name: str, values) -> None:
        arr = np.ascontiguousarray(values, dtype=np.float64).reshape(self._FIELD_SHAPES[name](self))
        check(self.lib.nsw_solver_set(self.h, name.encode(), _lib.dptr(arr), arr.size), f"set {name}")

    def set_scalar(self, name: str, value: int) -> None:
        check(self.lib.nsw_solver_set_scalar(self.h, name.encode(), int(value)), f"set {name}")

    def top_positions(self) -> np.ndarray:
        """Top-m ranking of the best policy, computed on the device:
        int32 [U][m-1], argmax over items per real position (lowest index on ties)."""
        out = np.empty((self.U, self.m - 1), dtype=np.int32)
        check(self.lib.nsw_solver_top_positions(self.h, out.ctypes.data_as(C.POINTER(C.c_int32))), "top_positions")
        return out

    def metrics(self, threshold: float = 0.10) -> dict:
        """Reference metrics (metrics.py) of the best policy, computed where it lives."""
        out = np.zeros(4)
        check(self.lib.nsw_solver_metrics(self.h, float(threshold), _lib.dptr(out)), "metrics")
        return {"user_utility": float(out[0]), "mean_max_envy": float(out[1]),
                "items_better_off": float(out[2]), "items_worse_off": float(out[3])}

    def result(self):
        """(best policy float64 [U][n][m], SolveTrace)."""
        J = self.config.outer_max_iters
        pol = _host_buffer((self.U, self.n, self.m))
        obj = np.zeros(J)
        gn = np.zeros(J)
        its = np.zeros(J, dtype=np.int32)
        wall = np.zeros(J)
        tr = _lib.TraceC(0, _lib.dptr(obj), _lib.dptr(gn), its.ctypes.data_as(C.POINTER(C.c_int32)),
                         _lib.dptr(wall))
        st = self.lib.nsw_solver_result(self.h, _lib.dptr(pol), C.byref(tr))
        k = tr.steps
        trace = SolveTrace([float(x) for x in obj[:k]], [float(x) for x in gn[:k]],
                           [int(x) for x in its[:k]], [float(x) for x in wall[:k]])
        try:
            check(st, "nsw_solver_result")
        except Exception as e:
            e.trace = trace  # the steps recorded before the failure
            raise
        return pol, trace


class _HostBlock:
    """Owner of a page-locked block from the library's host cache; freed
    (returned to the cache) when the last array viewing it goes away."""

    def __init__(self, lib, ptr):
        self.lib, self.ptr = lib, ptr

    def __del__(self):
        try:
            self.lib.nsw_host_free(self.ptr)
        except Exception:
            pass


def _host_buffer(shape) -> np.ndarray:
    """float64 host array for a device result, page-locked (the copy runs at
    full link speed and repeated solves reuse the block); pageable if the
    allocation fails."""
    count = int(np.prod(shape))
    lib = _lib.load()
    ptr = lib.nsw_host_alloc(count * 8)
    if not ptr:
        return np.empty(shape, dtype=np.float64)
    buf = (C.c_double * count).from_address(ptr)
    buf._owner = _HostBlock(lib, ptr)
    return np.ctypeslib.as_array(buf).reshape(shape)


def solve_fair_ranking(relevance, exposure, shape, config, options: DeviceOptions | None = None):
    """Maximise the log Nash social welfare over ranking policies on the GPU.

    Drop-in for the reference ``solve_fair_ranking`` (solver.py:138-241):
    Adam ascent on the per-user transport costs, one Sinkhorn solve per user
    per outer step, gradients by the exact reverse mode of the unrolled
    iterations, returning the best-objective policy and the trace.
    """
    relevance, exposure, shape, config = _coerce(relevance, exposure, shape, config)
    rel = relevance.values
    expo = exposure.values
    _check_instance(rel, expo, shape)
    options = options or DeviceOptions()
    lib = _lib.load()
    U, n, m = shape.num_users, shape.num_items, shape.num_positions
    J = config.outer_max_iters
    rel_c = np.ascontiguousarray(rel, dtype=np.float64)
    expo_c = np.ascontiguousarray(expo, dtype=np.float64)
    pol = _host_buffer((U, n, m))
    obj = np.zeros(J)
    gn = np.zeros(J)
    its = np.zeros(J, dtype=np.int32)
    wall = np.zeros(J)
    tr = _lib.TraceC(0, _lib.dptr(obj), _lib.dptr(gn), its.ctypes.data_as(C.POINTER(C.c_int32)), _lib.dptr(wall))
    cfg = _config_c(config)
    opt = options.to_c()
    check(lib.nsw_solve_fair_ranking(_lib.dptr(rel_c), _lib.dptr(expo_c), U, n, m, C.byref(cfg), C.byref(opt),
                                     _lib.dptr(pol), C.byref(tr)), "solve_fair_ranking")
    k = tr.steps
    trace = SolveTrace([float(x) for x in obj[:k]], [float(x) for x in gn[:k]], [int(x) for x in its[:k]],
                       [float(x) for x in wall[:k]])
    # float32 solves verify finiteness on the device while widening the policy
    return RankingPolicy._adopt(pol, finite_checked=options.dtype == "float32"), trace


# ---------------------------------------------------------------------------
# Building blocks of the ascent as standalone device ops (reference
# solver.py:46-122): the same names and semantics, for callers that compose
# their own loop.  numpy in -> numpy out; CUDA torch tensors stay on device.
# ---------------------------------------------------------------------------
def _as_dev(x, dtype=None):
    import torch
    if isinstance(x, torch.Tensor):
        t = x if dtype is None else x.to(dtype)
        return t.to("cuda").contiguous(), True
    a = np.asarray(x)
    if dtype is None:
        dtype = torch.float32 if a.dtype == np.float32 else torch.float64
    if not a.flags.writeable or not a.flags.c_contiguous:
        a = np.array(a, copy=True, order="C")
    return torch.as_tensor(a, device="cuda").to(dtype), False


def impact(policy, relevance, exposure) -> np.ndarray:
    """Expected impact per item, Imp_i = sum_{u,k<m-1} r_ui e_k x_uik
    (reference solver.py:46-53), float64 [n], computed on the device."""
    import torch
    x = policy if isinstance(policy, torch.Tensor) else getattr(policy, "values", policy)
    X, _ = _as_dev(x)
    R, _ = _as_dev(relevance if isinstance(relevance, torch.Tensor) else _values(relevance, "relevance"), X.dtype)
    e = np.ascontiguousarray(getattr(exposure, "values", exposure), dtype=np.float64)
    U, n, m = X.shape
    if tuple(R.shape) != (U, n) or e.shape != (m - 1,):
        raise ShapeError(f"relevance {tuple(R.shape)} / exposure {e.shape} do not match policy {tuple(X.shape)}")
    out = np.zeros(n)
    lib = _lib.load()
    fn = lib.nsw_policy_impact_f32 if X.dtype == torch.float32 else lib.nsw_policy_impact_f64
    check(fn(X.data_ptr(), R.data_ptr(), _lib.dptr(e), U, n, m, _lib.dptr(out),
             torch.cuda.current_stream(X.device).cuda_stream), "impact")
    return out


def nsw_objective(impacts) -> float:
    """Log Nash social welfare sum_i log Imp_i (reference solver.py:56-65); an
    n-vector reduction, done on the host like the reference."""
    imp = np.asarray(impacts, dtype=np.float64)
    if imp.size == 0 or imp.min() <= 0.0:
        raise DomainError("impacts must be strictly positive")
    return float(np.log(imp).sum())


def nsw_gradient_wrt_policy(policy, relevance, exposure):
    """r_ui e_k / Imp_i at real positions, 0 at the dummy (reference
    solver.py:68-90), computed on the device."""
    import torch
    x = policy if isinstance(policy, torch.Tensor) else getattr(policy, "values", policy)
    imp = impact(x, relevance, exposure)
    if imp.min() <= 0.0:
        raise DomainError("impacts must be strictly positive to differentiate the welfare")
    X, as_t = _as_dev(x)
    R, _ = _as_dev(relevance if isinstance(relevance, torch.Tensor) else _values(relevance, "relevance"), X.dtype)
    e = np.ascontiguousarray(getattr(exposure, "values", exposure), dtype=np.float64)
    U, n, m = X.shape
    grad = torch.empty_like(X)
    lib = _lib.load()
    fn = lib.nsw_welfare_gradient_f32 if X.dtype == torch.float32 else lib.nsw_welfare_gradient_f64
    check(fn(R.data_ptr(), _lib.dptr(e), _lib.dptr(imp), U, n, m, grad.data_ptr(),
             torch.cuda.current_stream(X.device).cuda_stream), "nsw_gradient_wrt_policy")
    return grad if as_t else grad.cpu().numpy()


@dataclass
class AdamState:
    """First/second moment accumulators (reference solver.py:92-102)."""

    m: object
    v: object
    step: int = 0

    @classmethod
    def zeros(cls, shape) -> "AdamState":
        return cls(m=np.zeros(shape), v=np.zeros(shape), step=0)


def adam_update(params, grads, state: AdamState, config):
    """One Adam ascent step (reference solver.py:105-122) on the device:
    returns (updated params, new AdamState); the inputs are not modified."""
    import torch
    P, as_t = _as_dev(params)
    G, _ = _as_dev(grads, P.dtype)
    Mm, _ = _as_dev(state.m, P.dtype)
    Vv, _ = _as_dev(state.v, P.dtype)
    if G.shape != P.shape or Mm.shape != P.shape or Vv.shape != P.shape:
        raise ShapeError("params, grads and state must share one shape")
    P, Mm, Vv = P.clone(), Mm.clone(), Vv.clone()
    step = state.step + 1
    b1, b2 = config.adam_beta1, config.adam_beta2
    lib = _lib.load()
    fn = lib.nsw_adam_update_f32 if P.dtype == torch.float32 else lib.nsw_adam_update_f64
    check(fn(P.data_ptr(), G.data_ptr(), Mm.data_ptr(), Vv.data_ptr(), P.numel(), config.adam_lr, b1, b2,
             config.adam_eps, 1.0 - b1 ** step, 1.0 - b2 ** step, torch.cuda.current_stream(P.device).cuda_stream),
          "adam_update")
    torch.cuda.current_stream(P.device).synchronize()
    if as_t:
        return P, AdamState(m=Mm, v=Vv, step=step)
    return P.cpu().numpy(), AdamState(m=Mm.cpu().numpy(), v=Vv.cpu().numpy(), step=step)
