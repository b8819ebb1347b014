"""ctypes binding of libnswrank_b200.so (the C ABI in include/nswrank_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of anything that needs it raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnswrank_b200.so")

NSW_OK, NSW_ERR_SHAPE, NSW_ERR_DOMAIN, NSW_ERR_STATE, NSW_ERR_SOLVER, NSW_ERR_UNSUPPORTED, NSW_ERR_CUDA, \
    NSW_ERR_ARG = range(8)
NSW_F32, NSW_F64 = 0, 1
NSW_SCHEDULE_FIXED, NSW_SCHEDULE_TOLERANCE = 0, 1


class NativeLibraryError(RuntimeError):
    """libnswrank_b200.so is missing or failed to load (no CPU fallback exists)."""


class SolverConfigC(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("sinkhorn_max_iters", C.c_int32), ("sinkhorn_tol", C.c_double),
                ("outer_max_iters", C.c_int32), ("grad_threshold", C.c_double), ("adam_lr", C.c_double),
                ("adam_beta1", C.c_double), ("adam_beta2", C.c_double), ("adam_eps", C.c_double),
                ("warm_start", C.c_int32)]


class DeviceOptionsC(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("schedule", C.c_int32), ("device", C.c_int32), ("variant", C.c_int32),
                ("use_graph", C.c_int32), ("check_every", C.c_int32), ("tol_chunk", C.c_int32),
                ("reabsorb", C.c_double)]


class TraceC(C.Structure):
    _fields_ = [("steps", C.c_int32), ("objective", C.POINTER(C.c_double)), ("grad_norm", C.POINTER(C.c_double)),
                ("sinkhorn_iterations", C.POINTER(C.c_int32)), ("wall_time", C.POINTER(C.c_double))]


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_vp = C.c_void_p
_i32 = C.c_int32

# name -> (restype, argtypes): every symbol declared in include/nswrank_b200.h
SIGNATURES = {
    "nsw_last_error": (C.c_char_p, []),
    "nsw_version": (C.c_char_p, []),
    "nsw_supported": (_i32, [_i32, _i32, _i32, _i32]),
    "nsw_tiled": (_i32, [_i32, _i32, _i32, _i32]),
    "nsw_datagen_latent": (C.c_int, [C.c_int64, _i32, _i32, _i32, _i32, C.c_double, C.c_uint64, _i32, _vp, _vp]),
    "nsw_datagen_sparse": (C.c_int, [C.c_int64, _i32, _i32, _i32, C.c_double, C.c_double, C.c_uint64, _i32, _vp,
                                     _vp]),
    "nsw_solve_fair_ranking": (C.c_int, [_dp, _dp, _i32, _i32, _i32, C.POINTER(SolverConfigC),
                                         C.POINTER(DeviceOptionsC), _dp, C.POINTER(TraceC)]),
    "nsw_solver_create": (C.c_int, [_dp, _dp, _i32, _i32, _i32, _dp, _i32, C.POINTER(SolverConfigC),
                                    C.POINTER(DeviceOptionsC), C.POINTER(_vp)]),
    "nsw_solver_destroy": (C.c_int, [_vp]),
    "nsw_solver_exchange_buffers": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp)]),
    "nsw_solver_bind_exchange": (C.c_int, [_vp, _vp, _vp]),
    "nsw_solver_local_step": (C.c_int, [_vp, _vp]),
    "nsw_solver_finalize": (C.c_int, [_vp, _vp]),
    "nsw_solver_run": (C.c_int, [_vp, _i32, C.POINTER(_i32)]),
    "nsw_solver_status": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "nsw_solver_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "nsw_solver_result": (C.c_int, [_vp, _dp, C.POINTER(TraceC)]),
    "nsw_solver_get": (C.c_int, [_vp, C.c_char_p, _dp, C.c_size_t]),
    "nsw_solver_set": (C.c_int, [_vp, C.c_char_p, _dp, C.c_size_t]),
    "nsw_solver_set_scalar": (C.c_int, [_vp, C.c_char_p, C.c_int64]),
    "nsw_solver_launch_count": (C.c_int64, [_vp]),
    "nsw_solver_variant": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "nsw_solver_tail_users": (_i32, [_vp]),
    "nsw_solver_time_steps": (C.c_int, [_vp, _i32, _i32, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "nsw_solver_time_fused": (C.c_int, [_vp, _i32, _i32, C.POINTER(C.c_float)]),
    "nsw_solver_phase_times": (C.c_int, [_vp, C.POINTER(C.c_uint64), _i32]),
    "nsw_solver_top_positions": (C.c_int, [_vp, C.POINTER(_i32)]),
    "nsw_solver_metrics": (C.c_int, [_vp, C.c_double, _dp]),
    "nsw_solver_flush_l2": (C.c_int, [_vp, _vp]),
    "nsw_host_alloc": (_vp, [C.c_size_t]),
    "nsw_host_free": (None, [_vp]),
    "nsw_release_cached": (None, []),
    "nsw_solver_bind_tol_exchange": (C.c_int, [_vp, _vp]),
    "nsw_solver_tol_local": (C.c_int, [_vp, _vp]),
    "nsw_solver_tol_decide": (C.c_int, [_vp, _vp, C.POINTER(_i32)]),
    "nsw_top_positions_f32": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "nsw_top_positions_f64": (C.c_int, [_vp, _i32, _i32, _i32, _vp, _vp]),
    "nsw_policy_impact_f32": (C.c_int, [_vp, _vp, _dp, _i32, _i32, _i32, _dp, _vp]),
    "nsw_policy_impact_f64": (C.c_int, [_vp, _vp, _dp, _i32, _i32, _i32, _dp, _vp]),
    "nsw_welfare_gradient_f32": (C.c_int, [_vp, _dp, _dp, _i32, _i32, _i32, _vp, _vp]),
    "nsw_welfare_gradient_f64": (C.c_int, [_vp, _dp, _dp, _i32, _i32, _i32, _vp, _vp]),
    "nsw_adam_update_f32": (C.c_int, [_vp, _vp, _vp, _vp, C.c_size_t] + [C.c_double] * 6 + [_vp]),
    "nsw_adam_update_f64": (C.c_int, [_vp, _vp, _vp, _vp, C.c_size_t] + [C.c_double] * 6 + [_vp]),
    "nsw_policy_metrics_f32": (C.c_int, [_vp, _vp, _dp, _i32, _i32, _i32, C.c_double, _dp, _vp]),
    "nsw_policy_metrics_f64": (C.c_int, [_vp, _vp, _dp, _i32, _i32, _i32, C.c_double, _dp, _vp]),
    "nsw_sinkhorn_solve_batch_f64": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, C.c_double, _vp, _vp,
                                               _vp, _vp, C.POINTER(_i32), C.POINTER(_i32), _dp, _vp]),
    "nsw_sinkhorn_solve_batch_f32": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, C.c_double, _vp, _vp,
                                               _vp, _vp, C.POINTER(_i32), C.POINTER(_i32), _dp, _vp]),
    "nsw_sinkhorn_backward_general_f64": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32,
                                                    _vp, _vp]),
    "nsw_sinkhorn_backward_general_f32": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32,
                                                    _vp, _vp]),
    "nsw_cost_from_policy_f64": (C.c_int, [_vp, C.c_size_t, C.c_double, _vp, _vp]),
    "nsw_cost_from_policy_f32": (C.c_int, [_vp, C.c_size_t, C.c_double, _vp, _vp]),
    "nsw_sinkhorn_batch_f64": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "nsw_sinkhorn_batch_f32": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "nsw_sinkhorn_backward_batch_f64": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "nsw_sinkhorn_backward_batch_f32": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
}

_LIB = None


def load(path: str | None = None):
    """Load (once) and return the native library; raises NativeLibraryError."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    # NSW_LIB_PATH: an A/B build of the same library (build.py --tag); experiments only
    p = path or os.environ.get("NSW_LIB_PATH") or LIB_PATH
    if not os.path.exists(p):
        raise NativeLibraryError(
            f"{p} not found: build it with `python -m paper_2406_10262_b200.build` (there is no CPU fallback)")
    try:
        lib = C.CDLL(p, mode=C.RTLD_LOCAL)
    except OSError as e:  # pragma: no cover - depends on the box
        raise NativeLibraryError(f"cannot load {p}: {e}") from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def last_error() -> str:
    return (load().nsw_last_error() or b"").decode()


def dptr(a):
    """ctypes double* of a C-contiguous float64 ndarray."""
    return a.ctypes.data_as(_dp)


def host_to_cuda(x, dtype=None):
    """numpy-like -> CUDA torch tensor (copies read-only / strided arrays first,
    which torch cannot wrap); torch tensors pass through (moved/cast if needed)."""
    import numpy as np
    import torch
    if isinstance(x, torch.Tensor):
        t = x if dtype is None else x.to(dtype)
        return t.to("cuda").contiguous()
    a = np.asarray(x)
    if not a.flags.writeable or not a.flags.c_contiguous:
        a = np.array(a, copy=True, order="C")
    t = torch.as_tensor(a, device="cuda")
    return t if dtype is None else t.to(dtype)
