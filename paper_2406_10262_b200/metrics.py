"""Policy evaluation metrics on the device (reference ``nswrank/metrics.py``).

Same names and signatures as the reference (metrics.py:16-63):

    user_utility(policy, relevance, exposure)
    mean_max_envy(policy, relevance, exposure)
    items_better_off(policy, relevance, exposure, threshold=0.10)
    items_worse_off(policy, relevance, exposure, threshold=0.10)

plus ``policy_metrics`` that returns all four from one device pass.  The
allocation masses, impacts and row maxima are kernels in
``csrc/nsw_metrics.cu``; the one dense product of ``mean_max_envy``
(n x n x |U|, metrics.py:38) is a hand-written FP64 tensor-core kernel
(mma.sync m8n8k4 f64) with the row maxima fused into its epilogue, so the
n x n matrix is never written.  float64 accumulation throughout; a
float32 policy tensor (e.g. a device solve's output) is read as is.
Inputs may be the reference-style objects, numpy arrays, or CUDA torch
tensors already on the device.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import ShapeError
from .solver import check

__all__ = ["user_utility", "mean_max_envy", "items_better_off", "items_worse_off", "policy_metrics"]


def _dev(x, dtype):
    return _lib.host_to_cuda(x, dtype)


def policy_metrics(policy, relevance, exposure, threshold: float = 0.10) -> dict:
    """{"user_utility", "mean_max_envy", "items_better_off", "items_worse_off"}."""
    import torch
    x = policy if isinstance(policy, torch.Tensor) else getattr(policy, "values", policy)
    r = relevance if isinstance(relevance, torch.Tensor) else getattr(relevance, "values", relevance)
    e = np.ascontiguousarray(getattr(exposure, "values", exposure), dtype=np.float64)
    dt = torch.float32 if getattr(x, "dtype", None) in (torch.float32, np.float32) else torch.float64
    X = _dev(x, dt)
    R = _dev(r, dt)
    if X.dim() != 3:
        raise ShapeError(f"policy must be 3-d (users x items x positions), got ndim={X.dim()}")
    U, n, m = X.shape
    if tuple(R.shape) != (U, n):
        raise ShapeError(f"relevance shape {tuple(R.shape)} does not match ({U}, {n})")
    if e.shape != (m - 1,):
        raise ShapeError(f"exposure is for m={e.size + 1}, shape has m={m}")
    out = np.zeros(4)
    lib = _lib.load()
    fn = lib.nsw_policy_metrics_f32 if dt == torch.float32 else lib.nsw_policy_metrics_f64
    stream = torch.cuda.current_stream(X.device).cuda_stream
    check(fn(X.data_ptr(), R.data_ptr(), _lib.dptr(e), U, n, m, float(threshold), _lib.dptr(out), stream),
          "policy_metrics")
    return {"user_utility": float(out[0]), "mean_max_envy": float(out[1]),
            "items_better_off": float(out[2]), "items_worse_off": float(out[3])}


def user_utility(policy, relevance, exposure) -> float:
    """Average per-user expected relevance-weighted exposure (metrics.py:16-22)."""
    return policy_metrics(policy, relevance, exposure)["user_utility"]


def mean_max_envy(policy, relevance, exposure) -> float:
    """Average over items of the largest impact gain from swapping allocations
    with any item, itself included (metrics.py:25-41)."""
    return policy_metrics(policy, relevance, exposure)["mean_max_envy"]


def items_better_off(policy, relevance, exposure, threshold: float = 0.10) -> float:
    """Fraction of items whose impact beats uniform by more than ``threshold`` (metrics.py:44-52)."""
    return policy_metrics(policy, relevance, exposure, threshold)["items_better_off"]


def items_worse_off(policy, relevance, exposure, threshold: float = 0.10) -> float:
    """Fraction of items whose impact trails uniform by more than ``threshold`` (metrics.py:55-63)."""
    return policy_metrics(policy, relevance, exposure, threshold)["items_worse_off"]
