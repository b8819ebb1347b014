"""Inner operator seam on the device: the reference's batched Sinkhorn
forward and its unrolled reverse mode, with the reference's log-domain inputs
and outputs (fixed schedule, ranking marginals of sinkhorn.py:55-60).

    sinkhorn_batch(log_kernel, log_v_init, iters)           ~ _sinkhorn_batch(..., tol=-1, record=True)
    sinkhorn_backward_batch(log_kernel, log_v_hist, log_v_init, grad_plan, plan, log_u_final)
                                                            ~ _sinkhorn_backward_batch (sinkhorn.py:258-309)

Arrays may be numpy (copied to the device, results returned as numpy) or
CUDA torch tensors (results returned as CUDA tensors on the same device).
float32 / float64 select the kernel instantiation.  No CPU fallback.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .solver import check

__all__ = ["sinkhorn_batch", "sinkhorn_backward_batch"]


def _to_dev(x, dtype):
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(dtype=dtype).contiguous(), True
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda"), False


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
    torch.cuda.synchronize(K.device)
    return tuple(_out(t, is_t) for t in (plan, lu, lv, hist))


def sinkhorn_backward_batch(log_kernel, log_v_hist, log_v_init, grad_plan, plan, log_u_final):
    """Gradient with respect to log_kernel (B,n,m)."""
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
    torch.cuda.synchronize(K.device)
    return _out(gk, is_t)
