"""Top-m ranking extraction on the device.

The reference returns the stochastic ranking tensor X and defines no
deterministic ranking; the north star's "final top-m ranking per user
bit-exact" check uses the definition SURVEY.md 8(a) recommends:
for every user u and real position k < m-1, the item argmax_i X[u, i, k],
lowest index on ties (numpy ``argmax`` semantics).  The oracle's
``top_positions`` is the CPU statement of the same rule.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .solver import check

__all__ = ["top_positions"]


def top_positions(policy):
    """int32 [U][m-1] ranking of a policy.

    ``policy`` may be a ``RankingPolicy`` (or anything with ``.values``), a
    numpy array (copied to the device; the result is numpy) or a CUDA torch
    tensor (the result is a CUDA int32 tensor).  float32 and float64 use
    their own kernel instantiation, so the comparison is on the exact values
    the solver produced."""
    import torch
    as_torch = isinstance(policy, torch.Tensor)
    x = policy if as_torch else getattr(policy, "values", policy)
    if not as_torch:
        arr = np.asarray(x)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        if not arr.flags.writeable or not arr.flags.c_contiguous:
            arr = np.array(arr, copy=True, order="C")   # torch wants a writable buffer
        x = torch.as_tensor(arr, device="cuda")
    elif x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    x = x.contiguous()
    if x.dim() != 3:
        from .core import ShapeError
        raise ShapeError(f"policy must be 3-d (users x items x positions), got ndim={x.dim()}")
    U, n, m = x.shape
    out = torch.empty((U, m - 1), dtype=torch.int32, device=x.device)
    lib = _lib.load()
    fn = lib.nsw_top_positions_f64 if x.dtype == torch.float64 else lib.nsw_top_positions_f32
    stream = torch.cuda.current_stream(x.device).cuda_stream
    check(fn(x.data_ptr(), U, n, m, out.data_ptr(), stream), "top_positions")
    torch.cuda.current_stream(x.device).synchronize()   # this call's stream only (a device-wide wait would break another thread's graph capture)
    return out if as_torch else out.cpu().numpy()
