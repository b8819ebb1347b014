"""On-device generation of the BASELINE synthetic relevance (
8(f) rank 4) through ``nsw_datagen_*`` (csrc/nsw_datagen.cu).

The host generators in ``data.py`` draw configs 3 / 4 in numpy (a per-user
loop for config 3's 50k users, 3.2 GB of float64 for config 4); here every
value is a counter-based function of (seed, stream, index), generated where it
is used, for any user slice -- a rank of a sharded solve generates exactly its
user block.  Same distributions as BASELINE.json (the values differ from the
numpy stream of ``data.make_instance``: a different, equally seeded RNG).
"""

from __future__ import annotations

from . import _lib
from .data import BASELINE_CONFIGS, exposure_model
from .solver import check

__all__ = ["GENERATORS", "generate_relevance", "make_instance_device"]

# config -> ("latent", d, bias_kind, bias_scale) | ("sparse", per_user, zipf_s, floor)
GENERATORS = {
    "cfg0": ("latent", 8, 0, 0.0),
    "cfg1": ("latent", 16, 1, 0.5),
    "cfg2": ("latent", 32, 2, 1.0),
    "cfg3": ("sparse", 50, 1.1, 1e-4),
    "cfg4": ("latent", 64, 1, 1.0),
}


def generate_relevance(name: str, seed: int = 0, user_slice=None, dtype=None, stream=None):
    """Relevance rows [start, stop) of BASELINE configuration ``name`` as a
    CUDA torch tensor (float32 for the fp32 configurations, rounded once;
    float64 for config 0)."""
    import torch
    cfg = BASELINE_CONFIGS[name]
    lo, hi = (0, cfg.num_users) if user_slice is None else (int(user_slice[0]), int(user_slice[1]))
    if not 0 <= lo < hi:
        raise ValueError(f"bad user slice {user_slice!r}")
    dtype = dtype or (torch.float64 if cfg.dtype == "float64" else torch.float32)
    out = torch.empty((hi - lo, cfg.num_items), dtype=dtype, device="cuda")
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    dt = _lib.NSW_F64 if dtype == torch.float64 else _lib.NSW_F32
    lib = _lib.load()
    kind = GENERATORS[name]
    if kind[0] == "latent":
        _, d, bias_kind, bias_scale = kind
        check(lib.nsw_datagen_latent(lo, hi - lo, cfg.num_items, d, bias_kind, bias_scale, seed, dt,
                                     out.data_ptr(), st), "nsw_datagen_latent")
    else:
        _, per_user, zipf_s, floor_value = kind
        check(lib.nsw_datagen_sparse(lo, hi - lo, cfg.num_items, per_user, zipf_s, floor_value, seed, dt,
                                     out.data_ptr(), st), "nsw_datagen_sparse")
    return out


def make_instance_device(name: str, seed: int = 0, user_slice=None):
    """(relevance CUDA tensor, exposure float64 ndarray, BaselineConfig)."""
    cfg = BASELINE_CONFIGS[name]
    return generate_relevance(name, seed, user_slice), exposure_model(cfg.num_positions).values.copy(), cfg
