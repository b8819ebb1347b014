"""Synthetic instances with the BASELINE.json shapes and distributions.

The paper's datasets (Saito & Joachims synthetic, Delicious) are not in this
container; the seeded generators below stand in for them.
One ``numpy.random.default_rng(seed)`` stream per instance; draw order: user
factors P, item factors Q, item bias b, then the sparse draws.  Relevance is
generated in float64 and, for the fp32 configurations, rounded to fp32 once so
that the device and the oracle see identical values.

``exposure_model`` follows the reference's ``log_decay`` semantics
(reference ``data.py:105-122``): e_k = 1/log2(k+1) for the m-1 real positions.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import RELEVANCE_FLOOR, DomainError, ExposureModel, RelevanceMatrix

__all__ = ["BASELINE_CONFIGS", "BaselineConfig", "make_instance", "exposure_model", "latent_relevance",
           "sparse_zipf_relevance"]


def exposure_model(num_positions: int, kind: str = "log_decay", p: float | None = None) -> ExposureModel:
    """Exposure of the m-1 real positions (reference data.py:105-122)."""
    if num_positions < 2:
        raise DomainError("num_positions must be >= 2")
    k = np.arange(1, num_positions, dtype=np.float64)
    if kind == "log_decay":
        vals = 1.0 / np.log2(k + 1.0)
    elif kind == "geometric":
        if p is None or not 0.0 < p <= 1.0:
            raise DomainError("geometric exposure needs p in (0, 1]")
        vals = np.float_power(p, k - 1)
    else:
        raise DomainError(f"unknown exposure kind {kind!r}")
    return ExposureModel(vals)


def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def latent_relevance(U, n, d, seed, bias=None, quantize_fp32=True, user_slice=None):
    """r_ui = sigmoid(<p_u, q_i> + b_i), p_u, q_i ~ N(0, I_d / d).

    ``bias``: None, ("normal", std) or ("lognormal_centered", sigma).
    ``user_slice``: optional (start, stop) — rows of the full instance (the
    full P is drawn so a slice equals the corresponding rows of the full
    matrix)."""
    rng = np.random.default_rng(seed)
    P = rng.standard_normal((U, d)) / np.sqrt(d)
    Q = rng.standard_normal((n, d)) / np.sqrt(d)
    b = np.zeros(n)
    if bias is not None:
        kind, s = bias
        if kind == "normal":
            b = rng.normal(0.0, s, n)
        elif kind == "lognormal_centered":
            L = rng.lognormal(0.0, s, n)
            b = L - L.mean()
        else:
            raise ValueError(kind)
    if user_slice is not None:
        P = P[user_slice[0]:user_slice[1]]
    r = _sigmoid(P @ Q.T + b[None, :])
    np.clip(r, RELEVANCE_FLOOR, 1.0, out=r)
    if quantize_fp32:
        r = r.astype(np.float32).astype(np.float64)
        np.clip(r, RELEVANCE_FLOOR, 1.0, out=r)
    return r


def sparse_zipf_relevance(U, n, per_user, zipf_s, seed, floor_value=1e-4, quantize_fp32=True,
                          user_slice=None):
    """Config 3: each user has ``per_user`` relevant items drawn without
    replacement with P(i) proportional to rank_i^-s (bounded Zipf over n items,
    rank = seeded permutation + 1), r ~ Beta(2, 5); every other entry is
    ``floor_value``; clamped into [RELEVANCE_FLOOR, 1]."""
    rng = np.random.default_rng(seed)
    rank = rng.permutation(n) + 1
    p = rank.astype(np.float64) ** (-zipf_s)
    p /= p.sum()
    lo, hi = (0, U) if user_slice is None else user_slice
    r = np.full((hi - lo, n), floor_value)
    for u in range(U):
        items = rng.choice(n, size=per_user, replace=False, p=p)
        vals = rng.beta(2.0, 5.0, size=per_user)
        if lo <= u < hi:
            r[u - lo, items] = vals
        elif u >= hi:
            break
    np.clip(r, RELEVANCE_FLOOR, 1.0, out=r)
    if quantize_fp32:
        r = r.astype(np.float32).astype(np.float64)
        np.clip(r, RELEVANCE_FLOOR, 1.0, out=r)
    return r


@dataclass(frozen=True)
class BaselineConfig:
    name: str
    num_users: int
    num_items: int
    num_positions: int          # m, including the dummy column
    epsilon: float
    outer_iters: int
    inner_iters: int
    dtype: str                  # arithmetic of the device run
    description: str

    @property
    def cells(self) -> int:
        return self.num_users * self.num_items * self.num_positions


BASELINE_CONFIGS = {
    "cfg0": BaselineConfig("cfg0", 100, 50, 11, 0.1, 200, 50, "float64",
                           "CPU-runnable reference: r=sigmoid(<p,q>), d=8, float64"),
    "cfg1": BaselineConfig("cfg1", 1000, 500, 11, 0.05, 500, 100, "float32",
                           "latent factors d=16 + item bias N(0,0.5), fp32, single GPU"),
    "cfg2": BaselineConfig("cfg2", 10000, 1000, 21, 0.02, 1000, 100, "float32",
                           "latent factors d=32 + centred log-normal bias, fp32, 1/2/4/8 GPUs"),
    "cfg3": BaselineConfig("cfg3", 50000, 2000, 11, 0.05, 500, 50, "float32",
                           "sparse Zipf(1.1) interactions, Beta(2,5), floor 1e-4, fp32"),
    "cfg4": BaselineConfig("cfg4", 100000, 4000, 51, 0.01, 200, 200, "float32",
                           "latent factors d=64 + bias N(0,1), fp32, 8 GPUs"),
}


def make_instance(name: str, seed: int = 0, num_users: int | None = None, user_slice=None):
    """Relevance (float64 ndarray, fp32-representable for fp32 configs) and
    exposure for a BASELINE configuration.

    ``num_users`` overrides |U| (the generator is re-drawn at that size);
    ``user_slice`` takes rows (start, stop) of the full-size instance."""
    cfg = BASELINE_CONFIGS[name]
    U = cfg.num_users if num_users is None else num_users
    n, m = cfg.num_items, cfg.num_positions
    if name == "cfg0":
        r = latent_relevance(U, n, 8, seed, None, quantize_fp32=False, user_slice=user_slice)
    elif name == "cfg1":
        r = latent_relevance(U, n, 16, seed, ("normal", 0.5), user_slice=user_slice)
    elif name == "cfg2":
        r = latent_relevance(U, n, 32, seed, ("lognormal_centered", 1.0), user_slice=user_slice)
    elif name == "cfg3":
        r = sparse_zipf_relevance(U, n, 50, 1.1, seed, user_slice=user_slice)
    elif name == "cfg4":
        r = latent_relevance(U, n, 64, seed, ("normal", 1.0), user_slice=user_slice)
    else:
        raise KeyError(name)
    return r, exposure_model(m).values.copy(), cfg
