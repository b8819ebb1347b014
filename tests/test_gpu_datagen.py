"""On-device BASELINE generator (csrc/nsw_datagen.cu) against its numpy port
(oracle/datagen_port.py) on user slices, plus the distribution properties
BASELINE.json states."""

import numpy as np
import pytest

from oracle import datagen_port as port
from paper_2406_10262_b200.datagen import GENERATORS, generate_relevance

pytestmark = pytest.mark.gpu


def _ulp_close(dev, ref):
    """equal up to 1 fp32 ulp (libm log/cos/exp may differ by an ulp before rounding)"""
    tol = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64) * 1.01
    bad = np.abs(dev - ref) > tol
    return bad.sum(), float((dev == ref).mean())


@pytest.mark.parametrize("name,lo,hi", [("cfg1", 0, 6), ("cfg2", 37, 41), ("cfg4", 99990, 99994), ("cfg0", 3, 9)])
def test_latent_slices_match_port(name, lo, hi):
    from paper_2406_10262_b200.data import BASELINE_CONFIGS
    cfg = BASELINE_CONFIGS[name]
    _, d, kind, scale = GENERATORS[name]
    dev = generate_relevance(name, seed=7, user_slice=(lo, hi)).double().cpu().numpy()
    ref = port.latent(lo, hi - lo, cfg.num_items, d, kind, scale, 7, quantize=cfg.dtype != "float64")
    if cfg.dtype == "float64":
        # unrounded float64 output: device libm (log / cos / exp) vs numpy's, ~1 ulp
        rel = float(np.abs(dev / ref - 1).max())
        print(f"{name} users {lo}..{hi}: float64, max rel diff {rel:.1e}")
        assert rel <= 1e-14
        return
    nbad, same = _ulp_close(dev, ref)
    print(f"{name} users {lo}..{hi}: bit-identical {same:.4f}, beyond 1 ulp: {nbad}")
    assert nbad == 0 and same > 0.99


def test_sparse_slice_matches_port():
    dev = generate_relevance("cfg3", seed=3, user_slice=(1000, 1004)).double().cpu().numpy()
    ref = port.sparse(1000, 4, 2000, 50, 1.1, 1e-4, 3)
    nbad, same = _ulp_close(dev, ref)
    print(f"cfg3 users 1000..1004: bit-identical {same:.4f}, beyond 1 ulp: {nbad}")
    assert nbad == 0
    # 50 relevant items per user, every other entry the floor
    assert np.all((dev > np.float32(1e-4) * 1.5).sum(axis=1) == 50)


def test_slices_are_consistent_and_distributions():
    """A slice equals the same rows of a larger slice (counter-based), and the
    drawn values follow BASELINE.json's distributions."""
    a = generate_relevance("cfg2", seed=0, user_slice=(0, 512)).cpu().numpy()
    b = generate_relevance("cfg2", seed=0, user_slice=(100, 200)).cpu().numpy()
    assert np.array_equal(a[100:200], b)
    assert a.min() >= 1e-6 and a.max() <= 1.0
    s = generate_relevance("cfg3", seed=0, user_slice=(0, 2000)).double().cpu().numpy()
    vals = s[s > 2e-4]
    assert vals.size == 2000 * 50
    assert abs(vals.mean() - 2 / 7) < 0.01            # Beta(2, 5) mean
    assert abs(vals.var() - 10 / (49 * 8)) < 0.005    # Beta(2, 5) variance
    # Zipf(1.1) popularity: the most popular item is chosen far more often than the median one
    counts = (s > 2e-4).sum(axis=0)
    assert counts.max() > 20 * max(1, np.median(counts))


def test_cfg4_full_generation_time():
    """Config 4's full 100k x 4000 relevance is generated on the device in well
    under a second (the host numpy path builds 3.2 GB of float64)."""
    import time
    import torch
    generate_relevance("cfg4", seed=0, user_slice=(0, 1024))
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = generate_relevance("cfg4", seed=0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"cfg4 100k x 4000 on device: {dt * 1e3:.1f} ms, {r.numel() * 4 / dt / 1e9:.1f} GB/s written")
    assert r.shape == (100000, 4000) and dt < 2.0
