"""Device evaluation metrics against the reference's own
values (tests/golden/metrics.npz, produced by oracle/gen_golden.py from
nswrank.metrics and pinned bit-exact to oracle.policy_metrics)."""

import numpy as np
import pytest

from oracle import nsw_oracle as orc
from paper_2406_10262_b200 import (items_better_off, items_worse_off, mean_max_envy, policy_metrics,
                                   user_utility)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag", ["cfg0", "cfg1s"])
def test_metrics_match_reference(golden, tag):
    g = golden("metrics")
    r, e, x, ref = g[f"{tag}_relevance"], g[f"{tag}_exposure"], g[f"{tag}_policy"], g[f"{tag}_metrics"]
    got = policy_metrics(x, r, e)
    got2 = policy_metrics(x, r, e, threshold=0.02)
    print(tag, got, ref)
    assert got["user_utility"] == pytest.approx(ref[0], rel=1e-13)
    assert got["mean_max_envy"] == pytest.approx(ref[1], rel=1e-11, abs=1e-13)
    assert got["items_better_off"] == ref[2] and got["items_worse_off"] == ref[3]
    assert got2["items_better_off"] == ref[4] and got2["items_worse_off"] == ref[5]
    # the reference-named entry points
    assert user_utility(x, r, e) == got["user_utility"]
    assert mean_max_envy(x, r, e) == got["mean_max_envy"]
    assert items_better_off(x, r, e, 0.02) == ref[4] and items_worse_off(x, r, e, 0.02) == ref[5]


def test_metrics_float32_policy_and_torch_inputs():
    import torch
    rng = np.random.default_rng(9)
    U, n, m = 37, 90, 8
    r = rng.random((U, n)).astype(np.float32)
    e = 1.0 / np.log2(np.arange(2, m + 1))
    x = rng.random((U, n, m)).astype(np.float32)
    ref = orc.policy_metrics(x.astype(np.float64), r.astype(np.float64), e, 0.05)
    got = policy_metrics(torch.as_tensor(x, device="cuda"), torch.as_tensor(r, device="cuda"), e, 0.05)
    assert got["user_utility"] == pytest.approx(ref[0], rel=1e-12)
    assert got["mean_max_envy"] == pytest.approx(ref[1], rel=1e-10)
    assert got["items_better_off"] == ref[2] and got["items_worse_off"] == ref[3]


def test_solver_metrics_on_device_policy(golden):
    """DeviceSolver.metrics() evaluates the best policy in place; equals the
    metrics of the downloaded policy."""
    from paper_2406_10262_b200 import DeviceOptions, DeviceSolver, SolverConfig
    g = golden("cfg0_fixed")
    rel, expo = g["relevance"], g["exposure"]
    cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=20, outer_max_iters=15, grad_threshold=1e-300)
    with DeviceSolver(rel, expo, rel.shape[1], expo.size + 1, cfg, DeviceOptions(dtype="float64",
                                                                                  schedule="fixed")) as s:
        s.run(16)
        pol, _ = s.result()
        m = s.metrics(0.1)
    ref = orc.policy_metrics(pol, rel, expo, 0.1)
    assert m["user_utility"] == pytest.approx(ref[0], rel=1e-13)
    assert m["mean_max_envy"] == pytest.approx(ref[1], rel=1e-11, abs=1e-13)
    assert (m["items_better_off"], m["items_worse_off"]) == (ref[2], ref[3])
