"""The operator seam (nsw_sinkhorn_batch_* / nsw_sinkhorn_backward_batch_*)
against the reference's own _sinkhorn_batch / _sinkhorn_backward_batch outputs
(tests/golden/ops_small.npz, produced by oracle/gen_golden.py)."""

import numpy as np
import pytest

from oracle import nsw_oracle as orc
from paper_2406_10262_b200.sinkhorn import sinkhorn_backward_batch, sinkhorn_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_forward_op_vs_reference(golden, tag):
    g = golden("ops_small")
    B, n, m, T = (int(v) for v in g[f"{tag}_shape"])
    plan, lu, lv, hist = sinkhorn_batch(g[f"{tag}_log_kernel"], g[f"{tag}_log_v_init"], T)
    assert np.abs(plan - g[f"{tag}_plan"]).max() < 1e-12
    assert np.abs(lu - g[f"{tag}_log_u"]).max() < 1e-11
    assert np.abs(lv - g[f"{tag}_log_v"]).max() < 1e-11
    assert np.abs(hist - g[f"{tag}_hist"]).max() < 1e-11


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_backward_op_vs_reference(golden, tag):
    g = golden("ops_small")
    gk = sinkhorn_backward_batch(g[f"{tag}_log_kernel"], g[f"{tag}_hist"], g[f"{tag}_log_v_init"],
                                 g[f"{tag}_grad_plan"], g[f"{tag}_plan"], g[f"{tag}_log_u"])
    ref = g[f"{tag}_grad_log_kernel"]
    assert np.abs(gk - ref).max() / np.abs(ref).max() < 1e-11


def test_ops_fp32_and_zero_upstream():
    rng = np.random.default_rng(4)
    B, n, m, T = 5, 40, 11, 30
    K = rng.uniform(-3, 3, (B, n, m))
    lvi = rng.uniform(-1, 1, (B, m))
    row, col, lr, lc = orc.ranking_marginals(n, m)
    fo = orc.sinkhorn_forward(K, lr, lc, row, col, -1.0, T, lvi)
    plan, lu, lv, hist = sinkhorn_batch(K.astype(np.float32), lvi.astype(np.float32), T)
    assert plan.dtype == np.float32
    assert np.abs(plan - fo.plan).max() < 1e-5
    gk = sinkhorn_backward_batch(K, fo.hist, lvi, np.zeros_like(K), fo.plan, fo.log_u)
    assert np.all(gk == 0)
