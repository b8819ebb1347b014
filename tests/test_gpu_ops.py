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


@pytest.mark.parametrize("B,n,m,T,tol,general,dtype", [
    (3, 120, 40, 12, -1.0, True, np.float64),      # m beyond the compiled tile widths, general marginals
    (40, 90, 64, 30, 1e-3, False, np.float64),     # tolerance stop (lock-step over the batch), ranking marginals
    (2, 3000, 16, 9, -1.0, False, np.float64),     # m has a tile, but 3000 rows do not fit shared memory
    (2, 700, 300, 4, -1.0, True, np.float64),      # more columns than threads
    (3, 150, 53, 10, -1.0, False, np.float32),     # float32
])
def test_streaming_operators_vs_oracle(B, n, m, T, tol, general, dtype):
    """Shapes no shared-memory tile of the operator seam holds run on the
    streaming operators (nsw_ops_generic.cuh): forward, finish and reverse
    mode against the oracle's restatement of sinkhorn.py:204-309."""
    from paper_2406_10262_b200.sinkhorn import sinkhorn_batch_solve
    rng = np.random.default_rng(B * 1000 + m)
    lk = -rng.uniform(0.0, 1.0, (B, n, m)) / 0.2
    if general:
        row = rng.uniform(0.5, 1.5, n)
        col = rng.uniform(0.5, 1.5, m)
        col *= row.sum() / col.sum()
    else:
        row, col, _, _ = orc.ranking_marginals(n, m)
    lvi = rng.normal(0.0, 0.3, (B, m))
    gp = rng.normal(0.0, 1.0, (B, n, m))
    ref = orc.sinkhorn_forward(lk, np.log(row), np.log(col), row, col, tol, T, lvi)
    gref = orc.sinkhorn_backward(lk, np.log(row), np.log(col), ref.hist, lvi, gp, ref.plan, ref.log_u)
    c = lambda a: np.ascontiguousarray(a, dtype=dtype)
    got = sinkhorn_batch_solve(c(lk), None, None, c(row), c(col), tol, T, c(lvi), True)
    ggot = sinkhorn_backward_batch(c(lk), got.log_v_hist, c(lvi), c(gp), got.plan, got.log_u, row=c(row), col=c(col))
    f64 = dtype is np.float64
    assert got.plan.dtype == dtype and got.iterations == ref.iterations
    assert np.array_equal(got.converged, ref.converged) or not f64
    dx = np.abs(got.plan - ref.plan).max()
    dv = np.abs(got.log_v_hist - ref.hist).max()
    dg = np.abs(ggot - gref).max() / np.abs(gref).max()
    print(f"streaming ops {B}x{n}x{m} {dtype.__name__}: |dX|={dx:.1e} |dhist|={dv:.1e} |dgK| rel {dg:.1e} "
          f"iterations {got.iterations}")
    assert dx <= (1e-12 if f64 else 2e-5) and dv <= (1e-10 if f64 else 2e-4) and dg <= (1e-10 if f64 else 2e-3)
    if f64:
        # (a converged residual is rounding noise of the largest mass: 3000 x 2^-52 ~ 7e-13)
        np.testing.assert_allclose(got.residual, ref.residual, rtol=1e-3, atol=1e-14 * max(row.max(), col.max(), 10.0) * 10)


def test_per_user_api_beyond_the_tiles():
    """sinkhorn_solve / sinkhorn_backward (sinkhorn.py:85-173) at m = 45."""
    from paper_2406_10262_b200.core import SolverConfig
    from paper_2406_10262_b200.sinkhorn import Marginals, sinkhorn_backward, sinkhorn_solve
    rng = np.random.default_rng(11)
    n, m = 70, 45
    cost = rng.uniform(0.0, 1.0, (n, m))
    mg = Marginals.for_shape(n, m)
    cfg = SolverConfig(epsilon=0.2, sinkhorn_tol=1e-5, sinkhorn_max_iters=200)
    plan, st = sinkhorn_solve(cost, mg, cfg)
    lk = (-cost / 0.2)[None]
    ref = orc.sinkhorn_forward(lk, np.log(mg.row), np.log(mg.col), mg.row, mg.col, 1e-5, 200, np.zeros((1, m)))
    assert st.iterations_used == ref.iterations and st.converged
    assert np.abs(plan - ref.plan[0]).max() <= 1e-12
    gp = rng.normal(0.0, 1.0, (n, m))
    grad = sinkhorn_backward(st, gp)
    gref = orc.sinkhorn_backward(lk, np.log(mg.row), np.log(mg.col), ref.hist, np.zeros((1, m)), gp[None], ref.plan,
                                 ref.log_u)[0] * (-1.0 / 0.2)
    assert np.abs(grad - gref).max() <= 1e-9 * max(1.0, np.abs(gref).max())
