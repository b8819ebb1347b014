"""Per-user Sinkhorn API and the full _sinkhorn_batch contract on the device
(SURVEY 8(f) rank 4): general marginals, the tolerance stop, the reverse mode
and the Theorem-1 map, against values the real reference produced
(tests/golden/api_small.npz, oracle/gen_golden.py case_api)."""

import numpy as np
import pytest

from paper_2406_10262_b200.core import DomainError, SolverConfig, StateError
from paper_2406_10262_b200.sinkhorn import (Marginals, cost_from_policy, sinkhorn_backward, sinkhorn_batch_solve,
                                            sinkhorn_solve)

pytestmark = pytest.mark.gpu


def test_sinkhorn_solve_general_marginals_tolerance(golden):
    g = golden("api_small")
    cfg = SolverConfig(epsilon=float(g["eps"]), sinkhorn_tol=float(g["tol"]), sinkhorn_max_iters=int(g["max_iters"]))
    plan, st = sinkhorn_solve(g["cost"], Marginals(g["row"], g["col"]), cfg)
    print("iterations", st.iterations_used, int(g["iterations"]), "residual", st.final_residual, float(g["residual"]))
    assert st.iterations_used == int(g["iterations"])
    assert st.converged == bool(g["converged"])
    assert np.abs(plan - g["plan"]).max() <= 1e-12
    assert np.abs(st.log_u - g["log_u"]).max() <= 1e-10
    assert np.abs(st.log_v - g["log_v"]).max() <= 1e-10
    assert st.final_residual == pytest.approx(float(g["residual"]), rel=1e-3, abs=1e-13)
    grad = sinkhorn_backward(st, g["grad_plan"])
    assert np.abs(grad - g["grad_cost"]).max() <= 1e-9 * max(1.0, np.abs(g["grad_cost"]).max())


def test_sinkhorn_backward_needs_iterates(golden):
    g = golden("api_small")
    cfg = SolverConfig(epsilon=float(g["eps"]), sinkhorn_tol=float(g["tol"]), sinkhorn_max_iters=50)
    _, st = sinkhorn_solve(g["cost"], Marginals(g["row"], g["col"]), cfg, record_iterates=False)
    with pytest.raises(StateError):
        sinkhorn_backward(st, g["grad_plan"])


def test_batch_lock_step_tolerance(golden):
    g = golden("api_small")
    lk, lv = g["b_log_kernel"], g["b_lvi"]
    B, n, m = lk.shape
    mg = Marginals.for_shape(n, m)
    res = sinkhorn_batch_solve(lk, np.log(mg.row), np.log(mg.col), mg.row, mg.col, 1e-6, 300, lv, True)
    assert res.iterations == int(g["b_iterations"])
    assert np.array_equal(res.converged, g["b_converged"])
    assert res.log_v_hist.shape == g["b_hist"].shape
    assert np.abs(res.plan - g["b_plan"]).max() <= 1e-12
    assert np.abs(res.log_v_hist - g["b_hist"]).max() <= 1e-10
    assert np.abs(res.log_u - g["b_log_u"]).max() <= 1e-10
    np.testing.assert_allclose(res.residual, g["b_residual"], rtol=1e-3, atol=1e-13)
    # float32 runs the same contract (tolerance is approximate at fp32 resolution)
    r32 = sinkhorn_batch_solve(lk.astype(np.float32), None, None, mg.row.astype(np.float32),
                               mg.col.astype(np.float32), -1.0, 40, lv.astype(np.float32))
    assert r32.iterations == 40 and np.isfinite(r32.plan).all()


def test_cost_from_policy_theorem1_map(golden):
    g = golden("api_small")
    got = cost_from_policy(g["policy"], 0.3)
    np.testing.assert_allclose(got, g["policy_cost"], rtol=1e-15, atol=1e-15)
    bad = g["policy"].copy()
    bad[0, 0, 0] = 0.0
    with pytest.raises(DomainError):
        cost_from_policy(bad, 0.3)
    with pytest.raises(DomainError):
        cost_from_policy(g["policy"], 0.0)


def test_ascent_building_blocks_match_oracle(golden):
    """impact / nsw_objective / nsw_gradient_wrt_policy / adam_update on the
    device vs the oracle (pinned bit-exact to the reference)."""
    from oracle import nsw_oracle as orc
    from paper_2406_10262_b200 import (AdamState, SolverConfig, adam_update, impact, nsw_gradient_wrt_policy,
                                       nsw_objective)
    g = golden("cfg0_fixed")
    rel, expo, x = g["relevance"], g["exposure"], g["policy"]
    imp_d = impact(x, rel, expo)
    imp_o = orc.impact(rel, expo, x)
    assert np.abs(imp_d / imp_o - 1).max() <= 1e-13
    assert nsw_objective(imp_d) == pytest.approx(float(np.log(imp_o).sum()), rel=1e-14)
    gd = nsw_gradient_wrt_policy(x, rel, expo)
    go = np.zeros_like(x)
    orc.welfare_gradient(rel, expo, imp_d, go)   # same impacts: the division is elementwise-exact
    assert np.array_equal(gd, go)
    cfg = SolverConfig()
    rng = np.random.default_rng(4)
    p0, g0 = rng.normal(size=(5, 7, 3)), rng.normal(size=(5, 7, 3))
    st = AdamState.zeros(p0.shape)
    p1, st1 = adam_update(p0, g0, st, cfg)
    p2, st2 = adam_update(p1, g0 * 0.5, st1, cfg)
    q1, m1, v1, s1 = orc.adam_ascent(p0, g0, np.zeros_like(p0), np.zeros_like(p0), 0, cfg.adam_lr, cfg.adam_beta1,
                                     cfg.adam_beta2, cfg.adam_eps)
    q2, m2, v2, s2 = orc.adam_ascent(q1, g0 * 0.5, m1, v1, s1, cfg.adam_lr, cfg.adam_beta1, cfg.adam_beta2,
                                     cfg.adam_eps)
    assert st2.step == s2 == 2
    assert np.array_equal(p2, q2) and np.array_equal(st2.m, m2) and np.array_equal(st2.v, v2)


def test_step_level_state_setters_validate():
    """nsw_solver_set_scalar: the step indexes the device's per-step trace and
    bias-correction arrays, so an out-of-range value is rejected (it used to be
    written through, and the next finalize wrote past the trace)."""
    from paper_2406_10262_b200 import DeviceOptions, DeviceSolver
    rng = np.random.default_rng(0)
    rel = np.clip(rng.uniform(0, 1, (5, 30)), 1e-4, 1)
    expo = 1.0 / np.log2(np.arange(2, 7))
    cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=5, outer_max_iters=3, grad_threshold=1e-300)
    with DeviceSolver(rel, expo, 30, 6, cfg, DeviceOptions(dtype="float64", schedule="fixed")) as s:
        for name, value in (("step", 3), ("step", -1), ("step", 99), ("phase", 7), ("phase", -1), ("improved", 2)):
            with pytest.raises(DomainError):
                s.set_scalar(name, value)
        with pytest.raises(ValueError):
            s.set_scalar("nope", 1)
        s.set_scalar("step", 2)      # in range
        s.set_scalar("step", 0)
        s.run(4)
        pol, tr = s.result()
        assert len(tr) == 3 and np.isfinite(pol).all()
