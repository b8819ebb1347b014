"""The streaming fused step (nsw_step_generic.cuh): every shape the reference
accepts that no on-chip tile holds -- float64 at config 4's 4000 x 51, m > 52,
n > 8192 -- against the float64 oracle (reference sinkhorn.py:204-309,
solver.py:138-241), in both schedules."""

import numpy as np
import pytest

from oracle import nsw_oracle as orc
from paper_2406_10262_b200 import (DeviceOptions, DeviceSolver, ExposureModel, ProblemShape, RelevanceMatrix,
                                   SolverConfig, SolverError, solve_fair_ranking)

pytestmark = pytest.mark.gpu

GEN64 = DeviceOptions(dtype="float64", schedule="fixed", variant=-3)


def _solve(rel, expo, eps, T, outer, opts, **kw):
    U, n = rel.shape
    m = expo.size + 1
    cfg = SolverConfig(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer,
                       grad_threshold=kw.pop("grad_threshold", 1e-300), **kw)
    pol, tr = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m), cfg, opts)
    return pol.values, tr


@pytest.mark.parametrize("U,n,m,T,outer,eps,warm", [
    (3, 7, 4, 9, 6, 0.1, True),       # ragged tiny
    (5, 37, 5, 13, 8, 0.2, False),    # warm start off
    (4, 9, 9, 5, 5, 0.1, True),       # m == n (dummy mass 1)
    (6, 12, 2, 7, 5, 0.3, True),      # m == 2
    (4, 20, 6, 1, 4, 0.1, True),      # one inner iteration
    (2, 30, 6, 10, 1, 0.1, True),     # one outer step: no backward
    (3, 300, 80, 12, 4, 0.1, True),   # m > 52 (no tile)
    (2, 70, 40, 8, 3, 0.1, True),     # m > 32 fp64
])
def test_streaming_fp64_vs_oracle(U, n, m, T, outer, eps, warm):
    rng = np.random.default_rng(U * 1000 + n + m)
    rel = np.clip(rng.uniform(0.0, 1.0, (U, n)), 1e-6, 1.0)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    p = orc.SolverParams(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300,
                         warm_start=warm)
    xo, tro, _ = orc.solve(rel, expo, p)
    xd, trd = _solve(rel, expo, eps, T, outer, GEN64, warm_start=warm)
    dx = np.abs(xd - xo).max()
    df = np.abs(np.array(trd.objective) / np.array(tro.objective) - 1).max()
    print(f"streaming fp64 U={U} n={n} m={m}: |dX|={dx:.2e} rel dF={df:.2e}")
    assert len(trd) == len(tro)
    assert dx <= 1e-9 and df <= 1e-12


def test_streaming_is_the_default_for_cfg4_float64():
    """Config 4's own shape (4000 x 51, eps 0.01, 200 inner iterations) in the
    default float64 drop-in: no float64 tile holds 4000 items, the streaming
    step runs it; 2 users x 3 outer steps against the oracle."""
    from paper_2406_10262_b200.data import make_instance
    rel, expo, cfg = make_instance("cfg4", seed=0, user_slice=(0, 2))
    U, n = rel.shape
    m = expo.size + 1
    scfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=200, outer_max_iters=3, grad_threshold=1e-300)
    with DeviceSolver(rel, expo, n, m, scfg, DeviceOptions(dtype="float64", schedule="fixed")) as s:
        assert s.variant().get("generic") is True
    p = orc.SolverParams(epsilon=cfg.epsilon, sinkhorn_max_iters=200, outer_max_iters=3, grad_threshold=1e-300)
    xo, tro, _ = orc.solve(rel, expo, p)
    xd, trd = _solve(rel, expo, cfg.epsilon, 200, 3, DeviceOptions(dtype="float64", schedule="fixed"))
    dx = np.abs(xd - xo).max()
    df = np.abs(np.array(trd.objective) / np.array(tro.objective) - 1).max()
    print(f"cfg4 float64 streaming: |dX|={dx:.2e} rel dF={df:.2e}")
    # eps = 0.01 (|K| ~ 1e2): float64 summation-order differences reach
    # ~1e-10 (the bars are 1e-5 on X and 1e-6 relative on F)
    assert dx <= 1e-9 and df <= 1e-9


def test_streaming_large_n_fp32():
    """n > 8192 (beyond the 16-CTA cluster tile) in float32, a few steps vs
    the float64 oracle."""
    rng = np.random.default_rng(9)
    U, n, m, T, outer, eps = 2, 9000, 11, 10, 3, 0.1
    rel = np.clip(rng.uniform(0.0, 1.0, (U, n)), 1e-6, 1.0).astype(np.float32).astype(np.float64)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    p = orc.SolverParams(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300)
    xo, tro, _ = orc.solve(rel, expo, p)
    xd, trd = _solve(rel, expo, eps, T, outer, DeviceOptions(dtype="float32", schedule="fixed"))
    dx = np.abs(xd - xo).max()
    df = np.abs(np.array(trd.objective) / np.array(tro.objective) - 1).max()
    print(f"streaming fp32 n={n}: |dX|={dx:.2e} rel dF={df:.2e}")
    assert dx <= 2e-4 and df <= 2e-6


def test_streaming_fp32_one_step():
    """fp32 one-step parity of the streaming step from a mid-trajectory
    oracle state, m > 52."""
    rng = np.random.default_rng(12)
    U, n, m, T = 3, 200, 64, 20
    rel = np.clip(rng.uniform(0.0, 1.0, (U, n)), 1e-6, 1.0).astype(np.float32).astype(np.float64)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    p = orc.SolverParams(epsilon=0.1, sinkhorn_max_iters=T, outer_max_iters=5, grad_threshold=1e-300)
    _, _, states = orc.solve(rel, expo, p, record_states={3})
    st = states[3]
    ref = orc.one_step(rel, expo, st, p)
    cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=T, outer_max_iters=8, grad_threshold=1e-300)
    with DeviceSolver(rel, expo, n, m, cfg, DeviceOptions(dtype="float32", schedule="fixed")) as s:
        assert s.variant().get("generic") is True
        s.set("cost", st["cost"])
        s.set("adam_m", st["m"])
        s.set("adam_v", st["v"])
        s.set("lvi", st["lvi"])
        s.set_scalar("step", 3)
        s.set_scalar("phase", 4)
        s.run(2)
        dx = np.abs(s.get("xbest") - ref["plan"]).max()
        dc = np.abs(s.get("cost") - ref["cost"]).max()
    print(f"streaming fp32 one-step: |dX|={dx:.2e} |dC|={dc:.2e}")
    assert dx <= 2e-6 and dc <= 5e-6


def test_streaming_tolerance_schedule_matches_reference(golden):
    """The reference's default tolerance schedule on the streaming step: the
    SPEC desk instance raises SolverError at the same outer step with the same
    inner-iteration counts as the reference (golden), like the tiled path."""
    g = golden("tolerance_desk")
    rel, expo = g["relevance"], g["exposure"]
    cfg = SolverConfig()
    s = DeviceSolver(rel, expo, rel.shape[1], expo.size + 1, cfg, DeviceOptions(dtype="float64", variant=-3))
    assert s.variant().get("generic") is True
    s.run(cfg.outer_max_iters + 1)
    with pytest.raises(SolverError) as ei:
        s.result()
    s.close()
    ref_its = [int(x) for x in g["sinkhorn_iterations"]]
    dev_its = ei.value.trace.sinkhorn_iterations
    assert len(dev_its) == int(g["failed_step"])
    assert dev_its == ref_its[: len(dev_its)]


def test_streaming_tolerance_eps03_golden(golden):
    g = golden("tolerance_eps03")
    rel, expo = g["relevance"], g["exposure"]
    U, n = rel.shape
    pol, tr = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, expo.size + 1),
                                 SolverConfig(epsilon=0.3, outer_max_iters=20), DeviceOptions(variant=-3))
    assert tr.sinkhorn_iterations == list(g["sinkhorn_iterations"])
    assert np.abs(pol.values - g["policy"]).max() <= 1e-9


# ---------------------------------------------------------------------------
# in-solve re-absorption (DeviceOptions.reabsorb): events forced with a tiny
# threshold so every 8th inner iteration folds the scalings into K~; the
# results must not move (it is a change of coordinates, forward and backward)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("U,n,m,T,outer,eps,warm", [
    (3, 37, 5, 40, 5, 0.1, False),
    (4, 60, 11, 33, 4, 0.05, True),
    (2, 90, 70, 26, 3, 0.2, False),
])
def test_reabsorption_is_a_change_of_coordinates_fp64(U, n, m, T, outer, eps, warm):
    rng = np.random.default_rng(U + n + m)
    rel = np.clip(rng.uniform(0.0, 1.0, (U, n)), 1e-6, 1.0)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    p = orc.SolverParams(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300,
                         warm_start=warm)
    xo, tro, _ = orc.solve(rel, expo, p)
    xd, trd = _solve(rel, expo, eps, T, outer, DeviceOptions(dtype="float64", schedule="fixed", reabsorb=1e-3),
                     warm_start=warm)
    dx = np.abs(xd - xo).max()
    df = np.abs(np.array(trd.objective) / np.array(tro.objective) - 1).max()
    print(f"re-absorbing fp64 U={U} n={n} m={m} T={T} warm={warm}: |dX|={dx:.2e} rel dF={df:.2e}")
    assert dx <= 1e-9 and df <= 1e-11


def test_reabsorption_fp32_cold_start_tracks_tiles():
    """Config-2 slice, cold start (warm_start=False), eps 0.02, float32: with
    events at 3 nats the streaming re-absorbing solve tracks the tiled float32
    solve within float32's own sensitivity at this eps (one outer step
    already amplifies rounding differences into ~1e-2 of X).

    What re-absorption cannot do: at eps = 0.01 a cold start absorbs at
    beta = 0, where whole columns of K~ = exp(K + alpha) already underflow
    float32 before the first iteration -- no change of coordinates recovers
    them (test_gpu_small_eps.py::test_cold_start_small_eps_fp32_fails_loudly:
    float32 raises, float64 runs)."""
    from paper_2406_10262_b200.data import make_instance
    rel, expo, cfg = make_instance("cfg2", seed=0, user_slice=(0, 64))
    U, n = rel.shape
    m = expo.size + 1
    # 3 outer steps: over tens of steps any two fp32 arithmetics drift apart
    # (SURVEY finding 4), so the comparison is short-horizon
    scfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=cfg.inner_iters, outer_max_iters=3,
                        grad_threshold=1e-300, warm_start=False)
    args = (RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m), scfg)
    pr, tr = solve_fair_ranking(*args, DeviceOptions(dtype="float32", schedule="fixed", reabsorb=3.0))
    pt, tt = solve_fair_ranking(*args, DeviceOptions(dtype="float32", schedule="fixed"))
    df = np.abs(np.array(tr.objective) / np.array(tt.objective) - 1).max()
    dx = np.abs(pr.values - pt.values).max()
    print(f"cfg2 cold start fp32, re-absorbing streaming vs tile: rel dF {df:.2e}, |dX| {dx:.2e}")
    assert np.isfinite(pr.values).all()
    assert df <= 2e-5 and dx <= 1e-2


def test_reabsorption_fp32_one_step():
    """fp32 one-step parity with events forced in the forward and crossed in the backward."""
    rng = np.random.default_rng(41)
    U, n, m, T = 3, 80, 9, 40
    rel = np.clip(rng.uniform(0.0, 1.0, (U, n)), 1e-6, 1.0).astype(np.float32).astype(np.float64)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    p = orc.SolverParams(epsilon=0.1, sinkhorn_max_iters=T, outer_max_iters=5, grad_threshold=1e-300)
    _, _, states = orc.solve(rel, expo, p, record_states={3})
    st = states[3]
    ref = orc.one_step(rel, expo, st, p)
    cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=T, outer_max_iters=8, grad_threshold=1e-300)
    with DeviceSolver(rel, expo, n, m, cfg, DeviceOptions(dtype="float32", schedule="fixed", reabsorb=1e-3)) as s:
        s.set("cost", st["cost"])
        s.set("adam_m", st["m"])
        s.set("adam_v", st["v"])
        s.set("lvi", st["lvi"])
        s.set_scalar("step", 3)
        s.set_scalar("phase", 4)
        s.run(2)
        dx = np.abs(s.get("xbest") - ref["plan"]).max()
        dc = np.abs(s.get("cost") - ref["cost"]).max()
    print(f"re-absorbing fp32 one-step: |dX|={dx:.2e} |dC|={dc:.2e}")
    assert dx <= 2e-6 and dc <= 5e-6


def test_reabsorption_needs_fixed_schedule():
    rng = np.random.default_rng(1)
    rel = np.clip(rng.uniform(0.0, 1.0, (2, 10)), 1e-6, 1.0)
    expo = 1.0 / np.log2(np.arange(2, 5))
    with pytest.raises(NotImplementedError):
        _solve(rel, expo, 0.1, 10, 2, DeviceOptions(dtype="float64", schedule="tolerance", reabsorb=30.0))
