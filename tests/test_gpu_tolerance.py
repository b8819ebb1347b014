"""The reference's default stopping rule on the device (schedule="tolerance").

sinkhorn.py:237-246: after every inner iteration the L-inf marginal residual
of every user's reconstructed plan is measured and all users stop together
once the largest is <= sinkhorn_tol; solver.py:200-205 raises SolverError when
more than half of the users miss the tolerance.  Pinned against fixtures the
real reference produced (oracle/gen_golden.py: tolerance_desk, tolerance_eps03).
"""

import numpy as np
import pytest

from paper_2406_10262_b200 import (DeviceOptions, DeviceSolver, ExposureModel, ProblemShape, RelevanceMatrix,
                                   SolverConfig, SolverError, solve_fair_ranking)

pytestmark = pytest.mark.gpu

TOL64 = DeviceOptions(dtype="float64", schedule="tolerance")


def test_reference_default_config_raises_at_the_same_step(golden):
    """Default SolverConfig on the SPEC desk instance (100 x 50 x 11): the
    reference raises SolverError on outer step 30 with the inner-iteration
    counts of the fixture; the device must do the same."""
    g = golden("tolerance_desk")
    rel, expo = g["relevance"], g["exposure"]
    cfg = SolverConfig()
    s = DeviceSolver(rel, expo, rel.shape[1], expo.size + 1, cfg, TOL64)
    s.run(cfg.outer_max_iters + 1)
    with pytest.raises(SolverError) as ei:
        s.result()
    s.close()
    ref_its = [int(x) for x in g["sinkhorn_iterations"]]
    dev_its = ei.value.trace.sinkhorn_iterations
    print("device inner iterations", dev_its[:12], "... reference", ref_its[:12])
    assert len(dev_its) == int(g["failed_step"])
    assert dev_its == ref_its[: len(dev_its)]
    assert "failed to converge" in str(ei.value)
    # the public entry point raises the same class
    with pytest.raises(SolverError):
        solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(100, 50, 11), cfg, TOL64)


def test_tolerance_mode_eps03_matches_reference(golden):
    g = golden("tolerance_eps03")
    rel, expo = g["relevance"], g["exposure"]
    cfg = SolverConfig(epsilon=0.3, outer_max_iters=20)
    pol, tr = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(100, 50, 11), cfg, TOL64)
    dx = np.abs(pol.values - g["policy"]).max()
    df = np.abs(np.array(tr.objective) / g["objective"] - 1).max()
    print(f"tolerance eps=0.3: |dX|={dx:.3e} rel dF={df:.3e} iterations {tr.sinkhorn_iterations}")
    assert tr.sinkhorn_iterations == [int(x) for x in g["sinkhorn_iterations"]]
    assert dx <= 1e-9 and df <= 1e-12


@pytest.mark.parametrize("chunk", [1, 7, 64])
def test_tolerance_chunking_is_invisible(golden, chunk):
    """The forward is launched in chunks of `tol_chunk` iterations; the result
    must not depend on the chunk size."""
    g = golden("tolerance_eps03")
    rel, expo = g["relevance"][:40], g["exposure"]
    cfg = SolverConfig(epsilon=0.3, outer_max_iters=8)
    ref = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(40, 50, 11), cfg,
                             DeviceOptions(dtype="float64", schedule="tolerance", tol_chunk=16))
    out = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(40, 50, 11), cfg,
                             DeviceOptions(dtype="float64", schedule="tolerance", tol_chunk=chunk))
    assert out[1].sinkhorn_iterations == ref[1].sinkhorn_iterations
    assert np.array_equal(out[0].values, ref[0].values)


def test_tolerance_mode_fp32_runs():
    g = np.random.default_rng(3)
    rel = np.clip(g.uniform(0.05, 1.0, (64, 80)), 1e-6, 1.0).astype(np.float32).astype(np.float64)
    expo = 1.0 / np.log2(np.arange(2, 12))
    cfg = SolverConfig(epsilon=0.3, outer_max_iters=10, sinkhorn_tol=1e-5)
    p32, t32 = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(64, 80, 11), cfg,
                                  DeviceOptions(dtype="float32", schedule="tolerance"))
    p64, t64 = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(64, 80, 11), cfg, TOL64)
    assert len(t32) == len(t64)
    assert max(abs(a - b) for a, b in zip(t32.sinkhorn_iterations, t64.sinkhorn_iterations)) <= 2
    assert np.abs(np.array(t32.objective) / np.array(t64.objective) - 1).max() < 1e-5


@pytest.mark.parametrize("dtype,tol,chunk", [("float64", 1e-2, 0), ("float64", 1e-6, 4), ("float32", 1e-2, 0)])
def test_tolerance_schedule_with_a_wave_tail(dtype, tol, chunk):
    """More users than one wave, so the fused step is a main launch plus a
    tail launch on the side stream: the tolerance schedule's per-step graph
    (a while-node whose body re-launches the fused step) must capture both --
    the side stream cannot join the body's capture, which used to crash the
    default drop-in call (found by scripts/fuzz_parity.py)."""
    from oracle import nsw_oracle as orc
    U, n, m, T, outer, eps = 310, 436, 21, 21, 5, 0.2
    rng = np.random.default_rng(40)
    rel = np.clip(rng.uniform(0.0, 1.0, (U, n)), 1e-4, 1.0).astype(np.float32).astype(np.float64)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    p = orc.SolverParams(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300,
                         warm_start=False, sinkhorn_tol=tol, fixed_schedule=False)
    xo, tro, _ = orc.solve(rel, expo, p)
    cfg = SolverConfig(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300,
                       warm_start=False, sinkhorn_tol=tol)
    opts = DeviceOptions(dtype=dtype, schedule="tolerance", **({"tol_chunk": chunk} if chunk else {}))
    with DeviceSolver(rel, expo, n, m, cfg, opts) as s:
        assert s.variant().get("tail_users", 0) > 0, s.variant()
    pol, tr = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m), cfg, opts)
    dx = np.abs(pol.values - xo).max()
    df = np.abs(np.array(tr.objective) / np.array(tro.objective) - 1).max()
    print(f"tolerance + tail {dtype} tol={tol}: |dX|={dx:.3e} rel dF={df:.3e} iterations {tr.sinkhorn_iterations}")
    assert tr.sinkhorn_iterations == tro.sinkhorn_iterations
    assert (dx <= 1e-9 and df <= 1e-12) if dtype == "float64" else (dx <= 1e-4 and df <= 1e-5)
