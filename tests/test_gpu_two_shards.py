"""The world >= 2 path of the sharded ascent on one GPU, without NCCL: two
DeviceSolvers (logical ranks 0 and 1, world = 2), each on its own stream and
user block, bound through nsw_solver_bind_exchange to ONE gathered
[2][n + 1] impact buffer -- each rank's local impact vector IS its slot of the
gathered buffer, which is what the NCCL all-gather produces on 2 GPUs.
finalize then sums the two partials in rank order (the coupling of reference
solver.py:206), so both logical ranks must hold bitwise-identical objective
traces, and the sharded solve must reproduce the unsharded one (the only
difference is the association order of the user sum in Imp)."""

import numpy as np
import pytest

from oracle import nsw_oracle as orc
from paper_2406_10262_b200 import DeviceOptions, DeviceSolver, SolverConfig, solve_fair_ranking
from paper_2406_10262_b200.distributed import shard_users

pytestmark = pytest.mark.gpu


def sharded_solve(rel, expo, cfg, opts, world=2):
    import torch
    U, n = rel.shape
    m = expo.size + 1
    rsq = (rel ** 2).sum(axis=0)
    gathered = torch.zeros(world * (n + 1), dtype=torch.float64, device="cuda")
    solvers = []
    for r in range(world):
        s0, s1 = shard_users(U, world, r)
        s = DeviceSolver(rel[s0:s1], expo, n, m, cfg, opts, rel_sq_sum=rsq, world=world)
        local = gathered[r * (n + 1):(r + 1) * (n + 1)]
        s.bind_exchange(local.data_ptr(), gathered.data_ptr())
        solvers.append(s)
    try:
        for _ in range(cfg.outer_max_iters + 1):
            for s in solvers:
                s.local_step()
            torch.cuda.synchronize()          # the "all-gather" is complete: both slots written
            for s in solvers:
                s.finalize()
            torch.cuda.synchronize()
            if all(s.status()[0] == 3 for s in solvers):
                break
        out = [s.result() for s in solvers]
    finally:
        for s in solvers:
            s.close()
    pol = np.concatenate([p for p, _ in out], axis=0)
    return pol, [t for _, t in out]


@pytest.mark.parametrize("dtype,U,n,m,T,outer", [("float64", 37, 60, 11, 20, 12), ("float32", 300, 500, 11, 15, 6)])
def test_two_logical_ranks_match_unsharded(dtype, U, n, m, T, outer):
    rng = np.random.default_rng(31)
    rel = np.clip(rng.uniform(0.05, 1.0, (U, n)), 1e-6, 1.0).astype(np.float32).astype(np.float64)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300)
    opts = DeviceOptions(dtype=dtype, schedule="fixed")
    pol, traces = sharded_solve(rel, expo, cfg, opts)
    # every logical rank computed F / grad-norm / best from the same two partials
    assert traces[0].objective == traces[1].objective
    assert traces[0].grad_norm == traces[1].grad_norm
    assert len(traces[0]) == outer
    from paper_2406_10262_b200 import ExposureModel, ProblemShape, RelevanceMatrix
    p1, t1 = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m), cfg, opts)
    dx = float(np.abs(pol - p1.values).max())
    df = float(np.abs(np.array(traces[0].objective) / np.array(t1.objective) - 1).max())
    print(f"{dtype} world=2 vs unsharded: |dX|={dx:.2e} rel dF={df:.2e}")
    if dtype == "float64":
        assert dx <= 1e-10 and df <= 1e-13
        p = orc.SolverParams(epsilon=0.1, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300)
        xo, tro, _ = orc.solve(rel, expo, p)
        assert np.abs(pol - xo).max() <= 1e-9
    else:
        # fp32: the association order of Imp's user sum is float64 in both, so
        # the runs stay within fp32 rounding of each other over a short horizon
        assert dx <= 1e-4 and df <= 1e-6


def test_two_logical_ranks_tolerance_schedule():
    """Tolerance schedule with two logical ranks on one buffer pair: the
    chunk residual maxima are combined (MAX) before each decide, the
    converged counts travel in slot n, and both ranks stop together with the
    same inner-iteration counts as the unsharded solve."""
    import torch
    rng = np.random.default_rng(2)
    U, n, m = 24, 30, 6
    rel = np.clip(rng.uniform(0.05, 1.0, (U, n)), 1e-6, 1.0)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    cfg = SolverConfig(epsilon=0.3, sinkhorn_max_iters=200, outer_max_iters=8, grad_threshold=1e-300)
    opts = DeviceOptions(dtype="float64", schedule="tolerance")
    rsq = (rel ** 2).sum(axis=0)
    world = 2
    gathered = torch.zeros(world * (n + 1), dtype=torch.float64, device="cuda")
    cmax = [torch.zeros(opts.tol_chunk, dtype=torch.float64, device="cuda") for _ in range(world)]
    solvers = []
    for r in range(world):
        s0, s1 = shard_users(U, world, r)
        s = DeviceSolver(rel[s0:s1], expo, n, m, cfg, opts, rel_sq_sum=rsq, world=world)
        s.bind_exchange(gathered[r * (n + 1):(r + 1) * (n + 1)].data_ptr(), gathered.data_ptr())
        s.set_scalar("users_total", U)
        s.bind_tol_exchange(cmax[r].data_ptr())
        solvers.append(s)
    try:
        for _ in range(cfg.outer_max_iters + 1):
            for s in solvers:
                s.local_step()
            while True:
                for s in solvers:
                    s.tol_local()
                torch.cuda.synchronize()
                mx = torch.maximum(cmax[0], cmax[1])      # the all-reduce MAX
                for c in cmax:
                    c.copy_(mx)
                torch.cuda.synchronize()
                phases = [s.tol_decide() for s in solvers]
                assert phases[0] == phases[1]
                if phases[0] == 5:
                    for s in solvers:
                        s.local_step()
                    continue
                if phases[0] == 6:
                    for s in solvers:
                        s.local_step()
                break
            torch.cuda.synchronize()
            for s in solvers:
                s.finalize()
            torch.cuda.synchronize()
            if all(s.status()[0] == 3 for s in solvers):
                break
        out = [s.result() for s in solvers]
    finally:
        for s in solvers:
            s.close()
    from paper_2406_10262_b200 import ExposureModel, ProblemShape, RelevanceMatrix
    p1, t1 = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m), cfg, opts)
    pol = np.concatenate([p for p, _ in out], axis=0)
    assert out[0][1].sinkhorn_iterations == out[1][1].sinkhorn_iterations == t1.sinkhorn_iterations
    assert out[0][1].objective == out[1][1].objective
    assert np.abs(pol - p1.values).max() <= 1e-10
