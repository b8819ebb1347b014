"""The multi-GPU code path (users sharded over ranks, impact all-gather inside
the captured CUDA graph) on this box's single GPU: a 1-rank NCCL group drives
ShardedAscent, which must reproduce the single-process solver exactly."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_world1_matches_single_process():
    import torch
    import torch.distributed as dist

    from paper_2406_10262_b200 import (DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix, SolverConfig,
                                       solve_fair_ranking)
    from paper_2406_10262_b200.distributed import solve_fair_ranking_distributed

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(8)
        rel = np.clip(rng.uniform(0.05, 1.0, (37, 60)), 1e-6, 1.0)
        expo = 1.0 / np.log2(np.arange(2, 12))
        cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=20, outer_max_iters=12, grad_threshold=1e-300)
        opts = DeviceOptions(dtype="float64", schedule="fixed")
        args = (RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(37, 60, 11), cfg)
        p1, t1 = solve_fair_ranking(*args, opts)
        p2, t2 = solve_fair_ranking_distributed(*args, opts)
        assert len(t2) == len(t1) == 12
        assert np.array_equal(p1.values, p2.values)
        assert t1.objective == t2.objective
    finally:
        dist.destroy_process_group()


def _nccl_world1():
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    return dist


def test_nccl_world1_tolerance_schedule_matches_single_process(golden):
    """Tolerance schedule through the sharded driver (chunk maxima all-reduced
    MAX, converged counts in the impact exchange): same inner-iteration counts
    and bitwise the same policy as the single-process solver, and the same
    SolverError on the reference's desk instance."""
    from paper_2406_10262_b200 import (DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix, SolverConfig,
                                       SolverError, solve_fair_ranking)
    from paper_2406_10262_b200.distributed import solve_fair_ranking_distributed

    dist = _nccl_world1()
    try:
        g = golden("tolerance_eps03")
        rel, expo = g["relevance"], g["exposure"]
        U, n = rel.shape
        cfg = SolverConfig(epsilon=0.3, outer_max_iters=20)
        opts = DeviceOptions(dtype="float64", schedule="tolerance", tol_chunk=7)
        args = (RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, expo.size + 1), cfg)
        p1, t1 = solve_fair_ranking(*args, opts)
        p2, t2 = solve_fair_ranking_distributed(*args, opts)
        assert t2.sinkhorn_iterations == t1.sinkhorn_iterations
        assert len(set(t1.sinkhorn_iterations)) > 1
        assert np.array_equal(p1.values, p2.values)
        assert t1.objective == t2.objective

        d = golden("tolerance_desk")
        rel, expo = d["relevance"], d["exposure"]
        U, n = rel.shape
        args = (RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, expo.size + 1), SolverConfig())
        with pytest.raises(SolverError) as ei:
            solve_fair_ranking_distributed(*args, DeviceOptions(dtype="float64", schedule="tolerance"))
        assert len(ei.value.trace) == int(d["failed_step"])
    finally:
        dist.destroy_process_group()
