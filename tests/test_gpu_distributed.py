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
