"""Device top-m ranking extraction (north star: "final top-m ranking per user
bit-exact").  The rule is the oracle's ``top_positions`` (argmax over items
per real position, lowest index on ties), checked against the reference's
golden ranking in float64 and against numpy on the same values in float32."""

import numpy as np
import pytest

from oracle import nsw_oracle as orc
from paper_2406_10262_b200 import (DeviceOptions, DeviceSolver, ExposureModel, ProblemShape, RelevanceMatrix,
                                   SolverConfig, top_positions)

pytestmark = pytest.mark.gpu


def test_cfg0_fp64_device_ranking_matches_reference(golden):
    g = golden("cfg0_fixed")
    rel, expo = g["relevance"], g["exposure"]
    U, n = rel.shape
    m = expo.size + 1
    cfg = SolverConfig(epsilon=float(g["epsilon"]), sinkhorn_max_iters=int(g["inner"]),
                       outer_max_iters=int(g["outer"]), grad_threshold=1e-300)
    with DeviceSolver(rel, expo, n, m, cfg, DeviceOptions(dtype="float64", schedule="fixed")) as s:
        assert s.run(cfg.outer_max_iters + 1)
        pol, _ = s.result()
        rank = s.top_positions()
    assert rank.dtype == np.int32 and rank.shape == (U, m - 1)
    assert np.array_equal(rank, g["top_positions"])
    assert np.array_equal(top_positions(pol), g["top_positions"])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("U,n,m", [(3, 7, 2), (5, 50, 11), (4, 33, 5), (2, 500, 11), (2, 130, 52)])
def test_ranking_matches_numpy_argmax_with_ties(dtype, U, n, m):
    rng = np.random.default_rng(U * 1000 + n + m)
    x = rng.random((U, n, m)).astype(dtype)
    # ties: coarse quantisation makes equal maxima common; plant exact ties too
    x = np.round(x * 8).astype(dtype) / dtype(8)
    x[0, n - 1, 0] = x[0, :, 0].max()
    x[-1, :, m - 2] = dtype(0.25)   # all items tied: index 0 wins
    got = top_positions(x)
    assert np.array_equal(got, orc.top_positions(x))
    assert np.array_equal(got[-1, m - 2], 0)


def test_ranking_torch_in_torch_out():
    import torch
    x = torch.rand((6, 40, 9), device="cuda", dtype=torch.float32)
    got = top_positions(x)
    assert isinstance(got, torch.Tensor) and got.is_cuda and got.dtype == torch.int32
    assert np.array_equal(got.cpu().numpy(), np.argmax(x.cpu().numpy()[:, :, :-1], axis=1))
