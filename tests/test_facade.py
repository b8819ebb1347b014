"""Package facade: the reference's boundary names (core.py:16-257) exist with
the same validation; validate_policy matches the reference's (CPU)."""
import os
import sys

import numpy as np
import pytest

import paper_2406_10262_b200 as nsw

REF_SRC = "/root/reference/pkg/src"


def test_boundary_names_exported():
    for name in ("CostTensor", "ValidationReport", "validate_policy", "FEASIBILITY_TOL", "RELEVANCE_FLOOR",
                 "RankingPolicy", "ProblemShape", "solve_fair_ranking", "SolveTrace", "uniform_policy"):
        assert hasattr(nsw, name), name
    assert nsw.FEASIBILITY_TOL == 1e-6


def test_cost_tensor_validation():
    c = nsw.CostTensor(np.zeros((2, 3, 2)))
    assert c.values.shape == (2, 3, 2) and not c.values.flags.writeable
    with pytest.raises(nsw.ShapeError):
        nsw.CostTensor(np.zeros((3, 2)))
    with pytest.raises(nsw.DomainError):
        nsw.CostTensor(np.full((1, 2, 2), np.inf))


def test_validate_policy_uniform_and_shape():
    shape = nsw.ProblemShape(3, 7, 4)
    rep = nsw.validate_policy(nsw.uniform_policy(shape), shape)
    assert rep.ok and rep.worst <= 1e-15
    with pytest.raises(nsw.ShapeError):
        nsw.validate_policy(nsw.uniform_policy(shape), nsw.ProblemShape(3, 7, 5))


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")
def test_validate_policy_matches_reference():
    sys.path.insert(0, REF_SRC)
    try:
        import nswrank
        rng = np.random.default_rng(4)
        for U, n, m in ((2, 5, 3), (4, 30, 11)):
            x = rng.random((U, n, m))
            x /= x.sum(axis=2, keepdims=True)
            x[0, 0, 0] = -1e-7
            ref = nswrank.validate_policy(nswrank.RankingPolicy(x), nswrank.ProblemShape(U, n, m), tol=0.5)
            mine = nsw.validate_policy(nsw.RankingPolicy(x), nsw.ProblemShape(U, n, m), tol=0.5)
            assert (ref.ok, ref.row_residual, ref.col_residual, ref.dummy_residual, ref.negativity, ref.worst) == \
                (mine.ok, mine.row_residual, mine.col_residual, mine.dummy_residual, mine.negativity, mine.worst)
    finally:
        sys.path.remove(REF_SRC)
