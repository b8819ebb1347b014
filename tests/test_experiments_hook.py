"""Experiment-runner hook: dispatch logic on CPU; the
device method itself on the GPU."""
import os
import sys
import types

import numpy as np
import pytest

from paper_2406_10262_b200 import experiments as ex

REF_SRC = "/root/reference/pkg/src"


def test_unknown_method_raises():
    with pytest.raises(ex.ConfigError):
        ex.compute_policy("nope", None, None, None, None)
    assert ex.METHODS[:4] == ex.REFERENCE_METHODS and ex.METHOD in ex.METHODS


def test_install_keeps_methods_and_delegates():
    calls = []
    fake = types.SimpleNamespace(METHODS=ex.REFERENCE_METHODS,
                                 _compute_policy=lambda *a: calls.append(a[0]) or "ref")
    ex.install(fake)
    ex.install(fake)   # idempotent
    assert fake.METHODS == ex.REFERENCE_METHODS   # the default method list is unchanged
    assert fake._compute_policy("uniform", 1, 2, 3, 4) == "ref" and calls == ["uniform"]


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")
def test_install_into_reference_runner():
    """The real reference runner keeps its own methods after the hook (CPU,
    'uniform' policy through the reference's code)."""
    sys.path.insert(0, REF_SRC)
    try:
        import importlib
        rexp = importlib.import_module("nswrank.experiments")
        core = importlib.import_module("nswrank.core")
        saved = (rexp.METHODS, rexp._compute_policy, rexp._methods)
        try:
            ex.install(rexp)
            assert ex.METHOD not in rexp.METHODS
            # a config without [methods] keeps the reference default list
            import configparser
            cfg = configparser.ConfigParser()
            assert rexp._methods(cfg) == list(ex.REFERENCE_METHODS)
            # a config naming the device method is accepted; unknown names still fail
            cfg.read_string("[methods]\nmethods = uniform, nsw_algo1_b200\n")
            assert rexp._methods(cfg) == ["uniform", ex.METHOD]
            bad = configparser.ConfigParser()
            bad.read_string("[methods]\nmethods = uniform, nope\n")
            with pytest.raises(rexp.ConfigError):
                rexp._methods(bad)
            shape = core.ProblemShape(3, 5, 3)
            pol = rexp._compute_policy("uniform", None, None, shape, None)
            assert pol.values.shape == (3, 5, 3)
        finally:
            rexp.METHODS, rexp._compute_policy, rexp._methods = saved
    finally:
        sys.path.remove(REF_SRC)


@pytest.mark.gpu
def test_device_method_matches_oracle():
    from oracle import nsw_oracle as orc
    from paper_2406_10262_b200 import (DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix,
                                       SolverConfig)
    from paper_2406_10262_b200.data import make_instance
    rel, expo, _ = make_instance("cfg0", seed=0, num_users=8)
    U, n = rel.shape
    cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=20, outer_max_iters=4, grad_threshold=1e-300)
    pol = ex.compute_policy(ex.METHOD, RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, expo.size + 1),
                            cfg, DeviceOptions(dtype="float64", schedule="fixed"))
    x, _, _ = orc.solve(rel, expo, orc.SolverParams(epsilon=0.1, sinkhorn_max_iters=20, outer_max_iters=4,
                                                   grad_threshold=1e-300))
    assert np.abs(pol.values - x).max() <= 1e-10
