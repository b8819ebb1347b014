"""Experiment-runner hook for the device solver.

The reference selects a policy by method name in
``nswrank.experiments._compute_policy`` (experiments.py:124-134) from the
``METHODS`` tuple (experiments.py:28), validated when a config is parsed
(experiments.py:93).  This module adds the device method ``"nsw_algo1_b200"``
next to ``"nsw_algo1"`` without changing the CSV schema: the runner still
gets a ``RankingPolicy`` (the best iterate, float64 [U][I][m]) and computes
its metrics exactly as for the CPU solver.  The CLI and the runner stay the
reference's (out of scope here); ``install`` is the one-line hook a
maintainer adds to them.
"""

from __future__ import annotations

from .solver import DeviceOptions, solve_fair_ranking

METHOD = "nsw_algo1_b200"
REFERENCE_METHODS = ("uniform", "max_rele", "nsw_greedy", "nsw_algo1")   # experiments.py:28
METHODS = REFERENCE_METHODS + (METHOD,)


class ConfigError(ValueError):
    """Unknown method name (mirrors ``nswrank.experiments.ConfigError``, experiments.py:43)."""


def compute_policy(method, rel, exposure, shape, solver_cfg, options: DeviceOptions | None = None, fallback=None):
    """``_compute_policy`` with the device method: ``"nsw_algo1_b200"`` runs
    :func:`solve_fair_ranking` on the B200 (``options``: dtype / schedule,
    default the reference's float64 tolerance schedule); any other name goes
    to ``fallback`` (the reference's own ``_compute_policy``) or raises
    :class:`ConfigError`."""
    if method == METHOD:
        policy, _ = solve_fair_ranking(rel, exposure, shape, solver_cfg, options)
        return policy
    if fallback is not None:
        return fallback(method, rel, exposure, shape, solver_cfg)
    raise ConfigError(f"unknown method {method!r}, expected one of {METHODS}")


def install(experiments_module, options: DeviceOptions | None = None):
    """Register the device method in a loaded ``nswrank.experiments`` module.

    ``_compute_policy`` dispatches ``"nsw_algo1_b200"`` to the device and every
    other method to the reference's original function; ``_methods``
    (experiments.py:88-96) additionally ACCEPTS the device method when a
    config names it.  ``METHODS`` -- and so the default method list of a
    config without a [methods] section -- is left unchanged: such configs
    keep running exactly the reference's methods (and need no GPU).
    Returns the module."""
    original = experiments_module._compute_policy
    if getattr(original, "_nsw_b200", False):
        return experiments_module

    def _compute_policy(method, rel, exposure, shape, solver_cfg):
        return compute_policy(method, rel, exposure, shape, solver_cfg, options, fallback=original)

    _compute_policy._nsw_b200 = True
    experiments_module._compute_policy = _compute_policy
    original_methods = getattr(experiments_module, "_methods", None)
    if original_methods is not None:
        def _methods(cfg):
            mod = experiments_module
            default = ", ".join(mod.METHODS)
            raw = mod._get(cfg, "methods", "methods", str, default) if hasattr(mod, "_get") else default
            names = [tok.strip() for tok in raw.split(",") if tok.strip()]
            if METHOD not in names:
                return original_methods(cfg)       # the reference's own validation and messages
            allowed = tuple(mod.METHODS) + (METHOD,)
            err = getattr(mod, "ConfigError", ConfigError)
            for name in names:
                if name not in allowed:
                    raise err(f"unknown method {name!r}, expected one of {allowed}")
            return names

        _methods._nsw_b200 = True
        experiments_module._methods = _methods
    return experiments_module
