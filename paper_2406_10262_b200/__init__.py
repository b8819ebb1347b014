"""B200-native drop-in for the NSW fair-ranking ascent path of arxiv 2406.10262.

Mirrors the reference package facade (``nswrank/__init__.py``): the same
public names for the hot path (``solve_fair_ranking`` and its boundary
types), resolved lazily.  The solver runs on hand-written sm_100a kernels in
``libnswrank_b200.so``; there is no CPU fallback.
"""

__version__ = "0.1.0"

_EXPORTS = {
    "core": ("ProblemShape", "RelevanceMatrix", "ExposureModel", "RankingPolicy", "SolverConfig",
             "ShapeError", "DomainError", "StateError", "SolverError", "RELEVANCE_FLOOR", "FEASIBILITY_TOL", "uniform_policy", "CostTensor",
             "ValidationReport", "validate_policy"),
    "solver": ("SolveTrace", "DeviceOptions", "DeviceSolver", "solve_fair_ranking", "NativeLibraryError",
               "impact", "nsw_objective", "nsw_gradient_wrt_policy", "AdamState", "adam_update"),
    "data": ("exposure_model", "make_instance", "BASELINE_CONFIGS"),
    "datagen": ("generate_relevance", "make_instance_device"),
    "sinkhorn": ("sinkhorn_batch", "sinkhorn_backward_batch", "sinkhorn_batch_solve", "Marginals", "SinkhornState",
                 "sinkhorn_solve", "sinkhorn_backward", "cost_from_policy"),
    "ranking": ("top_positions",),
    "metrics": ("user_utility", "mean_max_envy", "items_better_off", "items_worse_off", "policy_metrics"),
    "distributed": ("solve_fair_ranking_distributed", "shard_users", "ShardedAscent"),
    "experiments": ("compute_policy", "install"),
}

_ATTR_TO_MODULE = {name: mod for mod, names in _EXPORTS.items() for name in names}
__all__ = sorted(_ATTR_TO_MODULE) + ["__version__"]


def __getattr__(name):
    mod = _ATTR_TO_MODULE.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib

    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return __all__
