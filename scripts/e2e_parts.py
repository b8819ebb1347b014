"""Timing breakdown of the public-API solve (diagnostics): create (H2D +
allocation), run (steps incl. graph capture), result (D2H + conversion)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2406_10262_b200 import DeviceOptions, SolverConfig
    from paper_2406_10262_b200.data import BASELINE_CONFIGS, make_instance
    from paper_2406_10262_b200.solver import DeviceSolver
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    cfg = BASELINE_CONFIGS[name]
    rel, expo, _ = make_instance(name, seed=0)
    for steps in (2, 30):
        scfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=cfg.inner_iters, outer_max_iters=steps,
                            grad_threshold=1e-300)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = DeviceSolver(rel, expo, cfg.num_items, cfg.num_positions, scfg,
                         DeviceOptions(dtype="float32", schedule="fixed"))
        t1 = time.perf_counter()
        s.run(steps + 1)
        t2 = time.perf_counter()
        pol, tr = s.result()
        t3 = time.perf_counter()
        s.close()
        t4 = time.perf_counter()
        print(f"DeviceSolver steps {steps}: create {1e3*(t1-t0):.1f} ms, run {1e3*(t2-t1):.1f} ms ({1e3*(t2-t1)/steps:.3f}/step), "
              f"result {1e3*(t3-t2):.1f} ms, close {1e3*(t4-t3):.1f} ms, e2e it/s {steps/(t4-t0):.0f}")


def api():
    import cProfile
    import pstats
    import torch
    from paper_2406_10262_b200 import (DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix, SolverConfig,
                                       solve_fair_ranking)
    from paper_2406_10262_b200.data import BASELINE_CONFIGS, make_instance
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    cfg = BASELINE_CONFIGS[name]
    rel, expo, _ = make_instance(name, seed=0)
    args = (RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(rel.shape[0], cfg.num_items, cfg.num_positions))
    opts = DeviceOptions(dtype="float32", schedule="fixed")
    for steps in (2, 30, 30):
        c = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=cfg.inner_iters, outer_max_iters=steps,
                         grad_threshold=1e-300)
        t0 = time.perf_counter()
        pr = cProfile.Profile()
        pr.enable()
        pol, tr = solve_fair_ranking(*args, c, opts)
        pr.disable()
        dt = time.perf_counter() - t0
        print(f"solve_fair_ranking steps {steps}: {1e3*dt:.1f} ms, e2e it/s {steps/dt:.0f}")
        if steps == 30:
            pstats.Stats(pr).sort_stats("cumulative").print_stats(8)


if __name__ == "__main__":
    api()
    main()
