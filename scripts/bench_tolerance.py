"""Timing of the reference's default (tolerance) schedule on the device
(diagnostics): per-outer-step wall time and inner-iteration counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    from paper_2406_10262_b200 import (DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix, SolverConfig,
                                       SolverError, solve_fair_ranking)
    from paper_2406_10262_b200.data import make_instance
    t0 = time.perf_counter()
    import torch
    torch.zeros(1, device="cuda")
    print(f"torch CUDA init {time.perf_counter() - t0:.2f} s")
    rel, expo, _ = make_instance("cfg0", seed=0, num_users=4)
    t0 = time.perf_counter()
    solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(4, 50, 11),
                       SolverConfig(outer_max_iters=2), DeviceOptions())
    print(f"first solve (module loading) {time.perf_counter() - t0:.2f} s")
    chunk = int(os.environ.get("TOL_CHUNK", "16"))
    for name, users, eps, dtype in (("cfg0", 100, 0.1, "float64"), ("cfg1", 1000, 0.05, "float64"),
                                    ("cfg1", 1000, 0.05, "float32")):
        rel, expo, _ = make_instance(name, seed=0, num_users=users)
        U, n = rel.shape
        cfg = SolverConfig(epsilon=eps, sinkhorn_tol=1e-6 if dtype == "float64" else 1e-5, outer_max_iters=25)
        args = (RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, expo.size + 1), cfg)
        for graph in (False, True, False, True):
            t0 = time.perf_counter()
            try:
                pol, tr = solve_fair_ranking(*args, DeviceOptions(dtype=dtype, schedule="tolerance", tol_chunk=chunk,
                                                                  use_graph=graph))
            except SolverError as e:
                tr = e.trace
            dt = time.perf_counter() - t0
            its = tr.sinkhorn_iterations
            print(f"chunk {chunk} {name} U={U} {dtype} {'device-driven graph' if graph else 'host-driven chunks'}: "
                  f"{len(tr)} steps in {dt*1e3:.1f} ms ({dt/len(tr)*1e3:.2f} ms/step), "
                  f"inner iterations {its[:3]}..{its[-3:]} total {sum(its)}, {sum(its)/dt:.0f} inner it/s")


if __name__ == "__main__":
    main()
