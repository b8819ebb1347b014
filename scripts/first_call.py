"""First-call latency of the public API in a fresh process (no torch import)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.perf_counter()
from paper_2406_10262_b200 import (DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix,  # noqa: E402
                                   SolverConfig, solve_fair_ranking)
from paper_2406_10262_b200.data import make_instance  # noqa: E402

rel, expo, _ = make_instance("cfg0", seed=0)
t1 = time.perf_counter()
pol, tr = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(100, 50, 11),
                             SolverConfig(epsilon=0.1, sinkhorn_max_iters=50, outer_max_iters=200,
                                          grad_threshold=1e-300), DeviceOptions(schedule="fixed"))
t2 = time.perf_counter()
pol, tr = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(100, 50, 11),
                             SolverConfig(epsilon=0.1, sinkhorn_max_iters=50, outer_max_iters=200,
                                          grad_threshold=1e-300), DeviceOptions(schedule="fixed"))
t3 = time.perf_counter()
print(f"import+data {t1 - t0:.2f} s, first cfg0 fp64 solve {t2 - t1:.3f} s, second {t3 - t2:.3f} s "
      f"(reference: ~35 s), torch imported: {'torch' in sys.modules}")
