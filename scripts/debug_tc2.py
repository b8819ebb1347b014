import sys, numpy as np
sys.path.insert(0, '.')
from paper_2406_10262_b200 import DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix, SolverConfig, solve_fair_ranking, DeviceSolver
from paper_2406_10262_b200.data import make_instance
rel, expo, cfg1 = make_instance('cfg1', seed=0)
res = {}
for var in (-1, -2):
    c = SolverConfig(epsilon=0.05, sinkhorn_max_iters=100, outer_max_iters=6, grad_threshold=1e-300)
    s = DeviceSolver(rel, expo, 500, 11, c, DeviceOptions(dtype='float32', schedule='fixed', variant=var))
    print(var, s.variant())
    s.run(10)
    pol, tr = s.result()
    s.close()
    res[var] = (pol, tr.objective)
    print(var, tr.objective)
print('TC vs FFMA cfg1 6 steps: |dX|', np.abs(res[-1][0] - res[-2][0]).max(), 'rel dF', np.abs(np.array(res[-1][1]) / np.array(res[-2][1]) - 1).max())
