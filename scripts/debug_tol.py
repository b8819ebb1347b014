import sys, numpy as np
sys.path.insert(0, '.')
from paper_2406_10262_b200 import DeviceOptions, DeviceSolver, SolverConfig
from oracle import nsw_oracle as orc
g = np.load('tests/golden/tolerance_desk.npz')
rel, expo = g['relevance'], g['exposure']
for steps in (1, 2, 3, 6):
    cfg = SolverConfig(outer_max_iters=steps)
    s = DeviceSolver(rel, expo, 50, 11, cfg, DeviceOptions(dtype='float64', schedule='tolerance'))
    s.run(steps + 1)
    try:
        pol, tr = s.result()
        print(steps, 'iters', tr.sinkhorn_iterations, 'F', tr.objective[-1])
    except Exception as e:
        print(steps, 'ERR', e, getattr(e, 'trace', None))
    print('   phase/step/err', s.status(), 'beta finite', np.isfinite(s.get('beta')).all(), 'hist finite', np.isfinite(s.get('hist')).all(),
          'alpha finite', np.isfinite(s.get('alpha')).all(), 'partial finite', np.isfinite(s.get('partial')).all())
    s.close()
p = orc.SolverParams(fixed_schedule=False, outer_max_iters=6)
x, tr, _ = orc.solve(rel, expo, p)
print('oracle iters', tr.sinkhorn_iterations, 'F', tr.objective)
