import sys, numpy as np
sys.path.insert(0, '.')
from paper_2406_10262_b200 import DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix, SolverConfig, solve_fair_ranking, DeviceSolver
from oracle import nsw_oracle as orc
g = np.load('tests/golden/cfg0_fixed.npz')
rel, expo = g['relevance'], g['exposure']
p = orc.SolverParams(epsilon=0.1, sinkhorn_max_iters=50, outer_max_iters=12, grad_threshold=1e-300)
_, _, states = orc.solve(rel, expo, p, record_states={10})
st = states[10]; ref = orc.one_step(rel, expo, st, p)
for var in (-1, -2):
    cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=50, outer_max_iters=15, grad_threshold=1e-300)
    s = DeviceSolver(rel, expo, 50, 11, cfg, DeviceOptions(dtype='float32', schedule='fixed', variant=var))
    print('variant', var, s.variant())
    s.set('cost', st['cost']); s.set('adam_m', st['m']); s.set('adam_v', st['v']); s.set('lvi', st['lvi'])
    s.set_scalar('step', 10); s.set_scalar('phase', 4); s.run(1); s.run(1)
    print('  |dX|', np.abs(s.get('xbest') - ref['plan']).max(), '|dC|', np.abs(s.get('cost') - ref['cost']).max())
    s.close()
# end-to-end fp32 TC vs non-TC on cfg1 slice
from paper_2406_10262_b200.data import make_instance
rel, expo, cfg1 = make_instance('cfg1', seed=0, user_slice=(0, 64))
res = {}
for var in (-1, -2):
    c = SolverConfig(epsilon=0.05, sinkhorn_max_iters=100, outer_max_iters=20, grad_threshold=1e-300)
    pol, tr = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(64, 500, 11), c,
                                 DeviceOptions(dtype='float32', schedule='fixed', variant=var))
    res[var] = (pol.values, tr.objective)
print('TC vs FFMA cfg1-slice 20 steps: |dX|', np.abs(res[-1][0] - res[-2][0]).max(), 'rel dF', np.abs(np.array(res[-1][1]) / np.array(res[-2][1]) - 1).max())
