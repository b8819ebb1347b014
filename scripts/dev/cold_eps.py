import sys, numpy as np
sys.path.insert(0, '.')
from paper_2406_10262_b200 import *
from paper_2406_10262_b200.data import make_instance
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
users = int(sys.argv[2]) if len(sys.argv) > 2 else 128
rel, expo, cfg = make_instance(name, seed=0, user_slice=(0, users))
U, n = rel.shape; m = expo.size + 1
for dt in ("float64", "float32"):
    scfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=cfg.inner_iters, outer_max_iters=60, grad_threshold=1e-300, warm_start=False)
    s = DeviceSolver(rel, expo, n, m, scfg, DeviceOptions(dtype=dt, schedule="fixed"))
    for st in range(1, 61):
        s.run(1)
        ph, steps, err = s.status()
        h = s.get("hist"); b = s.get("beta")
        lv = np.log(np.abs(h) + 1e-300)
        if err or not np.isfinite(h).all() or st % 10 == 0:
            print(dt, "step", steps, "err", err, "max|log v~|", np.nanmax(np.abs(lv)), "beta range", b.min(), b.max(),
                  "finite", np.isfinite(h).all(), flush=True)
        if err: break
    s.close()
