import numpy as np, sys, os
sys.path.insert(0, '.')
from paper_2406_10262_b200 import *
from paper_2406_10262_b200.data import make_instance
rel, expo, _ = make_instance("cfg0", seed=0, num_users=8)
U, n = rel.shape
for dt in sys.argv[1:] or ("float64", "float32"):
    cfg = SolverConfig(epsilon=0.1, sinkhorn_max_iters=20, outer_max_iters=4, grad_threshold=1e-300)
    print(dt, flush=True)
    s = DeviceSolver(rel, expo, n, expo.size + 1, cfg, DeviceOptions(dtype=dt, schedule="fixed"))
    print("created", s.variant(), flush=True)
    s.run(1); print("step 1 ok", flush=True)
    s.run(5); print("steps ok", flush=True)
    s.result(); print("result ok", flush=True)
    s.close(); print("closed", dt, flush=True)
