"""Diagnostics (build: python -m paper_2406_10262_b200.build --tag xtime -D NSW_EXP_XTIME=1 --only inst_cl_f32;
run with NSW_LIB_PATH=paper_2406_10262_b200/libnswrank_b200_xtime.so): per-rank arrival and
completion stamps of 24 consecutive column exchanges of one config-4 user
(9-CTA cluster) -- how much of an exchange is the ranks arriving unevenly."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NSW_PHASE_TIMING", "1")


def main():
    import torch
    from paper_2406_10262_b200 import DeviceOptions, SolverConfig
    from paper_2406_10262_b200.datagen import make_instance_device
    from paper_2406_10262_b200.data import BASELINE_CONFIGS
    from paper_2406_10262_b200.solver import DeviceSolver
    cfg = BASELINE_CONFIGS["cfg4"]
    relt, expo, _ = make_instance_device("cfg4", seed=0, user_slice=(0, 30))
    rel = relt.double().cpu().numpy()
    scfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=cfg.inner_iters, outer_max_iters=8, grad_threshold=1e-300)
    s = DeviceSolver(rel, expo, cfg.num_items, cfg.num_positions, scfg, DeviceOptions(dtype="float32", schedule="fixed"))
    s.run(4)
    torch.cuda.synchronize()
    st = s.phase_times().astype(np.int64).reshape(-1)
    E = 24
    x = st[:9 * 2 * E].reshape(9, E, 2)
    arr, done = x[:, :, 0], x[:, :, 1]
    t0 = arr.min()
    print("rank  mean arrival after the first rank (ns)   per exchange: max-min arrival, done - last arrival")
    lag = arr - arr.min(axis=0, keepdims=True)
    for r in range(9):
        print(f"{r:4d}  {lag[r].mean():8.0f}  (late-most in {int((lag[r] == lag.max(axis=0)).sum())} of {E})")
    spread = arr.max(axis=0) - arr.min(axis=0)
    tail = done.max(axis=0) - arr.max(axis=0)
    period = np.diff(arr.min(axis=0))
    print(f"arrival spread: median {np.median(spread):.0f} ns, done after last arrival: median {np.median(tail):.0f} ns,"
          f" exchange period (first arrival to first arrival): median {np.median(period):.0f} ns")


if __name__ == "__main__":
    main()
