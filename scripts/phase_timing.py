"""Per-phase timeline of the fused step kernel (diagnostics, not product code).

    NSW_PHASE_TIMING=1 python scripts/phase_timing.py [--config 1] [--users N] [--inner T]

Runs a few fixed-schedule steps, then prints, for the main and tail launches,
the median / max duration of each phase of the last step across users, and
the spread of CTA start / end times."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NSW_PHASE_TIMING", "1")

NAMES = ["load hist/alpha/beta", "rebuild K~", "u~^T", "policy write", "seed W", "backward levels",
         "gK epilogue", "Adam", "absorb K~", "forward iterations", "impact terms"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--users", type=int, default=None)
    ap.add_argument("--inner", type=int, default=None)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--variant", type=int, default=-1)
    a = ap.parse_args()
    import torch
    from paper_2406_10262_b200 import DeviceOptions, SolverConfig
    from paper_2406_10262_b200.data import BASELINE_CONFIGS, make_instance
    from paper_2406_10262_b200.solver import DeviceSolver

    cfg = BASELINE_CONFIGS[a.config]
    rel, expo, _ = make_instance(a.config, seed=0, num_users=a.users)
    T = a.inner or cfg.inner_iters
    scfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=T, outer_max_iters=a.steps + 4, grad_threshold=1e-300)
    s = DeviceSolver(rel, expo, cfg.num_items, cfg.num_positions, scfg,
                     DeviceOptions(dtype="float32", schedule="fixed", variant=a.variant))
    s.run(a.steps)
    torch.cuda.synchronize()
    st = s.phase_times().astype(np.int64)
    U = st.shape[0]
    tail = s.lib.nsw_solver_tail_users(s.h)
    print("variant", s.variant(), "users", U, "tail", tail)
    t0 = st[:, 0].min()
    for lo, hi, name in ((0, U - tail, "main"), (U - tail, U, "tail")):
        if hi <= lo:
            continue
        blk = st[lo:hi]
        print(f"== {name} launch: users {lo}..{hi - 1}; start spread {(blk[:, 0].max() - blk[:, 0].min()) / 1e3:.1f} us,"
              f" first start +{(blk[:, 0].min() - t0) / 1e3:.1f} us, last end +{(blk[:, 11].max() - t0) / 1e3:.1f} us")
        for p in range(1, 12):
            d = (blk[:, p] - blk[:, p - 1]) / 1e3
            print(f"  {p:2d} {NAMES[p - 1]:22s} median {np.median(d):8.2f} us  max {d.max():8.2f} us")
        tot = (blk[:, 11] - blk[:, 0]) / 1e3
        print(f"  total per CTA: median {np.median(tot):.1f} us, max {tot.max():.1f} us")


if __name__ == "__main__":
    main()
