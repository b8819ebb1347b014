"""Timing of the device evaluation metrics at BASELINE
shapes, against the oracle port on the host (measurement helper)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from oracle import nsw_oracle as orc
    from paper_2406_10262_b200.data import BASELINE_CONFIGS, make_instance
    from paper_2406_10262_b200.metrics import policy_metrics
    for name in ("cfg1", "cfg2", "cfg3"):
        cfg = BASELINE_CONFIGS[name]
        rel, expo, _ = make_instance(name, seed=0)
        U, n, m = rel.shape[0], cfg.num_items, cfg.num_positions
        g = torch.Generator(device="cuda").manual_seed(0)
        X = torch.rand((U, n, m), generator=g, device="cuda", dtype=torch.float32)
        R = torch.as_tensor(rel.astype(np.float32), device="cuda")
        policy_metrics(X, R, expo)  # warm (cuBLAS handle, pool)
        torch.cuda.synchronize()
        t = time.perf_counter()
        reps = 5
        for _ in range(reps):
            out = policy_metrics(X, R, expo)
        torch.cuda.synchronize()
        dev = (time.perf_counter() - t) / reps
        # host oracle on a user slice, extrapolated linearly in |U| (envy GEMM is linear in |U| too)
        us = min(U, 200)
        xs = X[:us].double().cpu().numpy()
        t = time.perf_counter()
        orc.policy_metrics(xs, rel[:us], expo)
        cpu = (time.perf_counter() - t) * U / us
        print(json.dumps({"config": name, "U": U, "n": n, "m": m, "device_s": dev, "cpu_oracle_s_extrapolated": cpu,
                          "speedup": cpu / dev, "cells_per_s": U * n * m / dev, "metrics": out}))


if __name__ == "__main__":
    main()
