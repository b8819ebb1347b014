"""How much of the config-4 cluster step is the cross-CTA exchange? Same tile,
same CTA count, same per-CTA work: n = 4000 on 8-CTA clusters vs n = 512 on one
CTA per user (no exchange).  Diagnostics, not product code."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2406_10262_b200 import DeviceOptions, SolverConfig
    from paper_2406_10262_b200.data import make_instance
    from paper_2406_10262_b200.solver import DeviceSolver

    rel, expo, _ = make_instance("cfg4", seed=0, num_users=1184)
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    for U, n in ((1184, 4000), (9472, 512)):
        r = np.ascontiguousarray(np.tile(rel[:, :n], (U // 1184, 1)))
        scfg = SolverConfig(epsilon=0.01, sinkhorn_max_iters=T, outer_max_iters=12, grad_threshold=1e-300)
        s = DeviceSolver(r, expo, n, 51, scfg, DeviceOptions(dtype="float32", schedule="fixed",
                                                             variant=int(os.environ.get("VAR", "-1"))))
        s.run(3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.run(5)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"U={U} n={n} tile={s.variant()} {dt * 1e3:.2f} ms/step")
        s.close()


if __name__ == "__main__":
    main()
