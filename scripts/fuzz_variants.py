"""Every compiled tile on ragged shapes (GPU box, not part of the test suite): random (users >= 2, items,
positions, inner iterations) instances, each solved with every forced tile variant of its width
(DeviceOptions.variant = 0, 1, ...) in both dtypes, fixed schedule, against the oracle -- the tiles the automatic
choice does not pick for the BASELINE shapes get the same parity check as the production ones.
usage: python scripts/fuzz_variants.py -> a summary line, exit 1 on a violation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import nsw_oracle as orc  # checker only
from paper_2406_10262_b200 import DeviceOptions, DeviceSolver, SolverConfig
rng = np.random.default_rng(0)
bad = 0; ran = 0; seen = set()
for c in range(36):
    m = int(rng.choice([3, 4, 7, 8, 11, 13, 16, 21, 30, 32, 45, 52]))
    n = int(rng.integers(m, 1500)) if m <= 32 else int(rng.integers(m, 3000))
    U = int(rng.integers(2, 5)); T = int(rng.integers(1, 9)); outer = 3
    eps = float(rng.choice([0.05, 0.2]))
    rel = np.clip(rng.uniform(0, 1, (U, n)), 1e-4, 1).astype(np.float32).astype(np.float64)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    p = orc.SolverParams(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300)
    xo, tro, _ = orc.solve(rel, expo, p)
    cfg = SolverConfig(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300)
    for dtype in ("float64", "float32"):
        prev = None
        for var in range(0, 12):
            with DeviceSolver(rel, expo, n, m, cfg, DeviceOptions(dtype=dtype, schedule="fixed", variant=var)) as s:
                v = s.variant()
                key = (dtype, v.get("M"), v.get("R"), v.get("NT"), v.get("smem"), v.get("generic", False))
                if var > 0 and key == first: break      # index beyond the candidates: the default again
                if var == 0: first = key
                s.run(outer + 1)
                x = s.get("xbest"); f = s.get("objective")[:outer]
            ran += 1; seen.add(key[:4])
            dx = np.abs(x - xo).max(); df = np.abs(f / np.array(tro.objective) - 1).max()
            ok = (dx <= 1e-9 and df <= 1e-11) if dtype == "float64" else (np.isfinite(x).all() and dx <= 5e-2 and (U == 1 or df <= 5e-5))
            if not ok:
                bad += 1; print("MISMATCH", c, U, n, m, T, dtype, var, v, f"{dx:.2e} {df:.2e}", flush=True)
print("forced variants done:", ran, "runs,", len(seen), "distinct tiles,", bad, "violations")
sys.exit(1 if bad else 0)
