"""Randomised sweep of the operator seam on the GPU box (not part of the test
suite): batched Sinkhorn forward (general marginals, fixed / tolerance stop),
its reverse mode, the device metrics and the top-m ranking on random shapes,
against the oracle's restatement of sinkhorn.py:204-309 / metrics.py.
usage: python scripts/fuzz_ops.py [cases] [seed] -> one line per case, exit 1 on a violation."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import nsw_oracle as orc  # checker only
from paper_2406_10262_b200 import top_positions
from paper_2406_10262_b200.metrics import policy_metrics
from paper_2406_10262_b200.sinkhorn import sinkhorn_backward_batch, sinkhorn_batch_solve

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
t0 = time.time()
for c in range(cases):
    m = int(rng.choice([2, 3, 5, 8, 11, 16, 21, 32, 33, 52, 53, 64]))
    n = int(rng.integers(m, m + 4)) if rng.random() < 0.2 else int(rng.integers(m, 600))
    B = int(rng.choice([1, 2, 3, 7, 40, 200])) if n * m < 12000 else int(rng.integers(1, 5))
    eps = float(rng.choice([0.05, 0.1, 0.3, 1.0]))
    T = int(rng.integers(1, 40))
    tolm = bool(rng.random() < 0.4)
    general = bool(rng.random() < 0.5)      # general (random, balanced) marginals vs the ranking marginals
    tag = f"case {c:3d} B={B} n={n} m={m} T={T} eps={eps} {'tolerance' if tolm else 'fixed'} {'general' if general else 'ranking'} marginals"
    cost = rng.uniform(0.0, 1.0, (B, n, m))
    lk = -cost / eps
    if general:
        row = rng.uniform(0.5, 1.5, n)
        col = rng.uniform(0.5, 1.5, m)
        col *= row.sum() / col.sum()
    else:
        row, col, _, _ = orc.ranking_marginals(n, m)
    lvi = rng.normal(0.0, 0.3, (B, m))
    tol = 1e-3 if tolm else -1.0
    ref = orc.sinkhorn_forward(lk, np.log(row), np.log(col), row, col, tol, T, lvi)
    got = sinkhorn_batch_solve(lk, np.log(row), np.log(col), row, col, tol, T, lvi, True)
    dx = float(np.abs(got.plan - ref.plan).max())
    du = float(np.abs(got.log_u - ref.log_u).max())
    dv = float(np.abs(got.log_v - ref.log_v).max())
    ok = got.iterations == ref.iterations and np.array_equal(got.converged, ref.converged)
    ok = ok and dx <= 1e-11 * max(1.0, float(row.max())) and du <= 1e-9 and dv <= 1e-9
    msg = f"iters {got.iterations}/{ref.iterations} |dX|={dx:.1e} |dlogu|={du:.1e} |dlogv|={dv:.1e}"
    # reverse mode through the recorded iterates
    gp = rng.normal(0.0, 1.0, (B, n, m))
    gref = orc.sinkhorn_backward(lk, np.log(row), np.log(col), ref.hist, lvi, gp, ref.plan, ref.log_u)
    ggot = sinkhorn_backward_batch(lk, got.log_v_hist, lvi, gp, got.plan, got.log_u, row=row, col=col)
    dg = float(np.abs(ggot - gref).max() / max(1.0, float(np.abs(gref).max())))
    ok = ok and dg <= 1e-9
    msg += f" |dgK| rel {dg:.1e}"
    # metrics and ranking of the plan as a policy (ranking marginals only: a policy needs them)
    if not general and m >= 2:
        rel = np.clip(rng.uniform(0.0, 1.0, (B, n)), 1e-4, 1.0)
        expo = 1.0 / np.log2(np.arange(2, m + 1))
        # same input on both sides (the device plan): the metrics' thresholds and the argmax are
        # discontinuous, a 1e-13 difference between two plans may legitimately flip them
        mo = orc.policy_metrics(got.plan, rel, expo)
        md = policy_metrics(got.plan, rel, expo)
        md = (md["user_utility"], md["mean_max_envy"], md["items_better_off"], md["items_worse_off"])
        dm = max(abs(a - b) / max(1.0, abs(b)) for a, b in zip(md, mo))
        same_rank = np.array_equal(top_positions(got.plan), orc.top_positions(got.plan))
        ok = ok and dm <= 1e-9 and same_rank
        msg += f" metrics rel {dm:.1e} ranking {'same' if same_rank else 'DIFFERS'}"
    print(tag, msg, "" if ok else "VIOLATION", flush=True)
    bad += not ok
print(f"{cases} cases, {bad} violations, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
