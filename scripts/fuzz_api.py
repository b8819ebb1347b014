"""Randomised sweep of the step-level API on the GPU box (not part of the test
suite): (1) checkpoint / resume -- a solve interrupted at a random step, its
state read back, a fresh solver resumed from it -- against the uninterrupted
solve; (2) the sharded ascent with 2-4 logical ranks on one GPU (one gathered
impact buffer, as tests/test_gpu_two_shards.py) against the unsharded solve;
(3) invalid inputs through the public call: the reference's exception classes,
never a crash; (4) the tolerance schedule across 2-3 logical ranks (chunk residual
maxima combined by MAX before every decide) against the unsharded solve.
usage: python scripts/fuzz_api.py [cases] [seed] -> one line per case, exit 1 on a violation."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_10262_b200 import (DeviceOptions, DeviceSolver, DomainError, ExposureModel, ProblemShape,
                                   RelevanceMatrix, ShapeError, SolverConfig, solve_fair_ranking)
from paper_2406_10262_b200.distributed import shard_users

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
t_start = time.time()


def instance():
    m = int(rng.choice([2, 4, 5, 11, 16, 21, 32, 40, 53]))
    n = int(rng.integers(m, 400))
    U = int(rng.choice([2, 3, 7, 20, 160, 320])) if n * m < 9000 else int(rng.integers(2, 8))
    T = int(rng.integers(1, 16))
    outer = int(rng.integers(3, 8))
    eps = float(rng.choice([0.05, 0.1, 0.3]))
    warm = bool(rng.random() < 0.7)
    dtype = "float32" if rng.random() < 0.4 else "float64"
    rel = np.clip(rng.uniform(0.0, 1.0, (U, n)), 1e-4, 1.0).astype(np.float32).astype(np.float64)
    expo = 1.0 / np.log2(np.arange(2, m + 1))
    cfg = SolverConfig(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=outer, grad_threshold=1e-300, warm_start=warm)
    return U, n, m, rel, expo, cfg, dtype


for c in range(cases):
    kind = c % 4
    U, n, m, rel, expo, cfg, dtype = instance()
    opts = DeviceOptions(dtype=dtype, schedule="fixed")
    outer = cfg.outer_max_iters
    tag = f"case {c:3d} U={U} n={n} m={m} T={cfg.sinkhorn_max_iters} outer={outer} eps={cfg.epsilon} warm={cfg.warm_start} {dtype}"
    if kind == 0:
        # ---- checkpoint / resume at step k (1 <= k < outer) ----
        k = int(rng.integers(1, outer))
        with DeviceSolver(rel, expo, n, m, cfg, opts) as s:
            s.run(outer + 1)
            full = {f: s.get(f) for f in ("xbest", "cost", "adam_m", "adam_v", "lvi")}
            f_full = s.get("objective")[:outer]
        with DeviceSolver(rel, expo, n, m, cfg, opts) as s:
            # k launches: the forward of step k-1 is done, its backward is not -- the state held now
            # (cost, Adam moments, the warm-start duals that forward started from) is the state at the
            # START of step k-1, which is what PHASE_RESUME takes
            s.run(k)
            ck = {f: s.get(f) for f in ("cost", "adam_m", "adam_v", "lvi")}
        with DeviceSolver(rel, expo, n, m, cfg, opts) as s:
            for f, v in ck.items():
                s.set(f, v)
            s.set_scalar("step", k - 1)
            s.set_scalar("phase", 4)    # PHASE_RESUME
            s.run(outer + 1)
            res = {f: s.get(f) for f in ("cost", "adam_m", "adam_v", "lvi")}
            f_res = s.get("objective")[k - 1:outer]
        d = max(float(np.abs(res[f] - full[f]).max()) for f in res)
        df = float(np.abs(f_res / f_full[k - 1:] - 1).max())
        # float64 state goes through float64 get/set: bitwise; float32 state is widened and narrowed exactly
        ok = d == 0.0 and df == 0.0
        print(tag, f"resume at step {k - 1}: max |d state| {d:.1e} rel dF {df:.1e}", "" if ok else "VIOLATION", flush=True)
    elif kind == 1:
        # ---- logical shards ----
        world = int(rng.integers(2, 5))
        if U < world:
            world = U
        rsq = (rel ** 2).sum(axis=0)
        gathered = torch.zeros(world * (n + 1), dtype=torch.float64, device="cuda")
        solvers = []
        for r in range(world):
            s0, s1 = shard_users(U, world, r)
            s = DeviceSolver(rel[s0:s1], expo, n, m, cfg, opts, rel_sq_sum=rsq, world=world)
            s.bind_exchange(gathered[r * (n + 1):(r + 1) * (n + 1)].data_ptr(), gathered.data_ptr())
            solvers.append(s)
        try:
            for _ in range(outer + 1):
                for s in solvers:
                    s.local_step()
                torch.cuda.synchronize()
                for s in solvers:
                    s.finalize()
                torch.cuda.synchronize()
                if all(s.status()[0] == 3 for s in solvers):
                    break
            out = [s.result() for s in solvers]
        finally:
            for s in solvers:
                s.close()
        pol = np.concatenate([p for p, _ in out], axis=0)
        p1, t1 = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m), cfg, opts)
        same = all(t.objective == out[0][1].objective for _, t in out)
        dx = float(np.abs(pol - p1.values).max())
        df = float(np.abs(np.array(out[0][1].objective) / np.array(t1.objective) - 1).max())
        ok = same and len(out[0][1]) == len(t1) and (dx <= 1e-9 and df <= 1e-12 if dtype == "float64" else dx <= 5e-2 and df <= 1e-5)
        print(tag, f"world={world}: ranks agree {same} |dX|={dx:.1e} rel dF={df:.1e}", "" if ok else "VIOLATION", flush=True)
    elif kind == 3:
        # ---- tolerance schedule across logical ranks (float64; SolverError on both sides or neither) ----
        from paper_2406_10262_b200 import SolverError
        world = min(int(rng.integers(2, 4)), U)
        chunk = int(rng.choice([1, 4, 16]))
        cfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=int(rng.integers(4, 40)), outer_max_iters=outer,
                           grad_threshold=1e-300, warm_start=cfg.warm_start, sinkhorn_tol=float(rng.choice([1e-2, 1e-4])))
        opts = DeviceOptions(dtype="float64", schedule="tolerance", tol_chunk=chunk)
        tag = tag.replace(dtype, "float64") + f" T={cfg.sinkhorn_max_iters} tol={cfg.sinkhorn_tol} chunk={chunk}"
        rsq = (rel ** 2).sum(axis=0)
        gathered = torch.zeros(world * (n + 1), dtype=torch.float64, device="cuda")
        cmax = [torch.zeros(chunk, dtype=torch.float64, device="cuda") for _ in range(world)]
        solvers = []
        for r in range(world):
            s0, s1 = shard_users(U, world, r)
            s = DeviceSolver(rel[s0:s1], expo, n, m, cfg, opts, rel_sq_sum=rsq, world=world)
            s.bind_exchange(gathered[r * (n + 1):(r + 1) * (n + 1)].data_ptr(), gathered.data_ptr())
            s.set_scalar("users_total", U)
            s.bind_tol_exchange(cmax[r].data_ptr())
            solvers.append(s)
        derr = oerr = None
        try:
            for _ in range(outer + 1):
                for s in solvers:
                    s.local_step()
                while True:
                    for s in solvers:
                        s.tol_local()
                    torch.cuda.synchronize()
                    mx = cmax[0].clone()
                    for cm in cmax[1:]:
                        mx = torch.maximum(mx, cm)
                    for cm in cmax:
                        cm.copy_(mx)
                    torch.cuda.synchronize()
                    phases = [s.tol_decide() for s in solvers]
                    assert len(set(phases)) == 1, phases
                    if phases[0] in (5, 6):
                        for s in solvers:
                            s.local_step()
                    if phases[0] != 5:
                        break
                torch.cuda.synchronize()
                for s in solvers:
                    s.finalize()
                torch.cuda.synchronize()
                if all(s.status()[0] == 3 for s in solvers):
                    break
            try:
                out = [s.result() for s in solvers]
            except SolverError as e:
                derr = e
        finally:
            for s in solvers:
                s.close()
        try:
            p1, t1 = solve_fair_ranking(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m), cfg, opts)
        except SolverError as e:
            oerr = e
        if derr is not None or oerr is not None:
            ok = (derr is None) == (oerr is None)
            print(tag, f"world={world}: SolverError sharded {derr is not None} unsharded {oerr is not None}",
                  "" if ok else "VIOLATION", flush=True)
        else:
            pol = np.concatenate([p for p, _ in out], axis=0)
            same = all(t.objective == out[0][1].objective and t.sinkhorn_iterations == t1.sinkhorn_iterations for _, t in out)
            dx = float(np.abs(pol - p1.values).max())
            ok = same and dx <= 1e-9
            print(tag, f"world={world}: traces and iteration counts agree {same} |dX|={dx:.1e} iterations {t1.sinkhorn_iterations}",
                  "" if ok else "VIOLATION", flush=True)
    else:
        # ---- invalid inputs: the reference's exception classes ----
        which = int(rng.integers(0, 7))
        r2, e2, shape = rel.copy(), expo.copy(), (U, n, m)
        want = (ShapeError, DomainError)
        if which == 0:
            r2[rng.integers(0, U), rng.integers(0, n)] = np.nan
        elif which == 1:
            r2[rng.integers(0, U), rng.integers(0, n)] = -0.1
        elif which == 2:
            e2 = e2[:-1] if m > 2 else np.concatenate([e2, [0.1]])
        elif which == 3:
            shape = (U, n + 1, m)
        elif which == 4:
            e2[0] = np.inf
        elif which == 5:
            r2 = r2[:, :-1]
        else:
            e2 = -e2
        try:
            solve_fair_ranking(RelevanceMatrix(r2), ExposureModel(e2), ProblemShape(*shape), cfg, opts)
            ok, what = False, "accepted"
        except want as e:
            ok, what = True, type(e).__name__
        except Exception as e:   # noqa: BLE001 -- anything else is the finding
            ok, what = False, f"{type(e).__name__}: {e}"
        print(tag, f"invalid input {which}: {what}", "" if ok else "VIOLATION", flush=True)
    bad += not ok
print(f"{cases} cases, {bad} violations, {time.time() - t_start:.0f} s")
sys.exit(1 if bad else 0)
