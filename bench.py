"""Benchmark of the NSW ascent hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1] [--impl ours|reference]

A "step" is one outer ascent iteration of solve_fair_ranking (reference
solver.py:186-240): one Sinkhorn solve per user (T inner iterations), the
impact reduction, the unrolled backward and the Adam update, over the whole
synthetic instance.  Metric: outer ascent iterations / s (BASELINE.json
"outer ascent iters/sec & Sinkhorn cell-updates/s"), whole job.

Our arm prints one JSON line with value (device-resident, CUDA-event timed,
L2 flushed between steps), e2e (public API with host buffers), roofline of
the dominant kernel (the fused step kernel, FP32-pipe bound), cpu_baseline
(the oracle port on a bounded user slice) and nvidia-smi clocks.
The reference arm (--impl reference) times the CPU oracle port (the
reference is pure Python and does not exist on the GPU box) with all host
cores on a bounded user sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2406_10262_b200.data import BASELINE_CONFIGS, make_instance  # noqa: E402

FP32_LANES_PER_SM_CLK = 128
SMS = 148
# canonical FP32-pipe instruction count of one outer step in
# the stabilised multiplicative form: forward 2 N T + backward 7 N T.
INSTR_PER_CELL_ITER = 9


def _peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                try:
                    rows.append((float(f[0]), float(f[1]), f[3:7]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        loaded = [r[0] for r in rows if r[0] > 500] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------------------
# CPU baseline: the oracle port (test infrastructure) on a bounded user slice
# ------------------------------------------------------------------------------
def _oracle_slice_worker(args):
    name, start, stop, steps = args
    from oracle import nsw_oracle as orc
    rel, expo, cfg = make_instance(name, seed=0, user_slice=(start, stop))
    p = orc.SolverParams(epsilon=cfg.epsilon, sinkhorn_max_iters=cfg.inner_iters, outer_max_iters=steps + 1,
                         grad_threshold=1e-300)
    t0 = time.perf_counter()
    _, tr, _ = orc.solve(rel, expo, p)
    total = time.perf_counter() - t0
    return total, list(tr.wall_time)


def cpu_baseline(name, users_per_proc, procs, steps):
    """Seconds per full outer step of the oracle port, extrapolated linearly
    in |U| from `procs` processes x `users_per_proc` users x `steps` steps
    (each process solves its own user slice; steps are fixed-schedule so
    every step does the same work)."""
    cfg = BASELINE_CONFIGS[name]
    jobs = [(name, i * users_per_proc, (i + 1) * users_per_proc, steps) for i in range(procs)]
    t0 = time.perf_counter()
    if procs == 1:
        res = [_oracle_slice_worker(jobs[0])]
    else:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_oracle_slice_worker, jobs)
    wall = time.perf_counter() - t0
    # per-step time of a non-final step (final step is forward only)
    per_step = max(float(np.mean(w[:-1])) for _, w in res)
    users_done = users_per_proc * procs
    t_full = per_step * cfg.num_users / users_done
    return {"value": 1.0 / t_full, "unit": "outer_iters/s", "cores": procs, "kind": "port",
            "sample": (f"oracle/nsw_oracle.py (numpy float64 restatement of the reference) on {procs} process(es) x "
                       f"{users_per_proc} users of {name} x {steps} outer steps (+1 forward), "
                       f"{per_step:.3f} s/step per process, extrapolated x{cfg.num_users / users_done:.1f} "
                       f"to |U|={cfg.num_users}; wall {wall:.1f} s"),
            "seconds_per_step": t_full}


def _ref_worker(conn, name, start, stop):
    """Persistent CPU worker: owns a user slice and runs one full outer step
    of the oracle port (forward, impact, gradient, backward, Adam) per 'step'."""
    from oracle import nsw_oracle as orc
    rel, expo, cfg = make_instance(name, seed=0, user_slice=(start, stop))
    U, n = rel.shape
    m = expo.size + 1
    row, col, lr, lc = orc.ranking_marginals(n, m)
    cost = orc.initial_cost(U, n, m, cfg.epsilon)
    am, av, step = np.zeros_like(cost), np.zeros_like(cost), 0
    lvi = np.zeros((U, m))
    gx = np.zeros_like(cost)
    nie = -1.0 / cfg.epsilon
    while conn.recv() == "step":
        K = cost * nie
        fwd = orc.sinkhorn_forward(K, lr, lc, row, col, -1.0, cfg.inner_iters, lvi)
        imp = orc.impact(rel, expo, fwd.plan)
        orc.welfare_gradient(rel, expo, imp, gx)
        g = orc.sinkhorn_backward(K, lr, lc, fwd.hist, lvi, gx, fwd.plan, fwd.log_u) * nie
        cost, am, av, step = orc.adam_ascent(cost, g, am, av, step, 0.05, 0.9, 0.999, 1e-8)
        lvi = fwd.log_v
        conn.send("done")


def run_reference(a):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    procs = max(1, cores)
    cfg = BASELINE_CONFIGS[a.config]
    # ~0.1-0.3 s of CPU work per process per timed step
    # (the port runs ~1e-7 s per cell per inner iteration for forward+backward)
    users = max(1, min(cfg.num_users // procs,
                       int(0.2 / (1e-7 * cfg.num_items * cfg.num_positions * cfg.inner_iters))))
    ctx = mp.get_context("fork")
    conns, ps = [], []
    for i in range(procs):
        pa, pb = ctx.Pipe()
        p = ctx.Process(target=_ref_worker, args=(pb, a.config, i * users, (i + 1) * users), daemon=True)
        p.start()
        conns.append(pa)
        ps.append(p)
    samples = []
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        for c in conns:
            c.send("step")
        for c in conns:
            c.recv()
        if i >= a.warmup:
            samples.append(time.perf_counter() - t0)
    for c in conns:
        c.send("stop")
    for p in ps:
        p.join(timeout=10)
    t_sample = float(np.mean(samples))
    t = t_sample * cfg.num_users / (procs * users)
    v = 1.0 / t
    line = {"impl": "reference", "metric": "outer_ascent_iters_per_s", "value": v, "unit": "outer_iters/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE generator, seed 0)",
            "config": {"workload": f"{a.config}: U={cfg.num_users} I={cfg.num_items} m={cfg.num_positions} "
                                   f"eps={cfg.epsilon} T_in={cfg.inner_iters}",
                       "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": v, "unit": "outer_iters/s", "cores": procs, "kind": "port",
                             "sample": f"{procs} processes x {users} users x 1 outer step (fwd+bwd+Adam, "
                                       f"float64 numpy) per timed step, {t_sample:.3f} s/step, extrapolated "
                                       f"x{cfg.num_users / (procs * users):.1f} to |U|={cfg.num_users} "
                                       f"(reference is pure Python; the oracle port stands in since "
                                       f"/root/reference is absent on the box)"},
            "e2e": {"value": v, "unit": "outer_iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------
def run_ours(a):
    import torch
    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1 or a.sharded:
        import socket
        import torch.distributed as dist
        if world == 1:   # --sharded outside torchrun: a 1-rank group
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if "MASTER_PORT" not in os.environ:
                with socket.socket() as sk:
                    sk.bind(("127.0.0.1", 0))
                    os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2406_10262_b200 import DeviceOptions, ExposureModel, ProblemShape, RelevanceMatrix, SolverConfig
    from paper_2406_10262_b200.solver import DeviceSolver, solve_fair_ranking

    cfg = BASELINE_CONFIGS[a.config]
    if a.slice:
        lo, hi = (int(x) for x in a.slice.split(":"))
        rel, expo, _ = make_instance(a.config, seed=0, user_slice=(lo, hi))
    else:
        rel, expo, _ = make_instance(a.config, seed=0, num_users=a.users)
    U, n, m, T = rel.shape[0], cfg.num_items, cfg.num_positions, a.inner or cfg.inner_iters
    opts = DeviceOptions(dtype=a.dtype, schedule="fixed", device=local, variant=a.variant)
    scfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=T, outer_max_iters=a.warmup + a.steps + 2,
                        grad_threshold=1e-300)
    peaks, peaks_kind = _peaks()

    if world == 1 and not a.sharded:
        solver = DeviceSolver(rel, expo, n, m, scfg, opts)
        solver.run(a.warmup)
        torch.cuda.synchronize()
        launches0 = solver.launch_count()
        with ClockSampler(local) as cs:
            ms_total, ms_fused = solver.time_steps(a.steps, flush_l2=True)
        torch.cuda.synchronize()
        launches = solver.launch_count() - launches0   # our kernels in the timed steps
        phase, steps_done, err = solver.status()
        variant = solver.variant()
        solver.close()
        users_local = U
    else:
        import torch.distributed as dist
        from paper_2406_10262_b200.distributed import ShardedAscent
        sa = ShardedAscent(RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m), scfg, opts)
        for _ in range(a.warmup):
            sa.step()
        torch.cuda.synchronize()
        dist.barrier()
        # every step timed on the solver's stream between CUDA events, the L2
        # evicted (outside the events) before each one, as in the 1-GPU path
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        with ClockSampler(local) as cs:
            for e0, e1 in evs:
                sa.solver.flush_l2(sa.stream.cuda_stream)
                e0.record(sa.stream)
                sa.step()
                e1.record(sa.stream)
            torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([sum(e0.elapsed_time(e1) for e0, e1 in evs)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        ms_fused = float("nan")
        variant = sa.solver.variant()
        # the step replays a torch-captured graph: main (+ tail) fused launch,
        # impact reduction and finalize (our kernels) around the NCCL all-gather
        launches = a.steps * ((2 if variant.get("tail_users", 0) else 1) + 2)
        users_local = sa.stop - sa.start
        sa.solver.close()

    value = a.steps / (ms_total / 1e3)
    cells = U * n * m
    cell_updates = cells * T * a.steps
    clocks = cs.summary()

    # roofline of the dominant kernel (fused step): FP32-pipe instruction rate
    line = {"metric": "outer_ascent_iters_per_s", "value": value, "unit": "outer_iters/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_total / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if a.dtype == "float32" else "f64",
            "data": "synthetic (BASELINE generator, seed 0)",
            "config": {"workload": f"{a.config}: U={U} I={n} m={m} eps={cfg.epsilon} T_in={T} (fixed schedule)",
                       "users_per_gpu": users_local, "l2": "flushed between timed steps (1 GiB write, then discard of those lines)",
                       "tile": variant},
            "sinkhorn_cell_updates_per_s": cell_updates / (ms_total / 1e3),
            "gpu_launches": launches, "clocks": clocks}
    if world == 1 and ms_fused == ms_fused:
        per_launch_s = ms_fused / 1e3 / a.steps
        instr = INSTR_PER_CELL_ITER * cells * T
        clk = peaks.get("sm_max_mhz", 1965.0)
        peak = SMS * FP32_LANES_PER_SM_CLK * clk * 1e6
        achieved = instr / per_launch_s
        traffic = None
        tfile = os.path.join(REPO, "profiles", "traffic.json")
        if os.path.exists(tfile):
            with open(tfile) as f:
                traffic = json.load(f).get(f"{a.config}_{a.dtype}")
        hbm_bytes = (28 if a.dtype == "float32" else 56) * cells
        line["roofline"] = {
            "bound": "fp32", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tinstr/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": "step_kernel (fused backward+Adam+forward)",
            "count": f"{INSTR_PER_CELL_ITER} FP32-pipe instr per cell per inner iteration (SURVEY 8(d) form B) x "
                     f"{cells} cells x {T} iterations per launch",
            "peak_note": f"148 SMs x 128 FP32 lanes x {clk:.0f} MHz (sm_max from MEASURED_PEAKS.json, "
                         f"{peaks_kind}); no measured FP32 peak exists, so the datasheet lane rate is used",
            "fused_ms_per_launch": per_launch_s * 1e3,
            "fused_share_of_step": ms_fused / ms_total,
            "hbm_secondary": {"algorithmic_bytes_per_launch": hbm_bytes,
                              "achieved_gbs": hbm_bytes / per_launch_s / 1e9,
                              "peak_gbs": peaks.get("hbm_gbs", 6650.0),
                              "frac": hbm_bytes / per_launch_s / 1e9 / peaks.get("hbm_gbs", 6650.0)}}
        line["sinkhorn_cell_updates_per_s_fused_kernel"] = cell_updates / (ms_fused / 1e3)

    # e2e: the public API with host buffers, K outer steps, copies included
    if (world > 1 or a.sharded) and not a.no_e2e:
        # e2e at N GPUs: the SPMD drop-in with host float64 arrays on every rank
        from paper_2406_10262_b200.distributed import solve_fair_ranking_distributed
        ecfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=T, outer_max_iters=a.steps,
                            grad_threshold=1e-300)
        R, E, S = RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m)
        solve_fair_ranking_distributed(R, E, S, SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=T,
                                                             outer_max_iters=2, grad_threshold=1e-300), opts,
                                       gather_policy=False)   # warm
        dist.barrier()
        t0 = time.perf_counter()
        pol, tr = solve_fair_ranking_distributed(R, E, S, ecfg, opts, gather_policy=False)
        t_local = time.perf_counter() - t0
        tt = torch.tensor([t_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
        es = 4 if a.dtype == "float32" else 8
        line["e2e"] = {"value": len(tr) / t_e2e, "unit": "outer_iters/s",
                       "h2d_bytes_per_step": (users_local * n * es + 2 * m * es + n * 8) / a.steps,
                       "d2h_bytes_per_step": (users_local * n * m * es + a.steps * 8 * 3) / a.steps,
                       "what": f"solve_fair_ranking_distributed(host float64 arrays) on {world} rank(s), "
                               f"{a.steps} outer steps, each rank's policy block returned; max over ranks",
                       "seconds": t_e2e}
    if world == 1 and not a.sharded and not a.no_e2e:
        ecfg = SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=T, outer_max_iters=a.steps,
                            grad_threshold=1e-300)
        R, E, S = RelevanceMatrix(rel), ExposureModel(expo), ProblemShape(U, n, m)
        solve_fair_ranking(R, E, S, SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=T, outer_max_iters=2,
                                                 grad_threshold=1e-300), opts)  # warm
        t0 = time.perf_counter()
        pol, tr = solve_fair_ranking(R, E, S, ecfg, opts)
        t_e2e = time.perf_counter() - t0
        es = 4 if a.dtype == "float32" else 8
        h2d = U * n * es + 2 * m * es + n * 8 + 2 * (a.steps + 1) * 8
        d2h = cells * es + a.steps * 8 * 3
        line["e2e"] = {"value": len(tr) / t_e2e, "unit": "outer_iters/s",
                       "h2d_bytes_per_step": h2d / a.steps, "d2h_bytes_per_step": d2h / a.steps,
                       "what": f"solve_fair_ranking(host float64 arrays) for {a.steps} outer steps: H2D, "
                               f"allocation, graph capture, all steps, policy D2H + float64 conversion",
                       "seconds": t_e2e}

    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(a.config, 20, 1, 2)
        line["cpu_baseline"].pop("seconds_per_step", None)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1 or a.sharded:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg1", choices=sorted(BASELINE_CONFIGS))
    ap.add_argument("--dtype", default=None, choices=["float32", "float64"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU driver (ShardedAscent over torch.distributed) even at N=1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # experiment knobs (not used by the driver): override |U|, inner iterations, tile variant
    ap.add_argument("--users", type=int, default=None)
    ap.add_argument("--inner", type=int, default=None)
    ap.add_argument("--variant", type=int, default=-1)
    ap.add_argument("--slice", default=None, help="START:STOP users of the full instance (e.g. one GPU's shard)")
    a = ap.parse_args(argv)
    if a.dtype is None:
        a.dtype = BASELINE_CONFIGS[a.config].dtype
    a.warmup = max(a.warmup, 3)
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
