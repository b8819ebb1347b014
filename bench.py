"""Benchmark of the NSW ascent hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

A "step" is one outer ascent iteration of solve_fair_ranking (reference
solver.py:186-240): one Sinkhorn solve per user (T inner iterations), the
impact reduction, the unrolled backward and the Adam update, over the whole
synthetic instance.  Metric: outer ascent iterations / s (BASELINE.json
"outer ascent iters/sec & Sinkhorn cell-updates/s"), whole job.

Workload: BASELINE config 2 by default (10k users x 1000 items x 21
positions, eps 0.02, 100 inner iterations) -- the largest BASELINE
configuration that BASELINE runs at 1/2/4/8 GPUs and that fits one GPU, so
the 1-GPU bench and the scaling runs measure the same job (users sharded over
ranks, strong scaling).  ``--config cfg1`` runs the single-GPU config.

Our arm prints one JSON line with value (device-resident, CUDA-event timed,
L2 flushed between steps), e2e (public API with host buffers), roofline of
the dominant kernel (the fused step kernel, FP32-pipe bound), cpu_baseline
(the oracle port on a bounded user slice) and nvidia-smi clocks.
``--gpus N`` outside torchrun re-launches itself under torch.distributed.run
with one rank per GPU (at most the visible GPU count).
The reference arm (--impl reference) runs the unmodified reference package
(``baseline/_ref``, its public ``solve_fair_ranking`` under the fixed-schedule
shim of SURVEY.md 8(c)) on every host core, one user sample per process.
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


DEFAULT_CONFIG = "cfg2"


def _spawn_ranks(a, argv):
    """--gpus N outside torchrun: re-launch under torch.distributed.run with
    one rank per GPU (clamped to the visible GPUs: ranks never share a GPU)."""
    import socket
    import torch
    n = min(a.gpus, max(1, torch.cuda.device_count()))
    if n <= 1:
        return None
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


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


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def _import_reference():
    """The unmodified reference package installed at baseline/_ref (pip
    --target), or None."""
    if os.path.isdir(os.path.join(REF_DIR, "nswrank")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import nswrank
            return nswrank
        except Exception:
            return None
    return None


def _ref_solve_worker(args):
    """One process: the reference's public solve_fair_ranking on a user
    sample, under the fixed-schedule shim (every solve runs exactly
    sinkhorn_max_iters iterations); returns its own per-step
    wall times (SolveTrace.wall_time)."""
    name, start, stop, outer = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    nswrank = _import_reference()
    rel, expo, cfg = make_instance(name, seed=0, user_slice=(start, stop))
    U, n = rel.shape
    m = expo.size + 1
    if nswrank is not None:
        import nswrank.solver as ref_solver
        real = ref_solver._sinkhorn_batch

        def fixed(*aa, **kw):
            kw["tol"] = -1.0
            r = real(*aa, **kw)
            r.converged[:] = True
            return r

        ref_solver._sinkhorn_batch = fixed
        scfg = nswrank.SolverConfig(epsilon=cfg.epsilon, sinkhorn_max_iters=cfg.inner_iters, outer_max_iters=outer,
                                    grad_threshold=1e-300)
        _, tr = nswrank.solve_fair_ranking(nswrank.RelevanceMatrix(rel), nswrank.ExposureModel(expo),
                                           nswrank.ProblemShape(U, n, m), scfg)
        return "reference", list(tr.wall_time)
    from oracle import nsw_oracle as orc   # fallback: the bit-exact port
    p = orc.SolverParams(epsilon=cfg.epsilon, sinkhorn_max_iters=cfg.inner_iters, outer_max_iters=outer,
                         grad_threshold=1e-300)
    _, tr, _ = orc.solve(rel, expo, p)
    return "port", list(tr.wall_time)


def run_reference(a):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import multiprocessing as mp
    procs = max(1, os.cpu_count() or 1)
    cfg = BASELINE_CONFIGS[a.config]
    # users per process so that one outer step of a process is ~0.3 s of
    # numpy work (measured ~45 ns per cell per inner iteration, fwd + bwd)
    users = max(1, min(cfg.num_users // procs,
                       int(0.3 / (45e-9 * cfg.num_items * cfg.num_positions * cfg.inner_iters))))
    outer = a.warmup + a.steps + 1          # the final step is forward only (solver.py:220-223)
    jobs = [(a.config, i * users, (i + 1) * users, outer) for i in range(procs)]
    # the reference as it ships: one process alone (1 core), 1 warm-up + 2 steps
    with mp.get_context("fork").Pool(1) as pool:
        _, w1 = pool.map(_ref_solve_worker, [(a.config, 0, users, 4)])[0]
    one_core_full = float(np.mean(w1[1:3])) * cfg.num_users / users
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_ref_solve_worker, jobs)
    wall = time.perf_counter() - t0
    kind = res[0][0]
    walls = np.array([w for _, w in res])                  # [procs][outer]
    timed = walls[:, a.warmup:a.warmup + a.steps]          # the K timed full steps
    # one sample step = the K timed steps of the slowest process / K (all
    # processes run concurrently; the per-step maximum over processes would
    # add up stragglers of different steps)
    sample_step_s = float(timed.sum(axis=1).max()) / a.steps
    users_done = users * procs
    factor = cfg.num_users / users_done
    t_full = sample_step_s * factor                        # whole workload, all host cores
    v = 1.0 / t_full
    sample = (f"{'baseline/_ref nswrank.solve_fair_ranking (unmodified reference, fixed-schedule shim)' if kind == 'reference' else 'oracle port (reference not installed)'}"
              f" in {procs} processes x {users} users of {a.config} (float64 numpy, 1 thread each), "
              f"{a.warmup} warm-up + {a.steps} timed outer steps + 1 final forward; {sample_step_s * 1e3:.1f} ms per "
              f"sample step, extrapolated x{factor:.1f} to |U|={cfg.num_users}; wall {wall:.1f} s")
    line = {"impl": "reference", "metric": "outer_ascent_iters_per_s", "value": v, "unit": "outer_iters/s",
            "n_gpus": max(world, a.gpus), "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": sample_step_s * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE generator, seed 0)",
            "config": {"workload": _workload(a.config, cfg.num_users, cfg.num_items, cfg.num_positions,
                                             cfg.epsilon, cfg.inner_iters),
                       "l2": "n/a (CPU)"},
            "extrapolation": {"sample_users": users_done, "factor": factor,
                              "ms_per_step_full_workload": t_full * 1e3,
                              "note": "ms_per_step is the measured time of one sample step; value is the "
                                      "whole-workload rate (fixed-schedule steps do identical work per user)"},
            "one_core": {"value": 1.0 / one_core_full, "unit": "outer_iters/s",
                         "note": "the reference alone in one process (it is single-threaded numpy): "
                                 "its per-step time on the same sample x |U| / sample users"},
            "cpu_baseline": {"value": v, "unit": "outer_iters/s", "cores": procs, "kind": kind, "sample": sample},
            "e2e": {"value": v, "unit": "outer_iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _workload(name, U, n, m, eps, T):
    return f"{name}: U={U} I={n} m={m} eps={eps} T_in={T}"


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
    datagen = a.datagen or ("device" if a.config in ("cfg3", "cfg4") else "host")
    if datagen == "device":
        # on-device counter-based generator (csrc/nsw_datagen.cu): configs 3 / 4
        # are slow or infeasible to draw on the host; the solver API takes host
        # arrays, so the generated block is copied back once, outside timing
        from paper_2406_10262_b200.datagen import make_instance_device
        lo, hi = (int(x) for x in a.slice.split(":")) if a.slice else (0, a.users or cfg.num_users)
        relt, expo, _ = make_instance_device(a.config, seed=0, user_slice=(lo, hi))
        rel = relt.double().cpu().numpy()
        del relt
    elif a.slice:
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
        # per-rank fused-kernel time for the roofline: the fused launches
        # alone (no exchange), replayed after the timed region, max over ranks
        tf = torch.tensor([sa.solver.time_fused(a.steps, flush_l2=True)], device="cuda")
        dist.all_reduce(tf, op=dist.ReduceOp.MAX)
        ms_fused = float(tf.item())
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
            "data": f"synthetic (BASELINE generator, seed 0, {datagen})",
            "config": {"workload": _workload(a.config, U, n, m, cfg.epsilon, T), "schedule": "fixed (BASELINE)",
                       "users_per_gpu": users_local, "l2": "flushed between timed steps (1 GiB write, then discard of those lines)",
                       "tile": variant},
            "sinkhorn_cell_updates_per_s": cell_updates / (ms_total / 1e3),
            "gpu_launches": launches, "clocks": clocks}
    if a.gpus != world:
        line["requested_gpus"] = a.gpus   # clamped to the visible GPUs (ranks never share a GPU)
    if ms_fused == ms_fused:
        per_launch_s = ms_fused / 1e3 / a.steps
        cells_rank = users_local * n * m      # one launch processes this rank's users
        instr = INSTR_PER_CELL_ITER * cells_rank * T
        clk = peaks.get("sm_max_mhz", 1965.0)
        peak = SMS * FP32_LANES_PER_SM_CLK * clk * 1e6
        achieved = instr / per_launch_s
        traffic = None
        tfile = os.path.join(REPO, "profiles", "traffic.json")
        if os.path.exists(tfile):
            with open(tfile) as f:
                traffic = json.load(f).get(f"{a.config}_{a.dtype}")
        hbm_bytes = (28 if a.dtype == "float32" else 56) * cells_rank
        line["roofline"] = {
            "bound": "fp32", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tinstr/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": "step_kernel (fused backward+Adam+forward)",
            "count": f"{INSTR_PER_CELL_ITER} FP32-pipe instr per cell per inner iteration (SURVEY 8(d) form B) x "
                     f"{cells_rank} cells x {T} iterations per launch"
                     + (f" (rank 0 of {world}: per-rank fused time, max over ranks)" if world > 1 else ""),
            "peak_note": f"148 SMs x 128 FP32 lanes x {clk:.0f} MHz (sm_max from MEASURED_PEAKS.json, "
                         f"{peaks_kind}); no measured FP32 peak exists, so the datasheet lane rate is used",
            "fused_ms_per_launch": per_launch_s * 1e3,
            "fused_share_of_step": ms_fused / ms_total,
            "hbm_secondary": {"algorithmic_bytes_per_launch": hbm_bytes,
                              "achieved_gbs": hbm_bytes / per_launch_s / 1e9,
                              "peak_gbs": peaks.get("hbm_gbs", 6650.0),
                              "frac": hbm_bytes / per_launch_s / 1e9 / peaks.get("hbm_gbs", 6650.0)}}
        line["sinkhorn_cell_updates_per_s_fused_kernel"] = cells_rank * T * a.steps / (ms_fused / 1e3) * world

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
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(BASELINE_CONFIGS))
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
    ap.add_argument("--datagen", default=None, choices=["host", "device"],
                    help="input generator: numpy (host) or the on-device Philox generator (default: device for "
                         "cfg3 / cfg4, host otherwise)")
    a = ap.parse_args(argv)
    if a.dtype is None:
        a.dtype = BASELINE_CONFIGS[a.config].dtype
    a.warmup = max(a.warmup, 3)
    if a.impl == "reference":
        return run_reference(a)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        rc = _spawn_ranks(a, argv)
        if rc is not None:
            return rc
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
