"""Multi-GPU ascent: users sharded over ranks, one impact exchange per step.

One process per GPU (torchrun / torch.distributed).  Users are independent
except through the item impacts Imp_i = sum_u ... (reference solver.py:206),
so each rank owns a contiguous user block, runs the fused step kernel on it,
reduces its users' impact terms to one float64 n-vector, and the ranks
exchange those vectors once per outer step (all-gather, then every rank sums
them in rank order, so all ranks hold bitwise-identical Imp, objective,
best-iterate and stop decisions without a broadcast).  The gradient-norm
needs sum_u r_ui^2 over all users, exchanged once at setup.

The exchange is torch.distributed (NCCL on GPUs, gloo in the CPU tests)
running on the solver's own CUDA stream, captured with the step in a CUDA
graph when the backend allows it.

In the reference's tolerance schedule (sinkhorn.py:237-246) the lock-step
stop is over ALL users: after every forward chunk the ranks all-reduce (MAX)
their per-iteration residual maxima before the device picks t*, and each
rank's converged-user count rides in the last slot of its exchanged impact
vector, so the SolverError guard (solver.py:200-205) sees every user.  That
step is host-driven (the number of chunks is data dependent), not captured.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from .core import ExposureModel, ProblemShape, RankingPolicy, RelevanceMatrix, SolverConfig, SolverError
from .solver import DeviceOptions, DeviceSolver, SolveTrace, _check_instance, _coerce

__all__ = ["shard_users", "solve_fair_ranking_distributed", "ShardedAscent", "combine_impacts"]


def shard_users(num_users: int, world: int, rank: int):
    """Contiguous user block [start, stop) of ``rank`` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(num_users, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def combine_impacts(gathered: np.ndarray) -> np.ndarray:
    """Rank-ordered sum of the gathered [world][n] impact partials (the same
    fixed order the device finalize kernel uses)."""
    out = np.zeros(gathered.shape[1])
    for g in range(gathered.shape[0]):
        out += gathered[g]
    return out


class ShardedAscent:
    """This rank's shard + the per-step exchange over a torch process group."""

    def __init__(self, relevance, exposure, shape, config, options=None, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        rel = relevance.values
        self.start, self.stop = shard_users(shape.num_users, self.world, self.rank)
        if self.stop <= self.start:
            raise SolverError("more ranks than users")
        dev = torch.device("cuda", torch.cuda.current_device())
        # sum_u r_ui^2 over all users (closed-form gradient norm, solver.py:211)
        rsq_local = torch.tensor((rel[self.start:self.stop] ** 2).sum(axis=0), dtype=torch.float64, device=dev)
        dist.all_reduce(rsq_local, group=group)
        rsq = rsq_local.cpu().numpy()
        # the drop-in's defaults (reference tolerance schedule, float64), on
        # this rank's current device
        opts = options or DeviceOptions()
        if opts.device is None:
            opts = dataclasses.replace(opts, device=dev.index)
        self.device = dev
        self.tolerance = opts.schedule == "tolerance"
        self.solver = DeviceSolver(rel[self.start:self.stop], exposure.values, shape.num_items,
                                   shape.num_positions, config, opts, rel_sq_sum=rsq, world=self.world)
        n = shape.num_items
        # impacts + this shard's converged-user count (tolerance schedule)
        self.local = torch.zeros(n + 1, dtype=torch.float64, device=dev)
        self.gathered = torch.zeros(self.world * (n + 1), dtype=torch.float64, device=dev)
        self.solver.bind_exchange(self.local.data_ptr(), self.gathered.data_ptr())
        if self.tolerance:
            self.solver.set_scalar("users_total", shape.num_users)
            self.cmax = torch.zeros(max(1, opts.tol_chunk), dtype=torch.float64, device=dev)
            self.solver.bind_tol_exchange(self.cmax.data_ptr())
        self.stream = torch.cuda.ExternalStream(self.solver.stream())
        self.graph = None

    def _step_body(self):
        s = self.stream.cuda_stream
        self.solver.local_step(s)
        self.dist.all_gather_into_tensor(self.gathered, self.local, group=self.group)
        self.solver.finalize(s)

    def _tolerance_step(self):
        s = self.stream.cuda_stream
        self.solver.local_step(s)            # [backward + Adam +] first forward chunk
        while True:
            self.solver.tol_local(s)
            self.dist.all_reduce(self.cmax, op=self.dist.ReduceOp.MAX, group=self.group)
            phase = self.solver.tol_decide(s)
            if phase == 5:                   # next chunk of this forward
                self.solver.local_step(s)
                continue
            if phase == 6:                   # t* known: finish launch + impact terms
                self.solver.local_step(s)
            break
        self.dist.all_gather_into_tensor(self.gathered, self.local, group=self.group)
        self.solver.finalize(s)

    def step(self, use_graph=True):
        torch = self.torch
        if self.tolerance:
            with torch.cuda.stream(self.stream):
                self._tolerance_step()
            return
        with torch.cuda.stream(self.stream):
            if use_graph and self.graph is None:
                try:
                    self._step_body()  # warm NCCL before capture
                    torch.cuda.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=self.stream):
                        self._step_body()
                    self.graph = g
                    return
                except Exception:
                    self.graph = False
            if self.graph:
                self.graph.replay()
            else:
                self._step_body()

    def run(self, max_steps, check_every=16, use_graph=True):
        for it in range(max_steps):
            self.step(use_graph)
            if (it + 1) % check_every == 0 or it + 1 == max_steps:
                phase, _, _ = self.solver.status()
                if phase == 3:
                    return True
        return self.solver.status()[0] == 3


def solve_fair_ranking_distributed(relevance, exposure, shape, config, options: DeviceOptions | None = None,
                                   group=None, gather_policy=False):
    """SPMD drop-in: every rank calls it with the full inputs and the same
    arguments as ``solve_fair_ranking`` (same defaults: the reference's
    tolerance schedule in float64); each rank solves its user block on its
    current CUDA device.

    Returns (RankingPolicy, SolveTrace).  The policy is this rank's user block
    [start, stop) (``gather_policy=False``, default: at config 4 the full
    float64 policy is 163 GB), or, with ``gather_policy=True``, the full
    [U][n][m] policy assembled on every rank by one device all-gather (NCCL)
    of the equal-size padded blocks -- for instances whose full policy fits
    host memory."""
    import torch

    relevance, exposure, shape, config = _coerce(relevance, exposure, shape, config)
    _check_instance(relevance.values, exposure.values, shape)
    options = options or DeviceOptions()
    sa = ShardedAscent(relevance, exposure, shape, config, options, group)
    try:
        done = sa.run(config.outer_max_iters + 1, use_graph=bool(options.use_graph))
        torch.cuda.synchronize()
        if not done:
            raise SolverError("distributed solve did not reach its stop state")
        pol, trace = sa.solver.result()
    finally:
        sa.solver.close()
    if not gather_policy:
        return RankingPolicy(pol), trace
    U, n, m = shape.num_users, shape.num_items, shape.num_positions
    per = -(-U // sa.world)
    block = torch.zeros((per, n, m), dtype=torch.float64, device=sa.device)
    block[: sa.stop - sa.start].copy_(torch.from_numpy(np.ascontiguousarray(pol)))
    full = torch.empty((sa.world * per, n, m), dtype=torch.float64, device=sa.device)
    sa.dist.all_gather_into_tensor(full, block, group=group)
    parts = []
    for r in range(sa.world):
        s0, s1 = shard_users(U, sa.world, r)
        parts.append(full[r * per: r * per + (s1 - s0)])
    return RankingPolicy(torch.cat(parts).cpu().numpy()), trace
