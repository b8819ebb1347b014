"""Generate the golden fixtures in tests/golden/ from the REAL reference.

TEST INFRASTRUCTURE.  Run in the build container (where /root/reference
exists):  ``python oracle/gen_golden.py``.  It

1. imports the reference package (``/root/reference/pkg/src/nswrank``) without
   installing it,
2. applies the fixed-schedule shim of SURVEY.md 8(c): ``_sinkhorn_batch`` is
   called with ``tol=-1`` (exactly ``sinkhorn_max_iters`` iterations) and every
   user is marked converged (disarms the >50% guard, reference solver.py:200-205),
3. runs the reference on the cases below, checks that the numpy restatement in
   ``oracle/nsw_oracle.py`` reproduces it BIT-FOR-BIT in float64 (the pin), and
4. writes the reference's outputs as .npz fixtures.

Nothing here runs on the GPU box; the fixtures travel instead.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"

sys.path.insert(0, REPO)
sys.path.insert(0, REF_SRC)

import nswrank  # noqa: E402  (the reference)
import nswrank.solver as ref_solver  # noqa: E402
import nswrank.sinkhorn as ref_sink  # noqa: E402

from oracle import nsw_oracle as orc  # noqa: E402
from paper_2406_10262_b200.data import make_instance  # noqa: E402

_REAL_BATCH = ref_sink._sinkhorn_batch


def _fixed_batch(*args, **kwargs):
    kwargs["tol"] = -1.0
    res = _REAL_BATCH(*args, **kwargs)
    res.converged[:] = True
    return res


def run_reference(rel, expo, eps, inner, outer, fixed=True, **cfg_kw):
    """The reference's own solve_fair_ranking (+ shim when ``fixed``)."""
    U, n = rel.shape
    m = expo.size + 1
    cfg = nswrank.SolverConfig(epsilon=eps, sinkhorn_max_iters=inner, outer_max_iters=outer,
                               grad_threshold=1e-300 if fixed else cfg_kw.pop("grad_threshold", 1e-3),
                               **cfg_kw)
    ref_solver._sinkhorn_batch = _fixed_batch if fixed else _REAL_BATCH
    try:
        pol, tr = nswrank.solve_fair_ranking(nswrank.RelevanceMatrix(rel), nswrank.ExposureModel(expo),
                                             nswrank.ProblemShape(U, n, m), cfg)
    finally:
        ref_solver._sinkhorn_batch = _REAL_BATCH
    return pol.values, tr


def run_restatement(rel, expo, eps, inner, outer, fixed=True, **kw):
    p = orc.SolverParams(epsilon=eps, sinkhorn_max_iters=inner, outer_max_iters=outer,
                         grad_threshold=1e-300 if fixed else kw.pop("grad_threshold", 1e-3),
                         fixed_schedule=fixed, **kw)
    x, tr, _ = orc.solve(rel, expo, p)
    return x, tr


def pin(name, x_ref, tr_ref, x_or, tr_or):
    dx = float(np.abs(x_ref - x_or).max())
    df = float(np.abs(np.array(tr_ref.objective) - np.array(tr_or.objective)).max())
    print(f"[pin] {name}: max|dX|={dx:.3e} max|dF|={df:.3e}")
    assert dx == 0.0 and df == 0.0, f"restatement is not bit-exact on {name}"


def checksums(x):
    U = x.shape[0]
    w = np.linspace(0.5, 1.5, x.shape[1] * x.shape[2]).reshape(x.shape[1], x.shape[2])
    return np.stack([x.reshape(U, -1).sum(1), (x * x).reshape(U, -1).sum(1),
                     (x * w[None]).reshape(U, -1).sum(1)], axis=1)


def case_cfg0():
    rel, expo, cfg = make_instance("cfg0", seed=0)
    t0 = time.time()
    x_ref, tr_ref = run_reference(rel, expo, cfg.epsilon, cfg.inner_iters, cfg.outer_iters)
    t_ref = time.time() - t0
    x_or, tr_or = run_restatement(rel, expo, cfg.epsilon, cfg.inner_iters, cfg.outer_iters)
    pin("cfg0", x_ref, tr_ref, x_or, tr_or)
    np.savez(os.path.join(OUT, "cfg0_fixed.npz"), relevance=rel, exposure=expo, policy=x_ref,
             objective=np.array(tr_ref.objective), grad_norm=np.array(tr_ref.grad_norm),
             sinkhorn_iterations=np.array(tr_ref.sinkhorn_iterations),
             top_positions=orc.top_positions(x_ref), epsilon=cfg.epsilon,
             inner=cfg.inner_iters, outer=cfg.outer_iters, ref_seconds=t_ref)


def case_cfg1_slice(users=20, outer=60):
    rel, expo, cfg = make_instance("cfg1", seed=0, user_slice=(0, users))
    x_ref, tr_ref = run_reference(rel, expo, cfg.epsilon, cfg.inner_iters, outer)
    x_or, tr_or = run_restatement(rel, expo, cfg.epsilon, cfg.inner_iters, outer)
    pin("cfg1-slice", x_ref, tr_ref, x_or, tr_or)
    # reference noise floor: same instance with items permuted, output un-permuted
    perm = np.random.default_rng(123).permutation(rel.shape[1])
    x_perm, tr_perm = run_reference(rel[:, perm], expo, cfg.epsilon, cfg.inner_iters, outer)
    inv = np.argsort(perm)
    floor = float(np.abs(x_perm[:, inv, :] - x_ref).max())
    print(f"[floor] cfg1-slice reorder noise floor max|dX| = {floor:.3e}")
    np.savez(os.path.join(OUT, "cfg1_slice.npz"), relevance=rel, exposure=expo,
             policy_head=x_ref[:4], policy_checksums=checksums(x_ref),
             objective=np.array(tr_ref.objective), grad_norm=np.array(tr_ref.grad_norm),
             top_positions=orc.top_positions(x_ref), epsilon=cfg.epsilon, inner=cfg.inner_iters,
             outer=outer, noise_floor=floor)


def case_ops():
    """Inner-operator seam: _sinkhorn_batch (fixed T) and _sinkhorn_backward_batch."""
    rng = np.random.default_rng(7)
    out = {}
    for tag, (B, n, m, T) in {"a": (3, 7, 4, 9), "b": (2, 33, 11, 25), "c": (1, 5, 2, 1)}.items():
        K = rng.uniform(-3, 3, (B, n, m))
        lvi = rng.uniform(-1, 1, (B, m))
        mg = ref_sink.Marginals.for_shape(n, m)
        lr, lc = np.log(mg.row), np.log(mg.col)
        res = _REAL_BATCH(K, lr, lc, mg.row, mg.col, tol=-1.0, max_iters=T, log_v_init=lvi, record=True)
        gp = rng.uniform(-1, 1, (B, n, m))
        gk = ref_sink._sinkhorn_backward_batch(K, lr, lc, res.log_v_hist, lvi, gp, res.plan, res.log_u)
        fo = orc.sinkhorn_forward(K, lr, lc, mg.row, mg.col, -1.0, T, lvi)
        go = orc.sinkhorn_backward(K, lr, lc, fo.hist, lvi, gp, fo.plan, fo.log_u)
        assert np.array_equal(fo.plan, res.plan) and np.array_equal(go, gk), tag
        for k, v in dict(log_kernel=K, log_v_init=lvi, plan=res.plan, log_u=res.log_u, log_v=res.log_v,
                         hist=res.log_v_hist, grad_plan=gp, grad_log_kernel=gk,
                         shape=np.array([B, n, m, T])).items():
            out[f"{tag}_{k}"] = v
    # tolerance-mode solve (the reference default stopping rule) on a small instance
    K = rng.uniform(-2, 2, (4, 12, 5))
    mg = ref_sink.Marginals.for_shape(12, 5)
    res = _REAL_BATCH(K, np.log(mg.row), np.log(mg.col), mg.row, mg.col, tol=1e-9, max_iters=400,
                      log_v_init=np.zeros((4, 5)), record=True)
    out.update(tol_log_kernel=K, tol_plan=res.plan, tol_iterations=res.iterations,
               tol_residual=res.residual)
    print("[pin] ops: restatement bit-exact on 3 fwd/bwd cases; tolerance case iterations",
          res.iterations)
    np.savez(os.path.join(OUT, "ops_small.npz"), **out)


def case_tolerance_desk():
    """Reference default (tolerance) mode on the SPEC desk instance: the
    reference raises SolverError at an outer step."""
    rel = nswrank.generate_synthetic(100, 50, seed=0).values
    expo = nswrank.exposure_model(11).values
    ref_solver._sinkhorn_batch = _REAL_BATCH
    cfg = nswrank.SolverConfig()
    trace_obj, trace_it = [], []
    orig = ref_solver._sinkhorn_batch

    def spy(*a, **k):
        r = orig(*a, **k)
        trace_it.append(r.iterations)
        return r

    ref_solver._sinkhorn_batch = spy
    err = None
    try:
        nswrank.solve_fair_ranking(nswrank.RelevanceMatrix(rel), nswrank.ExposureModel(expo),
                                   nswrank.ProblemShape(100, 50, 11), cfg)
    except nswrank.SolverError as e:
        err = str(e)
    finally:
        ref_solver._sinkhorn_batch = _REAL_BATCH
    print(f"[tol] reference default mode: {err!r} after {len(trace_it)} forwards; iters {trace_it[:8]}...")
    # the restatement must fail at the same outer step with the same inner counts
    p = orc.SolverParams(fixed_schedule=False)
    its = []
    try:
        orc.solve(rel, expo, p, on_step=lambda it, fwd, imp: its.append(fwd.iterations))
        raise AssertionError("restatement did not raise")
    except orc.OracleSolverError:
        pass
    assert its == trace_it[:-1], (its[:10], trace_it[:10])
    np.savez(os.path.join(OUT, "tolerance_desk.npz"), relevance=rel, exposure=expo,
             sinkhorn_iterations=np.array(trace_it), error=np.array(err or ""),
             failed_step=len(trace_it) - 1)
    # a short tolerance-mode run that does NOT fail: eps=0.3, 20 outer steps
    cfg2 = dict(epsilon=0.3, outer_max_iters=20)
    ref_solver._sinkhorn_batch = _REAL_BATCH
    pol, tr = nswrank.solve_fair_ranking(nswrank.RelevanceMatrix(rel), nswrank.ExposureModel(expo),
                                         nswrank.ProblemShape(100, 50, 11), nswrank.SolverConfig(**cfg2))
    x_or, tr_or, _ = orc.solve(rel, expo, orc.SolverParams(fixed_schedule=False, **cfg2))
    pin("tolerance-eps0.3", pol.values, tr, x_or, tr_or)
    np.savez(os.path.join(OUT, "tolerance_eps03.npz"), relevance=rel, exposure=expo, policy=pol.values,
             objective=np.array(tr.objective), grad_norm=np.array(tr.grad_norm),
             sinkhorn_iterations=np.array(tr.sinkhorn_iterations))


def case_metrics():
    """The reference's metrics (metrics.py) on the cfg0 golden policy and on
    a cfg1-slice policy; pins oracle.policy_metrics against them."""
    import nswrank.metrics as ref_metrics
    out = {}
    g = np.load(os.path.join(OUT, "cfg0_fixed.npz"))
    rel, expo, pol = g["relevance"], g["exposure"], g["policy"]
    rel2, expo2, _ = make_instance("cfg1", seed=0, user_slice=(0, 16))
    rng = np.random.default_rng(3)
    pol2 = rng.random((16, rel2.shape[1], expo2.size + 1))
    pol2 /= pol2.sum(axis=1, keepdims=True)       # any nonnegative tensor is a valid metric input
    for tag, (r, e, x) in {"cfg0": (rel, expo, pol), "cfg1s": (rel2, expo2, pol2)}.items():
        U, n = r.shape
        R, E, P = nswrank.RelevanceMatrix(r), nswrank.ExposureModel(e), nswrank.RankingPolicy(x)
        ref = np.array([ref_metrics.user_utility(P, R, E), ref_metrics.mean_max_envy(P, R, E),
                        ref_metrics.items_better_off(P, R, E), ref_metrics.items_worse_off(P, R, E),
                        ref_metrics.items_better_off(P, R, E, threshold=0.02),
                        ref_metrics.items_worse_off(P, R, E, threshold=0.02)])
        mine = np.array(orc.policy_metrics(x, r, e) + orc.policy_metrics(x, r, e, 0.02)[2:])
        assert np.array_equal(ref, mine), (tag, ref, mine)
        out[f"{tag}_relevance"], out[f"{tag}_exposure"], out[f"{tag}_policy"] = r, e, x
        out[f"{tag}_metrics"] = ref
        print(f"metrics {tag}: {ref}")
    np.savez(os.path.join(OUT, "metrics.npz"), **out)


def case_api():
    """Per-user API with general marginals (sinkhorn.py:85-188): the
    reference's sinkhorn_solve / sinkhorn_backward / cost_from_policy and a
    tolerance-mode _sinkhorn_batch over a small batch; pins the oracle's
    general-marginal forward/backward against them bit-for-bit."""
    from nswrank.sinkhorn import Marginals, cost_from_policy, sinkhorn_backward, sinkhorn_solve
    rng = np.random.default_rng(21)
    n, m = 23, 7
    row = rng.uniform(0.5, 2.0, n)
    col = rng.uniform(0.5, 2.0, m)
    col *= row.sum() / col.sum()
    cost = rng.normal(0.0, 1.0, (n, m))
    cfg = nswrank.SolverConfig(epsilon=0.2, sinkhorn_tol=1e-7, sinkhorn_max_iters=400)
    mg = Marginals(row, col)
    plan, st = sinkhorn_solve(cost, mg, cfg)
    gp = rng.normal(0.0, 1.0, (n, m))
    grad = sinkhorn_backward(st, gp)
    # pin the oracle (same arithmetic, general masses)
    lk = -cost / cfg.epsilon
    fw = orc.sinkhorn_forward(lk[None], np.log(row), np.log(col), row, col, cfg.sinkhorn_tol,
                              cfg.sinkhorn_max_iters, np.zeros((1, m)))
    assert fw.iterations == st.iterations_used and np.array_equal(fw.plan[0], plan)
    g_or = orc.sinkhorn_backward(lk[None], np.log(row), np.log(col), fw.hist, np.zeros((1, m)), gp[None],
                                 np.exp(fw.log_u[0][:, None] + lk + fw.log_v[0][None, :])[None],
                                 fw.log_u) / (-cfg.epsilon)
    assert np.array_equal(g_or[0], grad), np.abs(g_or[0] - grad).max()
    # a lock-step batch in tolerance mode with the ranking marginals
    B, nb, mb = 5, 30, 6
    lkb = rng.normal(0.0, 3.0, (B, nb, mb))
    lvb = rng.normal(0.0, 0.3, (B, mb))
    mr = Marginals.for_shape(nb, mb)
    rb = ref_sink._sinkhorn_batch(lkb, np.log(mr.row), np.log(mr.col), mr.row, mr.col, 1e-6, 300, lvb, True)
    pol = rng.random((3, nb, mb)) + 0.01
    np.savez(os.path.join(OUT, "api_small.npz"), cost=cost, row=row, col=col, eps=cfg.epsilon, tol=cfg.sinkhorn_tol,
             max_iters=cfg.sinkhorn_max_iters, plan=plan, log_u=st.log_u, log_v=st.log_v,
             iterations=st.iterations_used, converged=st.converged, residual=st.final_residual, grad_plan=gp,
             grad_cost=grad, b_log_kernel=lkb, b_lvi=lvb, b_plan=rb.plan, b_log_u=rb.log_u, b_log_v=rb.log_v,
             b_hist=rb.log_v_hist, b_iterations=rb.iterations, b_converged=rb.converged, b_residual=rb.residual,
             policy=pol, policy_cost=cost_from_policy(pol, 0.3))
    print(f"api: solve {st.iterations_used} iterations (converged {st.converged}), batch {rb.iterations}")


def _long_job(args):
    kind, users, outer = args
    rel, expo, cfg = make_instance("cfg1", seed=0, user_slice=(0, users))
    if kind == "ref":
        return run_reference(rel, expo, cfg.epsilon, cfg.inner_iters, outer)
    if kind == "perm":
        perm = np.random.default_rng(123).permutation(rel.shape[1])
        x, tr = run_reference(rel[:, perm], expo, cfg.epsilon, cfg.inner_iters, outer)
        return x[:, np.argsort(perm), :], tr
    return run_restatement(rel, expo, cfg.epsilon, cfg.inner_iters, outer)


def case_cfg1_long(users=100, outer=200):
    """the config-1 generator's first 100 users over 200
    outer steps x 100 inner iterations (eps 0.05), the reference itself, its
    item-permuted twin (the reference's own reorder noise floor) and the
    restatement pin, run as three processes."""
    import multiprocessing as mp
    with mp.get_context("fork").Pool(3) as pool:
        (x_ref, tr_ref), (x_perm, tr_perm), (x_or, tr_or) = pool.map(
            _long_job, [("ref", users, outer), ("perm", users, outer), ("or", users, outer)])
    pin("cfg1-100x200", x_ref, tr_ref, x_or, tr_or)
    floor = float(np.abs(x_perm - x_ref).max())
    floor_f = float(np.abs(np.array(tr_perm.objective) / np.array(tr_ref.objective) - 1).max())
    print(f"[floor] cfg1 100x200 reorder noise floor max|dX| = {floor:.3e}, rel dF = {floor_f:.3e}")
    rel, expo, cfg = make_instance("cfg1", seed=0, user_slice=(0, users))
    np.savez(os.path.join(OUT, "cfg1_long.npz"), relevance=rel, exposure=expo,
             policy_head=x_ref[:8], policy_checksums=checksums(x_ref),
             objective=np.array(tr_ref.objective), grad_norm=np.array(tr_ref.grad_norm),
             top_positions=orc.top_positions(x_ref), epsilon=cfg.epsilon, inner=cfg.inner_iters,
             outer=outer, noise_floor=floor, noise_floor_objective=floor_f,
             perm_objective=np.array(tr_perm.objective))


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["ops", "cfg0", "tol", "cfg1", "metrics", "api"]
    for w in which:
        t = time.time()
        {"ops": case_ops, "cfg0": case_cfg0, "tol": case_tolerance_desk, "cfg1": case_cfg1_slice,
         "metrics": case_metrics, "api": case_api, "cfg1long": case_cfg1_long}[w]()
        print(f"  {w}: {time.time() - t:.1f}s")
