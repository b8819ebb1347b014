"""Oracle parity of every fp32 tile that produces a credited number.

Each production instantiation of the fused step kernel -- the ones bench.py
times at configs 1-4, including the wave-tail tiles that run beside them on
the side stream -- is forced and compared, one outer step (forward, impact,
gradient, backward, Adam) from a mid-trajectory state of the float64 oracle,
against that oracle (reference sinkhorn.py:204-309, solver.py:186-240).

Tolerance: the float32 restatement of the reference (the oracle in float32,
log-domain like the reference) run from the same state measures the error
floor that fp32 arithmetic itself has at that config's eps; the device must be
within 2x of it, and never looser than the cfg-0 bars |dX| <= 2e-6,
|dC_{t+1}| <= 5e-6 where that floor is below them.
"""

import numpy as np
import pytest

from oracle import nsw_oracle as orc
from paper_2406_10262_b200 import DeviceOptions, DeviceSolver, SolverConfig
from paper_2406_10262_b200.data import make_instance

pytestmark = pytest.mark.gpu

F32 = DeviceOptions(dtype="float32", schedule="fixed")


def resume_one_step(rel, expo, p, state, step, opts=F32):
    U, n = rel.shape
    m = expo.size + 1
    cfg = SolverConfig(epsilon=p.epsilon, sinkhorn_max_iters=p.sinkhorn_max_iters, outer_max_iters=step + 5,
                       grad_threshold=1e-300)
    s = DeviceSolver(rel, expo, n, m, cfg, opts)
    try:
        variant = s.variant()
        s.set("cost", state["cost"])
        s.set("adam_m", state["m"])
        s.set("adam_v", state["v"])
        s.set("lvi", state["lvi"])
        s.set_scalar("step", step)
        s.set_scalar("phase", 4)  # PHASE_RESUME
        s.run(1)
        obj = s.get("objective")[step]
        s.run(1)
        return dict(plan=s.get("xbest"), cost=s.get("cost"), objective=obj, variant=variant)
    finally:
        s.close()


def check_one_step(name, rel, expo, eps, T, step=3):
    p = orc.SolverParams(epsilon=eps, sinkhorn_max_iters=T, outer_max_iters=step + 2, grad_threshold=1e-300)
    _, _, states = orc.solve(rel, expo, p, record_states={step})
    st = states[step]
    ref = orc.one_step(rel, expo, st, p)
    r32 = orc.one_step(rel, expo, st, p, dtype=np.float32)
    dev = resume_one_step(rel, expo, p, st, step)
    dx = float(np.abs(dev["plan"] - ref["plan"]).max())
    dx32 = float(np.abs(r32["plan"].astype(np.float64) - ref["plan"]).max())
    # C_{t+1}: Adam's step m^/(sqrt(v^) + 1e-8) is scale-free, so cells whose
    # gradient lies below fp32 resolution relative to the tile's largest
    # (|g| < 1e-6 max|g|, e.g. plans of 1e-80 at eps = 0.01) take an O(lr)
    # step of arbitrary sign in ANY fp32 arithmetic; C parity is
    # judged on the resolvable cells, and every cell must stay within 1e-3
    g = ref["grad_cost"]
    ok = np.abs(g) >= 1e-6 * np.abs(g).max()
    dcell = np.abs(dev["cost"] - ref["cost"])
    dc = float(dcell[ok].max())
    dc32 = float(np.abs(r32["cost"].astype(np.float64) - ref["cost"])[ok].max())
    df = abs(dev["objective"] / st["objective"] - 1)
    print(f"{name} {dev['variant']}: |dX|={dx:.2e} (fp32 oracle {dx32:.2e}) |dC|={dc:.2e} "
          f"(fp32 oracle {dc32:.2e}; {int((~ok).sum())} unresolvable cells, worst {dcell.max():.1e}) "
          f"rel dF={df:.2e}")
    assert dx <= max(2e-6, 2 * dx32), (dx, dx32)
    assert dc <= max(5e-6, 2 * dc32), (dc, dc32)
    assert (dcell > 1e-3).sum() == 0
    assert df <= 1e-6
    return dev["variant"]


# (config, users, inner iterations, NSW_MAIN_TILE, NSW_SPLIT_USERS, expected main (M, R, NT), tail (R, NT))
PRODUCTION = [
    ("cfg1", 12, 30, "8,64,6", 6, (11, 8, 64), (2, 256)),     # bench cfg1: main wave + concurrent tail
    ("cfg2", 6, 30, "4,256,1", 3, (21, 4, 256), (2, 512)),    # bench cfg2 main tile + its tail
    ("cfg3", 4, 30, "8,256,1", None, (11, 8, 256), None),     # cfg3 main tile (2048 rows: it is its own wide tile)
]


@pytest.mark.parametrize("name,users,T,main,split,want,tail", PRODUCTION)
def test_production_tile_one_step(monkeypatch, name, users, T, main, split, want, tail):
    monkeypatch.setenv("NSW_MAIN_TILE", main)
    if split is not None:
        monkeypatch.setenv("NSW_SPLIT_USERS", str(split))
    rel, expo, cfg = make_instance(name, seed=0, user_slice=(0, users))
    v = check_one_step(name, rel, expo, cfg.epsilon, T)
    assert (v["M"], v["R"], v["NT"]) == want
    if tail is not None:
        assert v.get("tail_users") == users - split
        assert (v["tail_R"], v["tail_NT"]) == tail
    else:
        assert "tail_users" not in v


@pytest.mark.parametrize("n,m,main", [(997, 21, "4,256,1"), (601, 17, "4,256,1"), (511, 11, "2,256,1")])
def test_wide_forward_ragged_one_step(monkeypatch, n, m, main):
    """The wide-row forward (half the warps, 2R rows each) on ragged shapes:
    n not a multiple of the tile's rows or of 4 (padding rows in both warp
    groups' row sets) and m below the tile's compile-time width (padding
    columns)."""
    monkeypatch.setenv("NSW_MAIN_TILE", main)
    monkeypatch.setenv("NSW_SPLIT_USERS", "5")   # 5 users on the forced tile (a lone 6th on the tail tile)
    rel, expo, cfg = make_instance("cfg2", seed=0, user_slice=(0, 6))
    rel = np.ascontiguousarray(rel[:, :n])
    expo = np.ascontiguousarray(expo[:m - 1])
    v = check_one_step(f"ragged-{n}x{m}", rel, expo, cfg.epsilon, 20)
    assert (v["R"], v["NT"]) == tuple(int(x) for x in main.split(",")[:2])
    assert v.get("tail_users", 0) <= 1


def test_cfg1_natural_tile_choice_one_step():
    """Full config-1 user count: the automatic choice is the bench's main tile
    on 888 users (6 per SM) plus a 112-user tail on the wide tile."""
    rel, expo, cfg = make_instance("cfg1", seed=0)
    v = check_one_step("cfg1-full", rel, expo, cfg.epsilon, 8, step=2)
    assert (v["M"], v["R"], v["NT"]) == (11, 8, 64)
    assert v.get("tail_users") == 112 and (v["tail_R"], v["tail_NT"]) == (2, 256)


def test_cfg2_natural_tile_choice_multi_wave_one_step():
    """Config 2 (the bench workload) on 600 users: the automatic choice is the
    bench's main tile over four whole waves (592 users, one CTA per SM) plus
    an 8-user tail on the wide tile -- the launch shape of the full 10 000-user
    run (67 waves + 84) at a size the oracle finishes in seconds."""
    rel, expo, cfg = make_instance("cfg2", seed=0, user_slice=(0, 600))
    v = check_one_step("cfg2-600", rel, expo, cfg.epsilon, 8, step=2)
    assert (v["M"], v["R"], v["NT"]) == (21, 4, 256)
    assert v.get("tail_users") == 8 and (v["tail_R"], v["tail_NT"]) == (2, 512)


def test_cfg4_cluster_tile_one_step():
    """Config-4 shape (4000 x 51, eps 0.01): the 9-CTA thread-block-cluster tile."""
    rel, expo, cfg = make_instance("cfg4", seed=0, user_slice=(0, 2))
    v = check_one_step("cfg4", rel, expo, cfg.epsilon, 30)
    assert v["M"] >= 51


@pytest.mark.parametrize("T", [30, 31, 29, 32])
def test_tensor_core_adjoint_cfg2_tile_one_step(monkeypatch, T):
    """The config-2 tile with the tensor-core adjoint (tcgen05 MMAs into TMEM,
    NSW_TC=1) and its concurrent tail; T = 29..32 ends the reverse sweep on
    every slot of the 4-level MMA chunk (short final chunks)."""
    monkeypatch.setenv("NSW_TC", "1")
    monkeypatch.setenv("NSW_MAIN_TILE", "4,256,1")
    monkeypatch.setenv("NSW_SPLIT_USERS", "3")
    rel, expo, cfg = make_instance("cfg2", seed=0, user_slice=(0, 6))
    v = check_one_step(f"cfg2-tc-T{T}", rel, expo, cfg.epsilon, T)
    assert (v["M"], v["R"], v["NT"]) == (21, 4, 256)
    assert v.get("tail_users") == 3


def test_tensor_core_adjoint_ragged_one_step(monkeypatch):
    """Tensor-core adjoint on a ragged shape: padding rows in the last
    128-row MMA block and padding columns in the accumulator."""
    monkeypatch.setenv("NSW_TC", "1")
    monkeypatch.setenv("NSW_MAIN_TILE", "4,256,1")
    monkeypatch.setenv("NSW_SPLIT_USERS", "5")
    rel, expo, cfg = make_instance("cfg2", seed=0, user_slice=(0, 6))
    rel = np.ascontiguousarray(rel[:, :997])
    expo = np.ascontiguousarray(expo[:16])
    v = check_one_step("ragged-tc-997x17", rel, expo, cfg.epsilon, 21)
    assert (v["R"], v["NT"]) == (4, 256)
