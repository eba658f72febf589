"""K2s -- the screened on-the-fly evaluation (csrc/screen.cu, DESIGN.md
"Screened K2") -- against the fp64 oracle and against the dense K2.

The screen skips entries below 2^-T (T = 48) of both their row and column
totals (a rigorous bound, Z30), so every solve gate of the dense
path (tests/test_gpu_parity.py _gates: cost within 1e-5 of the oracle's solve,
the oracle's fp64 re-evaluation of the GPU potentials within 2 eps) must hold
unchanged.  MDOT_SCREEN_FMAX=2 forces the screened kernel at every density
(the solver would otherwise fall back to K2 where it keeps more than 0.8 %
of the entries), so the list path, the dense-region path and short tiles are
all exercised."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import synthetic as S
import paper_2307_08507_b200 as M
from tests.test_gpu_parity import DEV, _gates, _t

pytestmark = pytest.mark.gpu


@pytest.fixture
def forced_screen(monkeypatch):
    monkeypatch.setenv("MDOT_SCREEN", "1")
    monkeypatch.setenv("MDOT_SCREEN_FMAX", "2")
    yield


def _solve(inst, gb, T, eps, recipe):
    U = torch.empty(inst.n, dtype=torch.float64, device=DEV)
    V = torch.empty_like(U)
    res = M.mdot_solve(X=_t(inst.X), Y=_t(inst.Y), scale=inst.scale, r=_t(inst.r), c=_t(inst.c),
                       schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=T), options=M.options(eps=eps),
                       u_out=U, v_out=V, recipe=recipe)
    torch.cuda.synchronize()
    return res, U.cpu().numpy(), V.cpu().numpy(), M.mdot_last_screen_stats()


@pytest.mark.parametrize("n,d,recipe,gb,T", [
    (1500, 16, "dot", 2048.0, 4),    # ragged columns (5 x 256 + 220), 2 chunks of the 512-row tiles
    (1000, 8, "diff", 2048.0, 4),    # the difference-form recipe, d = 8
    (600, 4, "dot", 1024.0, 2),      # row tiles shorter than the 128-row MMA chunk (masked lanes), d = 4
])
def test_screened_solve_matches_oracle(forced_screen, n, d, recipe, gb, T):
    inst = S.config5(2, n=n, d=d)
    prob = O.OracleProblem(inst, recipe=recipe)
    eps = 1e-5
    res, U, V, st = _solve(inst, gb, T, eps, recipe)
    assert st["evals"] > 0, st                       # K2s ran
    assert st["kept_frac"] is not None and st["kept_frac"] < 0.9, st   # ... and skipped entries
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=T), O.make_options(eps=eps))
    _gates(res, ores, inst, prob, U, V, eps)


def test_screened_and_dense_solves_agree(monkeypatch):
    """Config-5-shaped instance at the BASELINE gbar: the screened solve and
    the dense one reach the same plan (cost within the 1e-5 gate, each at its
    own L1 <= eps) and the screen keeps well under 1 % of the entries."""
    inst = S.config5(3, n=4096, d=16)
    eps = 1e-5
    monkeypatch.setenv("MDOT_SCREEN", "0")
    rd, Ud, Vd, _ = _solve(inst, 4096.0, 16, eps, "dot")
    monkeypatch.setenv("MDOT_SCREEN", "1")
    rs, Us, Vs, st = _solve(inst, 4096.0, 16, eps, "dot")
    assert rd["status"] == 0 and rs["status"] == 0, (rd, rs)
    assert rs["l1_final"] <= eps and rd["l1_final"] <= eps
    assert abs(rs["cost_unrounded"] - rd["cost_unrounded"]) <= 1e-5 * rd["cost_unrounded"]
    assert st["evals"] > 0 and st["kept_frac"] < 0.01, st
    # the oracle's fp64 re-evaluation of the screened solve's potentials (all n^2 entries)
    prob = O.OracleProblem(inst, recipe="dot")
    lr, lc, _ = O.log_marginals(prob, Us, Vs, rs["gamma_bar"])
    l1 = np.abs(np.exp(lr) - inst.r).sum() + np.abs(np.exp(lc) - inst.c).sum()
    assert l1 <= 2 * eps, l1


def test_screen_disabled_is_the_dense_kernel(monkeypatch):
    """MDOT_SCREEN=0 leaves the dense path bit for bit (no screened evaluation)."""
    inst = S.config5(4, n=1024, d=16)
    monkeypatch.setenv("MDOT_SCREEN", "0")
    r1, U1, _, st = _solve(inst, 2048.0, 4, 1e-5, "dot")
    assert st["evals"] == 0
    r2, U2, _, _ = _solve(inst, 2048.0, 4, 1e-5, "dot")
    assert np.array_equal(U1, U2) and r1["evaluations"] == r2["evaluations"]


def test_screened_sharded_nccl_one_rank(forced_screen, monkeypatch):
    """Row-sharded path (the config-5 multi-GPU layout) with K2s: a 1-rank NCCL
    communicator forced onto the sharded code (MDOT_SHARDED_SELFTEST) runs the
    graph slots with the allreduced screen bound and decisions; gates against
    the oracle."""
    monkeypatch.setenv("MDOT_SHARDED_SELFTEST", "1")
    n, d, gb, T, eps = 1200, 16, 2048.0, 4, 1e-5
    inst = S.config5(5, n=n, d=d)
    r, c = _t(inst.r), _t(inst.c)
    comm = M.mdot_comm_create(M.mdot_get_unique_id(), 1, 0, 0)
    try:
        U = torch.empty(n, dtype=torch.float64, device=DEV)
        V = torch.empty_like(U)
        res = M.mdot_solve_sharded(comm, 0, n, X_local=_t(inst.X), Y=_t(inst.Y), scale=float(inst.scale), r=r, c=c,
                                   n=n, schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=T),
                                   options=M.options(eps=eps), u_local_out=U, v_out=V, recipe="dot")
        torch.cuda.synchronize()
        st = M.mdot_last_screen_stats()
    finally:
        M.mdot_comm_destroy(comm)
    assert res["control_path"] == 1, res["control_path"]
    assert st["evals"] > 0 and st["kept_frac"] < 0.9, st
    prob = O.OracleProblem(inst, recipe="dot")
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=T), O.make_options(eps=eps))
    _gates(res, ores, inst, prob, U.cpu().numpy(), V.cpu().numpy(), eps)


@pytest.mark.parametrize("projector", ["sinkhorn", "ncg"])
def test_screened_other_projectors_match_oracle(forced_screen, projector):
    """The graph slots of Alg. 3 (Sinkhorn half-steps: only one side's
    potentials move, the other side's shift is 0) and of vanilla NCG use K2s
    like PNCG; gates against the oracle's same projector."""
    n, d, gb, T, eps = 800, 8, 1024.0, 2, 1e-5
    inst = S.config5(6, n=n, d=d)
    prob = O.OracleProblem(inst, recipe="dot")
    U = torch.empty(n, dtype=torch.float64, device=DEV)
    V = torch.empty_like(U)
    if projector == "sinkhorn":
        res = M.mdot_sinkhorn(X=_t(inst.X), Y=_t(inst.Y), scale=inst.scale, r=_t(inst.r), c=_t(inst.c),
                              schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=T), options=M.options(eps=eps),
                              u_out=U, v_out=V, recipe="dot")
        oopts = O.make_options(eps=eps, projector=O.SINKHORN)
    else:
        res = M.mdot_solve(X=_t(inst.X), Y=_t(inst.Y), scale=inst.scale, r=_t(inst.r), c=_t(inst.c),
                           schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=T),
                           options=M.options(eps=eps, projector=M.MDOT_PROJ_NCG), u_out=U, v_out=V, recipe="dot")
        oopts = O.make_options(eps=eps, projector=O.NCG)
    torch.cuda.synchronize()
    st = M.mdot_last_screen_stats()
    assert st["evals"] > 0, st
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=T), oopts)
    _gates(res, ores, inst, prob, U.cpu().numpy(), V.cpu().numpy(), eps)


def test_screened_adaptive_schedule_matches_oracle(forced_screen):
    """MDOT_SCHED_ADAPTIVE (Z29) realises its steps on the fly; every
    projection after the first runs K2s (forced); Lemma 2 fixes the plan."""
    n, d, gb, eps = 1000, 16, 2048.0, 1e-5
    inst = S.config5(7, n=n, d=d)
    prob = O.OracleProblem(inst, recipe="dot")
    U = torch.empty(n, dtype=torch.float64, device=DEV)
    V = torch.empty_like(U)
    res = M.mdot_solve(X=_t(inst.X), Y=_t(inst.Y), scale=inst.scale, r=_t(inst.r), c=_t(inst.c),
                       schedule=M.schedule(M.MDOT_SCHED_ADAPTIVE, gb, step_max=256.0), options=M.options(eps=eps),
                       u_out=U, v_out=V, recipe="dot")
    torch.cuda.synchronize()
    st = M.mdot_last_screen_stats()
    assert st["evals"] > 0, st
    Uf, Vf, fres, _ = O.mdot(prob, O.schedule_fixed(gb, T=8), O.make_options(eps=eps))
    _gates(res, fres, inst, prob, U.cpu().numpy(), V.cpu().numpy(), eps)


@pytest.mark.parametrize("recipe", ["dot", "diff"])
def test_screened_non_power_of_two_scale(forced_screen, recipe):
    """A cost scale that is not a power of two (0.1): the recipe multiplies
    C~ by the scale (no fold into gh / gl) in K2s's exact path as in K2."""
    import dataclasses
    n, d, gb, T, eps = 700, 8, 1024.0, 2, 1e-5
    inst = dataclasses.replace(S.config5(8, n=n, d=d), scale=0.1)
    prob = O.OracleProblem(inst, recipe=recipe)
    res, U, V, st = _solve(inst, gb, T, eps, recipe)
    assert st["evals"] > 0, st
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=T), O.make_options(eps=eps))
    _gates(res, ores, inst, prob, U, V, eps)
