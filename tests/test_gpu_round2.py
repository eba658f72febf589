"""GPU parity, round 2 (VERDICT r1 "Next round"): the CUDA path through the C
ABI against the fp64 oracle at the BASELINE configs' stated parameters, the
beta variants / adaptive schedule / per-iteration trace against the oracle,
the solve-path rounding (G in U(r,c)), and the error paths (NaN injection).

Tolerances as in test_gpu_parity.py; stored
oracle solves come from tests/golden/*.json, written by scripts/make_golden.py
(which calls only oracle/).
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import synthetic as S

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_08507_b200 as M  # noqa: E402
from tests.test_gpu_parity import COST_GATE, DEV, _gates, _t  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        g = json.load(f)
    assert g["status"] == "OK" and g["generator"].startswith("scripts/make_golden.py")
    return g


def _oracle_l1(prob, inst, U, V, gb):
    lr, lc, st = O.log_marginals(prob, U, V, gb)
    assert st == 0
    return np.abs(np.exp(lr) - inst.r).sum() + np.abs(np.exp(lc) - inst.c).sum()


def _solve(inst, gb, T, eps, **kw):
    U = torch.empty(inst.n, dtype=torch.float64, device=DEV)
    V = torch.empty_like(U)
    sched = kw.pop("sched", None) or M.schedule(M.MDOT_SCHED_FIXED, gb, T=T)
    P = kw.pop("P_out", None)
    opts = kw.pop("opts", None) or M.options(eps=eps, **kw)
    res = M.mdot_solve(_t(inst.C), _t(inst.r), _t(inst.c), schedule=sched, options=opts, u_out=U, v_out=V,
                       P_out=P)
    return res, U.cpu().numpy(), V.cpu().numpy()


# ------------------------------------------------------------ rounding
@pytest.mark.parametrize("n", [2048, 300])
def test_solve_path_rounding_is_feasible_and_matches_oracle(n):
    """a10 on the solve path: x is computed from an exact fp64 r(F), so the
    rounded plan G lies in U(r,c): G >= 0, its
    marginals equal r and c to the fp32 resolution of the dense output, and the
    rounded cost equals the oracle's rounding of the SAME (U, V) to 1e-10.
    n = 2048: the persistent grid path with a dense P_out; n = 300: the one-CTA
    K8 route (no P_out)."""
    inst = S.config4(2, n=n)
    eps, gb = 1e-6, 4096.0
    P = torch.empty((n, n), dtype=torch.float32, device=DEV) if n > 512 else None
    res, U, V = _solve(inst, gb, 16, eps, P_out=P)
    assert res["status"] == 0 and res["l1_final"] <= eps
    assert res["control_path"] == (2 if n > 512 else 3)
    prob = O.OracleProblem(inst)
    rp = O.round_plan(prob, U, V, gb)
    assert abs(res["cost_rounded"] - rp["cost_G"]) <= 1e-10 * rp["cost_G"], (res["cost_rounded"], rp["cost_G"])
    assert abs(res["cost_unrounded"] - rp["cost_F"]) <= 1e-10 * rp["cost_F"]
    if P is not None:
        G = P.double().cpu().numpy()
        assert G.min() >= 0.0
        np.testing.assert_allclose(G.sum(1), inst.r, rtol=2e-6, atol=1e-12)
        np.testing.assert_allclose(G.sum(0), inst.c, rtol=2e-6, atol=1e-12)


# ------------------------------------------------------------ beta variants / NCG
@pytest.mark.parametrize("beta,projector,n", [(M.MDOT_BETA_PPR_AF, 0, 600), (M.MDOT_BETA_PFR, 0, 600),
                                              (M.MDOT_BETA_PPR_PLUS, 0, 600), (M.MDOT_BETA_PPR_PLUS, 0, 300),
                                              (M.MDOT_BETA_PFR, 0, 300), (M.MDOT_BETA_PPR, 2, 300)])
def test_beta_variants_and_ncg_match_oracle(beta, projector, n):
    """PPR with the Al-Baali-Fletcher denominator, preconditioned FR
    (PAPER.md:496-498), PR+ and vanilla NCG on the CUDA
    path (n = 600: persistent kernel; n = 300: K8 route) against the oracle's
    same variant (Z20 gates)."""
    inst = S.uniform_points_instance(3, n, 2, 60 + n % 7 + beta, marg="dirichlet")
    prob = O.OracleProblem(inst)
    eps, gb, T = 1e-6, 512.0, 4
    res, U, V = _solve(inst, gb, T, eps, beta=beta, projector=projector)
    obeta = {M.MDOT_BETA_PPR: O.BETA_PPR, M.MDOT_BETA_PPR_AF: O.BETA_PPR_AF, M.MDOT_BETA_PFR: O.BETA_PFR,
             M.MDOT_BETA_PPR_PLUS: O.BETA_PPR_PLUS}[beta]
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=T),
                             O.make_options(eps=eps, beta=obeta, projector=O.NCG if projector == 2 else O.PNCG))
    _gates(res, ores, inst, prob, U, V, eps)


# ------------------------------------------------------------ per-iteration trace
@pytest.mark.parametrize("route", ["host", "graph", "k8"])
def test_trace_matches_oracle_in_fp64_entry_mode(route, monkeypatch):
    """SolveTrace: with fp64 entries the CUDA controller and
    the oracle run the same algorithm on marginals equal to ~1e-15, so the
    first iterations' beta, alpha, phi'(0), phi'(alpha) and trial counts must
    agree (host loop, CUDA-graph device control, the one-CTA K8 route)."""
    n = 200
    inst = S.uniform_points_instance(3, n, 2, 70, marg="dirichlet")
    prob = O.OracleProblem(inst)
    gb, eps = 256.0, 1e-9
    if route == "graph":
        monkeypatch.setenv("MDOT_SMALL_N", "0")
    opts = M.options(eps=eps, precision=M.MDOT_PREC_F64P, device_control=0 if route == "host" else 1,
                     trace_cap=4096)
    res, U, V = _solve(inst, gb, 1, eps, opts=opts)
    assert res["status"] == 0
    assert res["control_path"] == {"host": 0, "graph": 1, "k8": 3}[route]
    tr = M.read_trace(opts)
    assert len(tr) == res["iterations"]
    _, _, ores, otr = O.mdot(prob, [gb], O.make_options(eps=eps), trace_cap=100000)
    K = 8
    for q, o in zip(tr[:K], otr[:K]):
        assert (q["t"], q["k"], q["trials"], q["reset"]) == (o["t"], o["k"], o["trials"], o["reset"]), (q, o)
        for f in ("alpha", "dphi0", "dphi_alpha", "gs", "l1"):
            assert abs(q[f] - o[f]) <= 1e-7 * abs(o[f]) + 1e-14, (f, q, o)
        assert abs(q["beta"] - o["beta"]) <= 1e-7 * abs(o["beta"]) + 1e-12, (q, o)


@pytest.mark.parametrize("n", [300, 1024])
def test_trace_direction_update_identity_on_gpu(n):
    """On the fp32-entry path (K8 route / persistent kernel) the traced scalars
    obey <p_k, g_k> = -<g_k, s_k> + beta_k phi'_{k-1}(alpha) (Alg. 2 line 6):
    the controller's direction, gradient reuse and trace are consistent."""
    inst = S.uniform_points_instance(3, n, 2, 71, marg="dirichlet")
    opts = M.options(eps=1e-6, trace_cap=1 << 16)
    res, U, V = _solve(inst, 1024.0, 4, 1e-6, opts=opts)
    assert res["status"] == 0
    tr = M.read_trace(opts)
    assert len(tr) == res["iterations"] and tr[0]["beta"] == 0.0
    checked = 0
    for prev, q in zip(tr, tr[1:]):
        if q["t"] != prev["t"] or q["reset"]:
            continue
        rhs = -q["gs"] + q["beta"] * prev["dphi_alpha"]
        assert abs(q["dphi0"] - rhs) <= 1e-9 * (abs(q["gs"]) + abs(q["beta"] * prev["dphi_alpha"])), (q, prev)
        assert q["dphi0"] < 0 and (2 * 0.1 - 1) * q["dphi0"] >= q["dphi_alpha"] >= 0.4 * q["dphi0"]
        checked += 1
    assert checked >= 10


# ------------------------------------------------------------ adaptive gamma
@pytest.mark.parametrize("n", [300, 1000])
def test_adaptive_schedule_matches_oracle(n):
    """MDOT_SCHED_ADAPTIVE (Z29): the realised steps sum to gbar
    exactly; by Lemma 2 the plan is the entropic plan at gbar, so the cost
    matches the oracle's fixed-schedule AND adaptive solves (Z20 gates)."""
    inst = S.uniform_points_instance(3, n, 2, 72, marg="dirichlet")
    prob = O.OracleProblem(inst)
    eps, gb = 1e-6, 4096.0
    res, U, V = _solve(inst, gb, 0, eps, sched=M.schedule(M.MDOT_SCHED_ADAPTIVE, gb, step_max=128.0))
    g = np.array(res["gammas"])
    assert res["status"] == 0 and g.sum() == gb and res["gamma_bar"] == gb and g[0] == 128.0 and len(g) >= 3
    Uo, Vo, ores, _, og = O.mdot_adaptive(prob, gb, 128.0, O.make_options(eps=eps))
    _gates(res, ores, inst, prob, U, V, eps)
    Uf, Vf, fres, _ = O.mdot(prob, O.schedule_fixed(gb), O.make_options(eps=eps))
    _gates(res, fres, inst, prob, U, V, eps)


# ------------------------------------------------------------ BASELINE configs at their stated parameters
@pytest.mark.parametrize("frac", [0.5, 0.9, 0.99])
def test_config3_at_baseline_parameters_against_stored_oracle_solve(frac):
    """BASELINE config 3 (n = 4096, H(r)/log n = frac, gbar 4096, T = 16, L1
    1e-6): the GPU solve against the stored full oracle
    solve (tests/golden): unrounded cost within 1e-5 (Z20 (i)), the oracle's
    re-evaluation of the GPU potentials within 2 eps, rounded cost within the
    Z20 (iii) allowance.  Also PNCG vs Sinkhorn on the same kernels."""
    g = _golden(f"cfg3_h{frac}_seed0")
    inst = S.config3(0, frac=frac)
    eps, gb = 1e-6, 4096.0
    res, U, V = _solve(inst, gb, 16, eps)
    assert res["status"] == 0 and res["l1_final"] <= eps
    rel = abs(res["cost_unrounded"] - g["cost_unrounded"]) / g["cost_unrounded"]
    assert rel <= 1e-5, (res["cost_unrounded"], g["cost_unrounded"])
    prob = O.OracleProblem(inst)
    assert _oracle_l1(prob, inst, U, V, gb) <= 2 * eps
    allow = max(1e-5 * g["cost_rounded"], 2 * (res["l1_final"] + g["l1_final"]) * float(inst.C.max()))
    assert abs(res["cost_rounded"] - g["cost_rounded"]) <= allow


def test_config3_secondary_gbar512_T4_against_stored_oracle_solve():
    g = _golden("cfg3_h0.5_gb512_T4_seed1")
    inst = S.config3(1, frac=0.5)
    eps, gb = 1e-6, 512.0
    for sink in (False, True):
        U = torch.empty(inst.n, dtype=torch.float64, device=DEV)
        V = torch.empty_like(U)
        fn = M.mdot_sinkhorn if sink else M.mdot_solve
        res = fn(_t(inst.C), _t(inst.r), _t(inst.c), schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=4),
                 options=M.options(eps=eps), u_out=U, v_out=V)
        assert res["status"] == 0 and res["l1_final"] <= eps
        assert abs(res["cost_unrounded"] - g["cost_unrounded"]) <= 1e-5 * g["cost_unrounded"]


def test_config4_headline_against_stored_oracle_solve():
    """BASELINE config 4 exactly as bench.py times it (n = 16384, 1 GiB C,
    gbar 4096, T = 16, L1 1e-6) against the stored FULL oracle solve
    (tests/golden/cfg4_seed0.json, Z20 (i) and (iii))."""
    g = _golden("cfg4_seed0")
    inst = S.config4(0)
    eps, gb = 1e-6, 4096.0
    res, U, V = _solve(inst, gb, 16, eps)
    assert res["status"] == 0 and res["control_path"] == 2 and res["l1_final"] <= eps
    rel = abs(res["cost_unrounded"] - g["cost_unrounded"]) / g["cost_unrounded"]
    assert rel <= 1e-5, (res["cost_unrounded"], g["cost_unrounded"], rel)
    allow = max(1e-5 * g["cost_rounded"], 2 * (res["l1_final"] + g["l1_final"]) * 1.0)
    assert abs(res["cost_rounded"] - g["cost_rounded"]) <= allow


def test_config2_eps1e8_at_baseline_parameters_against_stored_oracle_solves():
    """BASELINE config 2 at eps 1e-8 with gbar 4096, T = 16 (fp64-entry K8
    batch): two blob pairs against their stored oracle solves, and the
    oracle's re-evaluation of the GPU potentials within 2 eps."""
    eps, gb = 1e-8, 4096.0
    pairs = [S.config2_pair(0, 0), S.config2_pair(0, 1)]
    C = pairs[0].C
    R = np.ascontiguousarray(np.stack([p.r for p in pairs]))
    Cm = np.ascontiguousarray(np.stack([p.c for p in pairs]))
    U = torch.empty((2, 784), dtype=torch.float64, device=DEV)
    V = torch.empty_like(U)
    res = M.mdot_solve_batch(_t(C), _t(R), _t(Cm), schedule=M.schedule(M.MDOT_SCHED_FIXED, gb, T=16),
                             options=M.options(eps=eps), u_out=U, v_out=V)
    for b, inst in enumerate(pairs):
        g = _golden(f"cfg2_s0_p{b}_eps1e-8")
        assert res[b]["status"] == 0 and res[b]["control_path"] == 3 and res[b]["l1_final"] <= eps
        assert abs(res[b]["cost_unrounded"] - g["cost_unrounded"]) <= 1e-5 * g["cost_unrounded"]
        # at eps <= 1e-8 the rounded costs agree to 1e-5 too (Z20 (ii))
        assert abs(res[b]["cost_rounded"] - g["cost_rounded"]) <= 1e-5 * g["cost_rounded"]
        prob = O.OracleProblem(inst)
        assert _oracle_l1(prob, inst, U[b].cpu().numpy(), V[b].cpu().numpy(), gb) <= 2 * eps


@pytest.mark.parametrize("recipe", ["diff", "dot"])
def test_config5_full_size_at_baseline_parameters_oracle_reevaluation(recipe):
    """BASELINE config 5 at its stated parameters (n = 65536, d = 16, C on the
    fly, gbar 4096, T = 16, L1 1e-5): the oracle re-evaluates the GPU
    potentials over the WHOLE matrix with the same fp32 cost recipe (Z22
    difference form, Z22b dot form -- the one bench.py times): marginal L1
    within max(2 eps, 1e-6) and <C, P(U,V)> within 1e-9 of the GPU's."""
    inst = S.config5(0)
    n = inst.n
    U = torch.empty(n, dtype=torch.float64, device=DEV)
    V = torch.empty_like(U)
    eps, gb = 1e-5, 4096.0
    res = M.mdot_solve(X=_t(inst.X), Y=_t(inst.Y), scale=inst.scale, r=_t(inst.r), c=_t(inst.c),
                       schedule=M.schedule(M.MDOT_SCHED_FIXED, gb), options=M.options(eps=eps), u_out=U, v_out=V,
                       recipe=recipe)
    assert res["status"] == 0 and res["md_steps"] == 16 and res["l1_final"] <= eps
    prob = O.OracleProblem(inst, recipe=recipe)
    Un, Vn = U.cpu().numpy(), V.cpu().numpy()
    assert _oracle_l1(prob, inst, Un, Vn, gb) <= max(2 * eps, 1e-6)
    cF = O.plan_cost(prob, Un, Vn, gb)
    assert abs(res["cost_unrounded"] - cF) <= 1e-9 * cF, (res["cost_unrounded"], cF)


# ------------------------------------------------------------ error paths
@pytest.mark.parametrize("n", [300, 1024])
def test_nan_injection_range_guard_recovers(n, monkeypatch):
    """MDOT_FAULT_NAN=1 poisons one partial total of the first fp32-entry
    evaluation: the range guard must send that evaluation to the exact fp64
    evaluator (fallbacks >= 1 on the grid path) and the solve still meets the
    oracle gates."""
    monkeypatch.setenv("MDOT_FAULT_NAN", "1")
    inst = S.uniform_points_instance(3, n, 2, 73, marg="dirichlet")
    prob = O.OracleProblem(inst)
    res, U, V = _solve(inst, 512.0, 2, 1e-6)
    monkeypatch.setenv("MDOT_FAULT_NAN", "0")
    if n > 512:
        assert res["fallbacks"] >= 1
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(512.0, T=2), O.make_options(eps=1e-6))
    _gates(res, ores, inst, prob, U, V, 1e-6)


@pytest.mark.parametrize("n,dc", [(300, 1), (1024, 1), (1024, 0), (1024, 2)])
def test_nan_injection_persistent_failure_returns_einstable(n, dc, monkeypatch):
    """MDOT_FAULT_NAN=2: a marginal stays NaN even on the exact evaluator -> the
    call returns MDOT_EINSTABLE (SPEC exit 3) promptly on every control path
    (K8, persistent kernel, host loop, graph slots) instead of hanging."""
    monkeypatch.setenv("MDOT_FAULT_NAN", "2")
    if dc == 2:
        monkeypatch.setenv("MDOT_NO_PERSIST", "1")
    inst = S.uniform_points_instance(3, n, 2, 74, marg="dirichlet")
    with pytest.raises(M.MdotError) as e:
        _solve(inst, 512.0, 2, 1e-6, device_control=min(dc, 1))
    monkeypatch.setenv("MDOT_FAULT_NAN", "0")
    assert e.value.status == 3
    # the library is usable afterwards
    res, U, V = _solve(inst, 512.0, 2, 1e-6)
    assert res["status"] == 0


def test_lockstep_batch_matches_single_solves_and_oracle(monkeypatch):
    """Throughput mode, lockstep variant (MDOT_BATCH_LOCKSTEP=1: one launch per
    phase for every instance sharing C, a persistent K1 over the virtual
    (instance, tile) list): each instance against its own
    single solve (Z20 gate) and one against the oracle."""
    monkeypatch.setenv("MDOT_BATCH_LOCKSTEP", "1")
    n, B, gb, T, eps = 1000, 4, 1024.0, 4, 1e-6
    base = S.uniform_points_instance(3, n, 2, 90, marg="dirichlet")
    R = np.stack([S.uniform_points_instance(3, n, 2, 90 + b, marg="dirichlet").r for b in range(B)])
    Cm = np.stack([S.uniform_points_instance(3, n, 2, 95 + b, marg="dirichlet").c for b in range(B)])
    U = torch.empty((B, n), dtype=torch.float64, device=DEV)
    V = torch.empty_like(U)
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=T)
    res = M.mdot_solve_batch(_t(base.C), _t(R), _t(Cm), schedule=sched, options=M.options(eps=eps),
                             u_out=U, v_out=V)
    assert all(x["status"] == 0 and x["control_path"] == 4 and x["l1_final"] <= eps for x in res)
    monkeypatch.setenv("MDOT_BATCH_LOCKSTEP", "0")
    for b in range(B):
        rs = M.mdot_solve(_t(base.C), _t(R[b]), _t(Cm[b]), schedule=sched, options=M.options(eps=eps))
        assert abs(res[b]["cost_unrounded"] - rs["cost_unrounded"]) <= COST_GATE * rs["cost_unrounded"]
    inst = S.Instance(n, R[1], Cm[1], C=base.C)
    prob = O.OracleProblem(inst)
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=T), O.make_options(eps=eps))
    _gates(res[1], ores, inst, prob, U[1].cpu().numpy(), V[1].cpu().numpy(), eps)
