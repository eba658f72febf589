"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Each test names the passage it pins.  None of them re-types the oracle's own
formula: they use closed forms, exact OT values, invariants and brute force.
"""
import math

import numpy as np
import pytest

import oracle as O
import synthetic as S
from tests import exact_ot as X


def _dense_C(prob):
    n = prob.n
    if prob.C is not None:
        return prob.C.astype(np.float64)
    return np.array([[prob.cost(i, j) for j in range(n)] for i in range(n)])


# ---------------------------------------------------------------- evaluation
def test_log_marginals_direct_sum():
    """r(P)=P1, c(P)=P^T1 for P=exp(A+B-gC); compare to a
    direct fp64 sum of the explicit matrix (no log-sum-exp)."""
    inst = S.random_small(13, seed=3)
    prob = O.OracleProblem(inst)
    rng = np.random.default_rng(0)
    A = rng.normal(size=13) - 3
    B = rng.normal(size=13) - 2
    g = 7.5
    P = np.exp(A[:, None] + B[None, :] - g * inst.C)
    lr, lc, st = O.log_marginals(prob, A, B, g)
    assert st == 0
    np.testing.assert_allclose(np.exp(lr), P.sum(1), rtol=1e-14)
    np.testing.assert_allclose(np.exp(lc), P.sum(0), rtol=1e-14)


def test_log_marginals_shift_invariance_and_extremes():
    """PAPER.md:231 gauge: (A+d, B-d) gives the same P.  Log domain must also
    survive exponents far outside fp64 exp range (A34; SPEC criterion 13 is
    inverted for a log-domain build)."""
    inst = S.random_small(17, seed=4)
    prob = O.OracleProblem(inst)
    rng = np.random.default_rng(1)
    A = rng.normal(size=17)
    B = rng.normal(size=17)
    lr0, lc0, _ = O.log_marginals(prob, A, B, 3.0)
    for d in (-10.0, 3.7, 10.0):
        lr, lc, _ = O.log_marginals(prob, A + d, B - d, 3.0)
        np.testing.assert_allclose(lr, lr0, atol=1e-12)
        np.testing.assert_allclose(lc, lc0, atol=1e-12)
    # huge gamma: exp(-4096 C) underflows fp64 for most entries; LSE must not.
    lr, lc, st = O.log_marginals(prob, A + 2000, B + 1000, 4096.0)
    assert st == 0 and np.all(np.isfinite(lr)) and np.all(np.isfinite(lc))


def test_rank_one_marginals_closed_form():
    """gbar = 0: P = e^A e^B^T is rank one, r(P) = e^A sum(e^B)."""
    inst = S.random_small(9, seed=5)
    prob = O.OracleProblem(inst)
    A = np.linspace(-3, 2, 9)
    B = np.linspace(1, -1, 9)
    lr, lc, _ = O.log_marginals(prob, A, B, 0.0)
    np.testing.assert_allclose(lr, A + np.log(np.exp(B).sum()), atol=1e-14)
    np.testing.assert_allclose(lc, B + np.log(np.exp(A).sum()), atol=1e-14)


def test_cost_sqeuclid_recipe_is_fp32_fma_chain():
    """DESIGN.md Z22: on-the-fly C is the fixed fp32 recipe; check against a
    numpy float32 emulation (fma emulated exactly via float64 arithmetic:
    d*d + acc is exact in fp64 for fp32 operands, then rounded once)."""
    inst = S.config5(0, n=64, d=16)
    prob = O.OracleProblem(inst)
    for (i, j) in [(0, 0), (3, 7), (63, 1), (10, 10)]:
        acc = np.float32(0.0)
        for k in range(16):
            dk = np.float32(inst.X[i, k] - inst.Y[j, k])
            acc = np.float32(np.float64(dk) * np.float64(dk) + np.float64(acc))
        ref = np.float32(acc * np.float32(1.0 / 16))
        assert prob.cost(i, j) == float(ref)


# --------------------------------------------------------------- divergences
def test_rho_worked_example_two_rc():
    """SPEC.md:84 (P = 2 r c^T) with D_h(y|x)=sum x - y + y log(y/x)
    (PAPER.md:82): rho = 2 (2 ln2 - 1) (SPEC.md:73 example doubled)."""
    inst = S.random_small(6, seed=6)
    prob = O.OracleProblem(inst)
    U = np.log(inst.r) + math.log(2.0)
    V = np.log(inst.c)
    # gbar = 0 so P = exp(U+V) = 2 r c^T; eps huge -> no iteration
    _, _, res, _ = O.project(prob, U, V, 0.0, opts=O.make_options(eps=1e9))
    assert res["iterations"] == 0
    assert abs(res["rho_final"] - 2 * (2 * math.log(2) - 1)) < 1e-14
    assert abs(res["l1_final"] - 2.0) < 1e-14


def test_descent_identity_first_direction():
    """<s, grad g> = D(r(P)|r)+D(r|r(P))+D(c(P)|c)+D(c|c(P)).
    The first PNCG direction is p = -s (beta_1 = 0), so the
    traced phi'(0) = <p, grad> must equal minus the four-divergence sum,
    computed here from independently obtained marginals."""
    inst = S.random_small(20, seed=7)
    prob = O.OracleProblem(inst)
    rng = np.random.default_rng(2)
    U = np.log(inst.r) + 0.3 * rng.normal(size=20)
    V = np.log(inst.c) + 0.3 * rng.normal(size=20)
    g = 5.0
    P = np.exp(U[:, None] + V[None, :] - g * inst.C)
    rP, cP = P.sum(1), P.sum(0)
    r, c = inst.r, inst.c

    def D(y, x):
        return float(np.sum(x - y + y * np.log(y / x)))

    four = D(rP, r) + D(r, rP) + D(cP, c) + D(c, cP)
    _, _, res, tr = O.project(prob, U, V, g, opts=O.make_options(eps=1e-9, max_evals=6),
                              trace_cap=10)
    assert tr, "no iteration traced"
    assert tr[0]["reset"] == 0 and tr[0]["beta"] == 0.0
    assert abs(tr[0]["dphi0"] + four) < 1e-12 * max(1.0, four)


def test_phi_prime_matches_finite_difference():
    """phi'(alpha) equals the derivative of the dual objective
    g(u,v) = sum P - <u,r> - <v,c> - 1 along p; checked with a
    central difference of g built from a direct dense sum."""
    n = 12
    inst = S.random_small(n, seed=8)
    prob = O.OracleProblem(inst)
    g = 4.0
    U, V = np.log(inst.r), np.log(inst.c)
    u0 = np.zeros(n)
    v0 = np.zeros(n)
    _, _, res, tr = O.project(prob, U, V, g, u0, v0, opts=O.make_options(eps=1e-9, max_evals=4),
                              trace_cap=4)
    # direction of the first iteration is -s at (u0, v0):
    P = np.exp(U[:, None] + V[None, :] - g * inst.C)
    s = np.concatenate([np.log(P.sum(1)) - np.log(inst.r), np.log(P.sum(0)) - np.log(inst.c)])
    p = -s

    def gobj(a):
        uu = u0 + a * p[:n]
        vv = v0 + a * p[n:]
        Pa = np.exp((U + uu)[:, None] + (V + vv)[None, :] - g * inst.C)
        return Pa.sum() - uu @ inst.r - vv @ inst.c - 1.0

    h = 1e-6
    fd0 = (gobj(h) - gobj(-h)) / (2 * h)
    assert abs(tr[0]["dphi0"] - fd0) <= 1e-6 * abs(fd0)
    a = tr[0]["alpha"]
    fda = (gobj(a + h) - gobj(a - h)) / (2 * h)
    assert abs(tr[0]["dphi_alpha"] - fda) <= 1e-6 * max(abs(fda), 1e-8) + 1e-9
    # phi(alpha) - phi(0) as traced
    assert abs(tr[0]["dphi_value"] - (gobj(a) - gobj(0.0))) < 1e-12


# ------------------------------------------------------------ projections
def test_2x2_closed_form():
    """SURVEY 8(c) 2x2 closed form of the entropic plan at gbar (Lemma 2
    reduces MD with P0 = r c^T to entropic OT)."""
    rng = np.random.default_rng(11)
    for trial in range(20):
        C = rng.uniform(0, 1, size=(2, 2))
        r = rng.dirichlet([1, 1])
        c = rng.dirichlet([1, 1])
        gbar = [1.0, 8.0, 64.0, 200.0][trial % 4]
        prob = O.OracleProblem(C=C, r=r, c=c)
        for proj in (O.PNCG, O.SINKHORN):
            U, V, res, _ = O.mdot(prob, [gbar], O.make_options(eps=1e-14, projector=proj))
            assert res["status"] == 0, res
            P = np.exp(U[:, None] + V[None, :] - gbar * C)
            Pref = X.entropic_2x2(C, r, c, gbar)
            np.testing.assert_allclose(P, Pref, atol=1e-13)


def test_sinkhorn_and_pncg_same_fixed_point():
    """Uniqueness of the Bregman projection."""
    inst = S.random_small(24, seed=12)
    prob = O.OracleProblem(inst)
    U, V = np.log(inst.r), np.log(inst.c)
    g = 30.0
    u1, v1, r1, _ = O.project(prob, U, V, g, opts=O.make_options(eps=1e-13, projector=O.PNCG))
    u2, v2, r2, _ = O.project(prob, U, V, g, opts=O.make_options(eps=1e-13, projector=O.SINKHORN))
    u3, v3, r3, _ = O.project(prob, U, V, g, opts=O.make_options(eps=1e-13, projector=O.NCG))
    assert r1["status"] == 0 and r2["status"] == 0 and r3["status"] == 0
    P1 = np.exp((U + u1)[:, None] + (V + v1)[None, :] - g * inst.C)
    P2 = np.exp((U + u2)[:, None] + (V + v2)[None, :] - g * inst.C)
    P3 = np.exp((U + u3)[:, None] + (V + v3)[None, :] - g * inst.C)
    assert np.abs(P1 - P2).sum() < 1e-11
    assert np.abs(P1 - P3).sum() < 1e-11
    # fewer PNCG iterations than Sinkhorn half-steps
    assert r1["iterations"] < r2["iterations"]


def test_line_search_wolfe_post_hoc_and_decrease():
    """Every accepted alpha satisfies the approximate Wolfe conditions
     and the decrease safeguard (Z9); the dual objective is
    monotone; mean phi' evaluations per search is in the paper's range
    ("typically between 2-4"; SPEC criterion 9 allows <= 6)."""
    inst = S.paper_sphere_instance(96, 4, 0.9, seed=13)
    prob = O.OracleProblem(inst)
    g = O.schedule_fixed(128.0, T=2)
    U, V, res, tr = O.mdot(prob, g, O.make_options(eps=1e-9), trace_cap=100000)
    assert res["status"] == 0
    assert len(tr) == res["iterations"]
    c1, c2 = 0.1, 0.4
    for q in tr:
        assert q["dphi0"] < 0
        assert (2 * c1 - 1) * q["dphi0"] >= q["dphi_alpha"] >= c2 * q["dphi0"]
        assert q["dphi_value"] <= 1e-12
    mean_trials = np.mean([q["trials"] for q in tr])
    assert mean_trials <= 6.0


def test_reset_rule_and_first_step():
    """PAPER.md:190 read as: reset when <p, grad> >= 0 (Z5).  Every traced
    direction is a descent direction; k=1 has beta = 0."""
    inst = S.paper_sphere_instance(64, 4, 0.5, seed=14)
    prob = O.OracleProblem(inst)
    U, V, res, tr = O.mdot(prob, [64.0], O.make_options(eps=1e-10), trace_cap=100000)
    assert res["status"] == 0
    assert tr[0]["beta"] == 0.0
    assert all(q["dphi0"] < 0 for q in tr)


# ------------------------------------------------------------------ MD loop
def _md_plan(prob, gammas, **kw):
    U, V, res, _ = O.mdot(prob, gammas, O.make_options(**kw))
    assert res["status"] == 0, res
    g = float(np.sum(gammas))
    return np.exp(U[:, None] + V[None, :] - g * _dense_C(prob)), res


def test_lemma2_schedule_invariance():
    """Lemma 2: equal gbar, rank-1 P0 -> the same plan,
    for fixed T in {1,4,16}, the doubling schedule and both projectors."""
    inst = S.random_small(8, seed=15)
    prob = O.OracleProblem(inst)
    gb = 32.0
    Pref, _ = _md_plan(prob, [gb], eps=1e-13)
    for sched in (O.schedule_fixed(gb, T=4), O.schedule_fixed(gb, T=16), O.schedule_doubling(gb)):
        for proj in (O.PNCG, O.SINKHORN):
            P, _ = _md_plan(prob, sched, eps=1e-13, projector=proj)
            assert np.abs(P - Pref).sum() < 1e-10
    # P0 = 1 1^T (classic Sinkhorn special case) gives the same plan
    P, _ = _md_plan(prob, [gb], eps=1e-13, p0_ones=True)
    assert np.abs(P - Pref).sum() < 1e-10


def test_adaptive_eps_md_reaches_the_same_plan():
    """SURVEY 8(f) rank 1 (adaptive eps): by Lemma 2 the
    final plan depends only on gbar, and the projection onto U(r,c) is
    invariant to diagonal scalings of its input, so loose intermediate steps
    (eps_md) change only where the last projection starts.  Pinned against
    the single-step solve (T = 1, which has no intermediate step) and the 2x2
    closed form."""
    inst = S.random_small(8, seed=15)
    prob = O.OracleProblem(inst)
    gb = 32.0
    Pref, _ = _md_plan(prob, [gb], eps=1e-13)
    for em in (1e-6, 1e-3, 1e-1, 0.5):
        P, res = _md_plan(prob, O.schedule_fixed(gb, T=8), eps=1e-13, eps_md=em)
        assert np.abs(P - Pref).sum() < 1e-10, em
    # the loose steps really stopped early: fewer evaluations than eps_md = 0
    _, r0 = _md_plan(prob, O.schedule_fixed(gb, T=8), eps=1e-13)
    _, r1 = _md_plan(prob, O.schedule_fixed(gb, T=8), eps=1e-13, eps_md=1e-2)
    assert r1["evaluations"] < r0["evaluations"]
    rng = np.random.default_rng(21)
    for trial in range(6):
        C = rng.uniform(0, 1, size=(2, 2))
        r = rng.dirichlet([1, 1])
        c = rng.dirichlet([1, 1])
        g = [8.0, 64.0, 200.0][trial % 3]
        prob2 = O.OracleProblem(C=C, r=r, c=c)
        U, V, res, _ = O.mdot(prob2, O.schedule_fixed(g, T=4), O.make_options(eps=1e-14, eps_md=1e-2))
        assert res["status"] == 0
        P = np.exp(U[:, None] + V[None, :] - g * C)
        np.testing.assert_allclose(P, X.entropic_2x2(C, r, c, g), atol=1e-13)


def test_lemma1_exact_improvement_and_cor1():
    """Lemma 1 equality and Cor. 1
    bound on consecutive MD iterates (n = 8, gamma_t = 8)."""
    inst = S.random_small(8, seed=16)
    prob = O.OracleProblem(inst)
    C = inst.C
    Hmin = min(-(inst.r * np.log(inst.r)).sum(), -(inst.c * np.log(inst.c)).sum())
    plans = [np.outer(inst.r, inst.c)]
    for t in range(1, 6):
        P, _ = _md_plan(prob, [8.0] * t, eps=1e-13)
        plans.append(P)

    def kl(a, b):
        return float(np.sum(a * np.log(a / b)))

    for t in range(0, 5):
        Pt, Pn = plans[t], plans[t + 1]
        lhs = float((Pt * C).sum() - (Pn * C).sum())
        rhs = (kl(Pt, Pn) + kl(Pn, Pt)) / 8.0
        assert abs(lhs - rhs) < 1e-9
        assert lhs >= -1e-12       # monotone improvement
        if t >= 1:
            bound = min(8.0, math.sqrt(Hmin * 8.0 / (8.0 * t)))
            assert np.abs(Pn - Pt).sum() <= bound + 1e-9


@pytest.mark.parametrize("n", [4, 5, 6])
def test_prop1_bound_vs_permutation_enumeration(n):
    """Prop. 1: 0 <= <G,C> - OT and <P,C> - OT <= H_min/gbar,
    OT by enumerating permutation vertices (uniform marginals)."""
    for seed in range(4):
        inst = S.random_small(n, seed=100 + seed, uniform_marginals=True)
        prob = O.OracleProblem(inst)
        ot = X.ot_enumerate_uniform(inst.C)
        Hmin = math.log(n)
        prev = None
        for gb in (4.0, 16.0, 64.0):
            U, V, res, _ = O.mdot(prob, O.schedule_fixed(gb, T=4), O.make_options(eps=1e-8))
            assert res["status"] == 0
            gap = res["cost_rounded"] - ot
            assert gap >= -1e-12                     # rounded plan is feasible
            assert res["cost_unrounded"] - ot <= Hmin / gb + 1e-9
            if prev is not None:
                assert res["cost_unrounded"] <= prev + 1e-12   # -> OT as gbar grows
            prev = res["cost_unrounded"]


def test_prop1_bound_vs_lp_nonuniform():
    for seed in range(3):
        inst = S.random_small(7, seed=200 + seed)
        prob = O.OracleProblem(inst)
        ot = X.ot_lp(inst.C, inst.r, inst.c)
        Hmin = min(-(inst.r * np.log(inst.r)).sum(), -(inst.c * np.log(inst.c)).sum())
        U, V, res, _ = O.mdot(prob, O.schedule_fixed(512.0), O.make_options(eps=1e-12))
        assert res["status"] == 0
        assert res["cost_rounded"] - ot >= -1e-10
        assert res["cost_unrounded"] - ot <= Hmin / 512.0 + 1e-9


def test_exact_ot_helpers_agree():
    inst = S.random_small(5, seed=300, uniform_marginals=True)
    assert abs(X.ot_enumerate_uniform(inst.C) - X.ot_lp(inst.C, inst.r, inst.c)) < 1e-12
    li = S.line_instance(7, seed=301)
    assert abs(X.ot_line_nw(li.C, li.r, li.c) - X.ot_lp(li.C, li.r, li.c)) < 1e-12


def test_prop1_bound_vs_1d_monotone_coupling():
    """1-D convex cost: exact OT by the north-west corner rule, any marginals,
    larger n (the pin the GPU tests reuse at scale)."""
    li = S.line_instance(128, seed=302)
    prob = O.OracleProblem(li)
    ot = X.ot_line_nw(li.C, li.r, li.c)
    Hmin = min(-(li.r * np.log(li.r)).sum(), -(li.c * np.log(li.c)).sum())
    gb = 4096.0
    U, V, res, _ = O.mdot(prob, O.schedule_fixed(gb), O.make_options(eps=1e-10))
    assert res["status"] == 0
    assert res["cost_rounded"] - ot >= -1e-12
    assert res["cost_unrounded"] - ot <= Hmin / gb + 1e-9


def test_near_delta_marginal_gives_independence_coupling():
    """if r is a delta, the only feasible plan is r c^T."""
    n = 10
    inst = S.random_small(n, seed=17)
    r = np.full(n, 1e-13)
    r[3] = 1.0 - (n - 1) * 1e-13
    prob = O.OracleProblem(C=inst.C, r=r, c=inst.c)
    U, V, res, _ = O.mdot(prob, O.schedule_fixed(256.0), O.make_options(eps=1e-12))
    assert res["status"] == 0
    ind = float((np.outer(r, inst.c) * inst.C).sum())
    assert abs(res["cost_rounded"] - ind) < 1e-10


def test_gamma_4096_single_step_is_stable():
    """SPEC criterion 13 inverted: the log-domain oracle must not fail at a
    single MD step of gamma_t = 4096 (PAPER.md:362 reports failure > 256 for
    the paper's non-log implementation)."""
    inst = S.uniform_points_instance(3, 96, 2, 0, marg="dirichlet")
    prob = O.OracleProblem(inst)
    U, V, res, _ = O.mdot(prob, [4096.0], O.make_options(eps=1e-8))
    assert res["status"] == 0
    U2, V2, res2, _ = O.mdot(prob, O.schedule_fixed(4096.0), O.make_options(eps=1e-8))
    assert res2["status"] == 0
    assert abs(res["cost_unrounded"] - res2["cost_unrounded"]) < 1e-6 * res["cost_unrounded"]


# ----------------------------------------------------------------- rounding
def test_rounding_worked_example_half_rc():
    """F = r c^T / 2 -> G = r c^T."""
    inst = S.random_small(7, seed=18)
    prob = O.OracleProblem(inst)
    U = np.log(inst.r) + math.log(0.5)
    V = np.log(inst.c)
    out = O.round_plan(prob, U, V, 0.0, dense=True)
    np.testing.assert_allclose(out["G"], np.outer(inst.r, inst.c), atol=1e-16)


def test_rounding_exact_marginals_bound_idempotent():
    """Altschuler et al. Alg. 2: r(G)=r, c(G)=c, G>=0,
    |G-F|_1 <= 2 (|r(F)-r|_1 + |c(F)-c|_1), idempotence."""
    rng = np.random.default_rng(19)
    for seed in range(10):
        inst = S.random_small(8, seed=400 + seed)
        prob = O.OracleProblem(inst)
        U = np.log(inst.r) + 0.05 * rng.normal(size=8)
        V = np.log(inst.c) + 0.05 * rng.normal(size=8)
        g = 3.0
        F = np.exp(U[:, None] + V[None, :] - g * inst.C)
        out = O.round_plan(prob, U, V, g, dense=True)
        G = out["G"]
        assert np.all(G >= 0)
        np.testing.assert_allclose(G.sum(1), inst.r, atol=1e-15)
        np.testing.assert_allclose(G.sum(0), inst.c, atol=1e-15)
        l1 = np.abs(F.sum(1) - inst.r).sum() + np.abs(F.sum(0) - inst.c).sum()
        assert np.abs(G - F).sum() <= 2 * l1 + 1e-15
        assert abs(out["cost_G"] - (G * inst.C).sum()) < 1e-15
        assert abs(out["cost_F"] - (F * inst.C).sum()) < 1e-15


# ---------------------------------------------------------------- schedules
def test_schedules_and_default_eps():
    """PAPER.md:356 rule gamma_t = gbar/max(1, floor(gbar/256))
    examples; doubling schedule of BASELINE config 1 (Z13)."""
    assert list(O.schedule_fixed(128.0)) == [128.0]
    assert list(O.schedule_fixed(1024.0)) == [256.0] * 4
    assert list(O.schedule_fixed(512.0, T=4)) == [128.0] * 4
    assert len(O.schedule_fixed(4096.0)) == 16
    d = O.schedule_doubling(4096.0)
    assert list(d) == [1.0, 1.0] + [2.0 ** k for k in range(1, 12)]
    assert np.cumsum(d)[-1] == 4096.0
    assert abs(O.default_eps(4.0, 4096.0) - 1e-5 / 1024 ** 2) < 1e-20
    assert O.default_eps(10.0, 5.0) == 1e-5


# ------------------------------------------------------ paper trend pins
def test_warm_start_rho0_decreases():
    """Fig. 2 left (SPEC criterion 12): with warm starts
    the initial infeasibility at the last MD step is below the first one."""
    for seed in range(3):
        inst = S.paper_sphere_instance(128, 4, 0.9, seed=500 + seed)
        prob = O.OracleProblem(inst)
        U, V, res, _ = O.mdot(prob, O.schedule_fixed(512.0, T=16),
                              O.make_options(eps=1e-9, stop_rho=True))
        assert res["status"] == 0
        assert res["rho0"][-1] < res["rho0"][0]


@pytest.mark.slow
def test_pncg_fewer_iterations_than_sinkhorn():
    """Fig. 2/4 direction (SPEC criterion 10): n = 256,
    m = 4, entropy 0.9, gbar = 256, T = 1, rho <= 1e-9: PNCG needs fewer
    iterations than SA on every instance and >= 3x fewer on average."""
    ratios = []
    for seed in range(2):
        inst = S.paper_sphere_instance(256, 4, 0.9, seed=600 + seed)
        prob = O.OracleProblem(inst)
        _, _, rp, _ = O.mdot(prob, [256.0], O.make_options(eps=1e-9, stop_rho=True))
        _, _, rs, _ = O.mdot(prob, [256.0], O.make_options(eps=1e-9, stop_rho=True,
                                                           projector=O.SINKHORN))
        assert rp["status"] == 0 and rs["status"] == 0
        assert rp["iterations"] <= rs["iterations"]
        ratios.append(rs["iterations"] / rp["iterations"])
    assert np.mean(ratios) >= 3.0


# ------------------------------------------------------------------ Fig. 3 diagnostics
def test_hessian_null_vector_and_psd():
    """(1_n, -1_n) spans the null space direction of the dual
    Hessian; the Hessian is PSD."""
    from oracle import diagnostics as D
    inst = S.random_small(10, seed=31)
    prob = O.OracleProblem(inst)
    rng = np.random.default_rng(0)
    U = np.log(inst.r) + 0.3 * rng.standard_normal(10)
    V = np.log(inst.c) + 0.3 * rng.standard_normal(10)
    H, P = D.hessian(prob, U, V, 5.0)
    z = np.concatenate([np.ones(10), -np.ones(10)])
    assert np.abs(H @ z).max() < 1e-14
    w = D.spectrum(H)
    assert w[0] > -1e-14 and abs(w[0]) < 1e-12 and w[1] > 1e-8


def test_preconditioned_spectrum_closed_form_at_fixed_point():
    """At the projection's solution (P in U(r,c)) both diagonal
    preconditioners equal D(1/r, 1/c) and M^1/2 H M^1/2 = [[I, K], [K^T, I]]
    with K = D(r)^-1/2 P D(c)^-1/2, whose eigenvalues are 1 -+ sigma_k(K)
    (block-matrix identity); sigma_1 = 1 (singular vectors sqrt r, sqrt c),
    so the spectrum spans [0, 2].  Pinned against an SVD of K."""
    from oracle import diagnostics as D
    inst = S.paper_sphere_instance(12, 4, 0.7, 5)
    prob = O.OracleProblem(inst)
    U, V, res, _ = O.mdot(prob, [16.0], O.make_options(eps=1e-14))
    assert res["status"] == 0
    H, P = D.hessian(prob, U, V, 16.0)
    t = np.concatenate([inst.r, inst.c])
    for kind in ("sinkhorn", "jacobi"):
        M = D.preconditioner(prob, U, V, 16.0, kind)
        np.testing.assert_allclose(M, 1.0 / t, rtol=1e-9)
    K = P / np.sqrt(np.outer(inst.r, inst.c))
    sig = np.linalg.svd(K, compute_uv=False)
    assert abs(sig[0] - 1.0) < 1e-10
    expect = np.sort(np.concatenate([1.0 - sig, 1.0 + sig]))
    got = D.spectrum(H, D.preconditioner(prob, U, V, 16.0))
    np.testing.assert_allclose(got, expect, atol=1e-10)
    assert abs(D.pseudo_condition(H, 1.0 / t) - 2.0 / (1.0 - sig[1])) < 1e-8 * 2.0 / (1.0 - sig[1])


def test_fig3_preconditioning_gain_grows_as_entropy_falls():
    """Fig. 3 right: the ratio of pseudo-condition numbers
    kappa(H) / kappa(M H) along PNCG iterations is larger for lower-entropy
    marginals (n = 32, m = 4, gbar = 32, T = 1; 4 seeds, 20 evaluations)."""
    from oracle import diagnostics as D
    means = []
    for frac in (0.3, 0.6, 0.9):
        rat = []
        for seed in range(4):
            inst = S.paper_sphere_instance(32, 4, frac, 100 + seed)
            prob = O.OracleProblem(inst)
            U0, V0 = np.log(inst.r), np.log(inst.c)
            u, v, _, _ = O.project(prob, U0, V0, 32.0, opts=O.make_options(eps=1e-12, max_evals=20))
            H, _ = D.hessian(prob, U0 + u, V0 + v, 32.0)
            rat.append(D.pseudo_condition(H) / D.pseudo_condition(H, D.preconditioner(prob, U0 + u, V0 + v, 32.0)))
        means.append(np.mean(np.log(rat)))
    assert means[0] > means[1] > means[2] > 0.0, means


def test_fig3_left_ncg_vs_pncg_and_jacobi_ablation():
    """Fig. 3 left: vanilla NCG needs far more iterations
    than PNCG at low entropy (n = 8, m = 4, gbar = 128, T = 1, rho <= 1e-5);
    the Jacobi-preconditioned ablation converges to the same plan as PNCG
    (uniqueness of the projection) in a comparable count."""
    its = {O.PNCG: [], O.NCG: [], O.PNCG_JACOBI: []}
    for seed in range(4):
        inst = S.paper_sphere_instance(8, 4, 0.2, 200 + seed)
        prob = O.OracleProblem(inst)
        plans = {}
        for p in its:
            U, V, res, _ = O.mdot(prob, [128.0], O.make_options(eps=1e-5, stop_rho=True, projector=p,
                                                                 max_evals=200000))
            assert res["status"] == 0, (p, res["status"])
            its[p].append(res["iterations"])
            U2, V2, res2, _ = O.mdot(prob, [128.0], O.make_options(eps=1e-13, projector=p, max_evals=400000))
            plans[p] = O.plan(prob, U2, V2, 128.0)
        assert np.abs(plans[O.PNCG_JACOBI] - plans[O.PNCG]).sum() < 1e-10
    assert np.mean(its[O.NCG]) > 5 * np.mean(its[O.PNCG])
    assert np.mean(its[O.PNCG_JACOBI]) < 3 * np.mean(its[O.PNCG])


# --------------------------------------------------- round-2 pins
@pytest.mark.parametrize("kind", ["f32", "f64", "sqeuclid"])
def test_log_marginal_subsets_bitwise_and_direct(kind):
    """orc_log_marginal_rows / _cols (the checker of the full-size GPU tests)
    must give the SAME bits as orc_log_marginals on every row / column, and
    both must equal a direct fp64 sum of the explicit matrix."""
    rng = np.random.default_rng(40)
    for n in (1, 7, 33, 64):
        if kind == "sqeuclid":
            inst = S.config5(0, n=n, d=3)
        else:
            inst = S.random_small(n, seed=41 + n, dtype=np.float64 if kind == "f64" else np.float32)
        prob = O.OracleProblem(inst)
        C = _dense_C(prob)
        A = np.log(inst.r) + 0.5 * rng.standard_normal(n)
        B = np.log(inst.c) + 0.5 * rng.standard_normal(n)
        g = 37.0
        lr, lc, st = O.log_marginals(prob, A, B, g)
        assert st == 0
        idx = rng.permutation(n)
        sub = O.log_marginal_subset(prob, A, B, g, rows=idx, cols=idx[::-1])
        assert np.array_equal(sub["rows"], lr[idx])
        assert np.array_equal(sub["cols"], lc[idx[::-1]])
        P = np.exp(A[:, None] + B[None, :] - g * C)
        np.testing.assert_allclose(np.exp(sub["rows"]), P.sum(1)[idx], rtol=1e-13)
        np.testing.assert_allclose(np.exp(sub["cols"]), P.sum(0)[idx[::-1]], rtol=1e-13)


def test_plan_cost_direct_sum_and_rounding_cost_F():
    """orc_plan_cost = sum_ij C_ij P_ij (the unrounded cost of the Z20 gate):
    direct dense sum, and the rounding routine's <C, F>."""
    for kind in ("f32", "sqeuclid"):
        inst = S.random_small(29, seed=44, dtype=np.float32) if kind == "f32" else S.config5(1, n=29, d=5)
        prob = O.OracleProblem(inst)
        C = _dense_C(prob)
        rng = np.random.default_rng(45)
        A = np.log(inst.r) + 0.2 * rng.standard_normal(29)
        B = np.log(inst.c) + 0.2 * rng.standard_normal(29)
        pc = O.plan_cost(prob, A, B, 11.0)
        assert abs(pc - float((C * np.exp(A[:, None] + B[None, :] - 11.0 * C)).sum())) <= 1e-14 * pc
        assert abs(pc - O.round_plan(prob, A, B, 11.0)["cost_F"]) <= 1e-14 * pc


def test_line_search_quadratic_phi_closed_form():
    """Appx. C on a quadratic phi(alpha) = a/2 (alpha - a*)^2 - a/2 a*^2: phi' is
    linear, so the secant step alpha_sec is the exact minimiser
    a* and the hybrid step is a*/2 + (lo + hi)/4.  From alpha0 = 1
    with a* = 5.3: doubling (Z8) 1, 2, 4, 8 brackets a* in [4, 8], the hybrid
    step is 5.3/2 + 3 = 5.65, accepted by approximate Wolfe with
    c1 = 0.45, c2 = 0.1.  A sign or index slip in either formula changes the
    trial sequence."""
    a, star = 2.0, 5.3

    def phi(al):
        return a * (al - star), 0.5 * a * (al - star) ** 2 - 0.5 * a * star ** 2

    al, dp, dv, tr, acc, seen = O.line_search(phi, -a * star, c1=0.45, c2=0.1)
    assert acc and tr == 5
    np.testing.assert_allclose(seen, [1.0, 2.0, 4.0, 8.0, 0.5 * star + 0.25 * 12.0], rtol=0, atol=1e-14)
    assert al == seen[-1] and dv < 0
    # a* < alpha0: the first trial overshoots; every later trial is
    # a*/2 + (lo + hi)/4 of the current bracket: [0, 1] -> 0.4 (phi' > 0),
    # [0, 0.4] -> 0.25 (phi' < c2 phi'(0)), [0.25, 0.4] -> 0.3125 (accepted)
    star = 0.3
    al, dp, dv, tr, acc, seen = O.line_search(phi, -a * star, c1=0.45, c2=0.1)
    assert acc
    np.testing.assert_allclose(seen, [1.0, 0.15 + 0.25, 0.15 + 0.1, 0.15 + 0.1625], rtol=0, atol=1e-15)
    # near-exact search (c1 -> 1/2, c2 -> 0): converges to the minimiser
    star = 13.7
    al, dp, dv, tr, acc, seen = O.line_search(phi, -a * star, c1=0.5 - 1e-9, c2=1e-9)
    assert acc and abs(al - star) < 1e-7 * star and tr <= 60
    # the decrease safeguard (Z9) rejects a trial whose phi rose even when phi'
    # satisfies the curvature window
    al, dp, dv, tr, acc, seen = O.line_search(lambda x: (0.0, 1.0), -1.0, max_trials=5)
    assert not acc


def _traced(inst, gb, T, beta, c1=0.1, c2=0.4, eps=1e-10, max_evals=0):
    prob = O.OracleProblem(inst)
    U, V, res, tr = O.mdot(prob, O.schedule_fixed(gb, T=T),
                           O.make_options(eps=eps, beta=beta, c1=c1, c2=c2, max_evals=max_evals), trace_cap=100000)
    assert res["status"] == 0 or (max_evals and res["status"] == 4), res
    return U, V, res, tr


@pytest.mark.parametrize("beta", [O.BETA_PPR, O.BETA_PPR_AF, O.BETA_PFR, O.BETA_PPR_PRINTED, O.BETA_PPR_PLUS])
def test_direction_update_identity_every_beta_variant(beta):
    """p_k = -s_k + beta_k p_{k-1} (Alg. 2 line 6) implies
    <p_k, g_k> = -<g_k, s_k> + beta_k <p_{k-1}, g_k>, and <p_{k-1}, g_k> is the
    previous search's phi'(alpha) (g_k is the gradient at the
    accepted trial).  Checked on the traced scalars of every beta variant
    (first 300 evaluations: on this instance FR stalls in the "unproductive
    directions" PAPER.md:499 describes, beta ~ 1 with tiny steps)."""
    inst = S.paper_sphere_instance(40, 4, 0.7, seed=50)
    _, _, _, tr = _traced(inst, 128.0, 2, beta, max_evals=300)
    checked = 0
    for prev, q in zip(tr, tr[1:]):
        if q["t"] != prev["t"] or q["reset"]:
            continue
        rhs = -q["gs"] + q["beta"] * prev["dphi_alpha"]
        assert abs(q["dphi0"] - rhs) <= 1e-10 * (abs(q["gs"]) + abs(q["beta"] * prev["dphi_alpha"])), (q, prev)
        checked += 1
        if beta == O.BETA_PPR_PLUS:
            assert q["beta"] >= 0.0
        if beta == O.BETA_PFR:
            assert q["beta"] >= 0.0      # ratio of <g, s> = four-divergence sums >= 0
    assert checked >= 5


def test_beta_denominators_agree_under_exact_line_search_and_at_k2():
    """Z6: the PPR denominator -<g_{k-1}, p_{k-1}> and the Al-Baali-Fletcher
    one <g_{k-1}, s_{k-1}> differ by beta_{k-1} <g_{k-1}, p_{k-2}>, which vanishes
    under an exact line search (c1 -> 1/2, c2 -> 0 squeeze phi'(alpha) to ~0).
    At k = 2 (p_1 = -s_1 for every variant) they are equal
    exactly, the printed sign of PAPER.md:262 gives -beta^PPR, and PR+ gives
    max(0, beta^PPR)."""
    inst = S.paper_sphere_instance(40, 4, 0.7, seed=51)
    _, _, _, tr = _traced(inst, 128.0, 1, O.BETA_PPR, c1=0.5 - 1e-6, c2=1e-6)
    rel = [abs(-q["dphi0"] - q["gs"]) / q["gs"] for q in tr[1:] if not q["reset"] and q["gs"] > 0]
    assert len(rel) >= 5 and max(rel) <= 1e-4, max(rel)
    k2 = {}
    for beta in (O.BETA_PPR, O.BETA_PPR_AF, O.BETA_PPR_PRINTED, O.BETA_PPR_PLUS):
        prob = O.OracleProblem(inst)
        _, _, res, trb = O.project(prob, np.log(inst.r), np.log(inst.c), 128.0,
                                   opts=O.make_options(eps=1e-12, beta=beta, max_evals=40), trace_cap=100)
        q = trb[1]
        assert q["k"] == 2 and trb[0]["beta"] == 0.0
        k2[beta] = q["beta"] if not q["reset"] else 0.0
    b = k2[O.BETA_PPR]
    assert b != 0.0
    assert k2[O.BETA_PPR_AF] == b
    assert k2[O.BETA_PPR_PLUS] == max(b, 0.0)
    assert k2[O.BETA_PPR_PRINTED] in (-b, 0.0)   # 0.0 when the printed sign forces a reset (Z5)


@pytest.mark.parametrize("beta", [O.BETA_PPR_AF, O.BETA_PFR, O.BETA_PPR_PRINTED, O.BETA_PPR_PLUS])
def test_every_beta_variant_reaches_the_2x2_closed_form_and_the_ppr_plan(beta):
    """Uniqueness of the Bregman projection: every beta variant
    (FR; PPR with either denominator, Z6; PR+) converges to
    the entropic plan, pinned by the 2x2 closed form and, at n = 20, by the
    default PPR solve."""
    rng = np.random.default_rng(52)
    for trial in range(8):
        C = rng.uniform(0, 1, size=(2, 2))
        r = rng.dirichlet([1, 1])
        c = rng.dirichlet([1, 1])
        gb = [4.0, 32.0, 150.0][trial % 3]
        prob = O.OracleProblem(C=C, r=r, c=c)
        U, V, res, _ = O.mdot(prob, [gb], O.make_options(eps=1e-14, beta=beta))
        assert res["status"] == 0
        np.testing.assert_allclose(np.exp(U[:, None] + V[None, :] - gb * C), X.entropic_2x2(C, r, c, gb), atol=1e-13)
    inst = S.random_small(20, seed=53)
    ref, _ = _md_plan(O.OracleProblem(inst), [30.0], eps=1e-13)
    P, _ = _md_plan(O.OracleProblem(inst), [30.0], eps=1e-13, beta=beta)
    assert np.abs(P - ref).sum() < 1e-11


def test_warm_start_modes_reach_the_same_plan():
    """Z4 warm-start readings (scaled / carried / zero potentials) only move
    where each projection starts: by Lemma 2 the final plan
    is the entropic plan at gbar for all three, on a variable (doubling)
    schedule where scaled and carried differ."""
    inst = S.random_small(10, seed=54)
    prob = O.OracleProblem(inst)
    sched = O.schedule_doubling(64.0)
    ref, r0 = _md_plan(prob, [64.0], eps=1e-13)
    evals = {}
    for warm in (O.WARM_SCALED, O.WARM_CARRY, O.WARM_ZERO):
        P, res = _md_plan(prob, sched, eps=1e-13, warm=warm)
        assert np.abs(P - ref).sum() < 1e-10, warm
        evals[warm] = res["evaluations"]
    assert evals[O.WARM_ZERO] > evals[O.WARM_SCALED]   # warm starts save work
    rng = np.random.default_rng(55)
    C = rng.uniform(0, 1, size=(2, 2))
    r, c = rng.dirichlet([1, 1]), rng.dirichlet([1, 1])
    for warm in (O.WARM_CARRY, O.WARM_ZERO):
        U, V, res, _ = O.mdot(O.OracleProblem(C=C, r=r, c=c), O.schedule_doubling(100.0),
                              O.make_options(eps=1e-14, warm=warm))
        np.testing.assert_allclose(np.exp(U[:, None] + V[None, :] - 100.0 * C), X.entropic_2x2(C, r, c, 100.0),
                                   atol=1e-13)


def test_adaptive_gamma_schedule_lemma2_and_budget():
    """Adaptive step rule (Z29, PAPER.md:371 future work): the realised steps
    sum to gbar exactly, follow the doubling / halving rule, and -- Lemma 2,
    PAPER.md:152-155 -- the final plan equals the single-step (T = 1) plan and
    the 2x2 closed form."""
    inst = S.random_small(12, seed=56)
    prob = O.OracleProblem(inst)
    gb = 512.0
    ref, _ = _md_plan(prob, [gb], eps=1e-12)
    U, V, res, _, g = O.mdot_adaptive(prob, gb, 16.0, O.make_options(eps=1e-12))
    assert res["status"] == 0 and res["gamma_bar"] == gb
    assert g.sum() == gb and len(g) == res["md_steps"] >= 3
    assert g[0] == 16.0 and g[1] == 32.0
    for a, b in zip(g[1:-1], g[2:-1]):
        assert b in (2 * a, max(a / 2, gb / 1024))
    P = np.exp(U[:, None] + V[None, :] - gb * inst.C)
    assert np.abs(P - ref).sum() < 1e-10
    # eps_md composes with it (both only move starting points)
    U2, V2, res2, _, g2 = O.mdot_adaptive(prob, gb, 16.0, O.make_options(eps=1e-12, eps_md=1e-3))
    assert np.abs(np.exp(U2[:, None] + V2[None, :] - gb * inst.C) - ref).sum() < 1e-10
    # a first step covering the budget is the T = 1 solve
    U3, V3, res3, _, g3 = O.mdot_adaptive(prob, gb, 4096.0, O.make_options(eps=1e-12))
    assert list(g3) == [gb]
    rng = np.random.default_rng(57)
    C = rng.uniform(0, 1, size=(2, 2))
    r, c = rng.dirichlet([1, 1]), rng.dirichlet([1, 1])
    U, V, res, _, g = O.mdot_adaptive(O.OracleProblem(C=C, r=r, c=c), 100.0, 4.0, O.make_options(eps=1e-14))
    assert res["status"] == 0 and len(g) >= 3
    np.testing.assert_allclose(np.exp(U[:, None] + V[None, :] - 100.0 * C), X.entropic_2x2(C, r, c, 100.0),
                               atol=1e-13)


def test_cost_sqeuclid_dot_recipe_is_its_fp32_chain():
    """Z22b (dot form of the config-5 cost): C = max(fl(nx + ny) - 2 s, 0) * scale
    with nx, ny, s fp32 fma chains in index order; checked against a numpy
    float32 emulation (each fma exact in fp64 for fp32 operands, rounded once),
    and against the exact squared distance to fp32 cancellation accuracy."""
    inst = S.config5(0, n=64, d=16)
    prob = O.OracleProblem(inst, recipe="dot")

    def fma32(a, b, c):
        return np.float32(np.float64(a) * np.float64(b) + np.float64(c))

    for (i, j) in [(0, 0), (3, 7), (63, 1), (10, 10), (5, 40)]:
        x, y = inst.X[i], inst.Y[j]
        nx = ny = s = np.float32(0.0)
        for k in range(16):
            nx = fma32(x[k], x[k], nx)
        for k in range(16):
            ny = fma32(y[k], y[k], ny)
        for k in range(16):
            s = fma32(x[k], y[k], s)
        t = np.float32(nx + ny)
        ref = np.float32(max(fma32(np.float32(-2.0), s, t), np.float32(0.0)) * np.float32(1.0 / 16))
        assert prob.cost(i, j) == float(ref)
        exact = float(np.sum((x.astype(np.float64) - y.astype(np.float64)) ** 2)) / 16
        assert abs(prob.cost(i, j) - exact) <= 4e-7 * max(1.0, 16 * exact)


def test_cost_sqeuclid_dot_recipe_clamps_cancellation_at_zero():
    """Z22b's max(., 0): for nearly coincident points the dot form can round
    below zero; the oracle must return exactly 0 there (C >= 0),
    and exactly 0 for coincident points (the chains cancel exactly)."""
    rng = np.random.default_rng(7)

    def fma32(a, b, c):
        return np.float32(np.float64(a) * np.float64(b) + np.float64(c))

    def raw(x, y):
        nx = ny = s = np.float32(0.0)
        for k in range(len(x)):
            nx = fma32(x[k], x[k], nx)
            ny = fma32(y[k], y[k], ny)
            s = fma32(x[k], y[k], s)
        return float(fma32(np.float32(-2.0), s, np.float32(nx + ny)))

    neg = None
    for _ in range(4000):
        x = rng.random(16, dtype=np.float32)
        y = (x + rng.normal(0, 1e-4, 16).astype(np.float32)).astype(np.float32)
        if raw(x, y) < 0.0:
            neg = (x, y)
            break
    assert neg is not None, "no cancelling pair found"
    X = np.stack([neg[0], neg[0]])
    Y = np.stack([neg[1], neg[0]])
    prob = O.OracleProblem(X=X, Y=Y, r=np.full(2, 0.5), c=np.full(2, 0.5), scale=1.0 / 16, recipe="dot")
    assert prob.cost(0, 0) == 0.0          # clamped (unclamped value < 0)
    assert prob.cost(1, 1) == 0.0          # coincident points
    diffp = O.OracleProblem(X=X, Y=Y, r=np.full(2, 0.5), c=np.full(2, 0.5), scale=1.0 / 16)
    assert diffp.cost(0, 0) > 0.0          # the difference form sees the distance
