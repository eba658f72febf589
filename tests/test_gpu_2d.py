"""2-D (row x column) sharding (mdot_solve_sharded_2d) on
one GPU: a Gr x Gc grid of virtual ranks = threads of this process, each with
its own stream and its own block C[rows_a, cols_b]; the row team of a rank is
an in-process communicator over the Gc ranks of its row block, the column team
one over the Gr ranks of its column block (host-side rank-ordered sums: no
device code waits on another rank, so the ranks may share the GPU).

Gates:
  * every rank takes identical decisions: identical evaluation counts, costs,
    and identical potential slices across the replicas of a block;
  * unrounded cost within the Z20 gate (1e-5 relative) of the single-GPU solve;
  * the oracle's fp64 re-evaluation of the assembled (U, V): L1 <= 2 eps;
  * rounding: the rounded and unrounded costs equal the oracle's rounding of
    the SAME assembled (U, V) to 1e-10 relative.
"""
import threading

import numpy as np
import pytest

import oracle as O
import synthetic as S

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_08507_b200 as M  # noqa: E402

DEV = torch.device("cuda:0")
COST_GATE = 1e-5


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def _solve_2d(inst, Gr, Gc, sched, opts_kw, tag, otf_recipe=None):
    n = inst.n
    rows = np.array_split(np.arange(n), Gr)
    cols = np.array_split(np.arange(n), Gc)
    out = {}
    err = []

    def run(a, b):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                r0, nr = int(rows[a][0]), len(rows[a])
                c0, nc = int(cols[b][0]), len(cols[b])
                if otf_recipe is None:
                    cost = dict(C_block=_t(inst.C[r0:r0 + nr, c0:c0 + nc]))
                else:
                    cost = dict(X_block=_t(inst.X[r0:r0 + nr]), Y_block=_t(inst.Y[c0:c0 + nc]),
                                scale=float(inst.scale), recipe=otf_recipe)
                U = torch.empty(nr, dtype=torch.float64, device=DEV)
                V = torch.empty(nc, dtype=torch.float64, device=DEV)
                rc = M.mdot_comm_create_local(f"{tag}_row{a}", Gc, b, 0)
                cc = M.mdot_comm_create_local(f"{tag}_col{b}", Gr, a, 0)
                res = M.mdot_solve_sharded_2d(rc, cc, r0, nr, c0, nc, r=_t(inst.r), c=_t(inst.c), n=n,
                                              schedule=sched, options=M.options(**opts_kw),
                                              u_local_out=U, v_local_out=V, check=False, **cost)
                s.synchronize()
                M.mdot_comm_destroy(rc)
                M.mdot_comm_destroy(cc)
                out[(a, b)] = (res, U.cpu().numpy(), V.cpu().numpy(), M.mdot_last_error())
        except Exception as e:  # noqa: BLE001
            err.append(e)

    ths = [threading.Thread(target=run, args=(a, b)) for a in range(Gr) for b in range(Gc)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out, rows, cols


@pytest.mark.parametrize("Gr,Gc,projector", [(2, 2, 0), (1, 3, 0), (3, 2, 0), (2, 2, 1)])
def test_2d_grid_matches_single_gpu_and_oracle(Gr, Gc, projector):
    n = 600                                   # ragged blocks for Gr, Gc = 3 (200 x 300, 300 x 200 ...)
    inst = S.uniform_points_instance(3, n, 2, 31, marg="dirichlet")
    gb, T, eps = 512.0, 2, 1e-6
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=T)
    kw = {"eps": eps, "projector": projector}
    out, rows, cols = _solve_2d(inst, Gr, Gc, sched, kw, f"g2d_{Gr}{Gc}{projector}")
    r00 = out[(0, 0)][0]
    assert all(o[0]["status"] == 0 for o in out.values()), [(k, o[0]["status_name"], o[3]) for k, o in out.items()]
    assert all(o[0]["control_path"] == 0 for o in out.values())      # in-process teams: host control loop
    # identical decisions and scalars on every rank of the grid
    assert all(o[0]["evaluations"] == r00["evaluations"] for o in out.values())
    assert all(o[0]["cost_unrounded"] == r00["cost_unrounded"] for o in out.values())
    assert all(o[0]["cost_rounded"] == r00["cost_rounded"] for o in out.values())
    # replicas: U slices identical across a row team, V slices across a column team
    for a in range(Gr):
        assert all(np.array_equal(out[(a, b)][1], out[(a, 0)][1]) for b in range(Gc))
    for b in range(Gc):
        assert all(np.array_equal(out[(a, b)][2], out[(0, b)][2]) for a in range(Gr))
    assert r00["l1_final"] <= eps
    ref = M.mdot_solve(_t(inst.C), _t(inst.r), _t(inst.c), schedule=sched, options=M.options(**kw))
    assert abs(r00["cost_unrounded"] - ref["cost_unrounded"]) <= COST_GATE * ref["cost_unrounded"]
    U = np.concatenate([out[(a, 0)][1] for a in range(Gr)])
    V = np.concatenate([out[(0, b)][2] for b in range(Gc)])
    prob = O.OracleProblem(inst)
    lr, lc, _ = O.log_marginals(prob, U, V, gb)
    l1 = np.abs(np.exp(lr) - inst.r).sum() + np.abs(np.exp(lc) - inst.c).sum()
    assert l1 <= 2 * eps, l1
    rp = O.round_plan(prob, U, V, gb)
    assert abs(r00["cost_unrounded"] - rp["cost_F"]) <= 1e-10 * rp["cost_F"], (r00["cost_unrounded"], rp["cost_F"])
    assert abs(r00["cost_rounded"] - rp["cost_G"]) <= 1e-10 * rp["cost_G"], (r00["cost_rounded"], rp["cost_G"])


@pytest.mark.parametrize("recipe", ["diff", "dot"])
def test_2d_grid_on_the_fly_cost(recipe):
    """Config-5-shaped on-the-fly cost (d = 16, C = ||x - y||^2 / 16 by the
    Z22 / Z22b fp32 recipe) on a 2 x 2 grid: block (i, j) evaluates X rows_i
    against Y rows_j in-kernel (K2).  Same gates as the dense grid, the oracle
    built on the same fp32 recipe."""
    n = 1000
    inst = S.config5(1, n=n, d=16)
    gb, eps = 1024.0, 1e-5                     # config 5 target
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=4)
    out, _, _ = _solve_2d(inst, 2, 2, sched, {"eps": eps}, f"g2d_otf_{recipe}", otf_recipe=recipe)
    r00 = out[(0, 0)][0]
    assert all(o[0]["status"] == 0 for o in out.values()), [(k, o[0]["status_name"], o[3]) for k, o in out.items()]
    assert all(o[0]["evaluations"] == r00["evaluations"] for o in out.values())
    assert all(o[0]["cost_rounded"] == r00["cost_rounded"] for o in out.values())
    assert r00["l1_final"] <= eps
    ref = M.mdot_solve(X=_t(inst.X), Y=_t(inst.Y), scale=inst.scale, r=_t(inst.r), c=_t(inst.c), schedule=sched,
                       options=M.options(eps=eps), recipe=recipe)
    assert abs(r00["cost_unrounded"] - ref["cost_unrounded"]) <= COST_GATE * ref["cost_unrounded"]
    U = np.concatenate([out[(a, 0)][1] for a in range(2)])
    V = np.concatenate([out[(0, b)][2] for b in range(2)])
    prob = O.OracleProblem(inst, recipe=recipe)
    lr, lc, _ = O.log_marginals(prob, U, V, gb)
    l1 = np.abs(np.exp(lr) - inst.r).sum() + np.abs(np.exp(lc) - inst.c).sum()
    assert l1 <= 2 * eps, l1
    rp = O.round_plan(prob, U, V, gb)
    assert abs(r00["cost_unrounded"] - rp["cost_F"]) <= 1e-9 * rp["cost_F"], (r00["cost_unrounded"], rp["cost_F"])
    assert abs(r00["cost_rounded"] - rp["cost_G"]) <= 1e-9 * rp["cost_G"], (r00["cost_rounded"], rp["cost_G"])


def test_2d_one_by_one_grid_equals_host_loop_solve():
    """A 1 x 1 grid is the unsharded problem on the 2-D code path: same
    decisions as the single-GPU host-loop solve (device_control = 0) up to the
    summation order of the reduced partials (Z20 gate), oracle rounding of its
    own (U, V) to 1e-10."""
    n = 1000
    inst = S.uniform_points_instance(3, n, 2, 32, marg="dirichlet")
    gb, eps = 1024.0, 1e-6
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=4)
    out, _, _ = _solve_2d(inst, 1, 1, sched, {"eps": eps}, "g2d_11")
    res, U, V, _ = out[(0, 0)]
    assert res["status"] == 0 and res["l1_final"] <= eps
    ref = M.mdot_solve(_t(inst.C), _t(inst.r), _t(inst.c), schedule=sched,
                       options=M.options(eps=eps, device_control=0))
    assert abs(res["cost_unrounded"] - ref["cost_unrounded"]) <= COST_GATE * ref["cost_unrounded"]
    rp = O.round_plan(O.OracleProblem(inst), U, V, gb)
    assert abs(res["cost_rounded"] - rp["cost_G"]) <= 1e-10 * rp["cost_G"]


@pytest.mark.parametrize("f64_cost", [False, True])
def test_2d_grid_fp64_entries(f64_cost):
    """fp64-entry solves on the 2-D path (eps 1e-9 < 5e-8 with AUTO; fp64 C
    implies fp64 entries): every evaluation is the exact evaluator, its row
    log-sums combined over the row team and its column (max, sum) pairs over
    the column team.  Gates as the dense grid; at eps 1e-9 the unrounded cost
    agrees with the ORACLE's own solve to 1e-5 (Z20 (ii))."""
    n = 300
    inst = S.uniform_points_instance(3, n, 2, 35, marg="dirichlet")
    if f64_cost:
        inst.C = inst.C.astype(np.float64)
    gb, eps = 256.0, 1e-9
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=1)
    out, _, _ = _solve_2d(inst, 2, 2, sched, {"eps": eps}, f"g2d_f64_{int(f64_cost)}")
    r00 = out[(0, 0)][0]
    assert all(o[0]["status"] == 0 for o in out.values()), [(k, o[0]["status_name"], o[3]) for k, o in out.items()]
    assert all(o[0]["evaluations"] == r00["evaluations"] for o in out.values())
    assert all(o[0]["cost_rounded"] == r00["cost_rounded"] for o in out.values())
    assert r00["l1_final"] <= eps
    U = np.concatenate([out[(a, 0)][1] for a in range(2)])
    V = np.concatenate([out[(0, b)][2] for b in range(2)])
    prob = O.OracleProblem(inst)
    lr, lc, _ = O.log_marginals(prob, U, V, gb)
    assert np.abs(np.exp(lr) - inst.r).sum() + np.abs(np.exp(lc) - inst.c).sum() <= 2 * eps
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=1), O.make_options(eps=eps))
    assert abs(r00["cost_unrounded"] - ores["cost_unrounded"]) <= COST_GATE * ores["cost_unrounded"]
    rp = O.round_plan(prob, U, V, gb)
    assert abs(r00["cost_rounded"] - rp["cost_G"]) <= 1e-10 * rp["cost_G"]


def test_2d_rejects_bad_blocks():
    """A block outside the problem, or marginals that do not match the global
    n: MDOT_EINVAL before any device work."""
    n = 64
    inst = S.uniform_points_instance(3, n, 2, 33, marg="dirichlet")
    rc = M.mdot_comm_create_local("g2d_rej_row", 1, 0, 0)
    cc = M.mdot_comm_create_local("g2d_rej_col", 1, 0, 0)
    try:
        sched = M.schedule(M.MDOT_SCHED_FIXED, 64.0, T=1)
        res = M.mdot_solve_sharded_2d(rc, cc, 0, n, 8, n - 4, _t(inst.C[:, 4:]), _t(inst.r), _t(inst.c), n=n,
                                      schedule=sched, options=M.options(eps=1e-6), check=False)
        assert res["status"] == 1 and "column range" in M.mdot_last_error()
        res = M.mdot_solve_sharded_2d(rc, cc, 0, n, 8, n - 8, _t(inst.C[:, 8:]), _t(inst.r), _t(inst.c), n=n - 4,
                                      schedule=sched, options=M.options(eps=1e-6), check=False)
        assert res["status"] == 1
    finally:
        M.mdot_comm_destroy(rc)
        M.mdot_comm_destroy(cc)


@pytest.mark.parametrize("dc", [1, 0])
def test_2d_nccl_teams_one_rank(dc, monkeypatch):
    """The NCCL transport on the 2-D path: both teams are 1-rank NCCL
    communicators, so every row / column / scalar reduction is a real
    ncclAllReduce on the solve's stream -- captured inside the CUDA-graph
    slots under device control (dc = 1, control_path 1), or issued by the host
    loop (dc = 0).  The multi-rank logic is covered by the virtual-rank grids
    above, the gloo test and tests/multi/."""
    monkeypatch.setenv("MDOT_SHARDED_SELFTEST", "1")   # a 1-rank comm keeps its NCCL communicator
    n = 800
    inst = S.uniform_points_instance(3, n, 2, 34, marg="dirichlet")
    gb, eps = 512.0, 1e-6
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=2)
    rc = M.mdot_comm_create(M.mdot_get_unique_id(), 1, 0, 0)
    cc = M.mdot_comm_create(M.mdot_get_unique_id(), 1, 0, 0)
    try:
        U = torch.empty(n, dtype=torch.float64, device=DEV)
        V = torch.empty(n, dtype=torch.float64, device=DEV)
        res = M.mdot_solve_sharded_2d(rc, cc, 0, n, 0, n, _t(inst.C), _t(inst.r), _t(inst.c), n=n, schedule=sched,
                                      options=M.options(eps=eps, device_control=dc), u_local_out=U, v_local_out=V)
    finally:
        M.mdot_comm_destroy(rc)
        M.mdot_comm_destroy(cc)
    assert res["status"] == 0 and res["l1_final"] <= eps
    assert res["control_path"] == dc
    prob = O.OracleProblem(inst)
    Uo, Vo, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=2), O.make_options(eps=eps))
    assert abs(res["cost_unrounded"] - ores["cost_unrounded"]) <= COST_GATE * ores["cost_unrounded"]
    rp = O.round_plan(prob, U.cpu().numpy(), V.cpu().numpy(), gb)
    assert abs(res["cost_rounded"] - rp["cost_G"]) <= 1e-10 * rp["cost_G"]
    lr, lc, _ = O.log_marginals(prob, U.cpu().numpy(), V.cpu().numpy(), gb)
    assert np.abs(np.exp(lr) - inst.r).sum() + np.abs(np.exp(lc) - inst.c).sum() <= 2 * eps


# ------------------------------------------------------------------ NC2
def _solve_1d(inst, G, sched, opts_kw, tag):
    n = inst.n
    rows = np.array_split(np.arange(n), G)
    out = {}
    err = []

    def run(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                r0, nr = int(rows[k][0]), len(rows[k])
                U = torch.empty(nr, dtype=torch.float64, device=DEV)
                V = torch.empty(n, dtype=torch.float64, device=DEV)
                cm = M.mdot_comm_create_local(tag, G, k, 0)
                res = M.mdot_solve_sharded(cm, r0, nr, _t(inst.C[r0:r0 + nr]), _t(inst.r), _t(inst.c), n=n,
                                           schedule=sched, options=M.options(**opts_kw), u_local_out=U, v_out=V)
                s.synchronize()
                M.mdot_comm_destroy(cm)
                out[k] = (res, U.cpu().numpy(), V.cpu().numpy())
        except Exception as e:  # noqa: BLE001
            err.append(e)

    ths = [threading.Thread(target=run, args=(k,)) for k in range(G)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("layout", ["1d3", "2d22"])
def test_nc2_scalar_only_trials(layout, monkeypatch):
    """NC2 (MDOT_NC2=1, sharded host loop): a line-search trial
    exchanges 4 scalars -- each rank's contributions to phi'(alpha) and the
    mass, linear in its partial marginals -- and only an
    accepted trial's row / column vectors are reduced (evaluate from the kept
    partials).  Same gates as the vector-per-trial path: identical decisions on
    every rank, Z20 cost gate against the single-GPU solve, oracle L1 <= 2 eps,
    and the accepted-trial count equal to the iteration count."""
    monkeypatch.setenv("MDOT_NC2", "1")
    n = 600
    inst = S.uniform_points_instance(3, n, 2, 36, marg="dirichlet")
    gb, eps = 512.0, 1e-6
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=2)
    kw = {"eps": eps}
    if layout == "1d3":
        out = _solve_1d(inst, 3, sched, kw, "nc2_1d3")
        res = [o[0] for o in out.values()]
        U = np.concatenate([out[k][1] for k in range(3)])
        V = out[0][2]
    else:
        o2, _, _ = _solve_2d(inst, 2, 2, sched, kw, "nc2_2d22")
        res = [o[0] for o in o2.values()]
        U = np.concatenate([o2[(a, 0)][1] for a in range(2)])
        V = np.concatenate([o2[(0, b)][2] for b in range(2)])
    r0 = res[0]
    assert all(x["status"] == 0 for x in res)
    assert all(x["evaluations"] == r0["evaluations"] and x["cost_unrounded"] == r0["cost_unrounded"] for x in res)
    assert r0["l1_final"] <= eps
    ref = M.mdot_solve(_t(inst.C), _t(inst.r), _t(inst.c), schedule=sched, options=M.options(eps=eps))
    assert abs(r0["cost_unrounded"] - ref["cost_unrounded"]) <= COST_GATE * ref["cost_unrounded"]
    prob = O.OracleProblem(inst)
    lr, lc, _ = O.log_marginals(prob, U, V, gb)
    assert np.abs(np.exp(lr) - inst.r).sum() + np.abs(np.exp(lc) - inst.c).sum() <= 2 * eps
    rp = O.round_plan(prob, U, V, gb)
    assert abs(r0["cost_rounded"] - rp["cost_G"]) <= 1e-10 * rp["cost_G"]


def test_2d_grid_config4_full_size():
    """Config 4 at its BASELINE size and parameters (n = 16384, 1 GiB fp32 C,
    Dirichlet(1), gbar 4096, T 16, L1 1e-6) on a 2 x 2 grid of 8192 x 8192
    blocks: identical decisions on every rank, the oracle's full fp64
    re-evaluation of the assembled (U, V) at L1 <= 2 eps, the unrounded cost
    within the Z20 gate of the stored full oracle solve (tests/golden), and the
    rounded / unrounded costs equal to the oracle's rounding of the same
    potentials to 1e-10."""
    import json
    import os
    inst = S.config4(0)
    n = inst.n
    gb, eps = 4096.0, 1e-6
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=16)
    out, _, _ = _solve_2d(inst, 2, 2, sched, {"eps": eps}, "g2d_cfg4")
    r00 = out[(0, 0)][0]
    assert all(o[0]["status"] == 0 for o in out.values()), [(k, o[0]["status_name"], o[3]) for k, o in out.items()]
    assert all(o[0]["evaluations"] == r00["evaluations"] for o in out.values())
    assert all(o[0]["cost_rounded"] == r00["cost_rounded"] for o in out.values())
    assert r00["l1_final"] <= eps
    U = np.concatenate([out[(a, 0)][1] for a in range(2)])
    V = np.concatenate([out[(0, b)][2] for b in range(2)])
    prob = O.OracleProblem(inst)
    lr, lc, _ = O.log_marginals(prob, U, V, gb)
    assert np.abs(np.exp(lr) - inst.r).sum() + np.abs(np.exp(lc) - inst.c).sum() <= 2 * eps
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg4_seed0.json")))
    gc = golden["cost_unrounded"]
    assert abs(r00["cost_unrounded"] - gc) <= COST_GATE * gc, (r00["cost_unrounded"], gc)
    rp = O.round_plan(prob, U, V, gb)
    assert abs(r00["cost_unrounded"] - rp["cost_F"]) <= 1e-10 * rp["cost_F"]
    assert abs(r00["cost_rounded"] - rp["cost_G"]) <= 1e-10 * rp["cost_G"]
