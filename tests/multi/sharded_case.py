"""One rank of a real multi-GPU sharded solve (launched by
tests/test_gpu_multi.py with torch.distributed.run, one process per GPU):
rows of C (dense, fused peer exchange over NVLink / CUDA IPC) or of X
(on-the-fly cost, NCCL allreduce in CUDA-graph slots) sharded over the
ranks, then a 2-D (row x column) grid of blocks (mdot_solve_sharded_2d, NCCL
team communicators); rank 0 gathers the potentials and checks them against the fp64 oracle
and the single-GPU solve.  Prints "MULTI OK" on rank 0."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle as O  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402


def _team_comm(members, rank, lr, dev):
    """mdot communicator over `members` (global ranks): the first member's
    NCCL unique id broadcast over a torch subgroup.  Every rank calls this for
    every team in the same order (new_group is collective)."""
    grp = dist.new_group(members)
    if rank not in members:
        return None
    uid = M.mdot_get_unique_id() if rank == members[0] else bytes(128)
    t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).to(dev)
    dist.broadcast(t, members[0], group=grp)
    return M.mdot_comm_create(bytes(t.cpu().numpy()), len(members), members.index(rank), lr)


def two_d(rank, world, lr, dev, sched, eps, gb):
    """2-D grid (mdot_solve_sharded_2d): Gr x Gc ranks, rank = a Gc + b owns
    block rows_a x cols_b; row team = same a, column team = same b."""
    Gr = 2 if world >= 4 else 1
    Gc = world // Gr
    if Gr * Gc != world:
        return True
    a, b = rank // Gc, rank % Gc
    rc = cc = None
    for aa in range(Gr):
        x = _team_comm([aa * Gc + bb for bb in range(Gc)], rank, lr, dev)
        rc = x if aa == a else rc
    for bb in range(Gc):
        x = _team_comm([aa * Gc + bb for aa in range(Gr)], rank, lr, dev)
        cc = x if bb == b else cc
    inst = S.uniform_points_instance(3, 3000, 2, 81, marg="dirichlet")
    n = inst.n
    rows = np.array_split(np.arange(n), Gr)[a]
    cols = np.array_split(np.arange(n), Gc)[b]
    r0, nr, c0, nc = int(rows[0]), len(rows), int(cols[0]), len(cols)
    Cb = torch.from_numpy(np.ascontiguousarray(inst.C[r0:r0 + nr, c0:c0 + nc])).to(dev)
    r, c = torch.from_numpy(inst.r).to(dev), torch.from_numpy(inst.c).to(dev)
    U = torch.empty(nr, dtype=torch.float64, device=dev)
    V = torch.empty(nc, dtype=torch.float64, device=dev)
    res = M.mdot_solve_sharded_2d(rc, cc, r0, nr, c0, nc, Cb, r, c, n=n, schedule=sched,
                                  options=M.options(eps=eps), u_local_out=U, v_local_out=V)
    M.mdot_comm_destroy(rc)
    M.mdot_comm_destroy(cc)
    got = [None] * world
    dist.all_gather_object(got, (a, b, res["cost_unrounded"], res["cost_rounded"], res["evaluations"],
                                 U.cpu().numpy(), V.cpu().numpy()))
    if rank != 0:
        return True
    same = len({(g[2], g[3], g[4]) for g in got}) == 1
    Ufull = np.concatenate([g[5] for g in got if g[1] == 0])
    Vfull = np.concatenate([g[6] for g in got if g[0] == 0])
    prob = O.OracleProblem(inst)
    lrr, lcc, _ = O.log_marginals(prob, Ufull, Vfull, gb)
    l1 = np.abs(np.exp(lrr) - inst.r).sum() + np.abs(np.exp(lcc) - inst.c).sum()
    rp = O.round_plan(prob, Ufull, Vfull, gb)
    relG = abs(res["cost_rounded"] - rp["cost_G"]) / rp["cost_G"]
    good = res["status"] == 0 and same and l1 <= 2 * eps and relG <= 1e-10
    print(f"2d {Gr}x{Gc}: status {res['status_name']} identical_on_ranks {same} oracle_L1 {l1:.2e} "
          f"rounded_cost_rel_vs_oracle_rounding {relG:.2e} evals {res['evaluations']}", flush=True)
    return good


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    dist.init_process_group("nccl", device_id=dev)
    uid = M.mdot_get_unique_id() if rank == 0 else bytes(128)
    t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).to(dev)
    dist.broadcast(t, 0)
    comm = M.mdot_comm_create(bytes(t.cpu().numpy()), world, rank, lr)
    eps, gb = 1e-6, 1024.0
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb, T=4)
    ok = True
    for kind in ("dense", "otf"):
        inst = S.uniform_points_instance(3, 3000, 2, 80, marg="dirichlet") if kind == "dense" else \
            S.config5(2, n=3000, d=16)
        n = inst.n
        rows = np.array_split(np.arange(n), world)[rank]
        row0, nloc = int(rows[0]), len(rows)
        r, c = torch.from_numpy(inst.r).to(dev), torch.from_numpy(inst.c).to(dev)
        U = torch.empty(nloc, dtype=torch.float64, device=dev)
        V = torch.empty(n, dtype=torch.float64, device=dev)
        if kind == "dense":
            st = M.mdot_comm_enable_peer(comm, n, check=False)
            C = torch.from_numpy(np.ascontiguousarray(inst.C[row0:row0 + nloc])).to(dev)
            res = M.mdot_solve_sharded(comm, row0, nloc, C, r, c, n=n, schedule=sched, options=M.options(eps=eps),
                                       u_local_out=U, v_out=V)
            path = res["control_path"]
            if rank == 0:
                print(f"dense: peer enable status {st}, control_path {path}", flush=True)
        else:
            X = torch.from_numpy(np.ascontiguousarray(inst.X[row0:row0 + nloc])).to(dev)
            Y = torch.from_numpy(inst.Y).to(dev)
            res = M.mdot_solve_sharded(comm, row0, nloc, X_local=X, Y=Y, scale=inst.scale, r=r, c=c, n=n,
                                       schedule=sched, options=M.options(eps=eps), u_local_out=U, v_out=V)
        # every rank took the same decisions: identical scalars and V
        chk = torch.tensor([res["cost_unrounded"], float(res["evaluations"]), V.sum().item()], dtype=torch.float64,
                           device=dev)
        lo, hi = chk.clone(), chk.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        same = bool(torch.equal(lo, hi))
        parts = [torch.empty(len(x), dtype=torch.float64, device=dev) for x in np.array_split(np.arange(n), world)]
        dist.all_gather(parts, U)
        if rank == 0:
            Ufull = torch.cat(parts).cpu().numpy()
            prob = O.OracleProblem(inst)
            lrr, lcc, _ = O.log_marginals(prob, Ufull, V.cpu().numpy(), gb)
            l1 = np.abs(np.exp(lrr) - inst.r).sum() + np.abs(np.exp(lcc) - inst.c).sum()
            _, _, ores, _ = O.mdot(prob, O.schedule_fixed(gb, T=4), O.make_options(eps=eps))
            rel = abs(res["cost_unrounded"] - ores["cost_unrounded"]) / ores["cost_unrounded"]
            good = res["status"] == 0 and same and l1 <= 2 * eps and rel <= 1e-5
            print(f"{kind}: status {res['status_name']} identical_on_ranks {same} oracle_L1 {l1:.2e} "
                  f"cost_rel {rel:.2e} evals {res['evaluations']}", flush=True)
            ok = ok and good
    M.mdot_comm_destroy(comm)
    ok = two_d(rank, world, lr, dev, sched, eps, gb) and ok
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("MULTI OK" if ok else "MULTI FAIL", flush=True)
        sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
