"""World-size-2 gloo test (CPU) of the row-sharding decomposition the CUDA
sharded path uses: each rank owns a row block, row
marginals stay local, column partial sums and the row-side scalars travel in
ONE packed allreduce [column partials | row scalars], column-side scalars are
computed redundantly on every rank.  The packed result must equal the
unsharded oracle evaluation."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import oracle as O
    import synthetic as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = S.uniform_points_instance(3, 97, 2, 11, marg="dirichlet")
    n = inst.n
    rng = np.random.default_rng(0)
    A = np.log(inst.r) + 0.1 * rng.standard_normal(n)
    B = np.log(inst.c) + 0.1 * rng.standard_normal(n)
    p = rng.standard_normal(2 * n)
    g = 30.0
    rows = np.array_split(np.arange(n), world)[rank]
    row0, nloc = rows[0], len(rows)
    # this rank's row block, direct fp64 evaluation
    Cl = inst.C[row0:row0 + nloc].astype(np.float64)
    P = np.exp(A[row0:row0 + nloc, None] + B[None, :] - g * Cl)
    rP_loc = P.sum(1)
    col_partial = P.sum(0)
    row_scalars = np.array([rP_loc.sum(), np.abs(rP_loc - inst.r[rows]).sum(),
                            (p[:n][rows] * (rP_loc - inst.r[rows])).sum(), float(nloc)])
    buf = torch.from_numpy(np.concatenate([col_partial, row_scalars]))
    dist.all_reduce(buf)   # the one packed collective per evaluation
    buf = buf.numpy()
    cP = buf[:n]
    rs = buf[n:]
    col_scalars = np.array([0.0, np.abs(cP - inst.c).sum(), (p[n:] * (cP - inst.c)).sum(), 0.0])
    tot = rs + col_scalars
    if rank == 0:
        prob = O.OracleProblem(inst)
        lr, lc, _ = O.log_marginals(prob, A, B, g)
        rr, cc = np.exp(lr), np.exp(lc)
        ref = np.array([rr.sum(), np.abs(rr - inst.r).sum() + np.abs(cc - inst.c).sum(),
                        (p[:n] * (rr - inst.r)).sum() + (p[n:] * (cc - inst.c)).sum(), float(n)])
        q.put((tot.tolist(), ref.tolist(), float(np.abs(cP - cc).max())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_packed_allreduce_decomposition(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    tot, ref, dcol = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_allclose(tot, ref, rtol=1e-12, atol=1e-15)
    assert dcol < 1e-15


def test_row_partition_covers_rows_once():
    """The partition bench.py and the tests use (np.array_split): contiguous,
    disjoint, covering, sizes differ by at most one."""
    for n in (1, 7, 97, 16384, 65536):
        for G in (1, 2, 3, 4, 8):
            parts = np.array_split(np.arange(n), G)
            cat = np.concatenate(parts)
            assert np.array_equal(cat, np.arange(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1


# ---------------------------------------------------------------------------
# Fused peer exchange (k_persist_peer)
# ---------------------------------------------------------------------------
def _peer_worker(rank, world, port, q):
    """Host model of one exchange of k_persist_peer over gloo: every rank's
    slot [column totals | row scalars] lands in every rank's receive block
    (all_gather stands in for the peer stores), each rank sums the slots in
    rank order 0..G-1.  The summed block must be bitwise identical on every
    rank (identical controller decisions) and equal the unsharded oracle."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import oracle as O
    import synthetic as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = S.uniform_points_instance(3, 101, 2, 12, marg="dirichlet")
    n = inst.n
    rng = np.random.default_rng(1)
    A = np.log(inst.r) + 0.1 * rng.standard_normal(n)
    B = np.log(inst.c) + 0.1 * rng.standard_normal(n)
    g = 25.0
    rows = np.array_split(np.arange(n), world)[rank]
    Cl = inst.C[rows[0]:rows[0] + len(rows)].astype(np.float64)
    P = np.exp(A[rows, None] + B[None, :] - g * Cl)
    rP = P.sum(1)
    slot = torch.from_numpy(np.concatenate([P.sum(0), [rP.sum(), np.abs(rP - inst.r[rows]).sum()]]))
    recv = [torch.empty_like(slot) for _ in range(world)]
    dist.all_gather(recv, slot)
    tot = torch.zeros_like(slot)
    for p in range(world):          # rank order, identical on every rank
        tot += recv[p]
    allt = [torch.empty_like(tot) for _ in range(world)]
    dist.all_gather(allt, tot)
    if rank == 0:
        same = all(torch.equal(allt[0], x) for x in allt)
        prob = O.OracleProblem(inst)
        lr, lc, _ = O.log_marginals(prob, A, B, g)
        t = tot.numpy()
        q.put((same, float(np.abs(t[:n] - np.exp(lc)).max()), float(abs(t[n] - np.exp(lr).sum())),
               float(abs(t[n + 1] - np.abs(np.exp(lr) - inst.r).sum()))))
    dist.destroy_process_group()


def test_peer_exchange_rank_ordered_sum_is_identical_on_every_rank():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    same, dcol, dmass, dl1 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert same
    assert dcol < 1e-15 and dmass < 1e-13 and dl1 < 1e-13


@pytest.mark.parametrize("G", [2, 3, 8])
def test_peer_exchange_protocol_double_buffering(G):
    """Threads model of the in-kernel protocol (k_persist_peer, LL records):
    per exchange e, every "CTA" (ncta per rank) of rank k writes its records
    tagged e into parity e & 1 of every rank's receive block, then reads its
    F2 chunk of every rank's records of its own block, polling each until it
    carries e, then passes the rank's grid barrier.  Random delays between
    steps; a record must never be overwritten (by exchange e + 2) before every
    reader of exchange e has consumed it -- a reader that finds e + 2 spins to
    the timeout and the test fails."""
    import random
    import threading
    import time
    E, ncta = 25, 3
    recv = [[[[0] * ncta for _ in range(G)] for _ in range(2)] for _ in range(G)]   # [rank][parity][src][cta]
    errors = []
    bars = [threading.Barrier(ncta) for _ in range(G)]   # one grid barrier per rank

    def cta_fn(k, c):
        rnd = random.Random(1000 * G + 10 * k + c)
        for e in range(1, E + 1):
            for p in range(G):   # F1: store this CTA's record to every rank
                time.sleep(rnd.random() * 1e-4)
                recv[p][e & 1][k][c] = e
            time.sleep(rnd.random() * 1e-4)
            for p in range(G):   # F2: poll own block, chunk c of every source rank
                t0 = time.time()
                while recv[k][e & 1][p][c] != e:
                    if recv[k][e & 1][p][c] > e or time.time() - t0 > 20:
                        errors.append((k, c, e, p, recv[k][e & 1][p][c]))
                        return
                    time.sleep(1e-5)
            bars[k].wait(timeout=60)   # grid barrier after F2 (before the next F1)

    ths = [threading.Thread(target=cta_fn, args=(k, c)) for k in range(G) for c in range(ncta)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors[:3]


def _worker_2d(rank, world, port, q, Gr, Gc):
    """2-D grid (mdot_solve_sharded_2d): rank (a, b) = (rank // Gc, rank % Gc)
    owns block rows_a x cols_b.  Row sums go over the row team (same a), column
    sums over the column team (same b); row-side scalars (replicated across the
    row team) are then summed over the column team, column-side scalars over
    the row team -- the order of collectives the CUDA path uses."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import oracle as O
    import synthetic as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    row_teams = [dist.new_group([a * Gc + b for b in range(Gc)]) for a in range(Gr)]
    col_teams = [dist.new_group([a * Gc + b for a in range(Gr)]) for b in range(Gc)]
    a, b = rank // Gc, rank % Gc
    inst = S.uniform_points_instance(3, 101, 2, 12, marg="dirichlet")
    n = inst.n
    rng = np.random.default_rng(1)
    A = np.log(inst.r) + 0.1 * rng.standard_normal(n)
    B = np.log(inst.c) + 0.1 * rng.standard_normal(n)
    p = rng.standard_normal(2 * n)
    g = 30.0
    rows = np.array_split(np.arange(n), Gr)[a]
    cols = np.array_split(np.arange(n), Gc)[b]
    Cb = inst.C[np.ix_(rows, cols)].astype(np.float64)
    P = np.exp(A[rows, None] + B[None, cols] - g * Cb)
    rsum = torch.from_numpy(P.sum(1).copy())
    csum = torch.from_numpy(P.sum(0).copy())
    dist.all_reduce(rsum, group=row_teams[a])     # rows: over the column blocks
    dist.all_reduce(csum, group=col_teams[b])     # columns: over the row blocks
    rP, cP = rsum.numpy(), csum.numpy()
    rs = torch.from_numpy(np.array([rP.sum(), np.abs(rP - inst.r[rows]).sum(), (p[:n][rows] * (rP - inst.r[rows])).sum()]))
    cs = torch.from_numpy(np.array([0.0, np.abs(cP - inst.c[cols]).sum(), (p[n:][cols] * (cP - inst.c[cols])).sum()]))
    dist.all_reduce(rs, group=col_teams[b])       # row items: replicated across the row team
    dist.all_reduce(cs, group=row_teams[a])       # column items: replicated across the column team
    tot = (rs + cs).numpy()
    prob = O.OracleProblem(inst)
    lr, lc, _ = O.log_marginals(prob, A, B, g)
    rr, cc = np.exp(lr), np.exp(lc)
    ref = np.array([rr.sum(), np.abs(rr - inst.r).sum() + np.abs(cc - inst.c).sum(),
                    (p[:n] * (rr - inst.r)).sum() + (p[n:] * (cc - inst.c)).sum()])
    q.put((rank, tot.tolist(), ref.tolist(), float(np.abs(rP - rr[rows]).max() / rr[rows].max()),
           float(np.abs(cP - cc[cols]).max() / cc[cols].max())))
    dist.destroy_process_group()


@pytest.mark.parametrize("Gr,Gc", [(2, 2), (1, 3)])
def test_2d_grid_decomposition(Gr, Gc):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = Gr * Gc
    procs = [ctx.Process(target=_worker_2d, args=(r, world, port, q, Gr, Gc)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, tot, ref, drow, dcol in got:
        # identical scalars on every rank, equal to the unsharded evaluation
        np.testing.assert_allclose(tot, ref, rtol=1e-12, atol=1e-15)
        assert drow < 1e-13 and dcol < 1e-13
