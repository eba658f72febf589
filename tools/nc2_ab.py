"""NC2 A/B on one GPU: the row-sharded (G = 4 virtual ranks) and 2-D (2 x 2)
host-loop solves of a config-3-shaped instance (n = 4096, gbar 4096, T 16,
L1 1e-6) with and without MDOT_NC2 (scalar-only line-search trials).  The
in-process transport moves every allreduce through host memory, so the
saving in exchanged bytes shows up in wall time; on NVLink the same bytes are
a few microseconds per exchange."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

DEV = torch.device("cuda:0")
inst = S.config3(0, frac=0.9)
n = inst.n
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(DEV)  # noqa: E731
r, c = t(inst.r), t(inst.c)


def run_grid(Gr, Gc, tag):
    rows = np.array_split(np.arange(n), Gr)
    cols = np.array_split(np.arange(n), Gc)
    blocks = {(a, b): t(inst.C[rows[a][0]:rows[a][-1] + 1, cols[b][0]:cols[b][-1] + 1])
              for a in range(Gr) for b in range(Gc)}
    out = {}

    def run(a, b):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            rc = M.mdot_comm_create_local(f"{tag}_r{a}", Gc, b, 0)
            cc = M.mdot_comm_create_local(f"{tag}_c{b}", Gr, a, 0)
            if Gc == 1:   # 1-D: the row-sharded call
                res = M.mdot_solve_sharded(cc, int(rows[a][0]), len(rows[a]), blocks[(a, b)], r, c, n=n,
                                           schedule=sched, options=M.options(eps=1e-6))
            else:
                res = M.mdot_solve_sharded_2d(rc, cc, int(rows[a][0]), len(rows[a]), int(cols[b][0]), len(cols[b]),
                                              blocks[(a, b)], r, c, n=n, schedule=sched, options=M.options(eps=1e-6))
            s.synchronize()
            M.mdot_comm_destroy(rc)
            M.mdot_comm_destroy(cc)
            out[(a, b)] = res

    ths = [threading.Thread(target=run, args=(a, b)) for a in range(Gr) for b in range(Gc)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return time.perf_counter() - t0, out[(0, 0)]


for Gr, Gc in ((4, 1), (2, 2)):
    for rep in range(2):
        for nc2 in ("0", "1"):
            os.environ["MDOT_NC2"] = nc2
            dt, res = run_grid(Gr, Gc, f"g{Gr}{Gc}_{nc2}_{rep}")
            print(f"{Gr}x{Gc} NC2={nc2} rep {rep}: {1000 * dt:8.1f} ms  evals {res['evaluations']}  "
                  f"ls_evals {res['ls_evaluations']}  iters {res['iterations']}  cost {res['cost_unrounded']:.10g}  "
                  f"L1 {res['l1_final']:.2e}  {res['status_name']}", flush=True)
