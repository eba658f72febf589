"""Crossover of the small-problem route (mdot_solve on the one-CTA K8
kernel) vs the grid-wide paths: time-to-eps at several n, device-timed."""
import os
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_08507_b200 as M  # noqa: E402
import synthetic as S  # noqa: E402

t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731


def timed(fn, reps=3):
    fn()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if best is None or ms < best[0]:
            best = (ms, r)
    return best


cases = [("cfg1 n64 fp64 doubling", S.config1(0), M.schedule(M.MDOT_SCHED_DOUBLING, 4096.0))]
for n in (64, 128, 192, 256, 384, 512, 784):
    cases.append((f"fp32 n{n} gbar1024 T4", S.uniform_points_instance(3, n, 2, 30, marg="dirichlet"),
                  M.schedule(M.MDOT_SCHED_FIXED, 1024.0, T=4)))
for name, inst, sched in cases:
    C, r, c = t(inst.C), t(inst.r), t(inst.c)
    row = []
    for lim in ("0", "100000"):
        os.environ["MDOT_SMALL_N"] = lim
        ms, res = timed(lambda: M.mdot_solve(C, r, c, schedule=sched, options=M.options(eps=1e-6)))
        row.append((res["control_path"], round(ms, 2), res["evaluations"], res["status_name"], res["cost_unrounded"]))
    print(name, row, flush=True)
