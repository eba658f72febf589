"""Per-stage host timestamps (MDOT_TRACE=1) of config-5 and config-4 solves capped at 48
evaluations: isolates the rounding stage (a10) cost."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
dev = torch.device("cuda:0")
inst = S.config5(0)
X, Y, r, c = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (inst.X, inst.Y, inst.r, inst.c)]
for me in (48, 48):
    res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0),
                       options=M.options(eps=1e-5, max_evals=me), check=False)
    print(res["status_name"], res["evaluations"], res["seconds"], flush=True)
inst = S.config4(0)
C, r, c = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (inst.C, inst.r, inst.c)]
for me in (48, 48):
    res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0), options=M.options(eps=1e-6, max_evals=me), check=False)
    print(res["status_name"], res["evaluations"], res["seconds"], flush=True)
