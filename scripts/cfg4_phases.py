import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2307_08507_b200 as M, synthetic as S
inst = S.config4(0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
C, r, c = t(inst.C), t(inst.r), t(inst.c)
for rep in range(2):
    res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0), options=M.options(eps=1e-6, time_kernels=1))
print(res["seconds"], res["evaluations"], [1000*x/res["stage_samples"] for x in res["stage_ms"]])
