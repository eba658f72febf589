"""Config-4 persistent-kernel phase and finalize sub-phase times (MDOT_DEBUG prints per projection)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
inst = S.config4(0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
C, r, c = t(inst.C), t(inst.r), t(inst.c)
for _ in range(2):
    res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0), options=M.options(eps=1e-6, time_kernels=1))
    torch.cuda.synchronize()
ns = res["stage_samples"]
print("slot stages us:", [round(1000 * x / ns, 2) for x in res["stage_ms"]], "evals", res["evaluations"], "s", res["seconds"])
