import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2307_08507_b200 as M
import synthetic as S
inst = S.config1(0)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
C, r, c = t(inst.C), t(inst.r), t(inst.c)
for rep in range(3):
    res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_DOUBLING, 4096.0), options=M.options(eps=1e-6))
    print(f"{1000*res['seconds']:.2f} ms", res["evaluations"], res["control_path"], flush=True)
