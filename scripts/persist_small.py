# one short solve (n=16384, 2 MD steps, loose eps) for profiling the persistent kernel
import sys
sys.path.insert(0, '/root/repo')
import torch
import synthetic as S, paper_2307_08507_b200 as M
inst = S.config4(0)
t = lambda x: torch.from_numpy(x).cuda()
res = M.mdot_solve(t(inst.C), t(inst.r), t(inst.c), schedule=M.schedule(M.MDOT_SCHED_FIXED, 512.0, T=2),
                   options=M.options(eps=1e-3))
print(res["evaluations"], res["status_name"])
