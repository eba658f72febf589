import sys
sys.path.insert(0, '/root/repo')
import torch
import synthetic as S, paper_2307_08507_b200 as M
inst = S.config4(0)
t = lambda x: torch.from_numpy(x).cuda()
C, r, c = t(inst.C), t(inst.r), t(inst.c)
for _ in range(2):
    res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                       options=M.options(eps=1e-6, time_kernels=1))
print(res["evaluations"], res["status_name"], [x/res['stage_samples']*1000 for x in res['stage_ms']])
