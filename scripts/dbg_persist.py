import os, sys, time
sys.path.insert(0, '/root/repo')
os.environ['MDOT_DEBUG'] = '1'
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
inst = S.config4(0)
t = lambda x: torch.from_numpy(x).cuda()
C, r, c = t(inst.C), t(inst.r), t(inst.c)
for dc in (1, 2):
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.time()
        res = M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0), options=M.options(eps=1e-6, device_control=dc, time_kernels=1))
        torch.cuda.synchronize(); dt = time.time() - t0
        print(f"dc={dc} {dt*1e3:.1f} ms evals={res['evaluations']} per-eval={dt/res['evaluations']*1e6:.1f}us k1={res['kernel_ms']/max(1,res['kernel_launches'])*1e3:.1f}us stages={[x/max(1,res['stage_samples'])*1e3 for x in res['stage_ms']]}", flush=True)
