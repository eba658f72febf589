"""Adaptive gamma schedule (MDOT_SCHED_ADAPTIVE, Z29) vs the paper's FIXED T = 16 on
configs 4 and 3: time-to-eps, evaluations, realised steps (device-timed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
for name, inst in (("cfg4", S.config4(0)), ("cfg3-0.9", S.config3(0, frac=0.9))):
    C, r, c = t(inst.C), t(inst.r), t(inst.c)
    legs = [("fixed T16", M.schedule(M.MDOT_SCHED_FIXED, 4096.0), 0.0)]
    for g1 in (64.0, 128.0, 256.0, 512.0):
        legs.append((f"adaptive g1={g1:g}", M.schedule(M.MDOT_SCHED_ADAPTIVE, 4096.0, step_max=g1), 0.0))
    legs.append(("fixed T16 eps_md 1e-3", M.schedule(M.MDOT_SCHED_FIXED, 4096.0), 1e-3))
    legs.append(("adaptive g1=256 eps_md 1e-3", M.schedule(M.MDOT_SCHED_ADAPTIVE, 4096.0, step_max=256.0), 1e-3))
    legs.append(("single step T1", M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=1), 0.0))
    for lab, sched, em in legs:
        o = M.options(eps=1e-6, eps_md=em)
        M.mdot_solve(C, r, c, schedule=sched, options=o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        res = M.mdot_solve(C, r, c, schedule=sched, options=o)
        e1.record(); torch.cuda.synchronize()
        print(f"{name} {lab:28s} tte {e0.elapsed_time(e1):8.2f} ms evals {res['evaluations']:5d} steps {res['md_steps']:2d} "
              f"cost {res['cost_unrounded']:.10g} {res['status_name']} gammas {[round(g) for g in res['gammas']]}", flush=True)
