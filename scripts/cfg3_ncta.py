"""Config 3 (n = 4096) time-to-eps and slot phases vs the persistent grid size (MDOT_PERSIST_NCTA A/B)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
inst = S.config3(0, frac=0.9)
C, r, c = t(inst.C), t(inst.r), t(inst.c)
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
for _ in range(2):
    M.mdot_solve(C, r, c, schedule=sched, options=M.options(eps=1e-6))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    res = M.mdot_solve(C, r, c, schedule=sched, options=M.options(eps=1e-6, time_kernels=1))
e1.record(); torch.cuda.synchronize()
ns = res["stage_samples"]
print(os.environ.get("MDOT_PERSIST_NCTA", "default"), "tte %.2f ms" % (e0.elapsed_time(e1) / 3), "evals", res["evaluations"],
      "slot us", [round(1000 * x / ns, 2) for x in res["stage_ms"]], flush=True)
