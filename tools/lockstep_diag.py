import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2307_08507_b200 as M, synthetic as S
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
B = 4
base = S.config3(0, frac=0.9)
C = t(base.C)
pairs = [S.config3(i, frac=0.9) for i in range(B)]
Rb = t(np.stack([p.r for p in pairs])); Cb = t(np.stack([p.c for p in pairs]))
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16)
lk = M.mdot_solve_batch(C, Rb, Cb, schedule=sched, options=M.options(eps=1e-6))
os.environ["MDOT_NO_PERSIST"] = "1"
for b in range(B):
    g = M.mdot_solve(C, Rb[b], Cb[b], schedule=sched, options=M.options(eps=1e-6))
    print(b, "lockstep evals", lk[b]["evaluations"], "iters", lk[b]["iterations"], "per-step", lk[b]["iters_step"][:6],
          "| graph evals", g["evaluations"], "iters", g["iterations"], "per-step", g["iters_step"][:6], flush=True)
