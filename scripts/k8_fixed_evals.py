"""One K8 batch (config 2, 64 pairs, eps 1e-6) capped at K8_EVALS evaluations per
instance (default 400): for MDOT_DEBUG_K8 phase clocks and ncu captures."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
C, R, Cm = S.config2(0, pairs=64)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
Cd, Rd, Cmd = t(C), t(R), t(Cm)
sched = M.schedule(M.MDOT_SCHED_FIXED, 4096.0)
res = M.mdot_solve_batch(Cd, Rd, Cmd, schedule=sched, options=M.options(eps=1e-6, max_evals=int(os.environ.get("K8_EVALS", "400"))), check=False)
torch.cuda.synchronize()
