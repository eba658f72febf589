"""One lockstep throughput batch (16 x n = 4096, eps_md 1e-3) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MDOT_BATCH_LOCKSTEP"] = "1"
import numpy as np, torch
import paper_2307_08507_b200 as M, synthetic as S
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
base = S.config3(0, frac=0.9)
pairs = [S.config3(i, frac=0.9) for i in range(16)]
C = t(base.C); Rb = t(np.stack([p.r for p in pairs])); Cb = t(np.stack([p.c for p in pairs]))
res = M.mdot_solve_batch(C, Rb, Cb, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                         options=M.options(eps=1e-6, eps_md=float(os.environ.get("EM", "1e-3"))))
torch.cuda.synchronize()
print("evals", sum(r["evaluations"] for r in res))
