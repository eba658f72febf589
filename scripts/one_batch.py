"""One K8 batched solve (config 2, 64 pairs) for ncu captures."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import synthetic as S, paper_2307_08507_b200 as M
C, R, Cm = S.config2(0, pairs=64)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 2
res = M.mdot_solve_batch(t(C), t(R), t(Cm), schedule=M.schedule(M.MDOT_SCHED_FIXED, 256.0 * T, T=T),
                         options=M.options(eps=1e-6), check=False)
torch.cuda.synchronize()
print("evals", sum(r["evaluations"] for r in res) / len(res))
