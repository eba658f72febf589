"""One K8 batched solve in the fp64-entry mode (config 2, 64 pairs, eps 1e-8, T = 1) for ncu captures."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synthetic as S  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402
C, R, Cm = S.config2(0, pairs=64)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
res = M.mdot_solve_batch(t(C), t(R), t(Cm), schedule=M.schedule(M.MDOT_SCHED_FIXED, 256.0, T=1),
                         options=M.options(eps=1e-8, max_evals=300), check=False)
torch.cuda.synchronize()
print("evals", sum(r["evaluations"] for r in res) / len(res))
