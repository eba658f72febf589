"""One config-5 solve (n = 65536, d = 16, dot recipe, gbar 4096 T 16, L1 1e-5);
MDOT_SCREEN from the environment.  Harness for ncu captures of K2 / K2s."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as S  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
inst = S.config5(0, n=n)
dev = torch.device("cuda:0")
X, Y = torch.from_numpy(inst.X).to(dev), torch.from_numpy(inst.Y).to(dev)
r, c = torch.from_numpy(inst.r).to(dev), torch.from_numpy(inst.c).to(dev)
res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                   options=M.options(eps=1e-5), check=False, recipe="dot")
print(res["status_name"], res["evaluations"], res["cost_unrounded"], M.mdot_last_screen_stats())
