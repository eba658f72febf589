"""Bounded config-5-shaped screened solve with per-graph screen statistics
(MDOT_SCREEN_DEBUG=1): python tools/screen_probe.py n max_evals"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as S  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402

n, me = int(sys.argv[1]), int(sys.argv[2])
os.environ.setdefault("MDOT_SCREEN_DEBUG", "1")
inst = S.config5(0, n=n)
dev = torch.device("cuda:0")
X, Y = torch.from_numpy(inst.X).to(dev), torch.from_numpy(inst.Y).to(dev)
r, c = torch.from_numpy(inst.r).to(dev), torch.from_numpy(inst.c).to(dev)
t0 = time.time()
res = M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 4096.0, T=16),
                   options=M.options(eps=1e-5, max_evals=me, time_kernels=1), check=False, recipe="dot")
torch.cuda.synchronize()
print(f"{time.time() - t0:.2f}s", res["status_name"], res["evaluations"], res["fallbacks"], res["md_steps"],
      M.mdot_last_screen_stats(), flush=True)
