"""Screened (K2s) vs dense (K2) solve on one small on-the-fly instance:
cost, evaluations, status for several screen windows T (MDOT_SCREEN_T)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as S  # noqa: E402
import paper_2307_08507_b200 as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda:0")
inst = S.config5(0, n=n)
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
for scr, T in [(0, 48), (1, 48), (1, 200), (1, 2000)]:
    os.environ["MDOT_SCREEN"] = str(scr)
    os.environ["MDOT_SCREEN_T"] = str(T)
    os.environ["MDOT_SCREEN_FMAX"] = "2"   # never fall back: exercise K2s at every density
    res = M.mdot_solve(X=t(inst.X), Y=t(inst.Y), scale=inst.scale, r=t(inst.r), c=t(inst.c),
                       schedule=M.schedule(M.MDOT_SCHED_FIXED, 1024.0, T=4), options=M.options(eps=1e-5),
                       check=False, recipe="dot")
    print(f"screen={scr} T={T} {res['status_name']} evals={res['evaluations']} cost={res['cost_unrounded']!r} "
          f"L1={res['l1_final']:.2e} stats={M.mdot_last_screen_stats()}", flush=True)
