import os, sys, hashlib
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"] if "GRAFT_REPO_ROOT" in os.environ else ".")
import numpy as np, torch
import paper_2307_08507_b200 as M, synthetic as S
DEV = torch.device("cuda:0")
t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
inst = S.config5(0, n=600, d=16)
U = torch.empty(600, dtype=torch.float64, device=DEV); V = torch.empty_like(U)
res = M.mdot_solve(X=t(inst.X), Y=t(inst.Y), scale=inst.scale, r=t(inst.r), c=t(inst.c), schedule=M.schedule(M.MDOT_SCHED_FIXED, 256.0, T=2), options=M.options(eps=1e-4), u_out=U, v_out=V)
print(os.environ.get("MDOT_LIB","rel")[-14:], os.environ.get("MDOT_SCREEN"), res["evaluations"], repr(res["cost_unrounded"]), M.mdot_last_screen_stats(), hashlib.sha1(U.cpu().numpy().tobytes()).hexdigest()[:12])
