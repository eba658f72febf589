import os, sys
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import synthetic as S, paper_2307_08507_b200 as M
inst = S.config4(0); n = inst.n
t = lambda x: torch.from_numpy(x).cuda()
C, r, c = t(inst.C), t(inst.r), t(inst.c)
U = torch.empty(n, dtype=torch.float64, device='cuda'); V = torch.empty_like(U)
M.mdot_solve(C, r, c, schedule=M.schedule(M.MDOT_SCHED_FIXED, 1024.0, T=1), options=M.options(eps=1e-3), u_out=U, v_out=V)
lr1, lc1, _ = M.mdot_marginals(U, V, 1024.0, C, r, c)
os.environ["MDOT_DISABLE_TMA"] = "1"
lr2, lc2, _ = M.mdot_marginals(U, V, 1024.0, C, r, c)
dr = (lr1 - lr2).abs().cpu().numpy(); dc = (lc1 - lc2).abs().cpu().numpy()
br = np.nonzero(dr > 1e-9)[0]; bc = np.nonzero(dc > 1e-9)[0]
print("bad rows", len(br), br[:40], "bad cols", len(bc), bc[:40])
print("row tiles", np.unique(br // 512)[:40], "col tiles", np.unique(bc // 256)[:70])
print("rows mod 512 unique count", len(np.unique(br % 512)), "cols mod 256", len(np.unique(bc % 256)))
